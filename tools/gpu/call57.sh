# generated sparse stencils (NVRTC) for wide layers: engine parity, c1 A/B (SKC_SPARSE=0/default), ncu of the new kernel and of c3's layers
mkdir -p gpurun_out
export SKC_CACHE_DIR=$PWD/gpurun_out/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse or c1 or golden or half or linearity or dense" > gpurun_out/pytest_gpu57.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu57.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b57_$name.json 2> gpurun_out/b57_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b57_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']], d['roofline'].get('fp32_pipe'))")"; }
BARGS="--config c1"; run c1sp SKC_X=0; run c1tap SKC_SPARSE=0; run c1sp2 SKC_X=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skc_sparse_stencil -c 2 -o gpurun_out/prof57_sparse python bench.py --config c1 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu57a.log 2>&1; echo "ncu a rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"layer_tap|layer_stencil|relayout" -c 4 -o gpurun_out/prof57_c3 python bench.py --config c3 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu57b.log 2>&1; echo "ncu b rc=$?"
