# sparse stencil: taller tiles (4 warps along y) and the output-8 exchange body (odd positions as 4 FFMA2)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
SKC_SPARSE_F2=2 SKC_SPARSE_WY=4 python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse or c1 or stencil_variants" > gpurun_out/pytest_gpu69.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu69.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b69_$name.json 2> gpurun_out/b69_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b69_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run base SKC_X=0; run wy4 SKC_SPARSE_WY=4; run wy4m2 SKC_SPARSE_WY=4 SKC_SPARSE_MINB=2; run wy4m1 SKC_SPARSE_WY=4 SKC_SPARSE_MINB=1; run x SKC_SPARSE_F2=2; run xwy4 SKC_SPARSE_F2=2 SKC_SPARSE_WY=4 SKC_SPARSE_MINB=2
