# fp16 planar loader: 4 rows per iteration (more loads in flight)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "fp16 or half or kawase" > gpurun_out/pytest_gpu68.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu68.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b68_$name.json 2> gpurun_out/b68_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b68_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run c3 SKC_X=0; run c3b SKC_X=0
BARGS="--config c3big"; run big SKC_X=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"layer_tap" -c 2 -o gpurun_out/prof68_c3 python bench.py --config c3 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu68.log 2>&1; echo "ncu rc=$?"
