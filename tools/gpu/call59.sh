# sparse stencil at KR=3 (code size vs instruction cache): CTAs/SM and KR=1; c3 back on the register-path fp16 loader
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q > gpurun_out/pytest_gpu59.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu59.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b59_$name.json 2> gpurun_out/b59_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b59_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"
run kr3 SKC_X=0; run kr3m3 SKC_SPARSE_MINB=3; run kr3m4 SKC_SPARSE_MINB=4; run kr3m6 SKC_SPARSE_MINB=6; run kr1 SKC_SPARSE_KR=1; run kr1m6 SKC_SPARSE_KR=1 SKC_SPARSE_MINB=6
run kr3s2 SKC_SPARSE_SYNC=2; run kr3s4m4 SKC_SPARSE_SYNC=4 SKC_SPARSE_MINB=4
BARGS="--config c3"; run c3h SKC_HALF_MID=1; run c3f SKC_HALF_MID=0
