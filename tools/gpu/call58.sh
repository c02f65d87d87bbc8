# sparse stencil knobs (KR, barrier period, CTAs/SM) on c1; fp16 mids with cp.async staging on c3/c3big
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "half or sparse or fp16 or epilogue" > gpurun_out/pytest_gpu58.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu58.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b58_$name.json 2> gpurun_out/b58_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b58_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"
run kr7 SKC_X=0; run kr5 SKC_SPARSE_KR=5; run kr3 SKC_SPARSE_KR=3; run kr9 SKC_SPARSE_KR=9
run s4 SKC_SPARSE_SYNC=4; run s2 SKC_SPARSE_SYNC=2; run s8 SKC_SPARSE_SYNC=8
run m1 SKC_SPARSE_MINB=1; run kr5s4 SKC_SPARSE_KR=5 SKC_SPARSE_SYNC=4; run kr5m3 SKC_SPARSE_KR=5 SKC_SPARSE_MINB=3
BARGS="--config c3"; run c3h SKC_HALF_MID=1; run c3f SKC_HALF_MID=0
BARGS="--config c3big"; run bigh SKC_HALF_MID=1
