# defaults now: packed-FP32 sparse body, 3 CTAs/SM.  Full GPU suite + smoke, c1 A/B of CTAs/SM, c0
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu62.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu62.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke62.log 2>&1; echo smoke_rc=$?
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b62_$name.json 2> gpurun_out/b62_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b62_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run m3 SKC_X=0; run m4 SKC_SPARSE_MINB=4; run m2 SKC_SPARSE_MINB=2; run m3b SKC_X=0
