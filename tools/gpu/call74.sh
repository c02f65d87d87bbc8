# c3: generated sparse stencils forced for the Kawase layers (SKC_SPARSE=1) vs the KR=3 tap tiles
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b74_$name.json 2> gpurun_out/b74_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b74_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run tap SKC_X=0; run sp SKC_SPARSE=1; run spm4 SKC_SPARSE=1 SKC_SPARSE_MINB=4; run spk5 SKC_SPARSE=1 SKC_SPARSE_KR=5
SKC_SPARSE=1 python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "kawase or half" > gpurun_out/pytest_gpu74.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu74.log
