# sparse stencil: larger KR for tall footprints (config 1's 116-position layer, Dy = 30)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b78_$name.json 2> gpurun_out/b78_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b78_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run k3 SKC_X=0; run w5 SKC_SPARSE_KR_WIDE=5; run w5m2 SKC_SPARSE_KR_WIDE=5 SKC_SPARSE_MINB=2; run w7m2 SKC_SPARSE_KR_WIDE=7 SKC_SPARSE_MINB=2
SKC_SPARSE_KR_WIDE=5 python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse" > gpurun_out/pytest_gpu78.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu78.log
