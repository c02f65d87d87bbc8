# default: 4 CTAs/SM for small narrow sparse bodies; sparse + chain tests, c1/c0
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse or c1 or c0 or stencil_variants or golden or ragged" > gpurun_out/pytest_gpu85.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu85.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b85_$name.json 2> gpurun_out/b85_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b85_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke85.log 2>&1; echo smoke_rc=$?
