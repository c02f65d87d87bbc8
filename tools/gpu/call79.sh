# defaults: KR 5 / 2 CTAs per SM for tall footprints, KR 3 / 3 CTAs otherwise
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse or c1 or stencil_variants or chain_io" > gpurun_out/pytest_gpu79.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu79.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b79_$name.json 2> gpurun_out/b79_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b79_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0; run c1b SKC_X=0
