# odd pitch for HWC-input dense stencils (c1's D5 head: bank conflicts)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "dense or golden or c0 or c1 or ragged or known" > gpurun_out/pytest_gpu67.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu67.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b67_$name.json 2> gpurun_out/b67_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b67_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run odd SKC_X=0; run even SKC_HEAD_ODD_PITCH=0; run odd2 SKC_X=0
BARGS="--config c0"; run c0 SKC_X=0
