# FFMA2 stencil: scalar FFMA for the half-empty first/last stencil rows
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "stencil_variants or dense" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b54_$name.json 2> gpurun_out/b54_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b54_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0
