# staged HWC epilogue (default) vs planar + relayout
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b34_$name.json 2> gpurun_out/b34_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b34_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0; run c1_nostage SKC_TAP_HWC_STAGE=0
BARGS="--config c3"; run c3 SKC_X=0; run c3_nostage SKC_TAP_HWC_STAGE=0
