# fp16 planar intermediates for fp16-storage chains: engine parity + c3/c3big A/B (SKC_HALF_MID=0/1)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q > gpurun_out/pytest_gpu56.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu56.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b56_$name.json 2> gpurun_out/b56_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b56_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run c3h SKC_HALF_MID=1; run c3f SKC_HALF_MID=0; run c3h2 SKC_HALF_MID=1
BARGS="--config c3big"; run bigh SKC_HALF_MID=1; run bigf SKC_HALF_MID=0
BARGS="--config c1"; run c1 SKC_X=0
