# packed-FP32 tap rows for planar KR=3 layers (SKC_TAP_F2=1): parity + c3 / c3big A/B
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
SKC_TAP_F2=1 python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "half or kawase or fp16 or ragged or chain_io" > gpurun_out/pytest_gpu87.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu87.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b87_$name.json 2> gpurun_out/b87_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b87_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run base SKC_X=0; run f2 SKC_TAP_F2=1
BARGS="--config c3big"; run bbase SKC_X=0; run bf2 SKC_TAP_F2=1
