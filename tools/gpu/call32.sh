# persistent double-buffered stencil / tap variants on c1
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "rolled or dense or chain" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b32_$name.json 2> gpurun_out/b32_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b32_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0; run c1_spipe SKC_STENCIL_PIPE=1; run c1_tpipe SKC_TAP_PIPE=1; run c1_tpipe5 SKC_TAP_PIPE=1 SKC_TAP_KR=5
BARGS="--config c3"; run c3_spipe SKC_STENCIL_PIPE=1
