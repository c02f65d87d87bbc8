# fp16 HWC chain head (interior-tile strided loader): policies agree; c3 with SKC_CHAIN_IO=2
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "policies or kawase or fp16" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b36_$name.json 2> gpurun_out/b36_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b36_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run c3 SKC_X=0; run c3_io2 SKC_CHAIN_IO=2; run c3_io0 SKC_CHAIN_IO=0
BARGS="--config c1"; run c1 SKC_X=0
