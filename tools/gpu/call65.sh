# c3: KR=3 tap tiles for planar <=16-tap layers (KR=5 for the HWC-epilogue layer); dense D3 head vs the tap kernel
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "fp16 or half or kawase or epilogue or chain_io or fused" > gpurun_out/pytest_gpu65.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu65.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b65_$name.json 2> gpurun_out/b65_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b65_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run c3 SKC_X=0; run c3nd SKC_DENSE=0; run c3f SKC_HALF_MID=0; run c3fnd SKC_HALF_MID=0 SKC_DENSE=0
BARGS="--config c3big"; run big SKC_X=0; run bignd SKC_DENSE=0
BARGS="--config c0"; run c0 SKC_X=0
