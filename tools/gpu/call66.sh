# c3: tap tile instead of the dense D3 kernel for planar fp16 small layers; c1: generated sparse head on HWC input (opt-in)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "fp16 or half or kawase or sparse or dense" > gpurun_out/pytest_gpu66.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu66.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b66_$name.json 2> gpurun_out/b66_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b66_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run c3 SKC_X=0
BARGS="--config c1"; run c1 SKC_X=0; run c1hwc SKC_SPARSE=1 SKC_SPARSE_HWC=1; run c1hwc1 SKC_SPARSE=1 SKC_SPARSE_HWC=1 SKC_SPARSE_KR=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stencil" -c 1 -o gpurun_out/prof66_head python bench.py --config c1 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu66.log 2>&1; echo "ncu rc=$?"
