# SV: one table read per tap for bracket-uniform threads; tap kernel KR=3 tiles for c3's 4-tap layers
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_sv_fit.py -m gpu -x -q -k "sv or SV or grid" > gpurun_out/pytest_gpu64.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu64.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b64_$name.json 2> gpurun_out/b64_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b64_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c2"; run c2 SKC_X=0; run c2b SKC_X=0
BARGS="--config c3"; run c3 SKC_X=0; run c3k3 SKC_TAP_KR=3; run c3k3f SKC_TAP_KR=3 SKC_HALF_MID=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sv_tile -c 4 -o gpurun_out/prof64_sv python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu64.log 2>&1; echo "ncu rc=$?"
