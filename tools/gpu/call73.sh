# SV: packed-FP32 pixel pairs on the bracket-uniform path (SKC_SV_PAIRS=0/1)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_sv_fit.py -m gpu -x -q -k "sv or SV or grid" > gpurun_out/pytest_gpu73.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu73.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b73_$name.json 2> gpurun_out/b73_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b73_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c2"; run p1 SKC_SV_PAIRS=1; run p0 SKC_SV_PAIRS=0; run p1b SKC_SV_PAIRS=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sv_tile -c 2 -o gpurun_out/prof73_sv python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu73.log 2>&1; echo "ncu rc=$?"
