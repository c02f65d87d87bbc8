# SV interleaved tile: parity + c2 bench both layouts
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sv_fit.py -m gpu -x -q -k "sv" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b33_$name.json 2> gpurun_out/b33_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b33_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c2"; run c2 SKC_X=0; run c2_planar SKC_SV_PLANAR=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sv_tile" -c 4 -o gpurun_out/prof33_sv python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu33.log 2>&1; echo ncu rc=$?
