# stencil-row-loop (aloop) D=7/9: parity tests + c1 bench with/without
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b30_$name.json 2> gpurun_out/b30_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b30_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0; run c1_noal SKC_STENCIL_ALOOP=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"aloop" -c 1 -o gpurun_out/prof30_aloop python bench.py --config c1 --steps 1 --warmup 0 --frames 8 --no-e2e --no-cpu > gpurun_out/ncu30a.log 2>&1; echo ncu_a rc=$?
