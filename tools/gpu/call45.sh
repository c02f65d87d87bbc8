# packed-FP32 (FFMA2) dense stencil
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "rolled or dense" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b45_$name.json 2> gpurun_out/b45_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b45_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0; run c1_f2 SKC_STENCIL_FFMA2=1
BARGS="--config c3"; run c3_f2 SKC_STENCIL_FFMA2=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"stencil2" -c 2 -o gpurun_out/prof45_f2 env SKC_STENCIL_FFMA2=1 python bench.py --config c1 --steps 1 --warmup 0 --frames 8 --no-e2e --no-cpu > gpurun_out/ncu45.log 2>&1; echo ncu rc=$?
