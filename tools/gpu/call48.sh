# row-pair FFMA2 tap kernel
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "epilogue" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b48_$name.json 2> gpurun_out/b48_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b48_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0; run c1_tf2 SKC_TAP_FFMA2=1; run c1_tf3 SKC_TAP_FFMA2=3; run c1_tf2_kr5 SKC_TAP_FFMA2=1 SKC_TAP_KR=5
BARGS="--config c3"; run c3_tf2 SKC_TAP_FFMA2=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"layer_tap" -c 1 -o gpurun_out/prof48_tf2 env SKC_TAP_FFMA2=1 python bench.py --config c1 --steps 1 --warmup 0 --frames 8 --no-e2e --no-cpu > gpurun_out/ncu48.log 2>&1; echo ncu rc=$?
