# fused chain in groups of layers (config 3)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "fused" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b50_$name.json 2> gpurun_out/b50_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b50_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run c3 SKC_X=0; run c3_f6 SKC_FUSED=1; run c3_g2 SKC_FUSED=1 SKC_FUSED_GROUP=2; run c3_g3 SKC_FUSED=1 SKC_FUSED_GROUP=3; run c3_g1 SKC_FUSED=1 SKC_FUSED_GROUP=1
