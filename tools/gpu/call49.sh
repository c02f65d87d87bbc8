# stencil register caps (D3: 3 CTAs/SM, others 4)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "dense or stencil or policies or kawase" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b49_$name.json 2> gpurun_out/b49_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b49_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run c3 SKC_X=0
BARGS="--config c1"; run c1 SKC_X=0
BARGS="--config c0"; run c0 SKC_X=0
