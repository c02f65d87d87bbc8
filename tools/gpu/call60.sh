# sparse stencil also for D<=9 layers that skip >20% zeros (c1 layer 2: 58 of 81); ncu of the sparse launches
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "stencil or sparse or c1 or c0 or dense or golden or epilogue" > gpurun_out/pytest_gpu60.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu60.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke60.log 2>&1; echo smoke_rc=$?
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b60_$name.json 2> gpurun_out/b60_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b60_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0; run c1b SKC_X=0
BARGS="--config c0"; run c0 SKC_X=0; run c0d SKC_SPARSE=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skc_sparse_stencil -c 3 -o gpurun_out/prof60_sparse python bench.py --config c1 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu60.log 2>&1; echo "ncu rc=$?"
