# packed-FP32 sparse stencil body (SKC_SPARSE_F2=1: FFMA2 on output pairs, two accumulator parities) vs scalar, KR 3/5/7
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
SKC_SPARSE_F2=1 python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse or stencil_variants or c1" > gpurun_out/pytest_gpu61.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu61.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b61_$name.json 2> gpurun_out/b61_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b61_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"
run s3 SKC_SPARSE_F2=0; run f3 SKC_SPARSE_F2=1; run f5 SKC_SPARSE_F2=1 SKC_SPARSE_KR=5; run f7 SKC_SPARSE_F2=1 SKC_SPARSE_KR=7
run f3m3 SKC_SPARSE_F2=1 SKC_SPARSE_MINB=3; run f5m3 SKC_SPARSE_F2=1 SKC_SPARSE_KR=5 SKC_SPARSE_MINB=3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skc_sparse_stencil -c 3 -o gpurun_out/prof61_f2 env SKC_SPARSE_F2=1 python bench.py --config c1 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu61.log 2>&1; echo "ncu rc=$?"
BARGS="--config c0"; run c0 SKC_X=0; run c0d SKC_SPARSE=0
