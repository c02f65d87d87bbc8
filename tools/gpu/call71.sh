# all-channel generated head v2 (SKC_SPARSE_HWC=2: interleaved tile via coalesced 4-byte cp.async, stride-C window loads)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
SKC_SPARSE_HWC=2 python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse or c1 or golden or ragged" > gpurun_out/pytest_gpu71.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu71.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b71_$name.json 2> gpurun_out/b71_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b71_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run base SKC_X=0; run allc SKC_SPARSE_HWC=2; run allcm1 SKC_SPARSE_HWC=2 SKC_SPARSE_MINB=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"skc_sparse" -c 1 -o gpurun_out/prof71_head env SKC_SPARSE_HWC=2 python bench.py --config c1 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu70.log 2>&1; echo "ncu rc=$?"
