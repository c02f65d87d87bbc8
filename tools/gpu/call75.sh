# fp16 all-channel generated head (no input relayout pass for fp16 chains)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "fp16 or half or kawase or fused or epilogue or chain_io or sparse" > gpurun_out/pytest_gpu75.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu75.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b75_$name.json 2> gpurun_out/b75_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b75_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run allc SKC_X=0; run old SKC_SPARSE_HWC=0
BARGS="--config c3big"; run big SKC_X=0
BARGS="--config c1"; run c1 SKC_X=0
