# sparse stencil: full-width LDS.128 window loads (no narrowed, conflicted LDS) and TMA bulk row copies for interior tiles
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "sparse or c1 or golden or stencil_variants" > gpurun_out/pytest_gpu77.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu77.log
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b77_$name.json 2> gpurun_out/b77_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b77_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run tma SKC_X=0; run notma SKC_SPARSE_TMA=0; run tma2 SKC_X=0
BARGS="--config c0"; run c0 SKC_X=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"skc_sparse" -c 4 -o gpurun_out/prof77 python bench.py --config c1 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu77.log 2>&1; echo "ncu rc=$?"
