# sparse stencil: 4 CTAs/SM for small (<= 64-position) layers
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b84_$name.json 2> gpurun_out/b84_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b84_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run m3 SKC_X=0; run m4 SKC_SPARSE_MINB_SMALL=4; run m5 SKC_SPARSE_MINB_SMALL=5
BARGS="--config c0"; run c0m3 SKC_X=0; run c0m4 SKC_SPARSE_MINB_SMALL=4
