# c3 / c3big: KR=3 for the HWC-epilogue tap layer too (SKC_TAP_KR=3) vs the default KR=5 there
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b89_$name.json 2> gpurun_out/b89_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b89_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run base SKC_X=0; run k3 SKC_TAP_KR=3; run k7 SKC_TAP_KR=7
BARGS="--config c3big"; run bbase SKC_X=0; run bk3 SKC_TAP_KR=3
