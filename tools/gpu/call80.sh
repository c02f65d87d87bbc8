# c3: staged HWC epilogue on the last tap layer vs planar + fp16 relayout pass; nested default cache dir
mkdir -p gpurun_out
export XDG_CACHE_HOME=$(mktemp -d)/nested/cache
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b80_$name.json 2> gpurun_out/b80_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b80_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c3"; run stage SKC_X=0; run relayout SKC_TAP_HWC_STAGE=0
BARGS="--config c3big"; run bstage SKC_X=0; run brelayout SKC_TAP_HWC_STAGE=0
ls -la $XDG_CACHE_HOME/skc | head -5
