# c1: one-warp-row tiles on the wide layers; KR_WIDE variants
mkdir -p gpurun_out/s4k
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline'].get('per_launch_ms', [])])
" $1; }
run() { n=$1; shift; env "$@" timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4k/$n.json 2> gpurun_out/s4k/$n.err; show gpurun_out/s4k/$n.json; }
run base X=1
run wy1 SKC_SPARSE_WY1=1
run wy1_kr3 SKC_SPARSE_WY1=1 SKC_SPARSE_KR_WIDE=3
run wy1_kr7 SKC_SPARSE_WY1=1 SKC_SPARSE_KR_WIDE=7
run kr7 SKC_SPARSE_KR_WIDE=7
