mkdir -p gpurun_out/s4t
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline'].get('per_launch_ms', [])])
" $1; }
run() { n=$1; shift; env "$@" timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4t/$n.json 2> gpurun_out/s4t/$n.err; show gpurun_out/s4t/$n.json; }
run base X=1
run hkr1 SKC_SPARSE_HEAD_KR=1
run hkr5 SKC_SPARSE_HEAD_KR=5
run hkr5_wy2 SKC_SPARSE_HEAD_KR=5 SKC_SPARSE_HEAD_WY=2
run hkr1_wy2 SKC_SPARSE_HEAD_KR=1 SKC_SPARSE_HEAD_WY=2
