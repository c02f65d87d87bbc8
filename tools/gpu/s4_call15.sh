# c0 (512^2, launch-latency bound): tile-size knobs
mkdir -p gpurun_out/s4o
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,4) for t in d['roofline'].get('per_launch_ms', [])])
" $1; }
run() { n=$1; shift; env "$@" timeout 300 python bench.py --config c0 --steps 30 --warmup 5 --no-e2e --no-cpu --no-others > gpurun_out/s4o/$n.json 2> gpurun_out/s4o/$n.err; show gpurun_out/s4o/$n.json; }
run base X=1
run kr1 SKC_SPARSE_KR=1
run sparse1 SKC_SPARSE=1
run kr1_sparse1 SKC_SPARSE_KR=1 SKC_SPARSE=1
run tapkr5 SKC_TAP_KR=5
run small0 SKC_SPARSE_SMALL=0
for v in base kr1 kr1_sparse1; do
  e=""; [ $v = kr1 ] && e="SKC_SPARSE_KR=1"; [ $v = kr1_sparse1 ] && e="SKC_SPARSE_KR=1 SKC_SPARSE=1"
  env $e X=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4o/l_$v.csv python bench.py --config c0 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/s4o/l_$v.csv')))
hdr=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
print('$v', [(r[ki][:18], r[gi], r[vi]) for r in rows[hdr+1:] if 'skc' in r[ki] or 'layer_' in r[ki]][-4:])
PY
done
