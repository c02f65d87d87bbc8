# Kawase: suspend-hint sweep (c3 and c3big, peel on/off); c1 HWC epilogue A/B
mkdir -p gpurun_out/s4e
export SKC_CACHE_DIR=$(mktemp -d)
for hint in 131072 16384 4096 1000 250 0; do
  echo "hint=$hint c3:    $(SKC_KAWASE_HINT=$hint timeout 120 python tools/gpu/kw_one.py 2>&1 | tail -1)"
  echo "hint=$hint c3big: $(SKC_KAWASE_HINT=$hint timeout 120 python tools/gpu/kw_one.py c3big 2>&1 | tail -1)"
done
echo "hint=1000 nopeel c3: $(SKC_KAWASE_PEEL=0 timeout 120 python tools/gpu/kw_one.py 2>&1 | tail -1)"
echo "hint=1000 H only: $(SKC_KAWASE_DBG=4 timeout 120 python tools/gpu/kw_one.py 2>&1 | tail -1)"
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline'].get('per_launch_ms', [])])
" $1; }
for e in 1 0 1 0; do
  SKC_SPARSE_EPI=$e timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4e/c1_epi$e.json 2> gpurun_out/s4e/c1_epi$e.err; show gpurun_out/s4e/c1_epi$e.json
done
