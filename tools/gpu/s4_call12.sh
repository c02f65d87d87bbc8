# Kawase: V row pointer kept opaque (2 instead of 6 integer instructions per row)
mkdir -p gpurun_out/s4l
export SKC_CACHE_DIR=$(mktemp -d)
timeout 900 python -m pytest tests/test_gpu_kawase.py tests/test_gpu_parity_bench.py -m gpu -q -p no:cacheprovider -x > gpurun_out/s4l/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4l/tests.log
echo "c3:    $(timeout 120 python tools/gpu/kw_one.py 2>&1 | tail -1)"
echo "c3big: $(timeout 120 python tools/gpu/kw_one.py c3big 2>&1 | tail -1)"
for dbg in 2 4; do echo "dbg=$dbg: $(SKC_KAWASE_DBG=$dbg timeout 120 python tools/gpu/kw_one.py 2>&1 | tail -1)"; done
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline'].get('per_launch_ms', [])], 'bind', round(d['roofline']['binding']['frac'],3))
" $1; }
for c in c3 c3big; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4l/$c.json 2> gpurun_out/s4l/$c.err; show gpurun_out/s4l/$c.json
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kawase_sep -c 1 -o gpurun_out/s4l/kawase python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s4l/ncu_kw.log 2>&1; echo "ncu rc=$?"
