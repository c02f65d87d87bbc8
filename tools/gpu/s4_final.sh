# final verification of the tree: GPU tests (as the driver runs them), smoke, timed default bench, reference arm
mkdir -p gpurun_out/s4z
export SKC_CACHE_DIR=$(mktemp -d)
( time timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider ) > gpurun_out/s4z/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/s4z/gpu_tests.log
unset SKC_CACHE_DIR
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/s4z/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/s4z/smoke.log
( time timeout 900 python bench.py > gpurun_out/s4z/bench_default.json 2> gpurun_out/s4z/bench_default.err ) 2> gpurun_out/s4z/bench_time.txt; echo "bench rc=$?"; cat gpurun_out/s4z/bench_time.txt
( time timeout 600 python bench.py --impl reference > gpurun_out/s4z/bench_ref.json 2> gpurun_out/s4z/bench_ref.err ) 2> gpurun_out/s4z/ref_time.txt; echo "ref rc=$?"; cat gpurun_out/s4z/ref_time.txt
python - <<'PY'
import json
d = json.loads(open('gpurun_out/s4z/bench_default.json').read().strip().splitlines()[-1])
def show(n, x):
    print(n, round(x['value'], 1), x['unit'], 'ms', round(x['ms_per_step'], 4), 'e2e', round(x.get('e2e', {}).get('value', 0), 1),
          'per', [round(t, 3) for t in x['roofline'].get('per_launch_ms', [])],
          'bind', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in x['roofline'].get('binding', {}).items() if k in ('resource', 'frac')})
show('c1', d)
for k, v in d.get('other_configs', {}).items(): show(k, v)
PY
