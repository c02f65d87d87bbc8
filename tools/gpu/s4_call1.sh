# session 4: HEAD health check -- all GPU tests, smoke, default bench line, reference arm
mkdir -p gpurun_out/s4a
export SKC_CACHE_DIR=$(mktemp -d)
for f in test_gpu_kawase test_gpu_round2 test_gpu_sv_fit test_gpu_parity_bench test_gpu_engine test_gpu_pair; do
  timeout 900 python -m pytest tests/$f.py -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/s4a/$f.log 2>&1; echo "$f rc=$?"; tail -1 gpurun_out/s4a/$f.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4a/smoke.log
timeout 900 python bench.py > gpurun_out/s4a/bench_default.json 2> gpurun_out/s4a/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/s4a/bench_ref.json 2> gpurun_out/s4a/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/s4a/bench_default.json').read().strip().splitlines()[-1])
def show(n, x):
    print(n, round(x['value'], 1), x['unit'], 'ms', round(x['ms_per_step'], 4), 'e2e', round(x.get('e2e', {}).get('value', 0), 1),
          'per', [round(t, 3) for t in x['roofline'].get('per_launch_ms', [])],
          'bind', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in x['roofline'].get('binding', {}).items() if k in ('resource', 'frac', 'achieved')},
          'cpu', x.get('cpu_baseline', {}).get('value'))
show('c1', d)
for k, v in d.get('other_configs', {}).items(): show(k, v)
PY
