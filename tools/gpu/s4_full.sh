# round 2 / session 4 evidence pass: GPU tests, smoke, default bench line (c1 + other configs), reference arm,
# ncu launch lists (DRAM bytes per launch) for every config, --set full of the dominant kernels
mkdir -p gpurun_out/s4f
export SKC_CACHE_DIR=$(mktemp -d)
( time timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider --durations=8 ) > gpurun_out/s4f/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/s4f/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4f/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4f/smoke.log
timeout 900 python bench.py > gpurun_out/s4f/bench_default.json 2> gpurun_out/s4f/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/s4f/bench_ref.json 2> gpurun_out/s4f/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/s4f/bench_default.json').read().strip().splitlines()[-1])
def show(n, x):
    print(n, round(x['value'], 1), x['unit'], 'ms', round(x['ms_per_step'], 4), 'e2e', round(x.get('e2e', {}).get('value', 0), 1),
          'per', [round(t, 3) for t in x['roofline'].get('per_launch_ms', [])],
          'bind', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in x['roofline'].get('binding', {}).items() if k in ('resource', 'frac', 'achieved')},
          'cpu', x.get('cpu_baseline', {}).get('value'))
show('c1', d)
for k, v in d.get('other_configs', {}).items(): show(k, v)
r = json.loads(open('gpurun_out/s4f/bench_ref.json').read().strip().splitlines()[-1])
print('ref', r['value'], r['unit'], r['cpu_baseline']['cores'])
PY
for c in c1 c0 c2 c3 c3big; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s4f/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s4f/ncu_l_$c.log 2>&1; echo "ncu list $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:fit_kernel --log-file gpurun_out/s4f/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --fit-steps 300 --no-e2e --no-cpu --no-others > gpurun_out/s4f/ncu_l_c4.log 2>&1; echo "ncu list c4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:skc_sparse_stencil -c 4 -o gpurun_out/s4f/c1_layers python bench.py --config c1 --steps 1 --warmup 0 --no-e2e --no-cpu --no-others > gpurun_out/s4f/ncu_f_c1.log 2>&1; echo "ncu full c1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fit_kernel -c 1 -o gpurun_out/s4f/c4_fit python bench.py --config c4 --steps 1 --warmup 1 --fit-steps 200 --no-e2e --no-cpu --no-others > gpurun_out/s4f/ncu_f_c4.log 2>&1; echo "ncu full c4 rc=$?"
