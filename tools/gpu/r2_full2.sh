# round 2 evidence pass: GPU tests, smoke, default bench line (c1 + other configs), reference arm,
# ncu launch lists (DRAM bytes per launch) for every config, --set full of the dominant kernels
mkdir -p gpurun_out/e2
export SKC_CACHE_DIR=$(mktemp -d)
for f in test_gpu_kawase test_gpu_round2 test_gpu_sv_fit test_gpu_parity_bench test_gpu_engine; do
  timeout 900 python -m pytest tests/$f.py -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/e2/$f.log 2>&1; echo "$f rc=$?"; tail -1 gpurun_out/e2/$f.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e2/smoke.log 2>&1; tail -1 gpurun_out/e2/smoke.log
timeout 900 python bench.py > gpurun_out/e2/bench_default.json 2> gpurun_out/e2/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/e2/bench_ref.json 2> gpurun_out/e2/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/e2/bench_default.json').read().strip().splitlines()[-1])
def show(n, x):
    print(n, round(x['value'], 1), x['unit'], 'ms', round(x['ms_per_step'], 4), 'e2e', round(x.get('e2e', {}).get('value', 0), 1),
          'bind', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in x['roofline'].get('binding', {}).items() if k in ('resource', 'frac', 'achieved')},
          'cpu', x.get('cpu_baseline', {}).get('value'))
show('c1', d)
for k, v in d.get('other_configs', {}).items(): show(k, v)
PY
for c in c1 c0 c2 c3 c3big; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/e2/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/e2/ncu_l_$c.log 2>&1; echo "ncu list $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:fit_kernel --log-file gpurun_out/e2/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --fit-steps 300 --no-e2e --no-cpu --no-others > gpurun_out/e2/ncu_l_c4.log 2>&1; echo "ncu list c4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:skc_sparse_stencil -s 3 -c 1 -o gpurun_out/e2/c1_layer4 python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/e2/ncu_f_c1.log 2>&1; echo "ncu full c1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sv_tile -c 1 -o gpurun_out/e2/c2_sv python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/e2/ncu_f_c2.log 2>&1; echo "ncu full c2 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fit_kernel -c 1 -o gpurun_out/e2/c4_fit python bench.py --config c4 --steps 1 --warmup 1 --fit-steps 200 --no-e2e --no-cpu --no-others > gpurun_out/e2/ncu_f_c4.log 2>&1; echo "ncu full c4 rc=$?"
