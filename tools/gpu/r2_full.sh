# Round 2 evidence pass: GPU tests, smoke, every config's bench line, reference arm, launch lists.
mkdir -p gpurun_out/full
export SKC_CACHE_DIR=$(mktemp -d)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/full/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/full/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1; tail -1 gpurun_out/full/smoke.log
for c in c1 c0 c2 c3 c3big c4; do
  timeout 600 python bench.py --config $c > gpurun_out/full/bench_$c.json 2> gpurun_out/full/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference --config c1 --steps 2 --warmup 1 > gpurun_out/full/bench_ref_c1.json 2> gpurun_out/full/bench_ref_c1.err; echo "ref rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/full/bench_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(d.get('value', 0), 1), d.get('unit'), 'ms', d.get('ms_per_step'), 'e2e', round(d.get('e2e', {}).get('value', 0), 1),
              'roofline', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.get('roofline', {}).items() if k in ('frac', 'bound')},
              'cpu', d.get('cpu_baseline', {}).get('value'))
    except Exception as e:
        print(f, 'ERR', e)
PY
for c in c1 c3; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/full/${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/full/ncu_launch_$c.log 2>&1; echo "ncu $c rc=$?"
done
