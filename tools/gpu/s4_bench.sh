# default bench line + reference arm (refresh of profiles/bench_r02/bench_default.json)
mkdir -p gpurun_out/s4y
( time timeout 900 python bench.py > gpurun_out/s4y/bench_default.json 2> gpurun_out/s4y/bench_default.err ) 2> gpurun_out/s4y/bench_time.txt; echo "bench rc=$?"; cat gpurun_out/s4y/bench_time.txt
( time timeout 600 python bench.py --impl reference > gpurun_out/s4y/bench_ref.json 2> gpurun_out/s4y/bench_ref.err ) 2> gpurun_out/s4y/ref_time.txt; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/s4y/bench_default.json').read().strip().splitlines()[-1])
def show(n, x):
    print(n, round(x['value'], 1), x['unit'], 'ms', round(x['ms_per_step'], 4), 'steps', x['steps'], 'e2e', round(x.get('e2e', {}).get('value', 0), 1),
          'bind', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in x['roofline'].get('binding', {}).items() if k in ('resource', 'frac')})
show('c1', d)
for k, v in d.get('other_configs', {}).items(): show(k, v)
PY
