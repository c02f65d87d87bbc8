# Final evidence pass (cold kernel cache at the default location): GPU tests, smoke, every config, reference arm, torchrun N=1, c1 launch list + full capture
# the reference arm, a torchrun N=1 launch, and the c1 ncu launch list.
mkdir -p gpurun_out/full
export XDG_CACHE_HOME=$(mktemp -d)  # cold kernel cache at the default location, as on a fresh box
SECONDS=0
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/full/pytest_gpu.log 2>&1; echo pytest_rc=$? suite_s=$SECONDS; tail -2 gpurun_out/full/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full/smoke.log 2>&1; tail -1 gpurun_out/full/smoke.log
for c in c1 c0 c2 c3 c3big c4; do
  python bench.py --config $c > gpurun_out/full/bench_$c.json 2> gpurun_out/full/bench_$c.err; echo "$c rc=$?"
done
python bench.py --impl reference --config c1 > gpurun_out/full/bench_ref_c1.json 2> gpurun_out/full/bench_ref_c1.err; echo "ref rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/full/bench_torchrun1.json 2> gpurun_out/full/bench_torchrun1.err; echo "torchrun rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/full/bench_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(d.get('value', 0), 1), d.get('unit'), 'e2e', round(d.get('e2e', {}).get('value', 0), 1),
              'roofline', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.get('roofline', {}).items() if k in ('frac', 'traffic')},
              'smem', round(d.get('roofline', {}).get('smem', {}).get('frac', 0), 3), 'cpu', d.get('cpu_baseline', {}).get('value'))
    except Exception as e:
        print(f, 'ERR', e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"layer|relayout|stencil" --clock-control none --csv --log-file gpurun_out/full/c1_launches.csv python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/full/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"skc_sparse" -c 4 -o gpurun_out/full/prof_c1_sparse python bench.py --config c1 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/full/ncu_full.log 2>&1; echo "ncu full rc=$?"
