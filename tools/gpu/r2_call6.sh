# round 2 call 6: Kawase with suspend-hint waits + pointer-stepped stores
mkdir -p gpurun_out/c6
export SKC_CACHE_DIR=$(mktemp -d)
timeout 300 python -m pytest tests/test_gpu_kawase.py -m gpu -q -p no:cacheprovider -x > gpurun_out/c6/t_kawase.log 2>&1; echo "kawase tests rc=$?"; tail -1 gpurun_out/c6/t_kawase.log
for c in c3 c3big; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c6/bench_$c.json 2> gpurun_out/c6/bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/c6/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), d['ms_per_step'], d['roofline']['binding'])"
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:kawase -c 1 -o gpurun_out/c6/kawase python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/c6/ncu_kawase.log 2>&1; echo "ncu rc=$?"
