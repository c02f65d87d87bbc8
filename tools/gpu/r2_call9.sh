# round 2 call 9: config 0 -- whole-chain timing, half-height tiles for small grids
mkdir -p gpurun_out/c9
export SKC_CACHE_DIR=$(mktemp -d)
for sm in 1 0; do
  SKC_SPARSE_SMALL=$sm timeout 300 python bench.py --config c0 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c9/bench_c0_s$sm.json 2> gpurun_out/c9/bench_c0_s$sm.err; echo "small=$sm rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/c9/bench_c0_s$sm.json').read().strip().splitlines()[-1]); print('small $sm', round(d['value']), d['ms_per_step'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"skc_|layer_|relayout|stencil" --log-file gpurun_out/c9/launches_c0.csv python bench.py --config c0 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/c9/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider -k "c0 or ragged or sparse_stencil or golden or known or chain_io or jit or pinned" > gpurun_out/c9/t_engine.log 2>&1; echo "engine rc=$?"; tail -1 gpurun_out/c9/t_engine.log
