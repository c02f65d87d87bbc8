# round 2 call 8: fit kernel with per-tap unchecked windows on edge blocks
mkdir -p gpurun_out/c8
export SKC_CACHE_DIR=$(mktemp -d)
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c8/bench_c4.json 2> gpurun_out/c8/bench_c4.err; echo "c4 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c8/bench_c4.json').read().strip().splitlines()[-1]); print('c4', round(d['value']), d['ms_per_step'])"
timeout 900 python -m pytest tests/test_gpu_sv_fit.py tests/test_gpu_parity_bench.py tests/test_gpu_round2.py -m gpu -q -p no:cacheprovider -k "fit or backward or adam or pst or basis or c4" > gpurun_out/c8/t_fit.log 2>&1; echo "fit tests rc=$?"; tail -2 gpurun_out/c8/t_fit.log

