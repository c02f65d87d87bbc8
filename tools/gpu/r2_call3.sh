# round 2 call 3: Kawase HS=1 vs HS=2, ncu of HS=2, then GPU test files
mkdir -p gpurun_out/c3
export SKC_CACHE_DIR=$(mktemp -d)
for hs in 2 1; do
  SKC_KAWASE_HS=$hs timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c3/bench_c3_hs$hs.json 2> gpurun_out/c3/bench_c3_hs$hs.err; echo "hs=$hs rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/c3/bench_c3_hs$hs.json').read().strip().splitlines()[-1]); print('hs $hs', round(d['value']), d['ms_per_step'])"
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:kawase -c 1 -o gpurun_out/c3/kawase_hs2 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/c3/ncu_kawase.log 2>&1; echo "ncu rc=$?"
timeout 600 python -m pytest tests/test_gpu_kawase.py tests/test_gpu_round2.py -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/c3/t_kawase_round2.log 2>&1; echo "kawase+round2 rc=$?"; tail -3 gpurun_out/c3/t_kawase_round2.log
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/c3/t_engine.log 2>&1; echo "engine rc=$?"; tail -3 gpurun_out/c3/t_engine.log
timeout 600 python -m pytest tests/test_gpu_sv_fit.py tests/test_gpu_parity_bench.py -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/c3/t_svfit_parity.log 2>&1; echo "svfit+parity rc=$?"; tail -3 gpurun_out/c3/t_svfit_parity.log
