# round 2 call 4: Kawase HS 1/2/4, ncu HS=2, c1 bench (hoisted weights), all GPU test files
mkdir -p gpurun_out/c4
export SKC_CACHE_DIR=$(mktemp -d)
for hs in 2 4 1; do
  SKC_KAWASE_HS=$hs timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c4/bench_c3_hs$hs.json 2> gpurun_out/c4/bench_c3_hs$hs.err; echo "hs=$hs rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/c4/bench_c3_hs$hs.json').read().strip().splitlines()[-1]); print('hs $hs', round(d['value']), d['ms_per_step'])"
done
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c4/bench_c1.json 2> gpurun_out/c4/bench_c1.err; echo "c1 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c4/bench_c1.json').read().strip().splitlines()[-1]); print('c1', round(d['value']), d['ms_per_step'], d['roofline']['per_launch_ms'])"
SKC_KAWASE_HS=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:kawase -c 1 -o gpurun_out/c4/kawase_hs2 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/c4/ncu_kawase.log 2>&1; echo "ncu rc=$?"
for f in test_gpu_kawase test_gpu_round2 test_gpu_sv_fit test_gpu_parity_bench test_gpu_engine; do
  timeout 900 python -m pytest tests/$f.py -m gpu -q -p no:cacheprovider --durations=6 > gpurun_out/c4/$f.log 2>&1; echo "$f rc=$?"; tail -2 gpurun_out/c4/$f.log
done
