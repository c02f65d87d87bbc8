# round 2 call 2: GPU tests file by file (durations), smoke, kawase ncu --set full
mkdir -p gpurun_out/c2
export SKC_CACHE_DIR=$(mktemp -d)
for f in test_gpu_round2 test_gpu_parity_bench test_gpu_kawase test_gpu_sv_fit test_gpu_engine; do
  timeout 900 python -m pytest tests/$f.py -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/c2/$f.log 2>&1; echo "$f rc=$?"; tail -3 gpurun_out/c2/$f.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c2/smoke.log 2>&1; tail -1 gpurun_out/c2/smoke.log
SKC_JIT=sync timeout 600 ncu --set full --import-source on --clock-control none -k regex:kawase -c 1 -o gpurun_out/c2/kawase_full python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/c2/ncu_kawase.log 2>&1; echo "ncu rc=$?"
