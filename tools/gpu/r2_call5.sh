# round 2 call 5: looped Kawase bodies: tests + HS sweep + ncu
mkdir -p gpurun_out/c5
export SKC_CACHE_DIR=$(mktemp -d)
timeout 300 python -m pytest tests/test_gpu_kawase.py -m gpu -q -p no:cacheprovider -x > gpurun_out/c5/t_kawase.log 2>&1; echo "kawase tests rc=$?"; tail -2 gpurun_out/c5/t_kawase.log
for hs in 2 4 1; do
  SKC_KAWASE_HS=$hs timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c5/bench_c3_hs$hs.json 2> gpurun_out/c5/bench_c3_hs$hs.err; echo "hs=$hs rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/c5/bench_c3_hs$hs.json').read().strip().splitlines()[-1]); print('hs $hs', round(d['value']), d['ms_per_step'])"
done
for hs in 2 4; do
SKC_KAWASE_HS=$hs timeout 300 ncu --set full --import-source on --clock-control none -k regex:kawase -c 1 -o gpurun_out/c5/kawase_hs$hs python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/c5/ncu_kawase_hs$hs.log 2>&1; echo "ncu rc=$?"
done
