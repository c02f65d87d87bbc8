# fused head pair: parity tests, c1/c0 bench with and without the pair, SASS/launch list
mkdir -p gpurun_out/s3b
export SKC_CACHE_DIR=$(mktemp -d)
timeout 600 python -m pytest tests/test_gpu_pair.py tests/test_gpu_parity_bench.py::test_c1_bench_frames_0_and_63 -m gpu -q -p no:cacheprovider -x > gpurun_out/s3b/test_pair.log 2>&1; echo "pair tests rc=$?"; tail -15 gpurun_out/s3b/test_pair.log
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline']['per_launch_ms']], 'bind', round(d['roofline']['binding']['frac'],3))
" $1; }
for kr in 3 5; do
  SKC_PAIR_KR=$kr timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3b/c1_kr$kr.json 2> gpurun_out/s3b/c1_kr$kr.err; echo "c1 kr$kr rc=$?"; show gpurun_out/s3b/c1_kr$kr.json
done
SKC_PAIR=0 timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3b/c1_nopair.json 2>&1; show gpurun_out/s3b/c1_nopair.json
timeout 300 python bench.py --config c0 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/s3b/c0.json 2>&1; show gpurun_out/s3b/c0.json
SKC_PAIR=0 timeout 300 python bench.py --config c0 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/s3b/c0_nopair.json 2>&1; show gpurun_out/s3b/c0_nopair.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:skc_sparse_pair -c 1 -o gpurun_out/s3b/c1_pair python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s3b/ncu_pair.log 2>&1; echo "ncu pair rc=$?"
