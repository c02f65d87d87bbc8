# head WY=1 default + streamlined HWC epilogue; F2=3 A/B; parity
mkdir -p gpurun_out/s3e
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline']['per_launch_ms']], 'bind', round(d['roofline']['binding']['frac'],3))
" $1; }
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3e/c1.json 2> gpurun_out/s3e/c1.err; echo "c1 rc=$?"; show gpurun_out/s3e/c1.json
SKC_SPARSE_F2=3 timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3e/c1_f23.json 2>&1; show gpurun_out/s3e/c1_f23.json
SKC_SPARSE_HEAD_WY=2 timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3e/c1_hwy2.json 2>&1; show gpurun_out/s3e/c1_hwy2.json
timeout 300 python bench.py --config c0 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/s3e/c0.json 2>&1; show gpurun_out/s3e/c0.json
timeout 900 python -m pytest tests/test_gpu_parity_bench.py tests/test_gpu_pair.py -m gpu -q -p no:cacheprovider > gpurun_out/s3e/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3e/tests.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:skc_sparse_stencil -s 3 -c 1 -o gpurun_out/s3e/c1_l4 python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s3e/ncu_l4.log 2>&1; echo "ncu l4 rc=$?"
