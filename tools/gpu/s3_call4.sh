# pair correctness (opt-in), head tile option, L4 source-level ncu
mkdir -p gpurun_out/s3d
export SKC_CACHE_DIR=$(mktemp -d)
timeout 300 python tools/gpu/pair_dbg.py > gpurun_out/s3d/dbg.log 2>&1; echo "dbg rc=$?"; grep -v tiles gpurun_out/s3d/dbg.log | head -20
timeout 600 python -m pytest tests/test_gpu_pair.py -m gpu -q -p no:cacheprovider > gpurun_out/s3d/test_pair.log 2>&1; echo "pair tests rc=$?"; tail -5 gpurun_out/s3d/test_pair.log
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline']['per_launch_ms']], 'bind', round(d['roofline']['binding']['frac'],3))
" $1; }
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3d/c1.json 2> gpurun_out/s3d/c1.err; echo "c1 rc=$?"; show gpurun_out/s3d/c1.json
SKC_SPARSE_HEAD_WY=1 timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3d/c1_hwy1.json 2>&1; show gpurun_out/s3d/c1_hwy1.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:skc_sparse_stencil -s 3 -c 1 -o gpurun_out/s3d/c1_l4 python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s3d/ncu_l4.log 2>&1; echo "ncu l4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:skc_sparse_stencil -s 0 -c 1 -o gpurun_out/s3d/c1_head python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s3d/ncu_head.log 2>&1; echo "ncu head rc=$?"
