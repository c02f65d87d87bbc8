# streaming fused head pair: parity, c1 bench variants, ncu
mkdir -p gpurun_out/s3c
export SKC_CACHE_DIR=$(mktemp -d)
timeout 300 python tools/gpu/pair_dbg.py > gpurun_out/s3c/dbg.log 2>&1; echo "dbg rc=$?"; cat gpurun_out/s3c/dbg.log | head -30
timeout 600 python -m pytest tests/test_gpu_pair.py -m gpu -q -p no:cacheprovider -x > gpurun_out/s3c/test_pair.log 2>&1; echo "pair tests rc=$?"; tail -5 gpurun_out/s3c/test_pair.log
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline']['per_launch_ms']], 'bind', round(d['roofline']['binding']['frac'],3))
" $1; }
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3c/c1.json 2> gpurun_out/s3c/c1.err; echo "c1 rc=$?"; show gpurun_out/s3c/c1.json; tail -3 gpurun_out/s3c/c1.err
SKC_PAIR_MINB=2 timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3c/c1_m2.json 2>&1; show gpurun_out/s3c/c1_m2.json
SKC_PAIR_KR=5 timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s3c/c1_kr5.json 2>&1; show gpurun_out/s3c/c1_kr5.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:skc_sparse_pair -c 1 -o gpurun_out/s3c/c1_pair python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s3c/ncu_pair.log 2>&1; echo "ncu pair rc=$?"
