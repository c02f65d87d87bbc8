# fit kernel: window loads as LDS from the shared arena
mkdir -p gpurun_out/s4m
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4))
" $1; }
timeout 600 python bench.py --config c4 --steps 3 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s4m/c4.json 2> gpurun_out/s4m/c4.err; show gpurun_out/s4m/c4.json
timeout 1200 python -m pytest tests/test_gpu_sv_fit.py tests/test_gpu_parity_bench.py tests/test_gpu_round2.py -m gpu -q -p no:cacheprovider > gpurun_out/s4m/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4m/tests.log
timeout 300 python tools/bench_pst.py > gpurun_out/s4m/pst.log 2>&1; tail -3 gpurun_out/s4m/pst.log
