# small-launch policy (wide layers prefer the generated stencil, KR 1 head): c0 bench + engine tests
mkdir -p gpurun_out/s4p
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,4) for t in d['roofline'].get('per_launch_ms', [])], 'e2e', d.get('e2e',{}).get('value'))
" $1; }
timeout 300 python bench.py --config c0 --steps 30 --warmup 5 --no-cpu --no-others > gpurun_out/s4p/c0.json 2> gpurun_out/s4p/c0.err; show gpurun_out/s4p/c0.json
SKC_SPARSE_SMALL_PREFER=0 SKC_SPARSE_SMALL_KR=0 timeout 300 python bench.py --config c0 --steps 30 --warmup 5 --no-cpu --no-others > gpurun_out/s4p/c0_old.json 2> gpurun_out/s4p/c0_old.err; show gpurun_out/s4p/c0_old.json
( time timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_pair.py tests/test_gpu_parity_bench.py -x -q -m gpu -p no:cacheprovider --durations=5 ) > gpurun_out/s4p/tests.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/s4p/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4p/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4p/smoke.log
