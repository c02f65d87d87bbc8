mkdir -p gpurun_out/s4s
export SKC_CACHE_DIR=$(mktemp -d)
timeout 600 python -m pytest tests/test_gpu_engine.py -q -m gpu -p no:cacheprovider -k "pinned" > gpurun_out/s4s/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/s4s/tests.log
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'e2e', d.get('e2e',{}))
" $1; }
timeout 300 python bench.py --config c3big --steps 5 --warmup 3 --no-cpu --no-others > gpurun_out/s4s/c3big.json 2> gpurun_out/s4s/c3big.err; show gpurun_out/s4s/c3big.json; tail -3 gpurun_out/s4s/c3big.err
