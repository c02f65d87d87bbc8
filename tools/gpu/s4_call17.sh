mkdir -p gpurun_out/s4q
export SKC_CACHE_DIR=$(mktemp -d)
timeout 600 python -m pytest tests/test_gpu_engine.py -q -m gpu -p no:cacheprovider -k "pinned or batch" > gpurun_out/s4q/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4q/tests.log
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'e2e', d.get('e2e',{}))
" $1; }
timeout 300 python bench.py --config c0 --steps 30 --warmup 5 --no-cpu --no-others > gpurun_out/s4q/c0.json 2> gpurun_out/s4q/c0.err; show gpurun_out/s4q/c0.json
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --no-others > gpurun_out/s4q/c2.json 2> gpurun_out/s4q/c2.err; show gpurun_out/s4q/c2.json
