mkdir -p gpurun_out/s4aa
export SKC_CACHE_DIR=$(mktemp -d)
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_sv_fit.py -q -m gpu -p no:cacheprovider -k "pinned or strips" > gpurun_out/s4aa/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4aa/tests.log
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3))
" $1; }
for c in c2 c0 c3big c1; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-others > gpurun_out/s4aa/$c.json 2> gpurun_out/s4aa/$c.err; show gpurun_out/s4aa/$c.json
done
