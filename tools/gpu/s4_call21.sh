mkdir -p gpurun_out/s4u
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'e2e', round(d.get('e2e',{}).get('value',0),1))
" $1; }
for v in 0 1 0 1; do
  SKC_PDL=$v timeout 300 python bench.py --config c0 --steps 30 --warmup 5 --no-cpu --no-others > gpurun_out/s4u/c0_pdl$v.json 2> gpurun_out/s4u/c0_pdl$v.err; show gpurun_out/s4u/c0_pdl$v.json
done
SKC_PDL=1 timeout 900 python -m pytest tests/test_gpu_engine.py -q -m gpu -p no:cacheprovider -x -k "not sparse_stencil_path and not fused_chain and not io_policies and not stencil_variants and not hwc_epilogue and not half_intermediates" > gpurun_out/s4u/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4u/tests.log
SKC_PDL=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4u/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4u/smoke.log
