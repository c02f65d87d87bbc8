# round 2 call 7: C1 generated stencils, odd-position end pairing (SKC_SPARSE_F2=3) vs default
mkdir -p gpurun_out/c7
export SKC_CACHE_DIR=$(mktemp -d)
for m in 3 1; do
  SKC_SPARSE_F2=$m timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/c7/bench_c1_f$m.json 2> gpurun_out/c7/bench_c1_f$m.err; echo "f2=$m rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/c7/bench_c1_f$m.json').read().strip().splitlines()[-1]); print('f2 $m', round(d['value']), round(d['ms_per_step'],3), [round(x,3) for x in d['roofline']['per_launch_ms']])"
done
SKC_SPARSE_F2=3 timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider -k "sparse_stencil or c1_frame or golden or stencil_variants or hwc_epilogue" > gpurun_out/c7/t_engine_f3.log 2>&1; echo "engine f3 rc=$?"; tail -1 gpurun_out/c7/t_engine_f3.log
timeout 300 python tools/bench_pst.py > gpurun_out/c7/pst.json 2> gpurun_out/c7/pst.err; echo "pst rc=$?"; cat gpurun_out/c7/pst.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"skc_|layer_|relayout|stencil" --log-file gpurun_out/c7/launches_c1.csv python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/c7/ncu_l_c1.log 2>&1; echo "ncu list c1 rc=$?"
