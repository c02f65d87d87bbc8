# fit A/B: box loss + SAT vs whole-canvas loss; small-box correlate split
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sv_fit.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
for v in 1 0 1 0; do SKC_FIT_SAT=$v python bench.py --config c4 --no-e2e --no-cpu > gpurun_out/b43_c4_$v.json 2> gpurun_out/b43_c4.err; echo "sat=$v $(python -c "import json;d=json.loads(open('gpurun_out/b43_c4_$v.json').read().strip().splitlines()[-1]);print(d['value'])")"; done
SKC_FIT_PROF=1 python bench.py --config c4 --fit-steps 300 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/b43_prof.json 2> gpurun_out/b43_prof.err; grep "skc fit prof" gpurun_out/b43_prof.err | tail -1
