# fit: loss fused into the last forward pass (+ summed-area table for the outside-box loss)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sv_fit.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
SKC_FIT_PROF=1 python bench.py --config c4 --fit-steps 300 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/b41_prof.json 2> gpurun_out/b41_prof.err; echo prof rc=$?; grep "skc fit prof" gpurun_out/b41_prof.err | tail -1
for i in 1 2; do python bench.py --config c4 --no-e2e --no-cpu > gpurun_out/b41_c4_$i.json 2> gpurun_out/b41_c4.err; echo c4 rc=$?; python -c "import json;d=json.loads(open('gpurun_out/b41_c4_$i.json').read().strip().splitlines()[-1]);print(d['value'])"; done
