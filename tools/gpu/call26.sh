set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py --config c1 > gpurun_out/b26_c1.json 2> gpurun_out/b26_c1.err; echo c1 rc=$?
SKC_STENCIL_ROLL=0 python bench.py --config c1 --no-e2e --no-cpu > gpurun_out/b26_c1_noroll.json 2>&1; echo c1nr rc=$?
python bench.py --config c3 --no-cpu > gpurun_out/b26_c3.json 2> gpurun_out/b26_c3.err; echo c3 rc=$?
python bench.py --config c0 --no-cpu > gpurun_out/b26_c0.json 2> gpurun_out/b26_c0.err; echo c0 rc=$?
python -c "import json;[print(n, json.loads(open(f'gpurun_out/b26_{n}.json').read().strip().splitlines()[-1])['value'], json.loads(open(f'gpurun_out/b26_{n}.json').read().strip().splitlines()[-1])['roofline']['per_launch_ms']) for n in ('c1','c1_noroll','c3','c0')]"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"layer|relayout|stencil|fused" --clock-control none --csv --log-file gpurun_out/c1_launches26.csv python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu26a.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"layer|relayout|stencil|fused" --clock-control none --csv --log-file gpurun_out/c3_launches26.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu26b.log 2>&1; echo ncu2 rc=$?
