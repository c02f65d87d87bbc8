# fit: tap-split gather passes for small boxes
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sv_fit.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py --config c4 --no-e2e --no-cpu > gpurun_out/b39_c4.json 2> gpurun_out/b39_c4.err; echo c4 rc=$?; python -c "import json;d=json.loads(open('gpurun_out/b39_c4.json').read().strip().splitlines()[-1]);print(d['value'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fit_kernel" -c 1 -o gpurun_out/prof39_fit python bench.py --config c4 --fit-steps 300 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu39.log 2>&1; echo ncu rc=$?
