# fit phase split (SKC_FIT_PROF) + c4 bench
mkdir -p gpurun_out
SKC_FIT_PROF=1 python bench.py --config c4 --fit-steps 300 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/b40_prof.json 2> gpurun_out/b40_prof.err; echo prof rc=$?; grep "skc fit prof" gpurun_out/b40_prof.err | tail -2
python bench.py --config c4 --no-e2e --no-cpu > gpurun_out/b40_c4.json 2> gpurun_out/b40_c4.err; echo c4 rc=$?; python -c "import json;d=json.loads(open('gpurun_out/b40_c4.json').read().strip().splitlines()[-1]);print(d['value'])"
