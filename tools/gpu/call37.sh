# fit kernel capture (config 4 at 300 steps)
mkdir -p gpurun_out
python bench.py --config c4 --fit-steps 300 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b37_c4.json 2> gpurun_out/b37_c4.err; echo c4 rc=$?; tail -c 300 gpurun_out/b37_c4.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fit_kernel" -c 1 -o gpurun_out/prof37_fit python bench.py --config c4 --fit-steps 300 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu37.log 2>&1; echo ncu rc=$?
