# c3 4-tap layer source-level capture
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"layer_tap" -s 1 -c 1 -o gpurun_out/prof52_c3tap python bench.py --config c3 --steps 1 --warmup 0 --frames 8 --no-e2e --no-cpu > gpurun_out/ncu52.log 2>&1; echo ncu rc=$?
