# ncu --set full of config 3's launches with the final defaults (fp16 all-channel head, KR=3 tap layers, HWC-epilogue last layer)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python bench.py --config c3 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skc_sparse|layer_tap" -c 6 -o gpurun_out/prof88_c3 python bench.py --config c3 --frames 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu88.log 2>&1; echo "ncu rc=$?"
