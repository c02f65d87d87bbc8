# Kawase: V chunks held back until the H warps finished the next chunk's warm-up (SKC_KAWASE_VDELAY)
mkdir -p gpurun_out/s4n
export SKC_CACHE_DIR=$(mktemp -d)
for vd in 0 1 0 1; do
  echo "vdelay=$vd c3:    $(SKC_KAWASE_VDELAY=$vd timeout 120 python tools/gpu/kw_one.py 2>&1 | tail -1)"
done
echo "vdelay=1 c3big: $(SKC_KAWASE_VDELAY=1 timeout 120 python tools/gpu/kw_one.py c3big 2>&1 | tail -1)"
timeout 900 python -m pytest tests/test_gpu_kawase.py -m gpu -q -p no:cacheprovider -x > gpurun_out/s4n/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4n/tests.log
SKC_KAWASE_VDELAY=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:kawase_sep -c 1 -o gpurun_out/s4n/kawase_vd python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s4n/ncu_kw.log 2>&1; echo "ncu rc=$?"
