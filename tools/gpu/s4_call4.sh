mkdir -p gpurun_out/s4d
for dbg in 0 2 4 6; do
  for v in "" old; do
    echo "dbg=$dbg $v: $(SKC_KAWASE_DBG=$dbg timeout 120 python tools/gpu/kw_one.py $v 2>&1 | tail -1)"
  done
done
echo "nopeel: $(SKC_KAWASE_PEEL=0 timeout 120 python tools/gpu/kw_one.py 2>&1 | tail -1)"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:kawase_sep -s 2 -c 1 -o gpurun_out/s4d/kw_old python tools/gpu/kw_one.py old > gpurun_out/s4d/ncu_old.log 2>&1; echo "ncu old rc=$?"
SKC_KAWASE_PEEL=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:kawase_sep -s 2 -c 1 -o gpurun_out/s4d/kw_new_nopeel python tools/gpu/kw_one.py > gpurun_out/s4d/ncu_new.log 2>&1; echo "ncu new rc=$?"
