mkdir -p gpurun_out/s4c
timeout 300 python tools/gpu/kw_order.py > gpurun_out/s4c/new.log 2>&1; echo "new rc=$?"; cat gpurun_out/s4c/new.log
timeout 300 python tools/gpu/kw_order.py old > gpurun_out/s4c/old.log 2>&1; echo "old rc=$?"; cat gpurun_out/s4c/old.log
SKC_KAWASE_PEEL=0 timeout 300 python tools/gpu/kw_order.py > gpurun_out/s4c/new_nopeel.log 2>&1; echo "new nopeel rc=$?"; cat gpurun_out/s4c/new_nopeel.log
