# defaults after call 27 (cluster epilogue opt-in, KR=5 for <=16-tap layers); ncu of the stencil layers
mkdir -p gpurun_out
run() { name=$1; shift; env "$@" python bench.py --no-e2e --no-cpu $BARGS > gpurun_out/b28_$name.json 2> gpurun_out/b28_$name.err; echo "$name rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/b28_$name.json').read().strip().splitlines()[-1]);print(round(d['value'],1), [round(x,3) for x in d['roofline']['per_launch_ms']])")"; }
BARGS="--config c1"; run c1 SKC_X=0
BARGS="--config c3"; run c3 SKC_X=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"stencil" -c 2 -o gpurun_out/prof28_stencil python bench.py --config c1 --steps 1 --warmup 0 --frames 8 --no-e2e --no-cpu > gpurun_out/ncu28a.log 2>&1; echo ncu_a rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"layer_tap" -c 1 -o gpurun_out/prof28_c3tap python bench.py --config c3 --steps 1 --warmup 0 --frames 8 --no-e2e --no-cpu > gpurun_out/ncu28b.log 2>&1; echo ncu_b rc=$?
