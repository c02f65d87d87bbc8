mkdir -p gpurun_out/s4r
export SKC_CACHE_DIR=$(mktemp -d)
timeout 600 python -m pytest tests/test_gpu_sv_fit.py -q -m gpu -p no:cacheprovider -k "sv_" > gpurun_out/s4r/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/s4r/tests.log
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'e2e', d.get('e2e',{}))
" $1; }
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --no-others > gpurun_out/s4r/c2.json 2> gpurun_out/s4r/c2.err; show gpurun_out/s4r/c2.json; tail -3 gpurun_out/s4r/c2.err
python - <<'PY'
import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2512_04556_b200 as skc
from paper_2512_04556_b200 import synth
basis = synth.c2_basis()
img = torch.from_numpy(synth.c1_frame(0)).pin_memory(); pm = torch.from_numpy(synth.c2_pmap()).pin_memory(); out = torch.empty_like(img).pin_memory()
for strips in (1, 2, 3, 4, 6, 8):
    for _ in range(2): skc.sv_filter(img, basis, pm, out=out, strips=strips)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): skc.sv_filter(img, basis, pm, out=out, strips=strips)
    torch.cuda.synchronize(); print('strips', strips, 'ms', round((time.perf_counter() - t) / 5 * 1e3, 3))
PY
