show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), 'ms', round(d['ms_per_step'],4))
" $1; }
mkdir -p gpurun_out/s4x
timeout 300 python bench.py --config c0 --steps 5 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4x/a.json 2>/dev/null; show gpurun_out/s4x/a.json
timeout 300 python bench.py --config c0 --steps 30 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4x/b.json 2>/dev/null; show gpurun_out/s4x/b.json
timeout 300 python bench.py --config c0 --steps 5 --warmup 3 --no-cpu --no-others > gpurun_out/s4x/c.json 2>/dev/null; show gpurun_out/s4x/c.json
timeout 300 python bench.py --config c0 --steps 5 --warmup 3 --no-others > gpurun_out/s4x/d.json 2>/dev/null; show gpurun_out/s4x/d.json
python - <<'PY'
import sys, argparse, json
sys.argv = ['bench.py']
sys.path.insert(0, '.')
import bench, torch
args = bench.parse()
dev = torch.device('cuda', 0)
from paper_2512_04556_b200 import _native as nat
nat.lib(); nat.set_jit_mode(True)
for cfg_seq in (['c2', 'c0'], ['c0']):
    for c in cfg_seq:
        sub = argparse.Namespace(**vars(args)); sub.config = c
        w = bench.make_workload(sub, dev, 0, 1)
        l = bench.measure(w, sub, 5, 3, 0, 1, dev, 0, with_e2e=False)
        print(cfg_seq, c, round(l['value'], 1), round(l['ms_per_step'], 4))
        del w; torch.cuda.empty_cache()
PY
