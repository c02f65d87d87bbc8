"""Bring-up probe for the Kawase kernel: run one small call per debug mode in a subprocess."""
import os, subprocess, sys
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2512_04556_b200 as skc
from paper_2512_04556_b200 import synth
cpx = synth.kawase_complex(int(sys.argv[1]))
img = np.random.default_rng(0).random((int(sys.argv[2]), int(sys.argv[3]), 4)).astype(np.float16)
out = skc.apply_complex(torch.from_numpy(img).cuda(), cpx)
torch.cuda.synchronize()
print("ok", float(out.float().abs().max()))
'''
for L in (6, 2):
    for dbg in ("7", "6", "5", "3", "1", "4", "2", "0"):
        for shp in (("64", "256"), ("300", "600")):
            env = dict(os.environ, SKC_KAWASE_DBG=dbg, CUDA_LAUNCH_BLOCKING="1")
            r = subprocess.run([sys.executable, "-c", code, str(L), *shp], env=env, capture_output=True, text=True, timeout=120)
            tail = (r.stdout + r.stderr).strip().splitlines()
            print(f"L={L} dbg={dbg} shape={shp}: rc={r.returncode} {tail[-1] if tail else ''}", flush=True)
