"""Diagnostic: config 3's fused Kawase launch, 4 timed calls (for ncu and for the SKC_KAWASE_DBG modes).
    python tools/gpu/kw_one.py [old] [c3big]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_2512_04556_b200 import _native as nat, synth
for a in sys.argv[1:]:
    if a == "old" or a.startswith("lib="):
        nat.LIB_PATH = ROOT / "tools" / "gpu" / "tmp" / ("libskc_%s.so" % (a[4:] if a.startswith("lib=") else "old"))
lib = nat.lib()
dev = torch.device("cuda", 0)
cpx = synth.kawase_complex()
taps = np.ascontiguousarray(cpx.taps()); lay = np.ascontiguousarray(cpx.layout, dtype=np.int32)
nf, h, w = (1, 16384, 16384) if "c3big" in sys.argv[1:] else (32, 2160, 3840)
fr = torch.rand((nf, h, w, 4), device=dev, dtype=torch.float16)
out = torch.empty_like(fr)
st = torch.cuda.current_stream()
ts = []
for r in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    rc = lib.skc_chain_fwd(nat.ptr(fr), nat.SKC_F16, nat.ptr(out), nat.SKC_F16, nf, h, w, 4, nat.dbl(taps),
                           nat.ints(lay), lay.size, 0, nat.stream_ptr(st))
    assert rc == 0, nat.last_error()
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(sys.argv[1:], "ms", [round(t, 3) for t in ts], flush=True)
