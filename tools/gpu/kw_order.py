"""Diagnostic: the fused Kawase launch timed per call in one process, under
different allocation histories (c3 first / after a big freed allocation / c3big).
    python tools/gpu/kw_order.py [old]    # 'old' loads tools/gpu/tmp/libskc_old.so
"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_2512_04556_b200 import _native as nat, synth
if len(sys.argv) > 1 and sys.argv[1] == "old":
    nat.LIB_PATH = ROOT / "tools" / "gpu" / "tmp" / "libskc_old.so"
lib = nat.lib()
dev = torch.device("cuda", 0)
cpx = synth.kawase_complex()
taps = np.ascontiguousarray(cpx.taps()); lay = np.ascontiguousarray(cpx.layout, dtype=np.int32)

def run(tag, nf, h, w, fill, reps=8):
    fr = torch.empty((nf, h, w, 4), dtype=torch.float16, device=dev)
    if fill == "noise":
        for i in range(nf):
            fr[i].copy_(synth.value_noise_frame_device(h, w, 4, i, dev, dtype=torch.float16))
    elif fill == "rand":
        fr.copy_(torch.rand(fr.shape, device=dev, dtype=torch.float16))
    else:
        fr.zero_()
    out = torch.empty_like(fr)
    st = torch.cuda.current_stream()
    ts = []
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rc = lib.skc_chain_fwd(nat.ptr(fr), nat.SKC_F16, nat.ptr(out), nat.SKC_F16, nf, h, w, 4, nat.dbl(taps),
                               nat.ints(lay), lay.size, 0, nat.stream_ptr(st))
        assert rc == 0, nat.last_error()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(tag, "ptr %x" % fr.data_ptr(), "ms", [round(t, 3) for t in ts], flush=True)
    del fr, out
    torch.cuda.empty_cache()

run("c3 first noise", 32, 2160, 3840, "noise")
run("c3 zeros", 32, 2160, 3840, "zero")
run("c3 rand", 32, 2160, 3840, "rand")
big = torch.empty(6 << 30, dtype=torch.uint8, device=dev); del big; torch.cuda.empty_cache()
run("c3 after 6GB alloc/free", 32, 2160, 3840, "noise")
run("c3big noise", 1, 16384, 16384, "noise")
run("c3 16 frames", 16, 2160, 3840, "noise")
run("c3 31 frames", 31, 2160, 3840, "noise")
run("c3 again", 32, 2160, 3840, "noise")
