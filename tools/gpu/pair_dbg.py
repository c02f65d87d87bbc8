"""Debug the fused pair on config 0 shapes: which tiles disagree with the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
os.environ.setdefault("SKC_JIT", "sync")
os.environ["SKC_PAIR_SMALL"] = "1"
os.environ["SKC_PAIR"] = "1"
from oracle import oracle as orc
from paper_2512_04556_b200 import _native as nat, synth

orc.set_threads(os.cpu_count() or 1)
lib = nat.lib()
for cfg, shape, bnd in (("c0", (1, 512, 512, 3), 1), ("c0", (1, 512, 512, 3), 0), ("c1", (1, 512, 512, 3), 1),
                        ("c0", (1, 200, 333, 3), 1), ("c0", (1, 97, 130, 3), 1)):
    cpx = synth.c1_complex() if cfg == "c1" else synth.c0_complex()
    t0, t1 = (np.ascontiguousarray(l.taps()) for l in cpx.layers[:2])
    host = np.random.default_rng(1).random(shape).astype(np.float32)
    fr = torch.from_numpy(host).cuda()
    b, h, w, c = shape
    out = torch.full((b, c, h, w), float("nan"), device="cuda")
    rc = lib.skc_layer_pair_fwd(nat.ptr(fr), nat.ptr(out), b, h, w, c, nat.dbl(t0), t0.shape[0], nat.dbl(t1),
                                t1.shape[0], bnd, None)
    torch.cuda.synchronize()
    ref = orc.apply_complex(host[0].astype(np.float64), [(l.offsets, l.weights) for l in cpx.layers[:2]],
                            orc.CLAMP if bnd else orc.ZERO)
    got = out[0].permute(1, 2, 0).cpu().numpy()
    err = np.abs(got - ref).max(axis=2)
    bad = ~(err < 1e-5)
    print(cfg, shape, "bnd", bnd, "rc", rc, nat.last_error() if rc else "", "nan", int(np.isnan(got).sum()),
          "bad px", int(bad.sum()), "of", h * w)
    if bad.any():
        ys, xs = np.nonzero(bad)
        print("  bad rows", ys.min(), ys.max(), "cols", xs.min(), xs.max())
        for th in (24, 48):
            tiles = sorted(set(zip((ys // th).tolist(), (xs // 128).tolist())))
            print("  tiles(th=%d)" % th, len(tiles), tiles[:20])
        print("  sample got", got[ys[0], xs[0]], "ref", ref[ys[0], xs[0]])
