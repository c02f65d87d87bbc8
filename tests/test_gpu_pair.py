"""The fused head pair (opt-in, SKC_PAIR=1; skc_layer_pair_fwd, csrc/skc_sparse.cu sparse_pair):
layers 0 and 1 of a chain in one launch, the intermediate kept in shared
memory.  Checked against the float64 oracle of the same two layers
(oracle/skc_oracle.c, reference engine.apply_complex engine.py:173-178 on the
first two layers) at 1e-5 normwise, on ragged shapes, both boundary modes
(zero: the reference's padding; clamp: config 0) and C = 1, 3, 4 -- the edge
tiles re-apply the boundary rule to the shared intermediate, which is where a
fused pair can go wrong."""

import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle import oracle as orc
    from paper_2512_04556_b200 import _native as nat
    from paper_2512_04556_b200 import synth
    import os
    orc.set_threads(os.cpu_count() or 1)
    return torch, orc, nat, synth


def _pair(torch, nat, frames, t0, t1, boundary):
    b, h, w, c = frames.shape
    out = torch.empty((b, c, h, w), dtype=torch.float32, device=frames.device)
    rc = nat.lib().skc_layer_pair_fwd(nat.ptr(frames), nat.ptr(out), b, h, w, c, nat.dbl(t0), t0.shape[0],
                                      nat.dbl(t1), t1.shape[0], boundary, nat.stream_ptr())
    return rc, out


@pytest.mark.parametrize("cfg,shape,bnd", [
    ("c1", (2, 301, 259, 3), 0), ("c1", (1, 97, 130, 3), 1), ("c1", (1, 64, 128, 1), 0),
    ("c0", (1, 512, 512, 3), 1), ("c0", (3, 77, 45, 4), 0), ("c0", (1, 200, 333, 3), 1),
])
def test_pair_vs_oracle(env, cfg, shape, bnd, monkeypatch):
    torch, orc, nat, synth = env
    monkeypatch.setenv("SKC_PAIR", "1")         # opt-in
    monkeypatch.setenv("SKC_PAIR_SMALL", "1")   # small frames run unfused by default
    cpx = synth.c1_complex() if cfg == "c1" else synth.c0_complex()
    t0, t1 = (np.ascontiguousarray(l.taps()) for l in cpx.layers[:2])
    rng = np.random.default_rng(hash((cfg, shape, bnd)) % 2**32)
    host = rng.random(shape).astype(np.float32)
    frames = torch.from_numpy(host).cuda()
    rc, out = _pair(torch, nat, frames, t0, t1, bnd)
    assert rc == 0, nat.last_error() if rc != nat.SKC_ENOTTAKEN else "pair not taken"
    torch.cuda.synchronize()
    layers = [(l.offsets, l.weights) for l in cpx.layers[:2]]
    for b in range(shape[0]):
        ref = orc.apply_complex(host[b].astype(np.float64), layers, orc.CLAMP if bnd else orc.ZERO)
        got = out[b].permute(1, 2, 0).cpu().numpy()
        assert normwise(got, ref) < 1e-5, (b, normwise(got, ref))


def test_chain_with_pair_equals_unfused(env, monkeypatch):
    """skc_chain_fwd with the pair equals the layer-by-layer chain (the unfused
    sequence through skc_layer_fwd_ex)."""
    torch, orc, nat, synth = env
    monkeypatch.setenv("SKC_PAIR", "1")
    monkeypatch.setenv("SKC_PAIR_SMALL", "1")
    import paper_2512_04556_b200 as skc
    cpx = synth.c1_complex()
    rng = np.random.default_rng(5)
    host = rng.random((2, 211, 300, 3)).astype(np.float32)
    frames = torch.from_numpy(host).cuda()
    fused = skc.apply_complex_batch(frames, cpx)
    lib = nat.lib()
    b, h, w, c = frames.shape
    src, lay = frames, nat.SKC_HWC
    for k, l in enumerate(cpx.layers):
        t = np.ascontiguousarray(l.taps())
        last = k == len(cpx.layers) - 1
        dst = torch.empty_like(frames) if last else torch.empty((b, c, h, w), dtype=torch.float32, device="cuda")
        rc = lib.skc_layer_fwd_ex(nat.ptr(src), nat.SKC_F32, lay, nat.ptr(dst), nat.SKC_F32,
                                  nat.SKC_HWC if last else nat.SKC_CHW, b, h, w, c, nat.dbl(t), t.shape[0], 0,
                                  nat.stream_ptr())
        assert rc == 0, nat.last_error()
        src, lay = dst, nat.SKC_CHW
    torch.cuda.synchronize()
    assert normwise(fused.cpu().numpy(), src.cpu().numpy()) < 2e-6
    ref = orc.apply_complex(host[1].astype(np.float64), [(l.offsets, l.weights) for l in cpx.layers], orc.ZERO)
    assert normwise(fused[1].cpu().numpy(), ref) < 1e-5


def test_pair_plan_query_and_bad_args(env, monkeypatch):
    torch, orc, nat, synth = env
    monkeypatch.setenv("SKC_PAIR", "1")
    lib = nat.lib()
    cpx = synth.c1_complex()
    t0, t1 = (np.ascontiguousarray(l.taps()) for l in cpx.layers[:2])
    assert lib.skc_layer_pair_fwd(None, None, 64, 2665, 1264, 3, nat.dbl(t0), t0.shape[0], nat.dbl(t1),
                                  t1.shape[0], 0, None) == 0
    # a second layer taller than the streamed block is declined
    t3 = np.array([[0.25, -40.5, 0.5], [-0.75, 40.25, 0.5]], dtype=np.float64)
    assert lib.skc_layer_pair_fwd(None, None, 64, 2665, 1264, 3, nat.dbl(t0), t0.shape[0], nat.dbl(t3),
                                  t3.shape[0], 0, None) == nat.SKC_ENOTTAKEN
    bad = t0.copy()
    bad[0, 0] = np.nan
    assert lib.skc_layer_pair_fwd(None, None, 1, 100, 100, 3, nat.dbl(bad), bad.shape[0], nat.dbl(t1),
                                  t1.shape[0], 0, None) == nat.SKC_EBADARG
