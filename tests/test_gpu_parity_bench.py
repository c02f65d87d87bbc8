"""Parity at the configurations bench.py times (VERDICT r1 "next round" item 1).

Each test drives the SAME code path the bench measures on the full benchmark
shapes and checks whole frames (edges included) against the float64 oracle
(oracle/skc_oracle.c, pinned to the reference by tests/test_oracle.py):

  C1  frames 0 and 63 of the batch-64 run: through bench.Chain's launch
      sequence (skc_layer_fwd_ex / skc_relayout, what the bench times) and
      through skc_chain_fwd (apply_complex_batch), 1e-5 normwise;
  C2  the full 2665 x 1264 frame, zero and clamp boundaries, 1e-5;
  C3  (tests/test_gpu_kawase.py: full frames 0 and 31);
  C3big  the 16384^2 RGBA fp16 image: oracle seam windows (22-row margins)
      at the 2/4/8-way strip boundaries at 2e-3, and each rank's extended
      strip (21-row halos, dist.strip_bounds) filtered alone reproduces the
      full-image rows bit for bit;
  C4  backward of all 256 config-4 targets at 4x32 on 129^2 canvases vs the
      oracle at 1e-5 (L1 made sign-stable by giving the oracle the fp32 sign
      pattern), the first 20 fit steps, and the fit canvas.
"""

import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu

TOL32 = 1e-5
TOL16 = 2e-3


@pytest.fixture(scope="module")
def skc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2512_04556_b200 as m
    return m


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    oracle.set_threads(os.cpu_count() or 1)
    return oracle


def _layers(cpx):
    return [(l.offsets, l.weights) for l in cpx.layers]


def test_c1_bench_frames_0_and_63(skc, orc):
    import torch
    import bench
    wl = bench.Chain("c1", SimpleNamespace(frames=64), torch.device("cuda", 0), 0)
    wl.step(torch.cuda.current_stream())
    torch.cuda.synchronize()
    via_chain = skc.apply_complex_batch(wl.frames, wl.cpx)
    for b in (0, 63):
        frame = wl.frames[b].cpu().numpy().astype(np.float64)
        ref = orc.apply_complex(frame, _layers(wl.cpx), orc.ZERO)
        assert normwise(wl.out[b].cpu().numpy(), ref) < TOL32, b
        assert normwise(via_chain[b].cpu().numpy(), ref) < TOL32, b
    del wl, via_chain
    torch.cuda.empty_cache()


def test_c2_full_frame_both_boundaries(skc, orc):
    from paper_2512_04556_b200 import synth
    from paper_2512_04556_b200.svfilter import stacked_params
    basis = synth.c2_basis()
    pmap = synth.c2_pmap()
    img = synth.c1_frame(0)
    for mode, oid in (("zero", orc.ZERO), ("clamp", orc.CLAMP)):
        out = skc.sv_filter(img, basis, pmap, boundary=mode)
        ref = orc.sv_filter(img.astype(np.float64), pmap, basis.params, stacked_params(basis), basis.layout,
                            boundary=oid)
        assert normwise(out, ref) < TOL32, mode


def test_c3big_seams_and_strip_decomposition(skc, orc):
    import torch
    from paper_2512_04556_b200 import synth
    from paper_2512_04556_b200.dist import corner_reach, strip_bounds
    h, w, c = synth.C3_BIG
    cpx = synth.kawase_complex()
    dev = torch.device("cuda", 0)
    full = synth.value_noise_frame_device(h, w, c, 100, dev, dtype=torch.float16)
    out = skc.apply_complex(full, cpx)
    top, bot = corner_reach(cpx)[:2]
    assert (top, bot) == (21, 21)
    margin = 22
    for seam in (4096, 8192, 12288, 14336):
        r0, r1 = seam - margin - 24, seam + margin + 24
        win = full[r0:r1].cpu().numpy().astype(np.float64)
        ref = orc.apply_complex(win, _layers(cpx), orc.ZERO)
        got = out[r0 + margin:r1 - margin].cpu().numpy().astype(np.float64)
        assert normwise(got, ref[margin:-margin]) < TOL16, seam
    for world in (2, 8):
        for rank in range(world):
            a, b = strip_bounds(h, rank, world)
            e0, e1 = max(0, a - top), min(h, b + bot)
            part = skc.apply_complex(full[e0:e1].contiguous(), cpx)
            assert torch.equal(part[a - e0:a - e0 + (b - a)], out[a:b]), (world, rank)
    del full, out
    torch.cuda.empty_cache()


def _c4_batch(skc, n):
    from paper_2512_04556_b200 import synth
    tg = [synth.c4_target(i) for i in range(n)]
    inits = [synth.c4_init(i) for i in range(n)]
    return tg, inits


def test_c4_backward_all_256_sign_stable(skc, orc):
    """optim.py:278-292 at the config-4 shape.  The L1 gradient sign(IR-tgt)
    flips wherever |IR - tgt| is below fp32 resolution, so the oracle's
    reverse sweep is fed the fp32 forward's sign pattern (its forward stays
    float64); loss values are compared directly."""
    tg, inits = _c4_batch(skc, 256)
    res = skc.backward_batch(inits, tg, skc.LossKind("l1"))
    canvas = max(max(skc.auto_canvas(c) for c in inits), 129)
    irs = skc.synthesize_ir_batch(np.stack([np.stack([l.offsets for l in c.layers]) for c in inits]),
                                  np.stack([np.stack([l.weights for l in c.layers]) for c in inits]), canvas)
    for i in range(256):
        emb = tg[i].embedded(canvas).weights
        ref_v, _ = orc.backward(_layers(inits[i]), emb, "l1")
        val, grads = res[i]
        assert abs(val - ref_v) <= TOL32 * abs(ref_v), i
        g = np.sign(np.asarray(irs[i], np.float32) - emb.astype(np.float32)).astype(np.float64)
        ref_g = orc.backward_with_grad(_layers(inits[i]), g)
        dof = np.concatenate([a for a, _ in grads])
        dw = np.concatenate([b for _, b in grads])
        rof = np.concatenate([a for a, _ in ref_g])
        rw = np.concatenate([b for _, b in ref_g])
        scale = max(np.abs(rof).max(), np.abs(rw).max())
        assert np.abs(dof - rof).max() <= TOL32 * scale, i
        assert np.abs(dw - rw).max() <= TOL32 * scale, i


def test_c4_fit_first_20_steps(skc, orc):
    """optim.py:390-469: the first 20 loss-trace entries of 16 config-4 fits
    (L1, SUM, the bench's 3000-step schedule) against the float64 oracle.
    Every target agrees to 1e-5 over the first 8 steps and most over all 20.
    A few drift further: Adam's early steps are lr * sign(g)/|g|-normalised, so
    a gradient component that is zero up to fp32 rounding (~1e-6 of the
    gradient's scale) can step the other way -- an fp32-vs-float64 effect the
    oracle's own 1e-7 init perturbation does not reproduce (it keeps every
    sign).  Those are held to 5e-3 and counted."""
    from paper_2512_04556_b200 import optim
    tg, inits = _c4_batch(skc, 16)
    steps = 20
    full = skc.TrainConfig(steps=3000)
    # a 20-step schedule whose lr(t) equals the 3000-step schedule's for t < 20
    cfg = skc.TrainConfig(steps=steps, lr_start=full.lr_at(0), lr_end=full.lr_at(steps - 1))
    _, trace, _ = optim.fit_batch(tg, (32,) * 4, inits, cfg, skc.ConstraintConfig("sum"), skc.LossKind("l1"),
                                  return_device=True)
    gpu = trace.cpu().numpy().astype(np.float64)
    off0 = np.stack([np.concatenate([l.offsets for l in c.layers]) for c in inits])
    w0 = np.stack([np.concatenate([l.weights for l in c.layers]) for c in inits])
    tgts = np.stack([t.weights for t in tg])
    ref = orc.fit_batch(tgts, off0, w0, [32] * 4, steps=steps, lr_start=cfg.lr_start, lr_end=cfg.lr_end,
                        weight_norm="sum", loss_kind="l1")["trace"]
    rel = np.abs(gpu - ref) / np.abs(ref)
    assert rel[:, :8].max() < TOL32, rel[:, :8].max(axis=0)
    within = (rel.max(axis=1) < TOL32).sum()
    assert within >= 8, (within, rel.max(axis=1))
    assert rel.max() < 5e-3, rel.max(axis=1)


def test_fit_canvas_matches_reference(skc, golden):
    """fit.embed_if_grown (optim.py:429-434): the final canvas of every golden
    fit, including the lr 1e-2 run whose canvas grows, equals the reference's."""
    from conftest import split_layers
    g = golden("optim")
    for j in range(int(g["n_fit"])):
        lay = tuple(g[f"f{j}_layout"].tolist())
        cpx = skc.KernelComplex(tuple(skc.SparseLayer(o, w) for o, w in split_layers(g[f"f{j}_off"], g[f"f{j}_w"],
                                                                                     lay)))
        lr0, lr1 = g[f"f{j}_lr"]
        cfg = skc.TrainConfig(steps=int(g[f"f{j}_steps"]), lr_start=float(lr0), lr_end=float(lr1))
        res = skc.fit(skc.DenseKernel(g[f"f{j}_tgt"]), lay, cpx, cfg,
                      skc.ConstraintConfig(str(g[f"f{j}_wn"]), str(g[f"f{j}_sym"])),
                      skc.LossKind(str(g[f"f{j}_loss"])))
        assert res.canvas == int(g[f"f{j}_canvas"]), j
        assert res.best_step == int(g[f"f{j}_best_step"]), j
        n = min(10, res.losses.size)
        rel = np.abs(res.losses[:n] - g[f"f{j}_trace"][:n, 1]) / np.abs(g[f"f{j}_trace"][:n, 1])
        assert rel.max() < 1e-4, (j, rel)


def test_c4_d5_batch_statistic(skc, golden):
    """SURVEY D5(iii) at full scale: all 256 config-4 targets x 3000 steps (the
    bench's workload) against the float64 oracle (tests/golden/d5_c4_fit.npz,
    tools/make_d5.py).  Under the reference's default schedule most of these
    fits pass their best loss (median step ~80) and then diverge -- in the
    float64 reference too (208 of 256 end above loss 10), and a relative 1e-7
    perturbation of the inits moves the median FINAL loss by 64%.  The
    statistic that is stable under the reference's own perturbation is the
    best loss (FitResult.best_loss: mean 0.16%, median 0.6% apart), so that
    is held to 1% (mean) / 2% (median); the final losses must show the same
    divergence pattern."""
    import pathlib
    if not (pathlib.Path(__file__).parent / "golden" / "d5_c4_fit.npz").exists():
        pytest.skip("d5 fixture not generated")
    g = golden("d5_c4_fit")
    n, steps = int(g["targets"]), int(g["steps"])
    tg, inits = _c4_batch(skc, n)
    res = skc.fit_batch(tg, (32,) * 4, inits, skc.TrainConfig(steps=steps), skc.ConstraintConfig("sum"),
                        skc.LossKind("l1"))
    best = np.array([r.best_loss for r in res])
    final = np.array([r.losses[-1] for r in res])
    ref, pert = g["exact_best"], g["perturbed_best"]
    assert abs(best.mean() / ref.mean() - 1) < 0.01, (best.mean(), ref.mean(), pert.mean())
    assert abs(np.median(best) / np.median(ref) - 1) < 0.02, (np.median(best), np.median(ref), np.median(pert))
    # per-kernel: of the order of the reference's own perturbation spread
    assert np.median(np.abs(best / ref - 1)) < 3 * np.median(np.abs(pert / ref - 1)) + 1e-3
    # the divergence after the best step is the reference's behaviour, not ours alone
    div_ours, div_ref = (final > 10).sum(), (g["exact_final"] > 10).sum()
    assert abs(div_ours - div_ref) <= 0.1 * n, (div_ours, div_ref)
    assert all(r.canvas >= 129 for r in res)
