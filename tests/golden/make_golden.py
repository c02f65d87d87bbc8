"""Generate golden fixtures by running the UNMODIFIED reference `sparsekern`.

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box, so the outputs are committed
as small compressed .npz files next to this script):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every case stores its inputs and the reference outputs.  The oracle
(oracle/skc_oracle.c) is pinned against these in tests/test_oracle.py, and the
host-side restatements in paper_2512_04556_b200 (kernel rasteriser, bracket,
canvas rules) are pinned in tests/test_host.py.
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import sparsekern as sk  # noqa: E402
from sparsekern import engine, optim, svfilter  # noqa: E402
from sparsekern._fastpath import HAVE_NUMBA, ir_batch_compiled, sv_filter_compiled  # noqa: E402

OUT = Path(__file__).resolve().parent


def f32(a):
    """Inputs are fp32-rounded first: the GPU sees exactly these values."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rand_complex(rng, layout, reach):
    layers = []
    for n in layout:
        off = f32(rng.uniform(-reach, reach, size=(n, 2)))
        w = rng.uniform(0.05, 1.0, size=n)
        layers.append(sk.SparseLayer(off, f32(w / w.sum())))
    return sk.KernelComplex(tuple(layers))


def cpx_arrays(cpx):
    off = np.concatenate([l.offsets for l in cpx.layers])
    w = np.concatenate([l.weights for l in cpx.layers])
    return off, w, np.array(cpx.layout, dtype=np.int64)


def clamp_layer(img, layer):
    """SURVEY D1 clamp-to-edge wrapper: edge-pad P, reference layer, crop."""
    p = int(math.floor(np.abs(layer.offsets).max())) + 1
    pad = ((p, p), (p, p)) + (((0, 0),) if img.ndim == 3 else ())
    out = sk.apply_sparse_layer(np.pad(img, pad, mode="edge"), layer)
    return out[p:-p, p:-p]


def clamp_complex(img, cpx):
    out = np.asarray(img, dtype=np.float64)
    for layer in cpx.layers:
        out = clamp_layer(out, layer)
    return out


def gen_engine():
    rng = np.random.default_rng(1001)
    cases = {}
    specs = [
        ((23, 31), (3,), 2.5),
        ((19, 17, 3), (4, 2), 3.0),
        ((32, 40, 3), (12, 12, 12, 12), 6.0),
        ((16, 16, 4), (4, 4, 4), 1.5),
        ((9, 11, 1), (5,), 7.5),           # reach comparable to the image
        ((40, 13, 2), (2, 6, 3), 4.0),
    ]
    for k, (shape, layout, reach) in enumerate(specs):
        img = f32(rng.uniform(size=shape))
        cpx = rand_complex(rng, layout, reach)
        off, w, lay = cpx_arrays(cpx)
        cases[f"c{k}_img"] = img
        cases[f"c{k}_off"] = off
        cases[f"c{k}_w"] = w
        cases[f"c{k}_layout"] = lay
        cases[f"c{k}_zero"] = sk.apply_complex(img, cpx)
        cases[f"c{k}_layer0"] = sk.apply_sparse_layer(img, cpx.layers[0])
        cases[f"c{k}_clamp"] = clamp_complex(img, cpx)
    # exact integer and half-pixel taps, negative weights, duplicate taps
    img = f32(rng.uniform(size=(12, 14, 3)))
    cpx = sk.KernelComplex((
        sk.SparseLayer(np.array([[1.0, 0.0], [0.0, -2.0], [0.5, 0.5], [0.5, 0.5]]),
                       np.array([0.5, -0.25, 0.5, 0.25])),
        sk.SparseLayer(np.array([[-1.5, 2.0], [3.0, -0.5]]), np.array([0.75, 0.25])),
    ))
    off, w, lay = cpx_arrays(cpx)
    cases.update(k_img=img, k_off=off, k_w=w, k_layout=lay, k_zero=sk.apply_complex(img, cpx),
                 k_clamp=clamp_complex(img, cpx))
    np.savez_compressed(OUT / "engine.npz", **cases)


def gen_ir():
    rng = np.random.default_rng(1002)
    cases = {}
    for k, (layout, reach) in enumerate([((3,), 2.5), ((4, 4), 3.0), ((5, 3, 4), 2.0),
                                          ((8, 8, 8, 8), 4.0)]):
        cpx = rand_complex(rng, layout, reach)
        off, w, lay = cpx_arrays(cpx)
        ir = sk.synthesize_ir(cpx)
        cases[f"i{k}_off"] = off
        cases[f"i{k}_w"] = w
        cases[f"i{k}_layout"] = lay
        cases[f"i{k}_ir"] = ir.weights
        cases[f"i{k}_canvas"] = np.int64(ir.size)
        cases[f"i{k}_required"] = np.int64(sk.required_canvas(cpx))
    # Kawase 6x4 chain: reference canvas truncation
    layers = []
    for l in range(6):
        r = 0.5 + l
        layers.append(sk.SparseLayer(np.array([[r, r], [-r, r], [-r, -r], [r, -r]]),
                                     np.full(4, 0.25)))
    kaw = sk.KernelComplex(tuple(layers))
    cases["kawase_auto"] = sk.synthesize_ir(kaw).weights
    cases["kawase_61"] = sk.synthesize_ir(kaw, canvas=61).weights
    # batched IR (numpy and numba paths), ragged layout via zero weights
    off = f32(rng.uniform(-3, 3, (4, 3, 5, 2)))
    wts = f32(rng.uniform(-0.2, 0.5, (4, 3, 5)))
    wts[1, 2, 3:] = 0.0
    cases["batch_off"] = off
    cases["batch_w"] = wts
    cases["batch_ir"] = engine.synthesize_ir_batch(off, wts, 41)
    if HAVE_NUMBA:
        cases["batch_ir_numba"] = ir_batch_compiled(off, wts, 41)
    np.savez_compressed(OUT / "ir.npz", **cases)


def stacked(basis):
    ox, oy, w = svfilter._stacked_params(basis)
    return np.stack([ox, oy, w], axis=-1)


def gen_sv():
    rng = np.random.default_rng(1003)
    cases = {}
    layout = (4, 3, 5)
    base = rand_complex(rng, layout, 3.0)
    filters = []
    for k in range(3):
        layers = []
        for lay in base.layers:
            off = f32(lay.offsets * (0.5 + 0.75 * k) + rng.uniform(-0.3, 0.3, lay.offsets.shape))
            w = lay.weights * rng.uniform(0.8, 1.2, lay.weights.shape)
            layers.append(sk.SparseLayer(off, f32(w / w.sum())))
        filters.append(sk.KernelComplex(tuple(layers)))
    ps = np.array([0.0, 0.4, 1.0])
    basis = sk.FilterBasis(ps, tuple(filters))
    img = f32(rng.uniform(size=(29, 37, 3)))
    yy, xx = np.mgrid[0:29, 0:37]
    pmap = f32(np.clip(np.hypot(xx - 18, yy - 14) / 20.0 - 0.1, -0.2, 1.2))
    pmap[3:7, 20:25] = 0.4   # exact knot hits
    cases.update(img=img, pmap=pmap, params=ps, basis=stacked(basis),
                 layout=np.array(layout, dtype=np.int64), out=sk.sv_filter(img, basis, pmap))
    # clamp mode: per layer, sv_filter_compiled on edge-padded img/k0/k1/t, crop
    k0, k1, t = svfilter._bracket(pmap, basis.params)
    ox, oy, w = svfilter._stacked_params(basis)
    outc = []
    for c in range(3):
        cur = img[:, :, c]
        for l, n in enumerate(layout):
            p = int(math.floor(max(np.abs(ox[:, l]).max(), np.abs(oy[:, l]).max()))) + 2
            cp = np.pad(cur, p, mode="edge")
            nxt = sv_filter_compiled(cp, np.pad(k0, p, mode="edge"), np.pad(k1, p, mode="edge"),
                                     np.pad(t, p, mode="edge"), ox[:, l:l + 1], oy[:, l:l + 1],
                                     w[:, l:l + 1], (n,))
            cur = nxt[p:-p, p:-p]
        outc.append(cur)
    cases["out_clamp"] = np.stack(outc, axis=2)
    # single-entry basis, 2-D image
    b1 = sk.FilterBasis(np.array([0.3]), (filters[1],))
    img2 = f32(rng.uniform(size=(15, 12)))
    pm2 = f32(rng.uniform(-1, 2, size=(15, 12)))
    cases.update(img1=img2, pmap1=pm2, params1=b1.params, basis1=stacked(b1),
                 out1=sk.sv_filter(img2, b1, pm2))
    # bracket KAT
    probe = np.array([-1.0, 0.0, 0.2, 0.4, 0.7, 1.0, 3.0])
    k0p, k1p, tp = svfilter._bracket(probe, ps)
    cases.update(bracket_p=probe, bracket_k0=k0p, bracket_t=tp)
    np.savez_compressed(OUT / "sv.npz", **cases)


def gen_optim():
    rng = np.random.default_rng(1004)
    cases = {}
    kinds = [sk.LossKind("charbonnier", 1e-3), sk.LossKind("l1"), sk.LossKind("l2"),
             sk.LossKind("charbonnier", 1e-6)]
    k = 0
    for layout, reach, tsize in [((3,), 2.0, 9), ((4, 2), 2.0, 9), ((2, 3, 4), 1.7, 11),
                                 ((8, 8, 8, 8), 3.0, 21)]:
        for kind in kinds:
            cpx = rand_complex(rng, layout, reach)
            tgt = sk.DenseKernel(rng.uniform(size=(tsize, tsize))).normalized()
            tgt = sk.DenseKernel(f32(tgt.weights))
            value, grads = sk.backward(cpx, tgt, kind)
            off, w, lay = cpx_arrays(cpx)
            canvas = max(sk.auto_canvas(cpx), tgt.size)
            cases[f"b{k}_off"] = off
            cases[f"b{k}_w"] = w
            cases[f"b{k}_layout"] = lay
            cases[f"b{k}_tgt"] = tgt.weights
            cases[f"b{k}_kind"] = np.array(kind.kind)
            cases[f"b{k}_eps"] = np.float64(kind.epsilon)
            cases[f"b{k}_canvas"] = np.int64(canvas)
            cases[f"b{k}_value"] = np.float64(value)
            cases[f"b{k}_doff"] = np.concatenate([g[0] for g in grads])
            cases[f"b{k}_dw"] = np.concatenate([g[1] for g in grads])
            k += 1
    cases["n_backward"] = np.int64(k)
    # short fits with explicit init (optim.py:404-405)
    fits = [
        ("sum", "none", "l1", (8, 8, 8), 25, 1e-3, 1e-4),
        ("none", "none", "l2", (4, 4), 30, 1e-3, 1e-4),
        ("sofm", "none", "charbonnier", (6, 6), 30, 1e-3, 1e-4),
        ("sum", "kws", "charbonnier", (8, 4), 30, 2e-3, 1e-4),
        ("sum", "none", "l1", (4, 4), 12, 1e-2, 1e-2),   # canvas growth
    ]
    for j, (wn, sym, lk, layout, steps, lr0, lr1) in enumerate(fits):
        tgt = sk.disk_kernel(4.0 + j, 2 * (6 + j) + 1)
        tgt = sk.DenseKernel(f32(tgt.weights))
        cpx = rand_complex(rng, layout, 2.0 + j)
        cfg = sk.TrainConfig(steps=steps, lr_start=lr0, lr_end=lr1)
        res = sk.fit(tgt, layout, cpx, cfg, sk.ConstraintConfig(wn, sym), sk.LossKind(lk))
        off, w, lay = cpx_arrays(cpx)
        boff, bw, _ = cpx_arrays(res.complex)
        cases.update({
            f"f{j}_tgt": tgt.weights, f"f{j}_off": off, f"f{j}_w": w, f"f{j}_layout": lay,
            f"f{j}_wn": np.array(wn), f"f{j}_sym": np.array(sym), f"f{j}_loss": np.array(lk),
            f"f{j}_steps": np.int64(steps), f"f{j}_lr": np.array([lr0, lr1]),
            f"f{j}_trace": res.trace, f"f{j}_best_off": boff, f"f{j}_best_w": bw,
            f"f{j}_best_loss": np.float64(res.best_loss), f"f{j}_best_step": np.int64(res.best_step),
            f"f{j}_canvas": np.int64(res.canvas),
        })
    cases["n_fit"] = np.int64(len(fits))
    # adam KATs (test_optim.py:186-199)
    cfg = sk.TrainConfig(steps=10, lr_start=1e-3, lr_end=1e-3)
    params = [[np.zeros((1, 2)), np.zeros(1)]]
    st = sk.AdamState.for_params(params)
    out = sk.adam_step(params, [[np.zeros((1, 2)), np.ones(1)]], st, 0, cfg,
                       sk.ConstraintConfig("none"))
    cases["adam_first_w"] = out[0][1]
    np.savez_compressed(OUT / "optim.npz", **cases)


def gen_kernels():
    rng = np.random.default_rng(1005)
    cases = {}
    cases["disk_60_129"] = sk.disk_kernel(60.0, 129).weights
    r = float(rng.uniform(20, 60))
    rot = float(rng.uniform(0, 2 * np.pi))
    cases["params"] = np.array([r, rot])
    cases["square_129"] = sk.polygon_kernel(4, r, 129, rot).weights
    cases["hex_129"] = sk.polygon_kernel(6, r, 129, rot).weights
    cases["ring_129"] = sk.ring_kernel(0.6 * r, r, 129).weights
    cases["star_129"] = sk.star_kernel(4, r, 129, rotation=rot).weights
    cases["disk_7"] = sk.disk_kernel(2.5).weights
    cases["gauss_15"] = sk.gaussian_kernel(1.5).weights
    cases["gauss_2_11"] = sk.gaussian_kernel(1.7, 11).weights
    np.savez_compressed(OUT / "kernels.npz", **cases)


def gen_init():
    """initializers.py strategies on a few targets (host restatement pin)."""
    cases = {}
    targets = {"gauss": sk.gaussian_kernel(2.0), "ring": sk.ring_kernel(5.0, 9.0, 23),
               "disk": sk.disk_kernel(6.0)}
    k = 0
    for tname, tgt in targets.items():
        for tag in ("rand", "ir", "ss", "ss-ir"):
            for layout, kws in (((8, 4, 4), False), ((8, 8), True)):
                if kws and tag not in ("ir", "ss-ir"):
                    continue
                cpx = sk.build_init(sk.InitStrategy(tag, seed=3 + k), tgt, layout, kws=kws)
                off, w, lay = cpx_arrays(cpx)
                cases[f"n{k}_tgt"] = tgt.weights
                cases[f"n{k}_tag"] = np.array(tag)
                cases[f"n{k}_seed"] = np.int64(3 + k)
                cases[f"n{k}_layout"] = np.array(layout, dtype=np.int64)
                cases[f"n{k}_kws"] = np.int64(kws)
                cases[f"n{k}_off"] = off
                cases[f"n{k}_w"] = w
                k += 1
    cases["n_init"] = np.int64(k)
    off, r = sk.support_rejection_sample(targets["ring"], 12, seed=5, return_radius=True)
    cases["srs_off"] = off
    cases["srs_r"] = np.float64(r)
    np.savez_compressed(OUT / "init.npz", **cases)


def gen_pst():
    """PST energies (baselines.py:175-191) and a short seeded pst_fit trace."""
    from sparsekern import baselines
    rng = np.random.default_rng(1006)
    tgt = sk.DenseKernel(f32(sk.disk_kernel(5.0, 15).weights))
    off = f32(rng.uniform(-3, 3, (6, 3, 4, 2)))
    w = f32(rng.uniform(0.05, 1.0, (6, 3, 4)))
    w /= w.sum(axis=2, keepdims=True)
    w = f32(w)
    off[5, 2, 0] = [40.0, 0.5]   # drifts off the canvas: leak wall -> inf
    canvas = 25
    irs = engine.synthesize_ir_batch(off, w, canvas)
    diffs = irs - tgt.embedded(canvas).weights[None]
    e = np.abs(diffs).sum(axis=(1, 2))
    expected = np.prod(w.sum(axis=2), axis=1)
    leak = np.abs(irs.sum(axis=(1, 2)) - expected) > 1e-6 * np.maximum(np.abs(expected), 1.0)
    e[leak] = np.inf
    res = baselines.pst_fit(tgt, (4, 4), baselines.PSTConfig(chains=4, iterations=20, seed=2),
                            sk.InitStrategy("ss", seed=1), sk.LossKind("l1"))
    np.savez_compressed(OUT / "pst.npz", tgt=tgt.weights, off=off, w=w, canvas=np.int64(canvas),
                        energies=e, trace=res.trace, best=np.float64(res.best_energy))


def gen_next():
    """2-D grid SV and the dense convolution oracle."""
    rng = np.random.default_rng(1007)
    layout = (3, 4)
    base = rand_complex(rng, layout, 2.0)
    rows = []
    for iu in range(2):
        row = []
        for iv in range(3):
            layers = []
            for lay in base.layers:
                off = f32(lay.offsets * (0.6 + 0.5 * iu + 0.3 * iv) + rng.uniform(-0.2, 0.2, lay.offsets.shape))
                w = lay.weights * rng.uniform(0.8, 1.2, lay.weights.shape)
                layers.append(sk.SparseLayer(off, f32(w / w.sum())))
            row.append(sk.KernelComplex(tuple(layers)))
        rows.append(tuple(row))
    grid = svfilter.FilterBasisGrid(np.array([0.0, 1.0]), np.array([0.0, 0.5, 1.0]), tuple(rows))
    img = f32(rng.uniform(size=(23, 27)))
    pm2 = f32(np.stack([rng.uniform(-0.2, 1.2, (23, 27)), rng.uniform(-0.2, 1.2, (23, 27))], axis=2))
    out = svfilter.sv_filter_grid(img, grid, pm2)
    stack = np.stack([np.stack([stacked(sk.FilterBasis(grid.params_v, rows[iu]))[iv] for iv in range(3)])
                      for iu in range(2)])
    k7 = sk.DenseKernel(f32(rng.uniform(-1, 1, (7, 7))))
    k21 = sk.DenseKernel(f32(rng.uniform(0, 1, (21, 21))))
    imgc = f32(rng.uniform(size=(30, 26, 3)))
    np.savez_compressed(OUT / "next.npz", grid_img=img, grid_pm2=pm2, grid_pu=grid.params_u, grid_pv=grid.params_v,
                        grid_stack=stack, grid_layout=np.array(layout), grid_out=out,
                        k7=k7.weights, k21=k21.weights, dc_img=imgc, dc7=sk.dense_convolve(imgc, k7),
                        dc21=sk.dense_convolve(imgc, k21))


def gen_round2():
    """Round-2 rows: bilinear_sample, sv_ground_truth, KernelSpec / netpbm
    formats, build_basis(_grid) with KernelSpec targets, a longer PST trace."""
    import io
    import tempfile
    from dataclasses import replace  # noqa: F401
    from sparsekern import baselines, kernels
    rng = np.random.default_rng(2001)
    cases = {}
    # bilinear_sample (engine.py:212-248): plain, batched, broadcast, general batch broadcast
    img = rng.uniform(size=(9, 11))
    x = rng.uniform(-2, 13, (5, 7))
    y = rng.uniform(-2, 11, (5, 7))
    x[0, 0], y[0, 0] = 3.0, 4.0          # integer read
    cases.update(bs0_img=img, bs0_x=x, bs0_y=y, bs0_out=engine.bilinear_sample(img, x, y))
    imgb = rng.uniform(size=(3, 6, 8))
    xb = rng.uniform(-1, 9, (3, 4, 5))
    yb = rng.uniform(-1, 7, (3, 4, 5))
    cases.update(bs1_img=imgb, bs1_x=xb, bs1_y=yb, bs1_out=engine.bilinear_sample(imgb, xb, yb))
    xr = rng.uniform(-1, 9, (4, 5))
    yr = rng.uniform(-1, 7, (1, 5))
    cases.update(bs2_img=img, bs2_x=xr, bs2_y=yr, bs2_out=engine.bilinear_sample(img, xr, yr))
    imgc = rng.uniform(size=(2, 3, 6, 8))
    xc = rng.uniform(-1, 9, (2, 3, 4))
    yc = rng.uniform(-1, 7, (2, 3, 4))
    cases.update(bs3_img=imgc, bs3_x=xc, bs3_y=yc, bs3_out=engine.bilinear_sample(imgc, xc, yc))
    # sv_ground_truth (svfilter.py:206-235) with a KernelSpec family and 3 map levels
    gimg = f32(rng.uniform(size=(26, 21, 2)))
    pm = np.choose(rng.integers(0, 3, (26, 21)), [0.0, 0.5, 1.0])
    fam = lambda p: sk.KernelSpec("disk", (1.5 + 3.0 * p,))   # noqa: E731
    cases.update(gt_img=gimg, gt_pmap=pm, gt_out=svfilter.sv_ground_truth(gimg, fam, pm))
    pm2 = np.choose(rng.integers(0, 2, (26, 21)), [0.2, 0.7])
    fam2 = lambda p: sk.gaussian_kernel(0.5 + 2.0 * p)        # noqa: E731
    cases.update(gt2_pmap=pm2, gt2_out=svfilter.sv_ground_truth(gimg[:, :, 0], fam2, pm2))
    # KernelSpec parse + generate_kernel
    specs = ["gaussian:1.5", "gaussian:1.2:11", "disk:4.5", "disk:3:11", "ring:2:5", "ring:2:5:15",
             "polygon:5:6", "polygon:6:7:19:30", "star:4:8", "star:5:8:21:15", "heart:7", "heart:6:17",
             "delta", "delta:5"]
    cases["spec_texts"] = np.array(specs)
    for j, t in enumerate(specs):
        sp = sk.KernelSpec.parse(t)
        cases[f"spec{j}_repr"] = np.array(repr(sp))
        cases[f"spec{j}_k"] = sk.generate_kernel(sp).weights
    # netpbm bytes
    with tempfile.TemporaryDirectory() as d:
        k = sk.disk_kernel(3.3)
        kernels.save_kernel_image(k, f"{d}/k.pgm")
        cases["pgm_kernel_bytes"] = np.frombuffer(open(f"{d}/k.pgm", "rb").read(), np.uint8)
        cases["pgm_kernel_loaded"] = kernels.load_kernel_image(f"{d}/k.pgm").weights
        im2 = rng.uniform(-0.1, 1.1, (5, 7))
        im3 = rng.uniform(0, 1, (4, 6, 3))
        kernels.write_image(im2, f"{d}/a.pgm")
        kernels.write_image(im3, f"{d}/b.ppm", maxval=255)
        cases.update(img2=im2, img3=im3,
                     pgm_img2_bytes=np.frombuffer(open(f"{d}/a.pgm", "rb").read(), np.uint8),
                     ppm_img3_bytes=np.frombuffer(open(f"{d}/b.ppm", "rb").read(), np.uint8),
                     img2_read=kernels.read_image(f"{d}/a.pgm"), img3_read=kernels.read_image(f"{d}/b.ppm"))
        with open(f"{d}/c.pgm", "w") as fh:
            fh.write("P2\n# a comment\n3 2\n# another\n10\n0 1 2\n3 4 10\n")
        cases["ascii_read"] = kernels.read_image(f"{d}/c.pgm")
    # basis building with KernelSpec targets (short fits: trajectories stay within fp32 noise)
    cfg = sk.TrainConfig(steps=6)
    lk = sk.LossKind("l1")
    b1 = svfilter.build_basis(lambda p: sk.KernelSpec("disk", (2.0 + 2.0 * p,), size=11), [0.0, 0.5, 1.0],
                              (4, 4), cfg=cfg, init=sk.InitStrategy("ss", seed=3), loss_kind=lk)
    cases["bb_stack"] = stacked(b1)
    b2 = svfilter.build_basis(lambda p: sk.KernelSpec("disk", (2.0 + 2.0 * p,), size=11), [0.0, 0.25, 1.0],
                              (4, 4), cfg=cfg, init=sk.InitStrategy("ss", seed=3), loss_kind=lk,
                              warm_start=False)
    cases["bb_nows_stack"] = stacked(b2)
    g = svfilter.build_basis_grid(lambda u, v: sk.KernelSpec("disk", (2.0 + u + 1.5 * v,), size=11),
                                  [0.0, 1.0], [0.0, 0.5, 1.0], (4, 4), cfg=cfg,
                                  init=sk.InitStrategy("ss", seed=5), loss_kind=lk)
    cases["bbg_stack"] = np.stack([np.stack([stacked(g.row_basis(iu))[iv] for iv in range(3)]) for iu in range(2)])
    # a longer seeded PST trace (numpy proposal stream) + best energies over seeds
    tgt = sk.DenseKernel(f32(sk.disk_kernel(4.0, 13).weights))
    res = baselines.pst_fit(tgt, (4, 4), baselines.PSTConfig(chains=5, iterations=300, seed=7),
                            sk.InitStrategy("ss", seed=2), sk.LossKind("l1"))
    cases.update(pst_tgt=tgt.weights, pst_trace=res.trace, pst_ladder=res.ladder, pst_best=np.float64(res.best_energy),
                 pst_best_stack=stacked(sk.FilterBasis([0.0], (res.complex,))))
    bests = []
    for sd in range(12):
        r = baselines.pst_fit(tgt, (4, 4), baselines.PSTConfig(chains=4, iterations=400, seed=100 + sd),
                              sk.InitStrategy("ss", seed=2), sk.LossKind("l1"))
        bests.append(r.best_energy)
    cases["pst_seed_bests"] = np.array(bests)
    np.savez_compressed(OUT / "round2.npz", **cases)


if __name__ == "__main__":
    gen_round2()
    gen_next()
    gen_pst()
    gen_init()
    gen_engine()
    gen_ir()
    gen_sv()
    gen_optim()
    gen_kernels()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
