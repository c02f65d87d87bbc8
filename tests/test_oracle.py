"""Pin the CPU float64 oracle (oracle/skc_oracle.c) to the reference's own outputs.

The fixtures in tests/golden were produced by the unmodified reference
(tests/golden/make_golden.py).  Forward filtering is restated in the
reference's summation order, so it must be bit-identical; everything that goes
through np.vdot / numpy pairwise sums in the reference is held to 1e-12.
"""

import numpy as np
import pytest

from conftest import split_layers
from oracle import oracle as orc


def test_engine_zero_mode_bit_exact(golden):
    g = golden("engine")
    n = 0
    for k in range(6):
        img, off, w, lay = g[f"c{k}_img"], g[f"c{k}_off"], g[f"c{k}_w"], g[f"c{k}_layout"]
        layers = split_layers(off, w, lay)
        assert np.array_equal(orc.apply_complex(img, layers), g[f"c{k}_zero"])
        assert np.array_equal(orc.apply_layer(img, *layers[0]), g[f"c{k}_layer0"])
        n += 1
    layers = split_layers(g["k_off"], g["k_w"], g["k_layout"])
    assert np.array_equal(orc.apply_complex(g["k_img"], layers), g["k_zero"])


def test_engine_clamp_mode(golden):
    g = golden("engine")
    for k in range(6):
        layers = split_layers(g[f"c{k}_off"], g[f"c{k}_w"], g[f"c{k}_layout"])
        out = orc.apply_complex(g[f"c{k}_img"], layers, boundary=orc.CLAMP)
        assert np.array_equal(out, g[f"c{k}_clamp"])
    layers = split_layers(g["k_off"], g["k_w"], g["k_layout"])
    assert np.array_equal(orc.apply_complex(g["k_img"], layers, orc.CLAMP), g["k_clamp"])


def test_ir_synthesis(golden):
    g = golden("ir")
    for k in range(4):
        layers = split_layers(g[f"i{k}_off"], g[f"i{k}_w"], g[f"i{k}_layout"])
        ir = orc.synthesize_ir(layers, int(g[f"i{k}_canvas"]))
        assert np.array_equal(ir, g[f"i{k}_ir"])
    kaw = [(np.array([[r, r], [-r, r], [-r, -r], [r, -r]]), np.full(4, 0.25))
           for r in (0.5 + l for l in range(6))]
    auto = g["kawase_auto"]
    assert np.array_equal(orc.synthesize_ir(kaw, auto.shape[0]), auto)
    assert np.array_equal(orc.synthesize_ir(kaw, 61), g["kawase_61"])
    # D3: the reference's auto canvas truncates the Kawase IR
    assert abs(g["kawase_61"].sum() - 1.0) < 1e-12 and auto.sum() < 0.9995


def test_ir_batch(golden):
    g = golden("ir")
    off, w = g["batch_off"], g["batch_w"]
    out = orc.ir_batch(off, w, [5, 5, 5], 41)
    assert np.abs(out - g["batch_ir"]).max() < 1e-15
    if "batch_ir_numba" in g:
        assert np.abs(out - g["batch_ir_numba"]).max() < 1e-15


def test_sv_filter(golden):
    g = golden("sv")
    out = orc.sv_filter(g["img"], g["pmap"], g["params"], g["basis"], g["layout"])
    assert np.abs(out - g["out"]).max() < 1e-12
    outc = orc.sv_filter(g["img"], g["pmap"], g["params"], g["basis"], g["layout"], orc.CLAMP)
    assert np.abs(outc - g["out_clamp"]).max() < 1e-12
    out1 = orc.sv_filter(g["img1"], g["pmap1"], g["params1"], g["basis1"], [4, 3, 5])
    assert np.abs(out1 - g["out1"]).max() < 1e-12


def _embed(t, canvas):
    p = (canvas - t.shape[0]) // 2
    return np.pad(t, p)


def test_backward(golden):
    g = golden("optim")
    for k in range(int(g["n_backward"])):
        layers = split_layers(g[f"b{k}_off"], g[f"b{k}_w"], g[f"b{k}_layout"])
        tgt = _embed(g[f"b{k}_tgt"], int(g[f"b{k}_canvas"]))
        value, grads = orc.backward(layers, tgt, str(g[f"b{k}_kind"]), float(g[f"b{k}_eps"]))
        assert value == pytest.approx(float(g[f"b{k}_value"]), rel=1e-12)
        doff = np.concatenate([a for a, _ in grads])
        dw = np.concatenate([b for _, b in grads])
        scale = max(np.abs(g[f"b{k}_doff"]).max(), np.abs(g[f"b{k}_dw"]).max())
        assert np.abs(doff - g[f"b{k}_doff"]).max() <= 1e-11 * scale
        assert np.abs(dw - g[f"b{k}_dw"]).max() <= 1e-11 * scale


def test_fit_traces(golden):
    g = golden("optim")
    for j in range(int(g["n_fit"])):
        lay = g[f"f{j}_layout"]
        off = g[f"f{j}_off"][None]
        w = g[f"f{j}_w"][None]
        lr0, lr1 = g[f"f{j}_lr"]
        steps = int(g[f"f{j}_steps"])
        res = orc.fit_batch(g[f"f{j}_tgt"][None], off, w, lay, steps=steps, lr_start=lr0,
                            lr_end=lr1, weight_norm=str(g[f"f{j}_wn"]),
                            kws=str(g[f"f{j}_sym"]) == "kws", loss_kind=str(g[f"f{j}_loss"]))
        assert res["rc"][0] == 0
        ref_trace = g[f"f{j}_trace"][:, 1]
        assert np.allclose(res["trace"][0], ref_trace, rtol=1e-9, atol=1e-12), j
        assert int(res["canvas"][0]) == int(g[f"f{j}_canvas"])
        assert int(res["best_step"][0]) == int(g[f"f{j}_best_step"])
        assert np.allclose(res["best_offsets"][0], g[f"f{j}_best_off"], rtol=1e-8, atol=1e-10)
        assert np.allclose(res["best_weights"][0], g[f"f{j}_best_w"], rtol=1e-8, atol=1e-10)
