"""Host-side logic of the package (no GPU): types, validation, rasterisers, recipes."""

import math

import numpy as np
import pytest

import paper_2512_04556_b200 as skc
from paper_2512_04556_b200 import synth
from paper_2512_04556_b200.svfilter import _bracket, stacked_params


def test_rasterisers_bit_exact_vs_reference(golden):
    g = golden("kernels")
    r, rot = g["params"]
    assert np.array_equal(skc.disk_kernel(60.0, 129).weights, g["disk_60_129"])
    assert np.array_equal(skc.polygon_kernel(4, r, 129, rot).weights, g["square_129"])
    assert np.array_equal(skc.polygon_kernel(6, r, 129, rot).weights, g["hex_129"])
    assert np.array_equal(skc.ring_kernel(0.6 * r, r, 129).weights, g["ring_129"])
    assert np.array_equal(skc.star_kernel(4, r, 129, rotation=rot).weights, g["star_129"])
    assert np.array_equal(skc.disk_kernel(2.5).weights, g["disk_7"])
    assert np.array_equal(skc.gaussian_kernel(1.5).weights, g["gauss_15"])
    assert np.array_equal(skc.gaussian_kernel(1.7, 11).weights, g["gauss_2_11"])


def test_dense_kernel_invariants():
    k = skc.DenseKernel(np.ones((3, 3)))
    assert k.normalized().weights.sum() == pytest.approx(1.0)
    e = k.embedded(7)
    assert e.size == 7 and e.weights[2:5, 2:5].sum() == 9
    with pytest.raises(skc.KernelError):
        skc.DenseKernel(np.ones((4, 4)))
    with pytest.raises(skc.KernelError):
        k.embedded(2)
    with pytest.raises(skc.KernelError):
        skc.disk_kernel(10.0, 21)   # violates the one-pixel border


def test_layer_and_complex_validation():
    with pytest.raises(skc.EngineError):
        skc.SparseLayer(np.zeros((0, 2)), np.zeros(0))
    with pytest.raises(skc.EngineError):
        skc.SparseLayer(np.array([[np.inf, 0.0]]), np.array([1.0]))
    with pytest.raises(skc.EngineError):
        skc.KernelComplex(())
    lay = skc.SparseLayer(np.array([[1.2, -0.4]]), np.array([1.0]))
    cpx = skc.KernelComplex((lay, lay))
    assert skc.required_canvas(cpx) == 7 and skc.auto_canvas(cpx) == 11
    assert cpx.taps().shape == (2, 3) and cpx.padded(4).shape == (2, 4, 3)


def test_config_recipes_deterministic_and_in_range():
    a = synth.disk_complex(4, 32, seed=1)
    b = synth.disk_complex(4, 32, seed=1)
    for la, lb in zip(a.layers, b.layers):
        assert np.array_equal(la.offsets, lb.offsets)
    for l, lay in enumerate(a.layers):
        assert np.hypot(*lay.offsets.T).max() <= 2 * 2 ** l + 1e-5
        assert abs(lay.weights.sum() - 1) < 1e-6 and (lay.weights > 0).all()
    kaw = synth.kawase_complex()
    assert kaw.layout == (4,) * 6 and kaw.reach == sum(0.5 + l for l in range(6))
    basis = synth.c2_basis()
    st = stacked_params(basis)
    np.testing.assert_allclose(st[2, :, :, :2], 4 * st[0, :, :, :2], rtol=1e-6, atol=1e-6)
    f = synth.value_noise_frame(300, 200, 3, seed=4)
    assert f.dtype == np.float32 and f.min() >= 0 and f.max() == 1.0
    assert np.array_equal(f, synth.value_noise_frame(300, 200, 3, seed=4))
    pm = synth.c2_pmap(200, 150)
    assert pm.min() >= 0 and pm.max() <= 1
    for i in range(5):
        t = synth.c4_target(i)
        assert t.size == 129 and abs(t.weights.sum() - 1) < 1e-12


def test_bracket_and_interp(golden):
    g = golden("sv")
    k0, k1, t = _bracket(g["bracket_p"], g["params"])
    assert np.array_equal(k0, g["bracket_k0"]) and np.array_equal(t, g["bracket_t"])
    basis = synth.c2_basis()
    np.testing.assert_array_equal(skc.interp_weights(0.5, basis), [0, 1, 0])
    np.testing.assert_allclose(skc.interp_weights(0.25, basis), [0.5, 0.5, 0])
    np.testing.assert_array_equal(skc.interp_weights(-3, basis), [1, 0, 0])
    np.testing.assert_array_equal(skc.interp_weights(9, basis), [0, 0, 1])
    f = skc.synthesize_filter([0, 0, 1], basis)
    assert np.array_equal(f.layers[0].offsets, basis.filters[2].layers[0].offsets)
    with pytest.raises(skc.EngineError, match="convex"):
        skc.synthesize_filter([0.7, 0.6, -0.3], basis)
    with pytest.raises(skc.EngineError, match="increasing"):
        skc.FilterBasis(np.array([1.0, 1.0]), basis.filters[:2])


def test_train_config_and_layout():
    cfg = skc.TrainConfig(steps=101, lr_start=1e-3, lr_end=1e-4)
    assert cfg.lr_at(0) == 1e-3
    assert cfg.lr_at(100) == pytest.approx(1e-4)
    assert cfg.lr_at(50) == pytest.approx((1e-3 + 1e-4) / 2)
    assert skc.parse_layout("4x32") == (32,) * 4
    for bad in ("0x4", "12", "3x-2"):
        with pytest.raises(skc.OptimError):
            skc.parse_layout(bad)
    with pytest.raises(skc.OptimError):
        skc.LossKind("huber")
    with pytest.raises(skc.OptimError):
        skc.TrainConfig(steps=0)


def test_loss_metric_known_answers():
    k = skc.gaussian_kernel(5)
    assert skc.loss(k, k, skc.LossKind("charbonnier", 1e-6)) == pytest.approx(961e-6, rel=1e-12)
    a = np.zeros((5, 5))
    b = a.copy()
    b[2, 3] = 0.3
    assert skc.loss(skc.DenseKernel(a), skc.DenseKernel(b), skc.LossKind("l2")) == pytest.approx(0.09)
    assert skc.psnr(a, a) == 99.0


def test_theta_roundtrip(tmp_path):
    cpx = synth.disk_complex(3, 5, seed=9)
    p = tmp_path / "t.json"
    skc.save_theta(cpx, p)
    back = skc.load_theta(p)
    for la, lb in zip(cpx.layers, back.layers):
        assert np.array_equal(la.offsets, lb.offsets) and np.array_equal(la.weights, lb.weights)


def test_kawase_exact_reach():
    """the strip halo is the exact corner reach sum(floor|o|+1) = 21."""
    from paper_2512_04556_b200.dist import corner_reach
    kaw = synth.kawase_complex()
    assert corner_reach(kaw) == (21, 21, 21, 21)
    assert math.ceil(kaw.reach) == 18


def test_initializers_bit_exact_vs_reference(golden):
    from paper_2512_04556_b200.initializers import InitStrategy, build_init, support_rejection_sample
    g = golden("init")
    for k in range(int(g["n_init"])):
        tgt = skc.DenseKernel(g[f"n{k}_tgt"])
        cpx = build_init(InitStrategy(str(g[f"n{k}_tag"]), seed=int(g[f"n{k}_seed"])), tgt,
                         tuple(g[f"n{k}_layout"].tolist()), kws=bool(g[f"n{k}_kws"]))
        off = np.concatenate([l.offsets for l in cpx.layers])
        w = np.concatenate([l.weights for l in cpx.layers])
        assert np.array_equal(off, g[f"n{k}_off"]), k
        assert np.array_equal(w, g[f"n{k}_w"]), k
    off, r = support_rejection_sample(skc.ring_kernel(5.0, 9.0, 23), 12, seed=5, return_radius=True)
    assert np.array_equal(off, g["srs_off"]) and r == float(g["srs_r"])


def test_kernelspec_parse_and_generate_vs_reference(golden):
    """KernelSpec.parse / generate_kernel (kernels.py:105-171), bit-exact."""
    g = golden("round2")
    for j, text in enumerate(g["spec_texts"].tolist()):
        sp = skc.KernelSpec.parse(text)
        assert repr(sp) == str(g[f"spec{j}_repr"]), text
        assert np.array_equal(skc.generate_kernel(sp).weights, g[f"spec{j}_k"]), text
    for bad in ("blob:3", "gaussian", "ring:3", "file", "polygon:x:3"):
        with pytest.raises(skc.KernelError):
            skc.generate_kernel(skc.KernelSpec.parse(bad))


def test_netpbm_bytes_match_reference(golden, tmp_path):
    """PGM/PPM writers and readers (kernels.py:314-435): identical bytes."""
    g = golden("round2")
    skc.save_kernel_image(skc.disk_kernel(3.3), tmp_path / "k.pgm")
    assert (tmp_path / "k.pgm").read_bytes() == g["pgm_kernel_bytes"].tobytes()
    assert np.array_equal(skc.load_kernel_image(tmp_path / "k.pgm").weights, g["pgm_kernel_loaded"])
    skc.write_image(g["img2"], tmp_path / "a.pgm")
    skc.write_image(g["img3"], tmp_path / "b.ppm", maxval=255)
    assert (tmp_path / "a.pgm").read_bytes() == g["pgm_img2_bytes"].tobytes()
    assert (tmp_path / "b.ppm").read_bytes() == g["ppm_img3_bytes"].tobytes()
    assert np.array_equal(skc.read_image(tmp_path / "a.pgm"), g["img2_read"])
    assert np.array_equal(skc.read_image(tmp_path / "b.ppm"), g["img3_read"])
    (tmp_path / "c.pgm").write_text("P2\n# a comment\n3 2\n# another\n10\n0 1 2\n3 4 10\n")
    assert np.array_equal(skc.read_image(tmp_path / "c.pgm"), g["ascii_read"])
    spec = skc.KernelSpec.parse(f"file:{tmp_path / 'k.pgm'}")
    assert np.array_equal(skc.generate_kernel(spec).weights, g["pgm_kernel_loaded"])
    (tmp_path / "bad.pgm").write_bytes(b"P7\n1 1\n255\n\x00")
    with pytest.raises(skc.KernelError):
        skc.read_image(tmp_path / "bad.pgm")
    (tmp_path / "trunc.pgm").write_bytes(b"P5\n4 4\n255\n\x00\x01")
    with pytest.raises(skc.KernelError):
        skc.read_image(tmp_path / "trunc.pgm")


def test_pst_config_validation_and_exports():
    """PSTConfig (baselines.py:93-114) and the top-level PST names (__init__.py:64-71)."""
    assert skc.PSTConfig().chains == 10 and skc.PSTConfig().iterations == 10000
    for kw in ({"chains": 1}, {"iterations": 0}, {"swap_interval": 0}, {"t_max": 1e-3, "t_min": 1e-2}):
        with pytest.raises(skc.KernelError):
            skc.PSTConfig(**kw)
    from paper_2512_04556_b200 import baselines
    assert skc.pst_fit is baselines.pst_fit and skc.PSTResult is baselines.PSTResult
    draws = baselines._numpy_draws(skc.PSTConfig(chains=3, iterations=4, swap_interval=2, seed=9), 2, 5)
    rng = np.random.default_rng(9)
    for it in range(4):   # the reference's draw order, one record per iteration
        assert np.array_equal(draws[it, :60], 1.0 * rng.normal(0.0, 1.0, size=60))
        assert np.array_equal(draws[it, 60:90], rng.normal(0.0, 1.0, size=30))
        assert np.array_equal(draws[it, 90:93], rng.uniform(size=3))
        if (it + 1) % 2 == 0:
            assert np.array_equal(draws[it, 93:], [rng.uniform(), rng.uniform()])
        else:
            assert not draws[it, 93:].any()


def test_kawase_generated_h_bodies():
    """The peeled horizontal pass bodies gen_kawase.py emits for the fused
    Kawase kernel equal the direct chain of 1-D sums (engine.py:173-178 in its
    separable form) for every instantiated ladder and row split."""
    import importlib.util
    from pathlib import Path
    spec = importlib.util.spec_from_file_location(
        "kawase_gen_check", Path(__file__).resolve().parent.parent / "tools" / "kawase_gen_check.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    for scalar in (False, True):
        mod.check_peel(scalar)
        mod.check_loop(scalar)
