"""GPU parity of the fused separable Kawase kernel (csrc/skc_kawase.cu): the
config-3 chain on fp16 RGBA against the float64 oracle of engine.apply_complex
(engine.py:173-178) on the same fp16-decoded inputs, tolerance 2e-3 normwise
(north star, fp16 storage).  Full benchmark frames, ragged shapes, every
instantiated ladder length, weights other than 1/4, and the fall-back cases
(clamp boundary, odd width, non-Kawase taps) that must take the per-layer path.
"""

import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu

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
    oracle.set_threads(0)
    return oracle


def _layers(cpx):
    return [(l.offsets, l.weights) for l in cpx.layers]


def _is_fused(cpx, h, w, c=4, dt=1):
    from paper_2512_04556_b200 import _native as nat
    taps = np.ascontiguousarray(cpx.taps())
    lay = np.ascontiguousarray(cpx.layout, dtype=np.int32)
    return bool(nat.lib().skc_chain_is_fused(nat.dbl(taps), nat.ints(lay), lay.size, h, w, c, dt))


def test_c3_full_frames_0_and_31(skc, orc):
    """Benchmark frames 0 and 31 of config 3 (2160 x 3840 x 4 fp16), both
    through one batched call as the bench runs them."""
    import torch
    from paper_2512_04556_b200 import synth
    cpx = synth.kawase_complex()
    assert _is_fused(cpx, 2160, 3840)
    frames = np.stack([synth.c3_frame(0), synth.c3_frame(31)])
    out = skc.apply_complex_batch(torch.from_numpy(frames).cuda(), cpx).cpu().numpy()
    for k in range(2):
        ref = orc.apply_complex(frames[k].astype(np.float64), _layers(cpx), orc.ZERO)
        assert normwise(out[k].astype(np.float64), ref) < TOL16
        # the bound holds per pixel too, relative to the image's peak
        assert np.abs(out[k].astype(np.float64) - ref).max() <= 2e-3 * np.abs(ref).max()


@pytest.mark.parametrize("shape", [(1, 2, 4), (3, 130, 4), (37, 258, 4), (300, 128, 4), (129, 384, 4), (2, 2, 4),
                                   (75, 1000, 4)])
def test_ragged_shapes(skc, orc, shape):
    from paper_2512_04556_b200 import synth
    cpx = synth.kawase_complex()
    rng = np.random.default_rng(sum(shape))
    img = rng.random(shape).astype(np.float16)
    assert _is_fused(cpx, shape[0], shape[1])
    out = skc.apply_complex(img, cpx)
    ref = orc.apply_complex(img.astype(np.float64), _layers(cpx), orc.ZERO)
    assert normwise(out.astype(np.float64), ref) < TOL16


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 6])
def test_every_ladder_and_weights(skc, orc, L):
    """L = 1..6 and per-layer weights w_l != 1/4 (scale prod w_l / 4), signed input."""
    rng = np.random.default_rng(L)
    layers = []
    for l in range(L):
        r = 0.5 + l
        w = rng.uniform(0.1, 0.6)
        layers.append(skc.SparseLayer(np.array([[r, r], [-r, r], [-r, -r], [r, -r]]), np.full(4, w)))
    cpx = skc.KernelComplex(tuple(layers))
    img = (rng.random((150, 270, 4)) - 0.3).astype(np.float16)
    assert _is_fused(cpx, 150, 270)
    out = skc.apply_complex(img, cpx)
    ref = orc.apply_complex(img.astype(np.float64), _layers(cpx), orc.ZERO)
    assert normwise(out.astype(np.float64), ref) < TOL16


def test_batch_of_frames_equals_single(skc):
    import torch
    from paper_2512_04556_b200 import synth
    cpx = synth.kawase_complex()
    rng = np.random.default_rng(5)
    frames = torch.from_numpy(rng.random((3, 97, 300, 4)).astype(np.float16)).cuda()
    batched = skc.apply_complex_batch(frames, cpx)
    for k in range(3):
        assert torch.equal(batched[k], skc.apply_complex(frames[k], cpx))


def test_fallbacks_keep_parity(skc, orc):
    """Clamp boundary, odd width, a non-ladder radius and fp32 storage take the
    per-layer path; results still match the oracle."""
    from paper_2512_04556_b200 import synth
    cpx = synth.kawase_complex()
    rng = np.random.default_rng(9)
    img = rng.random((64, 91, 4)).astype(np.float16)
    assert not _is_fused(cpx, 64, 91)
    out = skc.apply_complex(img, cpx)
    assert normwise(out.astype(np.float64), orc.apply_complex(img.astype(np.float64), _layers(cpx))) < TOL16
    img = rng.random((64, 90, 4)).astype(np.float16)
    out = skc.apply_complex(img, cpx, boundary="clamp")
    ref = orc.apply_complex(img.astype(np.float64), _layers(cpx), orc.CLAMP)
    assert normwise(out.astype(np.float64), ref) < TOL16
    odd = skc.KernelComplex((skc.SparseLayer(np.array([[1.5, 1.5], [-1.5, 1.5], [-1.5, -1.5], [1.5, -1.5]]),
                                             np.full(4, 0.25)),))
    assert not _is_fused(odd, 64, 90)
    out = skc.apply_complex(img, odd)
    assert normwise(out.astype(np.float64), orc.apply_complex(img.astype(np.float64), _layers(odd))) < TOL16


def test_kernel_variants_keep_parity(skc, orc):
    """The Kawase kernel's switches -- SKC_KAWASE_LV=1 (the V lanes apply the
    last horizontal layer), SKC_KAWASE_PEEL=0 (rolled H loop everywhere),
    SKC_KAWASE_SC=1 (one channel per H lane, setmaxnreg), SKC_KAWASE_HS=1 (whole
    band rows per lane) -- each in a fresh process, against the oracle on frames
    with image edges inside a band, more than one band and more than one row
    segment; interior pixels of the variants that share the summation order
    agree bit for bit."""
    import os
    import subprocess
    import sys
    import tempfile
    from paper_2512_04556_b200 import synth
    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "import paper_2512_04556_b200 as skc; from paper_2512_04556_b200 import synth;"
            "img = np.load(sys.argv[1]); np.save(sys.argv[2], skc.apply_complex(img, synth.kawase_complex()))")
    root = str(__import__("pathlib").Path(__file__).parent.parent)
    cpx = synth.kawase_complex()
    rng = np.random.default_rng(11)
    variants = ({"SKC_KAWASE_LV": "1"}, {}, {"SKC_KAWASE_PEEL": "0"}, {"SKC_KAWASE_LV": "1", "SKC_KAWASE_PEEL": "0"},
                {"SKC_KAWASE_SC": "1"}, {"SKC_KAWASE_HS": "1"})
    with tempfile.TemporaryDirectory() as td:
        for shape in ((700, 300, 4), (90, 130, 4), (333, 1026, 4)):
            img = (rng.random(shape) - 0.2).astype(np.float16)
            np.save(f"{td}/in.npy", img)
            ref = orc.apply_complex(img.astype(np.float64), _layers(cpx), orc.ZERO)
            outs = []
            for var in variants:
                subprocess.run([sys.executable, "-c", code, f"{td}/in.npy", f"{td}/o.npy"], check=True,
                               env=dict(os.environ, **var), cwd=root)
                out = np.load(f"{td}/o.npy")
                assert normwise(out.astype(np.float64), ref) < TOL16, (shape, var)
                outs.append(out)
            # with and without the peeled warm-up the same additions run in the same order
            assert np.array_equal(outs[1], outs[2]), shape
            assert np.array_equal(outs[0], outs[3]), shape
