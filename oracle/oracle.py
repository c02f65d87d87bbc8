"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU float64 oracle.

The oracle (oracle/skc_oracle.c) restates the reference `sparsekern` hot path
(/root/reference/pkg/src/sparsekern: engine.py, svfilter.py, _fastpath.py,
optim.py) in float64 C.  It is the parity checker for the CUDA product path
and the CPU baseline of bench.py.  Nothing under paper_2512_04556_b200/ may
import this module; only tests/, __graft_entry__.smoke() and bench.py do.

Pinning: tests/test_oracle.py compares every function here with fixtures the
unmodified reference produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libskc_oracle.so"

ZERO, CLAMP = 0, 1
LOSS_IDS = {"charbonnier": 0, "l1": 1, "l2": 2}
WN_IDS = {"none": 0, "sum": 1, "sofm": 2}

_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)


class FitCfg(ctypes.Structure):
    _fields_ = [
        ("steps", ctypes.c_int64),
        ("lr_start", ctypes.c_double),
        ("lr_end", ctypes.c_double),
        ("beta1", ctypes.c_double),
        ("beta2", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("weight_norm", ctypes.c_int),
        ("kws", ctypes.c_int),
        ("loss_kind", ctypes.c_int),
        ("loss_eps", ctypes.c_double),
    ]


def build() -> Path:
    """Compile the oracle with its Makefile (gcc only; seconds)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(LIB_PATH))
        _lib.or_num_threads.restype = ctypes.c_int
        _lib.or_backward.restype = ctypes.c_int64
        _lib.or_backward_g.restype = ctypes.c_int64
        _lib.or_fit.restype = ctypes.c_int
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def num_threads() -> int:
    return int(lib().or_num_threads())


def _d(a):
    return a.ctypes.data_as(_D)


def _i(a):
    return a.ctypes.data_as(_I)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _as_hwc(img):
    img = _f64(img)
    if img.ndim == 2:
        return img[:, :, None], True
    return img, False


def _flat_taps(layers):
    """layers: sequence of (offsets (N,2), weights (N,)) -> flat arrays + layout."""
    offs = [np.asarray(o, dtype=np.float64).reshape(-1, 2) for o, _ in layers]
    wts = [np.asarray(w, dtype=np.float64).reshape(-1) for _, w in layers]
    layout = np.array([o.shape[0] for o in offs], dtype=np.int64)
    return _f64(np.concatenate(offs)), _f64(np.concatenate(wts)), layout


def apply_layer(img, offsets, weights, boundary=ZERO):
    """engine.py:160-170 apply_sparse_layer (boundary=CLAMP: SURVEY D1)."""
    x, squeeze = _as_hwc(img)
    h, w, c = x.shape
    off = _f64(np.asarray(offsets).reshape(-1, 2))
    wt = _f64(np.asarray(weights).reshape(-1))
    out = np.empty_like(x)
    lib().or_apply_layer(_d(x), _d(out), ctypes.c_int64(h), ctypes.c_int64(w), ctypes.c_int64(c),
                         _d(off), _d(wt), ctypes.c_int64(off.shape[0]), ctypes.c_int(boundary))
    return out[:, :, 0] if squeeze else out


def apply_complex(img, layers, boundary=ZERO):
    """engine.py:173-178 apply_complex; layers = [(offsets, weights), ...]."""
    x, squeeze = _as_hwc(img)
    h, w, c = x.shape
    off, wt, layout = _flat_taps(layers)
    out = np.empty_like(x)
    lib().or_apply_complex(_d(x), _d(out), ctypes.c_int64(h), ctypes.c_int64(w),
                           ctypes.c_int64(c), _d(off), _d(wt), _i(layout),
                           ctypes.c_int64(layout.size), ctypes.c_int(boundary))
    return out[:, :, 0] if squeeze else out


def ir_batch(offsets, weights, layout, canvas):
    """engine.py:251-303 synthesize_ir_batch: offsets (B,L,N,2), weights (B,L,N)."""
    off = _f64(offsets)
    wt = _f64(weights)
    b, nl, nmax = wt.shape
    lay = np.asarray(layout, dtype=np.int64)
    out = np.empty((b, canvas, canvas))
    lib().or_ir_batch(_d(off), _d(wt), _i(lay), ctypes.c_int64(nl), ctypes.c_int64(b),
                      ctypes.c_int64(nmax), ctypes.c_int64(canvas), _d(out))
    return out


def synthesize_ir(layers, canvas):
    off, wt, layout = _flat_taps(layers)
    nmax = int(layout.max())
    L = layout.size
    o = np.zeros((1, L, nmax, 2))
    w = np.zeros((1, L, nmax))
    base = 0
    for l, n in enumerate(layout):
        o[0, l, :n] = off[base:base + n]
        w[0, l, :n] = wt[base:base + n]
        base += n
    return ir_batch(o, w, layout, canvas)[0]


def sv_filter(img, pmap, params, basis, layout, boundary=ZERO):
    """svfilter.py:171-203 / _fastpath.py:97-150.  basis (Mb, L, Nmax, 3)."""
    x, squeeze = _as_hwc(img)
    h, w, c = x.shape
    pm = _f64(pmap)
    ps = _f64(params)
    bs = _f64(basis)
    lay = np.asarray(layout, dtype=np.int64)
    out = np.empty_like(x)
    lib().or_sv_filter(_d(x), _d(out), ctypes.c_int64(h), ctypes.c_int64(w), ctypes.c_int64(c),
                       _d(pm), _d(ps), ctypes.c_int64(ps.size), _d(bs), _i(lay),
                       ctypes.c_int64(lay.size), ctypes.c_int64(bs.shape[2]),
                       ctypes.c_int(boundary))
    return out[:, :, 0] if squeeze else out


class OracleError(RuntimeError):
    pass


def backward(layers, tgt_embedded, kind="charbonnier", eps=1e-6):
    """optim.py:278-292 backward() at the canvas of `tgt_embedded` (odd square)."""
    off, wt, layout = _flat_taps(layers)
    tgt = _f64(tgt_embedded)
    canvas = tgt.shape[0]
    d_off = np.zeros_like(off)
    d_w = np.zeros_like(wt)
    value = ctypes.c_double(0.0)
    bad = ctypes.c_int64(-1)
    rc = lib().or_backward(_d(off), _d(wt), _i(layout), ctypes.c_int64(layout.size),
                           ctypes.c_int64(canvas), _d(tgt), ctypes.c_int(LOSS_IDS[kind]),
                           ctypes.c_double(eps), ctypes.byref(value), _d(d_off), _d(d_w),
                           ctypes.byref(bad))
    if rc >= 0:
        raise OracleError(f"non-finite intermediate at layer {rc}")
    grads, base = [], 0
    for n in layout:
        grads.append((d_off[base:base + n].copy(), d_w[base:base + n].copy()))
        base += n
    return float(value.value), grads


def backward_with_grad(layers, g):
    """_backward_pass (optim.py:231-263) driven by an explicit upstream
    gradient g (canvas, canvas) -- e.g. the sign pattern an fp32 forward
    produced -- instead of the loss gradient.  Returns the per-layer grads."""
    off, wt, layout = _flat_taps(layers)
    g = _f64(g)
    canvas = g.shape[0]
    d_off = np.zeros_like(off)
    d_w = np.zeros_like(wt)
    bad = ctypes.c_int64(-1)
    rc = lib().or_backward_g(_d(off), _d(wt), _i(layout), ctypes.c_int64(layout.size), ctypes.c_int64(canvas),
                             _d(g), _d(d_off), _d(d_w), ctypes.byref(bad))
    if rc >= 0:
        raise OracleError(f"non-finite intermediate at layer {rc}")
    grads, base = [], 0
    for n in layout:
        grads.append((d_off[base:base + n].copy(), d_w[base:base + n].copy()))
        base += n
    return grads


def _cfg(steps, lr_start, lr_end, beta1, beta2, eps, weight_norm, kws, loss_kind, loss_eps):
    return FitCfg(int(steps), float(lr_start), float(lr_end), float(beta1), float(beta2),
                  float(eps), WN_IDS[weight_norm], int(bool(kws)), LOSS_IDS[loss_kind],
                  float(loss_eps))


def fit_batch(tgts, init_offsets, init_weights, layout, steps=1000, lr_start=1e-3, lr_end=1e-4,
              beta1=0.9, beta2=0.999, eps=1e-8, weight_norm="sum", kws=False,
              loss_kind="charbonnier", loss_eps=1e-6):
    """optim.py:390-469 fit() with explicit inits, for B independent targets.

    tgts (B,M,M); init_offsets (B,P,2); init_weights (B,P) where P = sum(layout).
    Returns dict(trace (B,steps+1), best_offsets, best_weights, best_loss,
    best_step, canvas, rc).
    """
    t = _f64(tgts)
    b, m, _ = t.shape
    off0 = _f64(init_offsets)
    w0 = _f64(init_weights)
    lay = np.asarray(layout, dtype=np.int64)
    P = int(lay.sum())
    cfg = _cfg(steps, lr_start, lr_end, beta1, beta2, eps, weight_norm, kws, loss_kind, loss_eps)
    trace = np.zeros((b, steps + 1))
    bo = np.zeros((b, P, 2))
    bw = np.zeros((b, P))
    bl = np.zeros(b)
    info = np.zeros((b, 2), dtype=np.int64)
    err = np.full(b, -1, dtype=np.int64)
    rcs = np.zeros(b, dtype=np.int32)
    lib().or_fit_batch(_d(t), ctypes.c_int64(b), ctypes.c_int64(m), _d(off0), _d(w0), _i(lay),
                       ctypes.c_int64(lay.size), ctypes.byref(cfg), _d(trace), _d(bo), _d(bw),
                       _d(bl), _i(info), _i(err), rcs.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return dict(trace=trace, best_offsets=bo, best_weights=bw, best_loss=bl,
                best_step=info[:, 0].copy(), canvas=info[:, 1].copy(), rc=rcs, err_layer=err)
