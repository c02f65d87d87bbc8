"""Differentiable fitting of kernel complexes on the B200.

Drop-in for the reference optim module (/root/reference/pkg/src/sparsekern/
optim.py).  `backward`, `adam_step` and `fit` keep the reference signatures and
semantics; the work runs in csrc/skc_fit.cu: one CTA per target kernel runs
the whole loop on device (forward on the impulse, loss, analytic backward,
Adam with the offset learning-rate scale, KWS/SUM projections, best-so-far
tracking, canvas growth).  `fit_batch` fits many targets in one launch -- the
BASELINE config-4 workload.

Arithmetic is fp32 (reductions in float64); the reference is float64.  Parity
is judged per step and on batch statistics: the L1 fit
is chaotic, so individual long trajectories diverge from any reordering of
the sums, including the reference's own.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from ._tensors import torch
from .engine import KernelComplex, SparseLayer, auto_canvas
from .kernels import DenseKernel

__all__ = [
    "OptimError",
    "LossKind",
    "ConstraintConfig",
    "TrainConfig",
    "FitResult",
    "loss",
    "backward",
    "backward_batch",
    "AdamState",
    "adam_step",
    "fit",
    "fit_batch",
    "parse_layout",
    "save_theta",
    "load_theta",
    "theta_to_dict",
    "theta_from_dict",
    "write_trace_csv",
]

SUM_DEGENERACY_EPS = 1e-8


class OptimError(RuntimeError):
    """optim.py:55-56"""


@dataclass(frozen=True)
class LossKind:
    kind: str = "charbonnier"  # charbonnier | l1 | l2
    epsilon: float = 1e-6

    def __post_init__(self):
        if self.kind not in ("charbonnier", "l1", "l2"):
            raise OptimError(f"unknown loss kind {self.kind!r}")
        if self.epsilon <= 0:
            raise OptimError(f"loss epsilon must be positive, got {self.epsilon}")


@dataclass(frozen=True)
class ConstraintConfig:
    weight_norm: str = "sum"  # none | sum | sofm
    symmetry: str = "none"    # none | kws

    def __post_init__(self):
        if self.weight_norm not in ("none", "sum", "sofm"):
            raise OptimError(f"unknown weight norm {self.weight_norm!r}")
        if self.symmetry not in ("none", "kws"):
            raise OptimError(f"unknown symmetry constraint {self.symmetry!r}")


@dataclass(frozen=True)
class TrainConfig:
    steps: int = 1000
    lr_start: float = 1e-3
    lr_end: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 0

    def __post_init__(self):
        if self.steps < 1:
            raise OptimError(f"steps must be >= 1, got {self.steps}")
        if not self.lr_start >= self.lr_end > 0:
            raise OptimError(f"need lr_start >= lr_end > 0, got {self.lr_start}, {self.lr_end}")

    def lr_at(self, step: int) -> float:
        """Linear decay (optim.py:101-105)."""
        if self.steps == 1:
            return self.lr_start
        t = min(max(step, 0), self.steps - 1)
        return self.lr_start + (self.lr_end - self.lr_start) * t / (self.steps - 1)


def parse_layout(text) -> tuple:
    """'LxN' or explicit per-layer counts (optim.py:108-122)."""
    if isinstance(text, str):
        try:
            nl, ns = (int(v) for v in text.lower().split("x"))
        except ValueError as exc:
            raise OptimError(f"cannot parse layout {text!r} (expected LxN)") from exc
        if nl < 1 or ns < 1:
            raise OptimError(f"layout must have positive layers and samples, got {text!r}")
        return (ns,) * nl
    layout = tuple(int(n) for n in text)
    if not layout or any(n < 1 for n in layout):
        raise OptimError(f"layout must have positive sample counts, got {layout}")
    return layout


def loss(k_syn: DenseKernel, k_tgt: DenseKernel, kind: LossKind = LossKind()) -> float:
    """Pixel-summed loss of two responses, smaller one embedded (optim.py:149-152).

    A host metric on two host kernels (like psnr/sse); the fit computes its
    loss inside the fit kernel."""
    size = max(k_syn.size, k_tgt.size)
    d = k_syn.embedded(size).weights - k_tgt.embedded(size).weights
    if kind.kind == "charbonnier":
        return float(np.sum(np.sqrt(d * d + kind.epsilon * kind.epsilon)))
    if kind.kind == "l1":
        return float(np.sum(np.abs(d)))
    return float(np.sum(d * d))


def _raise_status(st, what: str):
    code, layer, sample = int(st[0]), int(st[1]), int(st[2])
    if code == nat.SKC_ENONFINITE:
        raise OptimError(f"non-finite intermediate at layer {layer}"
                         + (f", sample {sample}" if sample >= 0 else " (accumulated overflow)"))
    if code == nat.SKC_EDEGENERATE:
        raise OptimError(f"SUM normalization degenerate at layer {layer}: |weight sum| < {SUM_DEGENERACY_EPS}")
    if code == nat.SKC_ETRUNC:
        raise OptimError(f"{what}: canvas grew beyond the device limit at step {int(st[3])} (diverging fit)")
    if code != nat.SKC_OK:
        raise OptimError(f"{what}: device status {code}")


def _targets(tgts):
    if isinstance(tgts, DenseKernel):
        tgts = [tgts]
    if isinstance(tgts, np.ndarray) and tgts.ndim == 3:
        arr = tgts
    else:
        arr = np.stack([t.weights if isinstance(t, DenseKernel) else np.asarray(t) for t in tgts])
    if arr.shape[1] != arr.shape[2] or arr.shape[1] % 2 == 0:
        raise OptimError(f"targets must be odd square, got {arr.shape[1:]}")
    return np.ascontiguousarray(arr, dtype=np.float32)


def backward_batch(cpxs, tgts, kind: LossKind = LossKind(), canvas: int | None = None):
    """Loss and gradients of B complexes against B targets in one launch."""
    t = torch()
    lib = nat.lib()
    cpxs = list(cpxs)
    layout = cpxs[0].layout
    if any(c.layout != layout for c in cpxs):
        raise OptimError("backward_batch needs one shared layout")
    tg = _targets(tgts)
    bsz, m = tg.shape[0], tg.shape[1]
    if canvas is None:
        canvas = max(max(auto_canvas(c) for c in cpxs), m)
    nmax = max(layout)
    taps = np.stack([c.padded(nmax) for c in cpxs])
    dev = t.device("cuda", t.cuda.current_device())
    d_taps = t.from_numpy(taps).to(dev)
    d_tg = t.from_numpy(tg).to(dev)
    d_loss = t.empty(bsz, dtype=t.float32, device=dev)
    d_grads = t.empty((bsz, len(layout), nmax, 3), dtype=t.float32, device=dev)
    d_st = t.zeros((bsz, 4), dtype=t.int32, device=dev)
    lay = np.ascontiguousarray(layout, dtype=np.int32)
    rc = lib.skc_backward_batch(nat.ptr(d_taps), bsz, nat.ints(lay), lay.size, nmax, nat.ptr(d_tg), m,
                                canvas, nat.LOSS_IDS[kind.kind], kind.epsilon, nat.ptr(d_loss),
                                nat.ptr(d_grads), nat.ptr(d_st), nat.stream_ptr())
    if rc == nat.SKC_EBADARG:
        raise OptimError(f"backward: {nat.last_error()}")
    nat.check(rc, "backward")
    st = d_st.cpu().numpy()
    for b in range(bsz):
        _raise_status(st[b], "backward")
    losses = d_loss.cpu().numpy().astype(np.float64)
    grads = d_grads.cpu().numpy().astype(np.float64)
    out = []
    for b in range(bsz):
        per = []
        for l, n in enumerate(layout):
            per.append((grads[b, l, :n, :2].copy(), grads[b, l, :n, 2].copy()))
        out.append((float(losses[b]), per))
    return out


def backward(cpx: KernelComplex, k_tgt: DenseKernel, kind: LossKind = LossKind(),
             canvas: int | None = None):
    """Loss and gradients over every offset and weight (optim.py:278-292).

    Returns (loss, [(d_offsets (N,2), d_weights (N,)) per layer])."""
    if canvas is None:
        canvas = max(auto_canvas(cpx), k_tgt.size)
    return backward_batch([cpx], [k_tgt], kind, canvas)[0]


@dataclass
class AdamState:
    """optim.py:298-309"""
    m: list
    v: list
    step: int = 0

    @classmethod
    def for_params(cls, params) -> "AdamState":
        return cls(m=[[np.zeros_like(o), np.zeros_like(w)] for o, w in params],
                   v=[[np.zeros_like(o), np.zeros_like(w)] for o, w in params])


def _pack(rows) -> np.ndarray:
    return np.ascontiguousarray(
        np.concatenate([np.concatenate([np.asarray(o, np.float64).reshape(-1, 2),
                                        np.asarray(w, np.float64).reshape(-1, 1)], axis=1)
                        for o, w in rows]), dtype=np.float32)


def _unpack(flat, layout, into=None):
    out, base = [], 0
    for l, n in enumerate(layout):
        o = flat[base:base + n, :2].astype(np.float64)
        w = flat[base:base + n, 2].astype(np.float64)
        if into is not None:
            into[l][0][...] = o
            into[l][1][...] = w
        out.append([o, w])
        base += n
    return out


def _cfg(cfg: TrainConfig, constraints: ConstraintConfig, loss_kind: LossKind):
    return nat.fit_cfg(cfg.steps, cfg.lr_start, cfg.lr_end, cfg.beta1, cfg.beta2, cfg.eps,
                       constraints.weight_norm, constraints.symmetry == "kws", loss_kind.kind,
                       loss_kind.epsilon)


def adam_step(params, grads, state: AdamState, step_index: int, cfg: TrainConfig,
              constraints: ConstraintConfig = ConstraintConfig(), offset_lr_scale: float = 1.0):
    """One Adam update with bias correction, then KWS/SUM projections (optim.py:338-369)."""
    t = torch()
    lib = nat.lib()
    layout = tuple(int(np.asarray(o).reshape(-1, 2).shape[0]) for o, _ in params)
    if constraints.symmetry == "kws" and any(n % 4 for n in layout):
        raise OptimError(f"KWS symmetry needs sample counts divisible by 4, got {layout}")
    dev = t.device("cuda", t.cuda.current_device())
    d_p = t.from_numpy(_pack(params)).to(dev)
    d_g = t.from_numpy(_pack(grads)).to(dev)
    d_m = t.from_numpy(_pack(state.m)).to(dev)
    d_v = t.from_numpy(_pack(state.v)).to(dev)
    d_st = t.zeros(4, dtype=t.int32, device=dev)
    lay = np.ascontiguousarray(layout, dtype=np.int32)
    c = _cfg(cfg, constraints, LossKind())
    nat.check(lib.skc_adam_step(nat.ptr(d_p), nat.ptr(d_g), nat.ptr(d_m), nat.ptr(d_v),
                                nat.ints(lay), lay.size, int(step_index), c,
                                float(offset_lr_scale), nat.ptr(d_st), nat.stream_ptr()),
              "adam_step")
    _raise_status(d_st.cpu().numpy(), "adam_step")
    _unpack(d_m.cpu().numpy(), layout, state.m)
    _unpack(d_v.cpu().numpy(), layout, state.v)
    state.step = step_index + 1
    return _unpack(d_p.cpu().numpy(), layout)


@dataclass
class FitResult:
    """optim.py:375-387"""
    complex: KernelComplex
    trace: np.ndarray          # rows of (step, loss, lr)
    best_loss: float
    best_step: int
    initial_loss: float
    final_loss: float
    canvas: int

    @property
    def losses(self) -> np.ndarray:
        return self.trace[:, 1]


def _resolve_init(init, k_tgt, layout, kws):
    if isinstance(init, KernelComplex):
        return init
    from .initializers import build_init
    return build_init(init, k_tgt, layout, kws=kws)


def fit_batch(targets, layout, inits, cfg: TrainConfig = TrainConfig(),
              constraints: ConstraintConfig = ConstraintConfig(),
              loss_kind: LossKind = LossKind(), return_device: bool = False):
    """Fit B independent targets in one persistent launch (one CTA per target).

    targets: sequence of DenseKernel (one size M) or array (B, M, M);
    inits: sequence of KernelComplex (optim.py:404-405 warm starts) or one
    init/InitStrategy applied to every target.  Returns a list of FitResult.
    """
    t = torch()
    lib = nat.lib()
    layout = parse_layout(layout)
    if constraints.symmetry == "kws" and any(n % 4 for n in layout):
        raise OptimError(f"KWS symmetry needs sample counts divisible by 4, got {layout}")
    tg = _targets(targets)
    bsz, m = tg.shape[0], tg.shape[1]
    if not isinstance(inits, (list, tuple)):
        inits = [inits] * bsz
    if len(inits) != bsz:
        raise OptimError(f"{len(inits)} inits for {bsz} targets")
    kt = [DenseKernel(tg[b].astype(np.float64)) for b in range(bsz)]
    starts = [_resolve_init(i, kt[b], layout, constraints.symmetry == "kws")
              for b, i in enumerate(inits)]
    for s in starts:
        if s.layout != layout:
            raise OptimError(f"init layout {s.layout} does not match requested {layout}")
    nmax = max(layout)
    nl = len(layout)
    dev = t.device("cuda", t.cuda.current_device())
    init_taps = t.from_numpy(np.stack([s.padded(nmax) for s in starts])).to(dev)
    d_tg = t.from_numpy(tg).to(dev)
    stride = nat.FIT_HDR + 6 * nl * nmax * 3
    state = t.zeros((bsz, stride), dtype=t.float32, device=dev)
    trace = t.full((bsz, cfg.steps + 1), float("nan"), dtype=t.float32, device=dev)
    status = t.zeros((bsz, 4), dtype=t.int32, device=dev)
    lay = np.ascontiguousarray(layout, dtype=np.int32)
    c = _cfg(cfg, constraints, loss_kind)
    sp = nat.stream_ptr()
    nat.check(lib.skc_fit_init(nat.ptr(state), nat.ptr(init_taps), bsz, nat.ints(lay), nl, nmax, m,
                               c, nat.ptr(status), sp), "fit_init")
    st = status.cpu().numpy()
    for b in range(bsz):
        _raise_status(st[b], "fit")
    nat.check(lib.skc_fit_run(nat.ptr(state), bsz, nat.ints(lay), nl, nmax, nat.ptr(d_tg), m, c,
                              nat.ptr(trace), nat.ptr(status), sp), "fit")
    if return_device:
        return state, trace, status
    return collect_fit(state, trace, status, layout, cfg)


def collect_fit(state, trace, status, layout, cfg: TrainConfig):
    """Host-side FitResults from the device fit state."""
    layout = tuple(layout)
    nl, nmax = len(layout), max(layout)
    st = status.cpu().numpy()
    sta = state.cpu().numpy()
    tr = trace.cpu().numpy().astype(np.float64)
    hdr = sta[:, :nat.FIT_HDR].copy().view(np.int32)
    blk = nl * nmax * 3
    lrs = np.array([cfg.lr_at(s) for s in range(cfg.steps)] + [cfg.lr_at(cfg.steps - 1)])
    results = []
    for b in range(sta.shape[0]):
        _raise_status(st[b], "fit")
        best = sta[b, nat.FIT_HDR + 3 * blk:nat.FIT_HDR + 4 * blk].reshape(nl, nmax, 3)
        layers = tuple(SparseLayer(best[l, :n, :2].astype(np.float64), best[l, :n, 2].astype(np.float64))
                       for l, n in enumerate(layout))
        trace_rows = np.stack([np.arange(cfg.steps + 1, dtype=np.float64), tr[b], lrs], axis=1)
        results.append(FitResult(
            complex=KernelComplex(layers), trace=trace_rows, best_loss=float(sta[b, 2]),
            best_step=int(hdr[b, 3]), initial_loss=float(tr[b, 0]), final_loss=float(tr[b, -1]),
            canvas=int(hdr[b, 1])))
    return results


def fit(k_tgt: DenseKernel, layout, init, cfg: TrainConfig = TrainConfig(),
        constraints: ConstraintConfig = ConstraintConfig(),
        loss_kind: LossKind = LossKind()) -> FitResult:
    """Optimise a complex against a target response (optim.py:390-469)."""
    return fit_batch([k_tgt], layout, [init], cfg, constraints, loss_kind)[0]


# ------------------------------------------------------- serialization ---
# Host JSON, same schema as optim.py:475-514.

def theta_to_dict(cpx: KernelComplex) -> dict:
    return {"layers": [{"samples": [{"ox": float(ox), "oy": float(oy), "w": float(w)}
                                    for (ox, oy), w in zip(l.offsets, l.weights)]}
                       for l in cpx.layers]}


def theta_from_dict(doc: dict) -> KernelComplex:
    layers = []
    for lay in doc["layers"]:
        off = np.array([[s["ox"], s["oy"]] for s in lay["samples"]], dtype=np.float64)
        wts = np.array([s["w"] for s in lay["samples"]], dtype=np.float64)
        layers.append(SparseLayer(off, wts))
    return KernelComplex(tuple(layers))


def save_theta(cpx: KernelComplex, path) -> None:
    with open(path, "w") as fh:
        json.dump(theta_to_dict(cpx), fh, indent=1)
        fh.write("\n")


def load_theta(path) -> KernelComplex:
    with open(path) as fh:
        return theta_from_dict(json.load(fh))


def write_trace_csv(trace: np.ndarray, path) -> None:
    with open(path, "w") as fh:
        fh.write("step,loss,lr\n")
        for step, value, lr in trace:
            fh.write(f"{int(step)},{float(value)!r},{float(lr)!r}\n")
