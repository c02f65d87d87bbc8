"""Spatially varying filtering through filter-space interpolation, on the B200.

Drop-in for the reference svfilter (/root/reference/pkg/src/sparsekern/
svfilter.py): `FilterBasis`, `interp_weights`, `synthesize_filter` and
`sv_filter` keep the reference names, validation and semantics; the per-pixel
bracket, slotwise lerp of offsets/weights and the bilinear gather of every
pass run in csrc/skc_filter.cu (sv_tile_kernel) through `skc_sv_fwd`.
Offline basis building (`build_basis`, a loop over `fit`) lives in optim's
batched fit; `sv_ground_truth` and the 2-D grid basis are SURVEY section 8(f)
"next" rows.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from ._tensors import Image, torch
from .engine import BOUNDARIES, EngineError, KernelComplex, SparseLayer

__all__ = [
    "FilterBasis",
    "interp_weights",
    "synthesize_filter",
    "sv_filter",
    "stacked_params",
]


def _check_shared_layout(filters) -> tuple:
    layouts = {f.layout for f in filters}
    if len(layouts) != 1:
        raise EngineError(f"basis filters must share one layout, got {sorted(layouts)}")
    return layouts.pop()


@dataclass(frozen=True, eq=False)
class FilterBasis:
    """Basis complexes at strictly increasing scalar parameters (svfilter.py:53-78)."""

    params: np.ndarray
    filters: tuple

    def __post_init__(self):
        ps = np.array(self.params, dtype=np.float64).reshape(-1)
        filters = tuple(self.filters)
        if ps.size != len(filters) or ps.size < 1:
            raise EngineError("basis needs one filter per parameter")
        if ps.size > 1 and not (np.diff(ps) > 0).all():
            raise EngineError("basis parameters must be strictly increasing")
        _check_shared_layout(filters)
        ps.flags.writeable = False
        object.__setattr__(self, "params", ps)
        object.__setattr__(self, "filters", filters)

    @property
    def size(self) -> int:
        return int(self.params.size)

    @property
    def layout(self) -> tuple:
        return self.filters[0].layout


def _bracket(p, ps: np.ndarray):
    """Bracketing entries and blend factor (svfilter.py:129-137), host version
    used by interp_weights; the per-pixel version runs on device."""
    if ps.size == 1:
        z = np.zeros_like(p, dtype=np.int64)
        return z, z, np.zeros_like(p, dtype=np.float64)
    pc = np.clip(p, ps[0], ps[-1])
    k0 = np.clip(np.searchsorted(ps, pc, side="right") - 1, 0, ps.size - 2)
    t = (pc - ps[k0]) / (ps[k0 + 1] - ps[k0])
    return k0, k0 + 1, t


def interp_weights(p: float, basis: FilterBasis) -> np.ndarray:
    """Hat weights over the grid, at most 2 nonzeros (svfilter.py:116-126)."""
    alpha = np.zeros(basis.size)
    k0, k1, t = _bracket(np.asarray(p, dtype=np.float64), basis.params)
    alpha[int(k0)] += 1.0 - float(t)
    alpha[int(k1)] += float(t)
    return alpha


def synthesize_filter(alpha, basis: FilterBasis) -> KernelComplex:
    """Slotwise convex blend of the basis (svfilter.py:140-152)."""
    alpha = np.asarray(alpha, dtype=np.float64).reshape(-1)
    if alpha.size != basis.size:
        raise EngineError(f"alpha has {alpha.size} entries for a basis of {basis.size}")
    if abs(float(alpha.sum()) - 1.0) > 1e-9 or (alpha < -1e-12).any():
        raise EngineError("alpha must be convex: nonnegative and summing to 1")
    layers = []
    for l in range(len(basis.layout)):
        off = sum(a * f.layers[l].offsets for a, f in zip(alpha, basis.filters))
        wts = sum(a * f.layers[l].weights for a, f in zip(alpha, basis.filters))
        layers.append(SparseLayer(off, wts))
    return KernelComplex(tuple(layers))


def stacked_params(basis: FilterBasis) -> np.ndarray:
    """(Mb, L, Nmax, 3) float64 (ox, oy, w), zero-padded (svfilter.py:155-168)."""
    layout = basis.layout
    out = np.zeros((basis.size, len(layout), max(layout), 3))
    for k, f in enumerate(basis.filters):
        for l, lay in enumerate(f.layers):
            out[k, l, :lay.sample_count] = lay.taps()
    return out


def sv_filter(img, basis: FilterBasis, pmap, boundary: str = "zero", out=None):
    """Per-pixel blended sparse filtering guided by a parameter map (svfilter.py:171-203).

    Each pass re-interpolates that layer's taps per pixel between the two
    bracketing basis entries and gathers bilinearly from the previous pass.
    Host torch tensors (pinned) with a pinned `out` move with async copies.
    """
    t = torch()
    lib = nat.lib()
    im = Image(img)
    b, h, w, c = im.dims
    pm_shape = tuple(pmap.shape)
    if pm_shape != (h, w):
        raise EngineError(f"parameter map {pm_shape} must match image {(h, w)}")
    if isinstance(pmap, t.Tensor):
        pm = pmap.to(device=im.tensor.device, dtype=t.float32, non_blocking=pmap.is_pinned()).contiguous()
    else:
        pm = t.from_numpy(np.ascontiguousarray(pmap, dtype=np.float32)).to(im.tensor.device)
    if boundary not in BOUNDARIES:
        raise EngineError(f"boundary must be one of {sorted(BOUNDARIES)}, got {boundary!r}")
    stack = np.ascontiguousarray(stacked_params(basis))
    ps = np.ascontiguousarray(basis.params, dtype=np.float64)
    layout = np.ascontiguousarray(basis.layout, dtype=np.int32)
    res = im.empty_like()
    rc = lib.skc_sv_fwd(nat.ptr(im.tensor), im.dtype_id, nat.ptr(res), im.dtype_id, h, w, c,
                        nat.ptr(pm), nat.dbl(ps), ps.size, nat.dbl(stack), stack.shape[2],
                        nat.ints(layout), layout.size, BOUNDARIES[boundary], nat.stream_ptr())
    if rc == nat.SKC_EBADARG:
        raise EngineError(f"sv_filter: {nat.last_error()}")
    nat.check(rc, "sv_filter")
    return im.restore(res, out)


# ---------------------------------------------------------------------------
# SURVEY 8(f) "next" rows: 2-D parameter grid, basis building, JSON I/O.

@dataclass(frozen=True, eq=False)
class FilterBasisGrid:
    """(u, v) grid of basis complexes sharing one layout (svfilter.py:242-269)."""

    params_u: np.ndarray
    params_v: np.ndarray
    filters: tuple   # filters[iu][iv]

    def __post_init__(self):
        pu = np.array(self.params_u, dtype=np.float64).reshape(-1)
        pv = np.array(self.params_v, dtype=np.float64).reshape(-1)
        rows = tuple(tuple(r) for r in self.filters)
        if len(rows) != pu.size or any(len(r) != pv.size for r in rows):
            raise EngineError("grid basis shape must match parameter axes")
        if (pu.size > 1 and not (np.diff(pu) > 0).all()) or (pv.size > 1 and not (np.diff(pv) > 0).all()):
            raise EngineError("grid parameters must be strictly increasing")
        _check_shared_layout([f for row in rows for f in row])
        pu.flags.writeable = False
        pv.flags.writeable = False
        object.__setattr__(self, "params_u", pu)
        object.__setattr__(self, "params_v", pv)
        object.__setattr__(self, "filters", rows)

    @property
    def layout(self) -> tuple:
        return self.filters[0][0].layout

    def row_basis(self, iu: int) -> FilterBasis:
        return FilterBasis(self.params_v, self.filters[iu])


def sv_filter_grid(img, grid: FilterBasisGrid, pmap2, boundary: str = "zero"):
    """SV filtering from a 2-channel map (H, W, 2) over a grid basis (svfilter.py:292-319).

    Each pass blends the four bracketing entries' taps per pixel with weights
    (1-tu)(1-tv), tu(1-tv), (1-tu)tv, tu tv, then gathers bilinearly."""
    t = torch()
    lib = nat.lib()
    im = Image(img if not isinstance(img, np.ndarray) else img.astype(np.float32, copy=False))
    if im.dtype_id != nat.SKC_F32:
        im.tensor = im.tensor.float()
        im.dtype_id = nat.SKC_F32
    b, h, w, c = im.dims
    if tuple(pmap2.shape) != (h, w, 2):
        raise EngineError(f"2D map must be {(h, w, 2)}, got {tuple(pmap2.shape)}")
    if boundary not in BOUNDARIES:
        raise EngineError(f"boundary must be one of {sorted(BOUNDARIES)}, got {boundary!r}")
    pm = (pmap2.to(device=im.tensor.device, dtype=t.float32).contiguous() if isinstance(pmap2, t.Tensor)
          else t.from_numpy(np.ascontiguousarray(pmap2, dtype=np.float32)).to(im.tensor.device))
    stack = np.ascontiguousarray(np.stack([stacked_params(grid.row_basis(iu))
                                           for iu in range(grid.params_u.size)]))   # (Mu, Mv, L, N, 3)
    pu = np.ascontiguousarray(grid.params_u)
    pv = np.ascontiguousarray(grid.params_v)
    layout = np.ascontiguousarray(grid.layout, dtype=np.int32)
    res = im.empty_like()
    rc = lib.skc_sv_grid_fwd(nat.ptr(im.tensor), nat.ptr(res), h, w, c, nat.ptr(pm), nat.dbl(pu), pu.size,
                             nat.dbl(pv), pv.size, nat.dbl(stack), stack.shape[3], nat.ints(layout), layout.size,
                             BOUNDARIES[boundary], nat.stream_ptr())
    if rc == nat.SKC_EBADARG:
        raise EngineError(f"sv_filter_grid: {nat.last_error()}")
    nat.check(rc, "sv_filter_grid")
    return im.restore(res)


def build_basis(target_family, params, layout, cfg=None, constraints=None, init=None, loss_kind=None,
                warm_start: bool = True) -> FilterBasis:
    """Fit one complex per grid parameter (svfilter.py:81-113); adjacent entries
    warm-start from the previous solution (slot correspondence).  Each fit runs
    on device; the chain of warm starts is inherently sequential."""
    from dataclasses import replace
    from .initializers import InitStrategy
    from .kernels import DenseKernel
    from .optim import ConstraintConfig, LossKind, TrainConfig, fit, parse_layout
    cfg = TrainConfig() if cfg is None else cfg
    constraints = ConstraintConfig() if constraints is None else constraints
    init = InitStrategy("ss-ir") if init is None else init
    loss_kind = LossKind() if loss_kind is None else loss_kind
    layout = parse_layout(layout)
    ps = np.array(sorted(params), dtype=np.float64)
    if ps.size > 1 and not (np.diff(ps) > 0).all():
        raise EngineError("basis parameters must be strictly increasing")
    step = float(np.min(np.diff(ps))) if ps.size > 1 else 0.0
    filters, prev = [], None
    for k, p in enumerate(ps):
        tgt = target_family(p)
        if not isinstance(tgt, DenseKernel):
            raise EngineError("target_family must return DenseKernel targets")
        adjacent = k > 0 and abs(float(ps[k] - ps[k - 1])) <= step * (1 + 1e-9)
        start = prev if (warm_start and prev is not None and adjacent) else replace(init, seed=init.seed + k)
        res = fit(tgt, layout, start, cfg, constraints, loss_kind)
        filters.append(res.complex)
        prev = res.complex
    return FilterBasis(ps, tuple(filters))


def save_basis(basis, path) -> None:
    """JSON, same schema as svfilter.py:325-341."""
    import json
    from .optim import theta_to_dict
    if isinstance(basis, FilterBasisGrid):
        doc = {"params_u": [float(p) for p in basis.params_u], "params_v": [float(p) for p in basis.params_v],
               "layout": {"samples_per_layer": list(basis.layout)},
               "filters": [[theta_to_dict(f) for f in row] for row in basis.filters]}
    else:
        doc = {"params": [float(p) for p in basis.params], "layout": {"samples_per_layer": list(basis.layout)},
               "filters": [theta_to_dict(f) for f in basis.filters]}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")


def load_basis(path):
    import json
    from .optim import theta_from_dict
    with open(path) as fh:
        doc = json.load(fh)
    if "params_u" in doc:
        return FilterBasisGrid(np.array(doc["params_u"]), np.array(doc["params_v"]),
                               tuple(tuple(theta_from_dict(f) for f in row) for row in doc["filters"]))
    return FilterBasis(np.array(doc["params"]), tuple(theta_from_dict(f) for f in doc["filters"]))
