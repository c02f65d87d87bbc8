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
    "FilterBasisGrid",
    "build_basis",
    "build_basis_grid",
    "sv_filter_grid",
    "sv_ground_truth",
    "save_basis",
    "load_basis",
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


def sv_vertical_reach(basis: FilterBasis) -> int:
    """Rows above / below a pixel that the whole SV chain can read: per layer
    floor(max |oy| over the basis entries) + 2 (the bilinear corner and one
    texel for the rounding of the lerped offset), summed over the layers.
    Lerping between entries never exceeds the larger |oy| of the two."""
    reach = 0
    for l in range(len(basis.layout)):
        m = max(float(np.abs(f.layers[l].offsets[:, 1]).max()) for f in basis.filters)
        reach += int(np.floor(m)) + 2
    return reach


def _sv_filter_strips(host_img, basis: FilterBasis, host_pmap, boundary: str, host_out, nstrips: int):
    """Pinned host (H, W, C) frame and (H, W) map -> pinned host result in row
    strips: the H2D copy of strip i+1, the passes on strip i and the D2H copy
    of strip i-1 overlap on three streams.  A strip is filtered as an image of
    its own rows plus sv_vertical_reach halo rows each side (real image rows,
    so the artefacts of its artificial edges stay inside the halo and the kept
    rows equal the whole-frame result bit for bit)."""
    t = torch()
    lib = nat.lib()
    dev = t.device("cuda", t.cuda.current_device())
    cur = t.cuda.current_stream(dev)
    h, w = int(host_img.shape[0]), int(host_img.shape[1])
    c = int(host_img.shape[2]) if host_img.dim() == 3 else 1
    dt = nat.SKC_F16 if host_img.dtype == t.float16 else nat.SKC_F32
    halo = sv_vertical_reach(basis)
    stack = np.ascontiguousarray(stacked_params(basis))
    ps = np.ascontiguousarray(basis.params, dtype=np.float64)
    layout = np.ascontiguousarray(basis.layout, dtype=np.int32)
    rows = -(-h // nstrips)
    cap = min(h, rows + 2 * halo)
    from .engine import side_streams
    s_in, s_cmp, s_out = side_streams(dev)
    for s in (s_in, s_cmp, s_out):
        s.wait_stream(cur)
    din = [t.empty((cap, w, c), dtype=host_img.dtype, device=dev) for _ in range(2)]
    dpm = [t.empty((cap, w), dtype=t.float32, device=dev) for _ in range(2)]
    dout = [t.empty((cap, w, c), dtype=host_img.dtype, device=dev) for _ in range(2)]
    h2d = [t.cuda.Event() for _ in range(2)]
    cmp = [t.cuda.Event() for _ in range(2)]
    d2h = [t.cuda.Event() for _ in range(2)]
    src = host_img.view(h, w, c)
    dst = host_out.view(h, w, c)
    for i, y0 in enumerate(range(0, h, rows)):
        k = i & 1
        y1 = min(h, y0 + rows)
        e0, e1 = max(0, y0 - halo), min(h, y1 + halo)
        n = e1 - e0
        with t.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(cmp[k])
            din[k][:n].copy_(src[e0:e1], non_blocking=True)
            dpm[k][:n].copy_(host_pmap[e0:e1], non_blocking=True)
            h2d[k].record(s_in)
        s_cmp.wait_event(h2d[k])
        if i >= 2:
            s_cmp.wait_event(d2h[k])
        rc = lib.skc_sv_fwd(nat.ptr(din[k]), dt, nat.ptr(dout[k]), dt, n, w, c, nat.ptr(dpm[k]), nat.dbl(ps),
                            ps.size, nat.dbl(stack), stack.shape[2], nat.ints(layout), layout.size,
                            BOUNDARIES[boundary], nat.stream_ptr(s_cmp))
        if rc == nat.SKC_EBADARG:
            raise EngineError(f"sv_filter: {nat.last_error()}")
        nat.check(rc, "sv_filter")
        cmp[k].record(s_cmp)
        with t.cuda.stream(s_out):
            s_out.wait_event(cmp[k])
            dst[y0:y1].copy_(dout[k][y0 - e0:y1 - e0], non_blocking=True)
            d2h[k].record(s_out)
    cur.wait_stream(s_out)
    for buf in din + dpm + dout:
        buf.record_stream(cur)
    return host_out


def sv_filter(img, basis: FilterBasis, pmap, boundary: str = "zero", out=None, strips: int = 4):
    """Per-pixel blended sparse filtering guided by a parameter map (svfilter.py:171-203).

    Each pass re-interpolates that layer's taps per pixel between the two
    bracketing basis entries and gathers bilinearly from the previous pass.
    Host torch tensors (pinned) with a pinned `out` move with async copies;
    a pinned float32 / float16 frame with a pinned float32 map and a pinned
    `out` of the frame's shape and dtype streams through in `strips` row
    strips (copies both ways overlapped with the passes; the call synchronises
    before it returns).
    """
    t = torch()
    lib = nat.lib()
    if boundary not in BOUNDARIES:
        raise EngineError(f"boundary must be one of {sorted(BOUNDARIES)}, got {boundary!r}")
    if (strips > 1 and isinstance(img, t.Tensor) and isinstance(pmap, t.Tensor) and isinstance(out, t.Tensor)
            and not img.is_cuda and not pmap.is_cuda and not out.is_cuda and img.is_pinned() and pmap.is_pinned()
            and out.is_pinned() and img.dim() in (2, 3) and img.dtype in (t.float32, t.float16)
            and out.dtype == img.dtype and tuple(out.shape) == tuple(img.shape) and pmap.dtype == t.float32
            and tuple(pmap.shape) == tuple(img.shape[:2]) and img.is_contiguous() and pmap.is_contiguous()
            and out.is_contiguous()
            and int(img.shape[0]) >= strips * max(64, 2 * sv_vertical_reach(basis))):
        _sv_filter_strips(img, basis, pmap, boundary, out, strips)
        t.cuda.current_stream().synchronize()
        return out
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


def _as_dense(tgt):
    from .kernels import DenseKernel, generate_kernel
    return tgt if isinstance(tgt, DenseKernel) else generate_kernel(tgt)


def _fit_round(jobs, layout, cfg, constraints, loss_kind):
    """Fit independent (target, init) jobs with one persistent batched launch
    per distinct target size (fit_batch); returns the complexes in order."""
    from .optim import fit_batch
    out = [None] * len(jobs)
    by_size = {}
    for j, (tgt, _) in enumerate(jobs):
        by_size.setdefault(tgt.size, []).append(j)
    for idx in by_size.values():
        res = fit_batch([jobs[j][0] for j in idx], layout, [jobs[j][1] for j in idx], cfg, constraints,
                        loss_kind)
        for j, r in zip(idx, res):
            out[j] = r.complex
    return out


def _basis_rows(families, params, layout, cfg, constraints, inits, loss_kind, warm_start):
    """Fit len(families) bases over the same parameter grid at once.

    Row i's entry k starts from row i's entry k-1 when warm_start holds and
    the two parameters are one grid step apart (svfilter.py:100-107), else
    from replace(inits[i], seed=inits[i].seed + k).  Rows never depend on
    each other, so entry k of every row is one batched fit: the warm-start
    chain is sequential along the grid only."""
    from dataclasses import replace
    ps = np.array(sorted(params), dtype=np.float64)
    if ps.size > 1 and not (np.diff(ps) > 0).all():
        raise EngineError("basis parameters must be strictly increasing")
    step = float(np.min(np.diff(ps))) if ps.size > 1 else 0.0
    rows = [[] for _ in families]
    for k, p in enumerate(ps):
        adjacent = k > 0 and abs(float(ps[k] - ps[k - 1])) <= step * (1 + 1e-9)
        jobs = []
        for i, fam in enumerate(families):
            start = rows[i][-1] if (warm_start and adjacent) else replace(inits[i], seed=inits[i].seed + k)
            jobs.append((_as_dense(fam(p)), start))
        for i, cpx in enumerate(_fit_round(jobs, layout, cfg, constraints, loss_kind)):
            rows[i].append(cpx)
    return ps, rows


def _fit_defaults(cfg, constraints, init, loss_kind):
    from .initializers import InitStrategy
    from .optim import ConstraintConfig, LossKind, TrainConfig
    return (TrainConfig() if cfg is None else cfg, ConstraintConfig() if constraints is None else constraints,
            InitStrategy("ss-ir") if init is None else init, LossKind() if loss_kind is None else loss_kind)


def build_basis(target_family, params, layout, cfg=None, constraints=None, init=None, loss_kind=None,
                warm_start: bool = True) -> FilterBasis:
    """Fit one complex per grid parameter (svfilter.py:81-113).  target_family
    maps a parameter to a DenseKernel or a KernelSpec.  Adjacent entries
    warm-start from the previous solution (slot correspondence); without warm
    starts every entry is fit in one batched launch."""
    from .optim import parse_layout
    cfg, constraints, init, loss_kind = _fit_defaults(cfg, constraints, init, loss_kind)
    ps, rows = _basis_rows([target_family], params, parse_layout(layout), cfg, constraints, [init], loss_kind,
                           warm_start)
    return FilterBasis(ps, tuple(rows[0]))


def build_basis_grid(target_family, params_u, params_v, layout, cfg=None, constraints=None, init=None,
                     loss_kind=None, warm_start: bool = True) -> FilterBasisGrid:
    """Fit a (u, v) grid of basis complexes (svfilter.py:272-289): every row is
    build_basis along v of target_family(u, .), row iu starting from
    replace(init, seed=init.seed + 1000 * iu) when warm_start, else from init.
    The rows are independent, so each v step fits all rows in one launch."""
    from dataclasses import replace
    from .optim import parse_layout
    cfg, constraints, init, loss_kind = _fit_defaults(cfg, constraints, init, loss_kind)
    pu = np.array(sorted(params_u), dtype=np.float64)
    inits = [replace(init, seed=init.seed + 1000 * iu) if (warm_start and iu > 0) else init
             for iu in range(pu.size)]
    fams = [(lambda v, u=float(u): target_family(u, v)) for u in pu]
    pv, rows = _basis_rows(fams, params_v, parse_layout(layout), cfg, constraints, inits, loss_kind, warm_start)
    return FilterBasisGrid(pu, pv, tuple(tuple(r) for r in rows))


def sv_ground_truth(img, target_family, pmap, *, levels: int | None = None, max_kernels: int = 8192):
    """Brute-force SV reference (svfilter.py:206-235): at every pixel the dense
    kernel target_family(pmap[y, x]) (DenseKernel or KernelSpec) applied as a
    zero-padded convolution.  The family is evaluated once per DISTINCT map
    value on the host and the per-pixel convolutions run on the device
    (skc_sv_ground_truth).  A continuous map has one value per pixel: pass
    `levels=N` to snap it to N evenly spaced values between its min and max
    first (an approximation the reference does not make)."""
    t = torch()
    lib = nat.lib()
    a = np.asarray(img, dtype=np.float64)
    pm = np.asarray(pmap, dtype=np.float64)
    if a.ndim not in (2, 3):
        raise EngineError(f"image must be (H, W) or (H, W, C), got {a.shape}")
    if pm.shape != a.shape[:2]:
        raise EngineError(f"parameter map {pm.shape} must match image {a.shape[:2]}")
    if levels is not None:
        if levels < 2:
            raise EngineError(f"levels must be >= 2, got {levels}")
        lo, hi = float(pm.min()), float(pm.max())
        if hi > lo:
            pm = lo + np.rint((pm - lo) / (hi - lo) * (levels - 1)) * ((hi - lo) / (levels - 1))
    vals, inv = np.unique(pm, return_inverse=True)
    if vals.size > max_kernels:
        raise EngineError(f"parameter map has {vals.size} distinct values (> max_kernels={max_kernels}); "
                          "pass levels=N to quantise it")
    ks = [_as_dense(target_family(float(v))).weights for v in vals]
    m = max(k.shape[0] for k in ks)
    bank = np.stack([np.pad(k, (m - k.shape[0]) // 2) for k in ks]).astype(np.float32)
    chans = a if a.ndim == 3 else a[:, :, None]
    h, w, c = chans.shape
    dev = t.device("cuda", t.cuda.current_device())
    d_img = t.from_numpy(np.ascontiguousarray(np.moveaxis(chans, 2, 0), dtype=np.float32)).to(dev)
    d_idx = t.from_numpy(np.ascontiguousarray(inv.reshape(h, w), dtype=np.int32)).to(dev)
    d_k = t.from_numpy(bank).to(dev)
    d_out = t.empty_like(d_img)
    rc = lib.skc_sv_ground_truth(nat.ptr(d_img), h, w, c, nat.ptr(d_idx), nat.ptr(d_k), len(ks), m,
                                 nat.ptr(d_out), nat.stream_ptr())
    if rc == nat.SKC_EBADARG:
        raise EngineError(f"sv_ground_truth: {nat.last_error()}")
    nat.check(rc, "sv_ground_truth")
    res = np.moveaxis(d_out.cpu().numpy().astype(np.float64), 0, 2)
    return res if a.ndim == 3 else res[:, :, 0]


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
