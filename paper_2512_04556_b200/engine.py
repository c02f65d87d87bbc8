"""Uniform sparse-layer filtering and impulse responses on the B200.

Drop-in for the reference engine (/root/reference/pkg/src/sparsekern/
engine.py): same types, names, validation and errors; the arithmetic runs in
libskc.so (csrc/skc_filter.cu, csrc/skc_fit.cu) through the C ABI.  New
keywords: `boundary` ("zero" = the reference's zero padding, "clamp" =
clamp-to-edge for BASELINE config 0) and the batched `apply_complex_batch`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from ._tensors import Image, torch
from .kernels import DenseKernel

__all__ = [
    "EngineError",
    "TruncationError",
    "SparseLayer",
    "KernelComplex",
    "apply_sparse_layer",
    "apply_complex",
    "apply_complex_batch",
    "dense_convolve",
    "bilinear_sample",
    "synthesize_ir",
    "synthesize_ir_batch",
    "required_canvas",
    "auto_canvas",
    "psnr",
    "sse",
    "BOUNDARIES",
]

BOUNDARIES = {"zero": nat.SKC_ZERO, "clamp": nat.SKC_CLAMP}


class EngineError(ValueError):
    """engine.py:35-36"""


class TruncationError(EngineError):
    """Requested impulse-response canvas cannot hold the composed support (engine.py:39-40)."""


@dataclass(frozen=True, eq=False)
class SparseLayer:
    """N taps: offsets (N, 2) as (ox, oy) pixels and weights (N,) (engine.py:43-71)."""

    offsets: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        off = np.array(self.offsets, dtype=np.float64, copy=True).reshape(-1, 2)
        wts = np.array(self.weights, dtype=np.float64, copy=True).reshape(-1)
        if off.shape[0] < 1:
            raise EngineError("sparse layer needs at least one sample")
        if off.shape[0] != wts.shape[0]:
            raise EngineError(f"offset/weight count mismatch: {off.shape[0]} vs {wts.shape[0]}")
        if not (np.isfinite(off).all() and np.isfinite(wts).all()):
            raise EngineError("sparse layer parameters must be finite")
        off.flags.writeable = False
        wts.flags.writeable = False
        object.__setattr__(self, "offsets", off)
        object.__setattr__(self, "weights", wts)

    @property
    def sample_count(self) -> int:
        return int(self.offsets.shape[0])

    @property
    def reach(self) -> float:
        """Max Chebyshev extent of the offsets."""
        return float(np.abs(self.offsets).max())

    def taps(self) -> np.ndarray:
        """(N, 3) float64 rows (ox, oy, w) -- the C ABI's tap table."""
        return np.ascontiguousarray(np.concatenate([self.offsets, self.weights[:, None]], axis=1))


@dataclass(frozen=True, eq=False)
class KernelComplex:
    """Layers applied input to output (engine.py:74-103)."""

    layers: tuple

    def __post_init__(self):
        layers = tuple(self.layers)
        if len(layers) < 1:
            raise EngineError("kernel complex needs at least one layer")
        if not all(isinstance(l, SparseLayer) for l in layers):
            raise EngineError("kernel complex layers must be SparseLayer instances")
        object.__setattr__(self, "layers", layers)

    @property
    def layer_count(self) -> int:
        return len(self.layers)

    @property
    def layout(self) -> tuple:
        return tuple(l.sample_count for l in self.layers)

    @property
    def total_samples(self) -> int:
        return sum(self.layout)

    @property
    def reach(self) -> float:
        return sum(l.reach for l in self.layers)

    def taps(self) -> np.ndarray:
        return np.ascontiguousarray(np.concatenate([l.taps() for l in self.layers], axis=0))

    def padded(self, nmax: int | None = None) -> np.ndarray:
        """(L, nmax, 3) float32 (ox, oy, w), zero-padded (zero weights are inert)."""
        nmax = max(self.layout) if nmax is None else nmax
        out = np.zeros((self.layer_count, nmax, 3), dtype=np.float32)
        for l, lay in enumerate(self.layers):
            out[l, :lay.sample_count] = lay.taps()
        return out


def _boundary(boundary) -> int:
    try:
        return BOUNDARIES[boundary]
    except KeyError:
        raise EngineError(f"boundary must be one of {sorted(BOUNDARIES)}, got {boundary!r}") from None


def _raise(rc: int, what: str):
    msg = f"{what}: {nat.last_error()}"
    if rc == nat.SKC_EBADARG:
        raise EngineError(msg)
    if rc == nat.SKC_ETRUNC:
        raise TruncationError(msg)
    raise nat.NativeError(rc, msg)


def apply_sparse_layer(img, layer: SparseLayer, boundary: str = "zero"):
    """out[y,x] = sum_i w_i bilinear(img, x+ox_i, y+oy_i) (engine.py:160-170)."""
    lib = nat.lib()
    im = Image(img)
    b, h, w, c = im.dims
    out = im.empty_like()
    taps = layer.taps()
    rc = lib.skc_layer_fwd(nat.ptr(im.tensor), im.dtype_id, nat.ptr(out), im.dtype_id, b, h, w, c,
                           nat.dbl(taps), taps.shape[0], _boundary(boundary), nat.stream_ptr())
    if rc:
        _raise(rc, "apply_sparse_layer")
    return im.restore(out)


def _chain(im: Image, cpx: KernelComplex, boundary: str, out_dtype=None):
    lib = nat.lib()
    b, h, w, c = im.dims
    out = im.empty_like(out_dtype)
    odt = nat.SKC_F16 if out.dtype == torch().float16 else nat.SKC_F32
    taps = cpx.taps()
    layout = np.ascontiguousarray(cpx.layout, dtype=np.int32)
    rc = lib.skc_chain_fwd(nat.ptr(im.tensor), im.dtype_id, nat.ptr(out), odt, b, h, w, c,
                           nat.dbl(taps), nat.ints(layout), layout.size, _boundary(boundary),
                           nat.stream_ptr())
    if rc:
        _raise(rc, "apply_complex")
    return out


def chain_into(src, dst, cpx: KernelComplex, boundary: str = "zero", stream=None):
    """skc_chain_fwd from one contiguous CUDA tensor into another (H, W[, C])
    or (B, H, W, C), fp32 or fp16, no allocation of the output: the building
    block of the overlapped strip pipeline (dist.StripPipeline)."""
    t = torch()
    lib = nat.lib()
    for name, ten in (("src", src), ("dst", dst)):
        if not (isinstance(ten, t.Tensor) and ten.is_cuda and ten.is_contiguous()
                and ten.dtype in (t.float32, t.float16)):
            raise EngineError(f"chain_into: {name} must be a contiguous fp32/fp16 CUDA tensor")
    if src.shape != dst.shape:
        raise EngineError(f"chain_into: shapes differ {tuple(src.shape)} vs {tuple(dst.shape)}")
    shp = tuple(src.shape)
    if len(shp) == 2:
        b, h, w, c = 1, shp[0], shp[1], 1
    elif len(shp) == 3:
        b, (h, w, c) = 1, shp
    elif len(shp) == 4:
        b, h, w, c = shp
    else:
        raise EngineError(f"chain_into: bad shape {shp}")
    dt = {t.float32: nat.SKC_F32, t.float16: nat.SKC_F16}
    taps = cpx.taps()
    layout = np.ascontiguousarray(cpx.layout, dtype=np.int32)
    rc = lib.skc_chain_fwd(nat.ptr(src), dt[src.dtype], nat.ptr(dst), dt[dst.dtype], b, h, w, c, nat.dbl(taps),
                           nat.ints(layout), layout.size, _boundary(boundary), nat.stream_ptr(stream))
    if rc:
        _raise(rc, "chain_into")
    return dst


def apply_complex(img, cpx: KernelComplex, boundary: str = "zero"):
    """All layers in order (engine.py:173-178); intermediates stay fp32 on device."""
    im = Image(img)
    return im.restore(_chain(im, cpx, boundary))


_ROW_STRIP_MIN_BYTES = 64 << 20
_SIDE_STREAMS = {}


def side_streams(dev):
    """The three side streams (H2D, compute, D2H) of the pinned-host pipelines,
    created once per device: creating them per call costs as much as a small
    frame's kernels."""
    t = torch()
    key = (dev.type, dev.index)
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = tuple(t.cuda.Stream(dev) for _ in range(3))
    return _SIDE_STREAMS[key]


def _pipelined_host_rows(host_in, cpx: KernelComplex, boundary: str, host_out, strips: int):
    """One large pinned host frame (1, H, W, C) in row strips: the H2D copy of
    strip i+1, the chain on strip i and the D2H copy of strip i-1 overlap on
    three streams.  A strip is filtered as an image of its own rows plus the
    chain's composed corner reach (dist.corner_reach) of real image rows each
    side, so the artefacts of its artificial edges stay inside the halo and
    the kept rows equal the whole-frame result bit for bit (the same argument
    as dist.StripPipeline's row strips across GPUs)."""
    from .dist import corner_reach
    t = torch()
    lib = nat.lib()
    dev = t.device("cuda", t.cuda.current_device())
    cur = t.cuda.current_stream(dev)
    h, w = (int(v) for v in host_in.shape[1:3])
    c = int(host_in.shape[3]) if host_in.dim() == 4 else 1
    idt = nat.SKC_F16 if host_in.dtype == t.float16 else nat.SKC_F32
    top, bottom, _, _ = corner_reach(cpx)
    taps = cpx.taps()
    layout = np.ascontiguousarray(cpx.layout, dtype=np.int32)
    bnd = _boundary(boundary)
    rows = -(-h // strips)
    cap = min(h, rows + top + bottom)
    s_in, s_cmp, s_out = side_streams(dev)
    for s in (s_in, s_cmp, s_out):
        s.wait_stream(cur)
    din = [t.empty((cap, w, c), dtype=host_in.dtype, device=dev) for _ in range(2)]
    dout = [t.empty((cap, w, c), dtype=host_in.dtype, device=dev) for _ in range(2)]
    h2d = [t.cuda.Event() for _ in range(2)]
    cmp = [t.cuda.Event() for _ in range(2)]
    d2h = [t.cuda.Event() for _ in range(2)]
    src = host_in.view(h, w, c)
    dst = host_out.view(h, w, c)
    for i, y0 in enumerate(range(0, h, rows)):
        k = i & 1
        y1 = min(h, y0 + rows)
        e0, e1 = max(0, y0 - top), min(h, y1 + bottom)
        n = e1 - e0
        with t.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(cmp[k])
            din[k][:n].copy_(src[e0:e1], non_blocking=True)
            h2d[k].record(s_in)
        s_cmp.wait_event(h2d[k])
        if i >= 2:
            s_cmp.wait_event(d2h[k])
        rc = lib.skc_chain_fwd(nat.ptr(din[k]), idt, nat.ptr(dout[k]), idt, 1, n, w, c, nat.dbl(taps),
                               nat.ints(layout), layout.size, bnd, nat.stream_ptr(s_cmp))
        if rc:
            _raise(rc, "apply_complex_batch")
        cmp[k].record(s_cmp)
        with t.cuda.stream(s_out):
            s_out.wait_event(cmp[k])
            dst[y0:y1].copy_(dout[k][y0 - e0:y1 - e0], non_blocking=True)
            d2h[k].record(s_out)
    cur.wait_stream(s_out)
    for buf in din + dout:
        buf.record_stream(cur)
    return host_out


def _pipelined_host_batch(host_in, cpx: KernelComplex, boundary: str, host_out, chunk: int):
    """Pinned host (B,H,W,C) -> device -> pinned host, overlapping the H2D copy
    of chunk i+1, the chain on chunk i and the D2H copy of chunk i-1 on three
    streams (copy engines both ways + SMs)."""
    t = torch()
    lib = nat.lib()
    dev = t.device("cuda", t.cuda.current_device())
    cur = t.cuda.current_stream(dev)
    b, h, w = (int(v) for v in host_in.shape[:3])
    c = int(host_in.shape[3]) if host_in.dim() == 4 else 1
    idt = nat.SKC_F16 if host_in.dtype == t.float16 else nat.SKC_F32
    odt = nat.SKC_F16 if host_out.dtype == t.float16 else nat.SKC_F32
    taps = cpx.taps()
    layout = np.ascontiguousarray(cpx.layout, dtype=np.int32)
    bnd = _boundary(boundary)
    if b == 1 and host_in.numel() * host_in.element_size() >= _ROW_STRIP_MIN_BYTES:
        # one large frame (config 3's 16384^2 image): overlap the copies over row strips
        from .dist import corner_reach
        top, bottom, _, _ = corner_reach(cpx)
        if h >= 8 * 8 * max(1, top + bottom):
            return _pipelined_host_rows(host_in, cpx, boundary, host_out, 8)
    if b <= chunk:
        # one chunk: nothing to overlap -- copy in, filter, copy out on the caller's stream
        # (three streams and six events cost more than a small frame's kernels)
        din1 = t.empty((b, h, w, c), dtype=host_in.dtype, device=dev)
        dout1 = t.empty((b, h, w, c), dtype=host_out.dtype, device=dev)
        din1.copy_(host_in.view(b, h, w, c), non_blocking=True)
        rc = lib.skc_chain_fwd(nat.ptr(din1), idt, nat.ptr(dout1), odt, b, h, w, c, nat.dbl(taps),
                               nat.ints(layout), layout.size, bnd, nat.stream_ptr(cur))
        if rc:
            _raise(rc, "apply_complex_batch")
        host_out.view(b, h, w, c).copy_(dout1, non_blocking=True)
        return host_out
    s_in, s_cmp, s_out = side_streams(dev)
    for s in (s_in, s_cmp, s_out):
        s.wait_stream(cur)
    n = min(chunk, b)
    din = [t.empty((n, h, w, c), dtype=host_in.dtype, device=dev) for _ in range(2)]
    dout = [t.empty((n, h, w, c), dtype=host_out.dtype, device=dev) for _ in range(2)]
    h2d = [t.cuda.Event() for _ in range(2)]
    cmp = [t.cuda.Event() for _ in range(2)]
    d2h = [t.cuda.Event() for _ in range(2)]
    src = host_in.view(b, h, w, c)
    dst = host_out.view(b, h, w, c)
    for i, f0 in enumerate(range(0, b, n)):
        k = i & 1
        f1 = min(b, f0 + n)
        m = f1 - f0
        with t.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(cmp[k])
            din[k][:m].copy_(src[f0:f1], non_blocking=True)
            h2d[k].record(s_in)
        s_cmp.wait_event(h2d[k])
        if i >= 2:
            s_cmp.wait_event(d2h[k])
        rc = lib.skc_chain_fwd(nat.ptr(din[k]), idt, nat.ptr(dout[k]), odt, m, h, w, c, nat.dbl(taps),
                               nat.ints(layout), layout.size, bnd, nat.stream_ptr(s_cmp))
        if rc:
            _raise(rc, "apply_complex_batch")
        cmp[k].record(s_cmp)
        with t.cuda.stream(s_out):
            s_out.wait_event(cmp[k])
            dst[f0:f1].copy_(dout[k][:m], non_blocking=True)
            d2h[k].record(s_out)
    cur.wait_stream(s_out)
    for buf in din + dout:
        buf.record_stream(cur)
    return host_out


def apply_complex_batch(imgs, cpx: KernelComplex, boundary: str = "zero", out=None,
                        chunk: int = 4):
    """Batched frames (B, H, W[, C]) through one complex in a single call per layer.

    Device tensors are filtered on the device.  A pinned, contiguous float32
    or float16 host tensor with a pinned host `out` of the same shape and
    dtype streams through the GPU in chunks of `chunk` frames, overlapping
    both copy directions with the kernels; the call synchronises before it
    returns, so `out` holds the result.  Every other input (numpy, other
    dtypes, pageable memory) goes through the generic path (fp32 on device,
    result converted back)."""
    t = torch()
    if (isinstance(imgs, t.Tensor) and not imgs.is_cuda and imgs.is_pinned() and isinstance(out, t.Tensor)
            and not out.is_cuda and out.is_pinned() and imgs.dim() in (3, 4)
            and imgs.dtype in (t.float32, t.float16) and out.dtype == imgs.dtype
            and tuple(out.shape) == tuple(imgs.shape) and imgs.is_contiguous() and out.is_contiguous()):
        _pipelined_host_batch(imgs, cpx, boundary, out, chunk)
        t.cuda.current_stream().synchronize()   # `out` is complete when the call returns
        return out
    im = Image(imgs, batched=True)
    res = _chain(im, cpx, boundary)
    if out is not None:
        if isinstance(out, np.ndarray):
            out[...] = im.restore(res)
        else:
            out.copy_(res.view(out.shape))
        return out
    return im.restore(res)


def dense_convolve(img, kernel: DenseKernel, boundary: str = "zero"):
    """Dense M x M convolution (engine.py:139-157): out[y,x] = sum_{j,i}
    img[y-j, x-i] K[c+j, c+i].  Runs as one sparse layer of integer taps
    (offset (-i, -j), weight K[c+j, c+i], zero entries dropped) through the
    same device kernels (dense-stencil path for M <= 9)."""
    w = np.asarray(kernel.weights, dtype=np.float64)
    r = kernel.radius
    jj, ii = np.nonzero(w)
    if jj.size == 0:
        im = Image(img)
        return im.restore(im.empty_like().zero_())
    off = np.stack([-(ii - r), -(jj - r)], axis=1).astype(np.float64)
    return apply_sparse_layer(img, SparseLayer(off, w[jj, ii]), boundary)


def bilinear_sample(img, x, y):
    """Bilinear lookup at per-element fractional coordinates, zero padding
    (engine.py:212-248).  img (..., H, W); x, y (..., A, B) broadcast
    together and share img's leading batch dims (every batch slice samples
    its own image).  One device gather (skc_bilinear_sample) in float64
    coordinates and weights, the reference's corner order; float64 images
    stay float64, so numpy inputs give the reference's values.  numpy in ->
    float64 numpy out; CUDA tensors in -> float64 CUDA tensor out."""
    t = torch()
    lib = nat.lib()
    on_dev = isinstance(img, t.Tensor) and img.is_cuda
    dev = img.device if on_dev else t.device("cuda", t.cuda.current_device())

    def dev_tensor(a, dtype):
        if isinstance(a, t.Tensor):
            return a.to(device=dev, dtype=dtype)
        return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(dev).to(dtype)

    im = dev_tensor(img, t.float32 if isinstance(img, t.Tensor) and img.dtype in (t.float16, t.float32)
                    else t.float64)
    if im.dim() < 2:
        raise EngineError(f"image must have at least 2 dims, got {tuple(im.shape)}")
    h, w = int(im.shape[-2]), int(im.shape[-1])
    batch = tuple(int(v) for v in im.shape[:-2])
    xs, ys = dev_tensor(x, t.float64), dev_tensor(y, t.float64)
    try:
        shape = tuple(np.broadcast_shapes(tuple(xs.shape), tuple(ys.shape)))
    except ValueError as exc:
        raise EngineError(f"x and y do not broadcast: {exc}") from exc
    xs = xs.expand(shape).contiguous()
    ys = ys.expand(shape).contiguous()
    nb = int(np.prod(batch)) if batch else 1
    bidx, inner = None, 0
    if batch:
        if shape[:len(batch)] == batch:
            inner = int(np.prod(shape[len(batch):])) if len(shape) > len(batch) else 1
        else:
            # general numpy broadcasting of the batch index (engine.py:234-237)
            b = np.arange(nb).reshape(batch + (1,) * (len(shape) - len(batch)))
            try:
                bb = np.broadcast_to(b, np.broadcast_shapes(b.shape, shape))
            except ValueError as exc:
                raise EngineError(f"batch dims {batch} do not broadcast with {shape}: {exc}") from exc
            shape = bb.shape
            xs = xs.expand(shape).contiguous()
            ys = ys.expand(shape).contiguous()
            bidx = t.from_numpy(np.ascontiguousarray(bb, dtype=np.int64)).to(dev)
    im = im.contiguous()
    out = t.empty(shape, dtype=t.float64, device=dev)
    n = int(out.numel())
    rc = lib.skc_bilinear_sample(nat.ptr(im), nat.SKC_F32 if im.dtype == t.float32 else nat.SKC_F64, nb, h, w,
                                 nat.ptr(xs), nat.ptr(ys), nat.ptr(bidx) if bidx is not None else None,
                                 n, inner, nat.ptr(out), nat.stream_ptr())
    if rc:
        _raise(rc, "bilinear_sample")
    return out if on_dev else out.cpu().numpy()


def required_canvas(cpx: KernelComplex) -> int:
    """Smallest odd canvas for the composed response (engine.py:181-183)."""
    return 2 * math.ceil(cpx.reach) + 1


def auto_canvas(cpx: KernelComplex) -> int:
    """required_canvas plus a 2-pixel guard (engine.py:186-188)."""
    return required_canvas(cpx) + 4


def _ir_device(padded: np.ndarray, layout, canvas: int):
    """padded (B, L, nmax, 3) float32 -> (B, canvas, canvas) CUDA float32."""
    t = torch()
    lib = nat.lib()
    taps = t.from_numpy(np.ascontiguousarray(padded, dtype=np.float32)).cuda()
    bsz, nl, nmax, _ = padded.shape
    out = t.empty((bsz, canvas, canvas), dtype=t.float32, device=taps.device)
    lay = np.ascontiguousarray(layout, dtype=np.int32)
    rc = lib.skc_ir_batch(nat.ptr(taps), bsz, nat.ints(lay), nl, nmax, canvas, nat.ptr(out),
                          nat.stream_ptr())
    if rc == nat.SKC_ENONFINITE:
        raise EngineError(f"synthesize_ir: {nat.last_error()}")
    if rc:
        _raise(rc, "synthesize_ir")
    return out


def synthesize_ir(cpx: KernelComplex, canvas: int | None = None) -> DenseKernel:
    """Impulse response on a centred delta canvas (engine.py:191-209)."""
    if canvas is None:
        canvas = auto_canvas(cpx)
    else:
        if canvas % 2 == 0:
            raise EngineError(f"canvas must be odd, got {canvas}")
        if canvas < required_canvas(cpx):
            raise TruncationError(f"canvas {canvas} would truncate impulse response "
                                  f"(needs >= {required_canvas(cpx)})")
    ir = _ir_device(cpx.padded()[None], cpx.layout, canvas)
    return DenseKernel(ir[0].cpu().numpy().astype(np.float64))


def synthesize_ir_batch(offsets, weights, canvas: int) -> np.ndarray:
    """Batched responses (engine.py:251-303): offsets (B,L,N,2), weights (B,L,N)."""
    off = np.asarray(offsets, dtype=np.float64)
    wts = np.asarray(weights, dtype=np.float64)
    bsz, nl, ns, _ = off.shape
    if canvas % 2 == 0:
        raise EngineError(f"canvas must be odd, got {canvas}")
    padded = np.concatenate([off, wts[..., None]], axis=-1).astype(np.float32)
    ir = _ir_device(padded, (ns,) * nl, canvas)
    return ir.cpu().numpy().astype(np.float64)


def sse(a, b) -> float:
    """Sum of squared differences (engine.py:306-313); host metric."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise EngineError(f"dimension mismatch: {a.shape} vs {b.shape}")
    d = a - b
    return float(np.sum(d * d))


PSNR_CAP_DB = 99.0


def psnr(a, b) -> float:
    """PSNR with peak max(|a|, 1), capped at 99 dB (engine.py:316-329); host metric."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise EngineError(f"dimension mismatch: {a.shape} vs {b.shape}")
    peak = max(float(np.abs(a).max(initial=0.0)), 1.0)
    mse = float(np.mean((a - b) ** 2))
    if mse == 0.0:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, 10.0 * math.log10(peak * peak / mse))
