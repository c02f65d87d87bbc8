"""Seeded synthetic inputs for the five BASELINE configurations.

The reference publishes no datasets for this path (the
paper's photographs and PSF kernels are absent), so every workload uses the
seeded stand-ins SURVEY section 8(d) specifies, with the draw order written
down here.  All inputs are rounded to fp32 (fp16 for config 3) before both the
GPU and the oracle see them.
"""

from __future__ import annotations

import math

import numpy as np

from .engine import KernelComplex, SparseLayer
from .kernels import disk_kernel, polygon_kernel, ring_kernel, star_kernel
from .svfilter import FilterBasis

C1_SHAPE = (2665, 1264, 3)      # (H, W, C) portrait, SURVEY D6
C3_SHAPE = (2160, 3840, 4)
C3_BIG = (16384, 16384, 4)


def disk_complex(layers: int, samples: int, seed: int, scale: float = 1.0) -> KernelComplex:
    """Increasing-step radial disk complex: layer l offsets uniform in a disk of
    radius 2*2^l*scale, weights uniform(0,1] normalised per layer.  Draws per
    layer: u, v ~ U[0,1)^S, then w = 1 - U[0,1)^S."""
    rng = np.random.default_rng(seed)
    out = []
    for l in range(layers):
        radius = 2.0 * (2 ** l) * scale
        u = rng.random(samples)
        v = rng.random(samples)
        r = radius * np.sqrt(u)
        th = 2.0 * math.pi * v
        off = np.stack([r * np.cos(th), r * np.sin(th)], axis=1)
        w = 1.0 - rng.random(samples)
        w = w / w.sum()
        out.append(SparseLayer(off.astype(np.float32).astype(np.float64),
                               w.astype(np.float32).astype(np.float64)))
    return KernelComplex(tuple(out))


def kawase_complex(layers: int = 6) -> KernelComplex:
    """Config 3: taps (+r,+r), (-r,+r), (-r,-r), (+r,-r), r_l = 0.5 + l, w = 1/4."""
    out = []
    for l in range(layers):
        r = 0.5 + l
        out.append(SparseLayer(np.array([[r, r], [-r, r], [-r, -r], [r, -r]]), np.full(4, 0.25)))
    return KernelComplex(tuple(out))


def _upsample_axis(lat: np.ndarray, n: int, cell: int, axis: int) -> np.ndarray:
    pos = np.arange(n, dtype=np.float64) / cell
    i = np.floor(pos).astype(np.int64)
    t = pos - i
    s = t * t * (3.0 - 2.0 * t)  # smoothstep
    a = np.take(lat, i, axis=axis)
    b = np.take(lat, i + 1, axis=axis)
    shape = [1] * lat.ndim
    shape[axis] = n
    s = s.reshape(shape)
    return a + (b - a) * s


def value_noise_frame(h: int, w: int, c: int, seed: int, rects: int = 200,
                      dtype=np.float32) -> np.ndarray:
    """4-octave value noise (cells 128/64/32/16 px, amplitudes 1/2/4/8ths,
    independent lattices per channel, smoothstep-bilinear upsampling, sum /
    sum(amp)) plus `rects` axis-aligned rectangles at 1.0 (sides U{8..128},
    top-left uniform)."""
    rng = np.random.default_rng(seed)
    acc = np.zeros((h, w, c), dtype=np.float64)
    amps = (1.0, 0.5, 0.25, 0.125)
    for cell, amp in zip((128, 64, 32, 16), amps):
        lat = rng.random((h // cell + 2, w // cell + 2, c))
        rows = _upsample_axis(lat, h, cell, 0)
        acc += amp * _upsample_axis(rows, w, cell, 1)
    acc /= sum(amps)
    for _ in range(rects):
        rh = int(rng.integers(8, 129))
        rw = int(rng.integers(8, 129))
        y0 = int(rng.integers(0, max(1, h - rh + 1)))
        x0 = int(rng.integers(0, max(1, w - rw + 1)))
        acc[y0:y0 + rh, x0:x0 + rw, :] = 1.0
    return acc.astype(dtype)


def value_noise_frame_device(h: int, w: int, c: int, seed: int, device, rects: int = 200,
                             dtype=None):
    """value_noise_frame with the upsampling done on the device (same draws,
    float64 arithmetic; used to build large benchmark batches quickly)."""
    import torch
    rng = np.random.default_rng(seed)
    acc = torch.zeros((h, w, c), dtype=torch.float64, device=device)
    amps = (1.0, 0.5, 0.25, 0.125)

    def up(lat, n, cell, axis):
        pos = torch.arange(n, dtype=torch.float64, device=device) / cell
        i = torch.floor(pos).long()
        t = pos - i
        s = t * t * (3.0 - 2.0 * t)
        a = lat.index_select(axis, i)
        b = lat.index_select(axis, i + 1)
        shape = [1] * lat.dim()
        shape[axis] = n
        return a + (b - a) * s.view(shape)

    for cell, amp in zip((128, 64, 32, 16), amps):
        lat = torch.from_numpy(rng.random((h // cell + 2, w // cell + 2, c))).to(device)
        acc += amp * up(up(lat, h, cell, 0), w, cell, 1)
    acc /= sum(amps)
    for _ in range(rects):
        rh = int(rng.integers(8, 129))
        rw = int(rng.integers(8, 129))
        y0 = int(rng.integers(0, max(1, h - rh + 1)))
        x0 = int(rng.integers(0, max(1, w - rw + 1)))
        acc[y0:y0 + rh, x0:x0 + rw, :] = 1.0
    return acc.to(torch.float32 if dtype is None else dtype)


def c0_image() -> np.ndarray:
    """Config 0: 512x512x3, iid U[0,1) from seed 0, fp32."""
    return np.random.default_rng(0).random((512, 512, 3)).astype(np.float32)


def c0_complex() -> KernelComplex:
    return disk_complex(4, 12, seed=1)


def c1_frame(b: int) -> np.ndarray:
    h, w, c = C1_SHAPE
    return value_noise_frame(h, w, c, seed=b)


def c1_complex() -> KernelComplex:
    return disk_complex(4, 32, seed=1)


def c2_basis() -> FilterBasis:
    """Three bases (4x24, seed 2, radius scale 0.5/1/2) at p = 0, 0.5, 1; the
    shared seed keeps slot correspondence."""
    filters = tuple(disk_complex(4, 24, seed=2, scale=s) for s in (0.5, 1.0, 2.0))
    return FilterBasis(np.array([0.0, 0.5, 1.0]), filters)


def c2_pmap(h: int = C1_SHAPE[0], w: int = C1_SHAPE[1], seed: int = 3, blobs: int = 20,
            sigma: float = 60.0) -> np.ndarray:
    """Radial gradient from the centre plus 20 Gaussian blobs (a = +-0.3), clipped to [0, 1]."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
    d = np.hypot(xx - cx, yy - cy)
    p = d / math.hypot(cx, cy)
    for _ in range(blobs):
        by = rng.random() * h
        bx = rng.random() * w
        a = 0.3 if rng.random() < 0.5 else -0.3
        p += a * np.exp(-((xx - bx) ** 2 + (yy - by) ** 2) / (2.0 * sigma * sigma))
    return np.clip(p, 0.0, 1.0).astype(np.float32)


def c3_frame(b: int, shape=C3_SHAPE) -> np.ndarray:
    h, w, c = shape
    return value_noise_frame(h, w, c, seed=b, dtype=np.float16)


C4_SHAPES = ("disk", "square", "hexagon", "ring", "star4")


def c4_target(i: int, size: int = 129):
    """Target i: shape i mod 5, R ~ U[20, 60], rotation ~ U[0, 2pi), seed 4 + i."""
    rng = np.random.default_rng(4 + i)
    r = float(rng.uniform(20.0, 60.0))
    rot = float(rng.uniform(0.0, 2.0 * math.pi))
    kind = C4_SHAPES[i % 5]
    if kind == "disk":
        k = disk_kernel(r, size)
    elif kind == "square":
        k = polygon_kernel(4, r, size, rot)
    elif kind == "hexagon":
        k = polygon_kernel(6, r, size, rot)
    elif kind == "ring":
        k = ring_kernel(0.6 * r, r, size)
    else:
        k = star_kernel(4, r, size, rotation=rot)
    return k


def c4_init(i: int) -> KernelComplex:
    return disk_complex(4, 32, seed=1000 + i)
