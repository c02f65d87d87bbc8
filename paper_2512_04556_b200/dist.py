"""Multi-GPU decomposition of the hot path (one process per GPU).

* Batched frames / batched fits (configs 1, 3, 4): independent units, sharded
  as contiguous blocks with no collective on the data path (`shard`).
* One very large image (config 3, 16384^2): row strips; before the chain each
  rank exchanges exactly the rows its neighbours' outputs depend on -- the
  composed corner reach of the complex (`corner_reach`: 21 rows for
  the Kawase 6x4 chain, not the 19 of sum(r_l)+1) -- over NCCL point-to-point
  (NVLink/NVSwitch on a B200 node), runs the chain on the extended strip and
  keeps its own rows.  Boundary effects of the artificial strip edges travel
  at most the corner reach inward, i.e. they stay inside the halo, so the kept
  rows are exactly the single-GPU result.

The reference is single-process; this module has no
reference counterpart.  Its host logic is covered with world-size-2 gloo
tests on CPU (tests/test_dist.py).
"""

from __future__ import annotations

import math

import numpy as np

from .engine import KernelComplex


def corner_reach(cpx: KernelComplex):
    """(top, bottom, left, right) rows/cols the chain reads beyond an output pixel.

    Layer l reads input rows y + [min floor(oy), max floor(oy) + 1] (bilinear
    corners, engine.py:118-130); the chain composes these ranges additively.
    """
    lo_y = hi_y = lo_x = hi_x = 0
    for lay in cpx.layers:
        fl = np.floor(lay.offsets)
        lo_x += int(fl[:, 0].min())
        hi_x += int(fl[:, 0].max()) + 1
        lo_y += int(fl[:, 1].min())
        hi_y += int(fl[:, 1].max()) + 1
    return max(0, -lo_y), max(0, hi_y), max(0, -lo_x), max(0, hi_x)


def shard(n: int, rank: int, world: int) -> slice:
    """Contiguous block of n independent units owned by `rank`."""
    per = n // world
    extra = n % world
    start = rank * per + min(rank, extra)
    return slice(start, start + per + (1 if rank < extra else 0))


def strip_bounds(height: int, rank: int, world: int):
    s = shard(height, rank, world)
    return s.start, s.stop


def exchange_halo(strip, top: int, bottom: int, rank: int, world: int, group=None):
    """Return (rows above, rows below) this rank's strip from its neighbours.

    `top` rows are needed above each strip and `bottom` rows below it.  The
    rank above receives our first `bottom` rows; the rank below receives our
    last `top` rows.  One batched NCCL/gloo send/recv group per call.
    """
    import torch
    import torch.distributed as dist

    h = strip.shape[0]
    if (rank > 0 and h < bottom) or (rank < world - 1 and h < top):
        raise ValueError(f"strip of {h} rows is shorter than the halo ({top}, {bottom})")
    rest = tuple(strip.shape[1:])
    above = strip.new_empty((top if rank > 0 else 0,) + rest)
    below = strip.new_empty((bottom if rank < world - 1 else 0,) + rest)
    ops = []
    if rank > 0:
        if bottom:
            ops.append(dist.P2POp(dist.isend, strip[:bottom].contiguous(), rank - 1, group))
        if top:
            ops.append(dist.P2POp(dist.irecv, above, rank - 1, group))
    if rank < world - 1:
        if top:
            ops.append(dist.P2POp(dist.isend, strip[h - top:].contiguous(), rank + 1, group))
        if bottom:
            ops.append(dist.P2POp(dist.irecv, below, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return above, below


def apply_complex_strips(strip, cpx: KernelComplex, rank: int, world: int, boundary: str = "zero",
                         group=None, compute=None):
    """Filter one row strip of a large image; returns this rank's output rows.

    `compute(img, cpx, boundary)` defaults to the device `apply_complex`.
    """
    import torch

    if compute is None:
        from .engine import apply_complex as compute
    top, bottom, _, _ = corner_reach(cpx)
    above, below = exchange_halo(strip, top, bottom, rank, world, group)
    ext = torch.cat([above, strip, below], dim=0) if (above.shape[0] or below.shape[0]) else strip
    out = compute(ext, cpx, boundary)
    return out[above.shape[0]:above.shape[0] + strip.shape[0]]
