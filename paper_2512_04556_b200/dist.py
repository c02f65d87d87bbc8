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

`StripPipeline` is the production form of the strip path: the rank's strip
lives inside a preallocated extended buffer, the neighbours' halo rows are
received straight into its ends (no concatenation), and the interior rows --
which do not depend on any halo -- are filtered while the exchange is in
flight; only two thin border bands wait for it.

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

    Convenience form of StripPipeline (it copies `strip` into a fresh
    pipeline).  `compute(img, cpx, boundary) -> tensor` overrides the device
    chain."""
    into = None
    if compute is not None:
        def into(src, dst, c, b):
            dst.copy_(compute(src, c, b))
    pipe = StripPipeline(strip.shape[0], strip.shape[1], strip.shape[2] if strip.dim() == 3 else 1, strip.dtype,
                         strip.device, cpx, rank, world, boundary, group, compute_into=into)
    pipe.strip.copy_(strip.reshape(pipe.strip.shape))
    return pipe.step().reshape(strip.shape)


def _halo_ops(ext, top_h, h, bot_h, top, bottom, rank, world, group):
    """P2P ops of one exchange: our first `bottom` rows go up, our last `top`
    rows go down; the neighbours' rows land in ext[:top_h] / ext[top_h+h:]."""
    import torch.distributed as dist
    ops = []
    if rank > 0:
        if bottom:
            ops.append(dist.P2POp(dist.isend, ext[top_h:top_h + bottom], rank - 1, group))
        if top_h:
            ops.append(dist.P2POp(dist.irecv, ext[:top_h], rank - 1, group))
    if rank < world - 1:
        if top:
            ops.append(dist.P2POp(dist.isend, ext[top_h + h - top:top_h + h], rank + 1, group))
        if bot_h:
            ops.append(dist.P2POp(dist.irecv, ext[top_h + h:], rank + 1, group))
    return ops


class StripPipeline:
    """One rank's row strip of a large image, filtered with an overlapped halo
    exchange.

    Output row y of the strip reads input rows [y - top, y + bottom]
    (`corner_reach`).  Per step:
      1. post the P2P exchange (our boundary rows out, the neighbours' rows
         into the preallocated ends of `ext`);
      2. filter the strip alone into `out` -- rows [top, h - bottom) only read
         the strip, so they are final (the image's own edges are final too);
      3. wait for the exchange (for NCCL a stream dependency, not a host
         block), then filter the two border bands -- 2*top+bottom and
         top+2*bottom rows of `ext` -- and copy their central `top` / `bottom`
         rows into `out`.
    With NCCL, step 2 runs on the compute stream while the transfer runs on
    NCCL's stream.  `compute_into(src, dst, cpx, boundary)` defaults to the
    device chain (engine.chain_into); tests inject a CPU oracle.

    Write the strip's rows into `strip` (a view into `ext`) before `step()`.
    """

    def __init__(self, rows: int, width: int, channels: int, dtype, device, cpx: KernelComplex,
                 rank: int, world: int, boundary: str = "zero", group=None, compute_into=None):
        import torch
        top, bottom = corner_reach(cpx)[:2]
        self.top, self.bottom = top, bottom
        self.top_h = top if rank > 0 else 0
        self.bot_h = bottom if rank < world - 1 else 0
        if world > 1 and rows < max(top, bottom):
            raise ValueError(f"strip of {rows} rows is shorter than the halo ({top}, {bottom})")
        self.h, self.rank, self.world = rows, rank, world
        self.cpx, self.boundary, self.group = cpx, boundary, group
        if compute_into is None:
            from .engine import chain_into as compute_into
        self.compute_into = compute_into
        shape = (width, channels)
        self.ext = torch.zeros((self.top_h + rows + self.bot_h,) + shape, dtype=dtype, device=device)
        self.strip = self.ext[self.top_h:self.top_h + rows]
        self.out = torch.empty((rows,) + shape, dtype=dtype, device=device)
        # border bands: (input rows of ext, their filtered copy, first kept
        # band row, first out row, rows kept).  A band clipped at an end of
        # ext ends at the image's own edge there, so it stays exact.
        n_ext = self.ext.shape[0]
        self._bands = []
        if self.top_h:
            src = self.ext[:min(n_ext, 2 * top + bottom)]
            self._bands.append((src, torch.empty_like(src), top, 0, top))
        if self.bot_h:
            a = max(0, self.top_h + rows - bottom - top)
            src = self.ext[a:]
            self._bands.append((src, torch.empty_like(src), self.top_h + rows - bottom - a, rows - bottom, bottom))

    def step(self):
        """Filter the strip; returns `out` (this rank's rows of the result)."""
        import torch.distributed as dist
        ops = _halo_ops(self.ext, self.top_h, self.h, self.bot_h, self.top, self.bottom, self.rank,
                        self.world, self.group)
        reqs = dist.batch_isend_irecv(ops) if ops else []
        self.compute_into(self.strip, self.out, self.cpx, self.boundary)    # interior, overlapped
        for r in reqs:
            r.wait()
        for src, dst, k0, o0, n in self._bands:
            self.compute_into(src, dst, self.cpx, self.boundary)
            self.out[o0:o0 + n].copy_(dst[k0:k0 + n])
        return self.out
