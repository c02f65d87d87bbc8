"""World-size-2 (and 3) gloo tests of the multi-GPU decomposition on CPU.

The per-strip compute is injected: here the float64 oracle stands in for the
device kernel (this file tests the sharding/halo logic; the device kernel has
its own parity tests).  Stitched strip outputs must equal the single-process
result bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_compute(ext, cpx, boundary):
    from oracle import oracle as orc
    layers = [(l.offsets, l.weights) for l in cpx.layers]
    out = orc.apply_complex(ext.numpy(), layers, orc.CLAMP if boundary == "clamp" else orc.ZERO)
    return torch.from_numpy(out)


def _worker(rank, world, port, img, cpx, boundary, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_04556_b200.dist import apply_complex_strips, strip_bounds
        r0, r1 = strip_bounds(img.shape[0], rank, world)
        strip = torch.from_numpy(img[r0:r1].copy())
        out = apply_complex_strips(strip, cpx, rank, world, boundary, compute=_oracle_compute)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, img, cpx, boundary):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, cpx, boundary, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return np.concatenate([res[r] for r in range(world)], axis=0)


@pytest.mark.parametrize("world,boundary", [(2, "zero"), (2, "clamp"), (3, "zero")])
def test_strip_halo_exchange_is_exact(world, boundary):
    from oracle import oracle as orc
    from paper_2512_04556_b200 import synth
    cpx = synth.kawase_complex()
    img = np.random.default_rng(3).random((97, 41, 2))
    stitched = _run(world, img, cpx, boundary)
    full = _oracle_compute(torch.from_numpy(img), cpx, boundary).numpy()
    assert np.array_equal(stitched, full)


def test_undersized_halo_would_be_caught():
    """Cutting the halo to sum(r_l)+1 = 19 rows (BASELINE's figure) breaks the seam."""
    from paper_2512_04556_b200 import dist as d
    from paper_2512_04556_b200 import synth
    cpx = synth.kawase_complex()
    img = np.random.default_rng(4).random((90, 30))
    full = _oracle_compute(torch.from_numpy(img), cpx, "zero").numpy()
    r1 = 45
    ext = torch.from_numpy(img[:r1 + 19])
    part = _oracle_compute(ext, cpx, "zero").numpy()[:r1]
    assert not np.array_equal(part, full[:r1])
    ext = torch.from_numpy(img[:r1 + d.corner_reach(cpx)[1]])
    part = _oracle_compute(ext, cpx, "zero").numpy()[:r1]
    assert np.array_equal(part, full[:r1])


def test_shard_covers_everything():
    from paper_2512_04556_b200.dist import shard
    for n in (0, 1, 7, 64, 256):
        for world in (1, 2, 3, 8):
            idx = []
            for r in range(world):
                idx.extend(range(n)[shard(n, r, world)])
            assert idx == list(range(n))


def _oracle_into(src, dst, cpx, boundary):
    dst.copy_(_oracle_compute(src, cpx, boundary).to(dst.dtype).reshape(dst.shape))


def _pipe_worker(rank, world, port, img, cpx, boundary, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_04556_b200.dist import StripPipeline, strip_bounds
        r0, r1 = strip_bounds(img.shape[0], rank, world)
        pipe = StripPipeline(r1 - r0, img.shape[1], img.shape[2], torch.float64, torch.device("cpu"), cpx, rank,
                             world, boundary, compute_into=_oracle_into)
        pipe.strip.copy_(torch.from_numpy(img[r0:r1]))
        out1 = pipe.step().clone()
        out2 = pipe.step().clone()          # buffers are reused step after step
        q.put((rank, out1.numpy(), bool(torch.equal(out1, out2))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,boundary", [(2, "zero"), (3, "clamp"), (4, "zero")])
def test_strip_pipeline_overlapped_is_exact(world, boundary):
    """dist.StripPipeline: halo rows received into the extended buffer,
    interior filtered before the exchange completes, border bands after --
    the stitched result equals the single-process chain bit for bit."""
    from paper_2512_04556_b200 import synth
    cpx = synth.kawase_complex()
    img = np.random.default_rng(11).random((260, 23, 2))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipe_worker, args=(r, world, port, img, cpx, boundary, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, same = q.get(timeout=180)
        res[r] = out
        assert same
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _oracle_compute(torch.from_numpy(img), cpx, boundary).numpy()
    assert np.array_equal(np.concatenate([res[r] for r in range(world)], 0), full)


def _bench_strips_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        wl = bench.Strips(None, torch.device("cpu"), rank, world, shape=(192, 40, 4),
                          compute_into=_oracle_into, dtype=torch.float64)
        wl.step(None)
        q.put((rank, wl.rows, wl.out.numpy()))
    finally:
        dist.destroy_process_group()


def test_bench_strips_rank_path_end_to_end():
    """bench.Strips -- the c3big multi-GPU workload -- driven through its own
    rank path (pipeline construction, strip upload, step) on world-size-2
    gloo: the two ranks' rows stitch to the single-process result."""
    from paper_2512_04556_b200 import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_strips_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, rows, out = q.get(timeout=180)
        res[r] = (rows, out)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    img = synth.value_noise_frame_device(192, 40, 4, 100, torch.device("cpu"), dtype=torch.float64)
    full = _oracle_compute(img, synth.kawase_complex(), "zero").numpy()
    assert res[0][0] == (0, 96) and res[1][0] == (96, 192)
    assert np.array_equal(np.concatenate([res[0][1], res[1][1]], 0), full)
