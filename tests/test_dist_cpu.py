"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel host
logic: the slice schedule, per-rank gradient scaling, the AoS-12 packing and
the single all-reduce reproduce the one-process mean-gradient step.  The
per-slice gradients come from the oracle (this box has no GPU); the code
under test is paper_2505_05643_b200.parallel, which the trainer uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cases
from oracle import oracle as O
from paper_2505_05643_b200.parallel import (SliceScheduler, allreduce_gradients,
                                            grad_scale, pack_aos12, unpack_aos12)

B, WORLD, N = 2, 2, 60


def _scene():
    rng = np.random.default_rng(77)
    cloud = cases.random_cloud(rng, N, extent=6.0)
    specs = [cases.random_pose(rng, 2.0) for _ in range(6)]
    consts = [O.slice_constants(R, t, 20, 18, 0.8, 0.95) for R, t in specs]
    dps = [np.random.default_rng(100 + i).standard_normal((18, 20)).astype(np.float32)
           for i in range(6)]
    return cloud, consts, dps


def _slice_grads(cloud, sc, dpix):
    args = (cloud["means"], cloud["l_raw"], cloud["intensity_raw"],
            cloud["opacity_raw"], cloud["bg_intensity_raw"], cloud["bg_opacity_raw"],
            cloud["beta"], sc)
    num, den, acc, G = O.rasterize(*args)
    g = O.backward(*args, num, den, dpix, gathered=G)
    touched = np.zeros(N, np.uint8)
    touched[acc] = 1
    return g, touched


def _rank_flat(rank, world, picks_per_step):
    cloud, consts, dps = _scene()
    flat = torch.zeros(12 * N + 2)
    touched = torch.zeros(N, dtype=torch.uint8)
    s = grad_scale(B, world)
    for i in picks_per_step[rank * B:(rank + 1) * B] if world > 1 else picks_per_step:
        g, t = _slice_grads(cloud, consts[i], dps[i])
        flat += s * pack_aos12(g["d_means"], g["d_l_raw"], g["d_intensity_raw"],
                               g["d_opacity_raw"], [g["d_bg_intensity_raw"],
                                                    g["d_bg_opacity_raw"]])
        touched |= torch.as_tensor(t)
    return flat, touched


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sched = SliceScheduler(np.random.default_rng(5), 6, B, world, rank)
        picks = sched.next_global()
        flat, touched = _rank_flat(rank, world, picks)
        allreduce_gradients(flat, touched)
        q.put((rank, picks, flat.numpy(), touched.numpy(), sched.next()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_scheduler_matches_reference_order():
    """world=1, batch=1 is the reference's permutation walk (trainer.py:375-386)."""
    rng_a, rng_b = np.random.default_rng(3), np.random.default_rng(3)
    s = SliceScheduler(rng_a, 5)
    order, cursor, ref = rng_b.permutation(5), 0, []
    for _ in range(12):
        if cursor >= len(order):
            order, cursor = rng_b.permutation(5), 0
        ref.append(int(order[cursor]))
        cursor += 1
    assert [s.next()[0] for _ in range(12)] == ref


def test_rank_partition_covers_global_batch():
    a = SliceScheduler(np.random.default_rng(9), 7, 3, 2, 0)
    b = SliceScheduler(np.random.default_rng(9), 7, 3, 2, 1)
    for _ in range(5):
        pa, pb = a.next(), b.next()
        assert len(pa) == len(pb) == 3
    g = SliceScheduler(np.random.default_rng(9), 7, 3, 2, 0)
    for _ in range(5):
        picks = g.next_global()
    assert picks[:3] == pa and picks[3:] == pb


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(1)
    parts = [rng.standard_normal((N, 3)), rng.standard_normal((N, 6)),
             rng.standard_normal(N), rng.standard_normal(N), rng.standard_normal(2)]
    flat = pack_aos12(*parts)
    back = unpack_aos12(flat, N)
    for k, p in zip(("d_means", "d_l_raw", "d_intensity_raw", "d_opacity_raw", "d_bg"), parts):
        np.testing.assert_allclose(back[k].numpy(), np.asarray(p, np.float32))


def test_two_rank_allreduce_equals_single_process():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(WORLD):
        r, picks, flat, touched, nxt = q.get(timeout=240)
        out[r] = (picks, flat, touched, nxt)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # both ranks hold the same reduced gradient and mask ...
    np.testing.assert_array_equal(out[0][1], out[1][1])
    np.testing.assert_array_equal(out[0][2], out[1][2])
    assert out[0][0] == out[1][0]            # same global picks on every rank
    assert out[0][3] != out[1][3]            # ... but disjoint next batches
    # ... equal to one process averaging the whole global batch
    picks = out[0][0]
    cloud, consts, dps = _scene()
    ref = torch.zeros(12 * N + 2)
    ref_t = np.zeros(N, np.uint8)
    for i in picks:
        g, t = _slice_grads(cloud, consts[i], dps[i])
        ref += grad_scale(B, WORLD) * pack_aos12(
            g["d_means"], g["d_l_raw"], g["d_intensity_raw"], g["d_opacity_raw"],
            [g["d_bg_intensity_raw"], g["d_bg_opacity_raw"]])
        ref_t |= t
    np.testing.assert_allclose(out[0][1], ref.numpy(), rtol=1e-6, atol=1e-7)
    np.testing.assert_array_equal(out[0][2], ref_t)
