"""Slice-batch data parallelism.

The training path shards by probe slices: parameters are replicated, every
rank draws the same host slice order and takes its own ``batch`` slices of
each global step, and the per-rank gradients (scaled 1/(batch*world)) are
summed with one all-reduce of the AoS-12 buffer before the identical Adam
update on every rank.  These helpers hold that host logic so it is shared by
``trainer.train``, ``bench.py`` and the CPU (gloo) tests.
"""

from __future__ import annotations

import numpy as np
import torch


class SliceScheduler:
    """The reference's slice order (ref trainer.py:375-386: a permutation per
    epoch from the training rng), cut into global batches of batch*world
    slices; rank r takes picks [r*batch, (r+1)*batch)."""

    def __init__(self, rng: np.random.Generator, n_slices: int, batch: int = 1,
                 world: int = 1, rank: int = 0):
        if n_slices < 1:
            raise ValueError("need at least one slice")
        self.rng, self.n, self.batch, self.world, self.rank = rng, n_slices, batch, world, rank
        self.order = rng.permutation(n_slices)
        self.cursor = 0

    def next_global(self) -> list:
        picks = []
        for _ in range(self.batch * self.world):
            if self.cursor >= len(self.order):
                self.order = self.rng.permutation(self.n)
                self.cursor = 0
            picks.append(int(self.order[self.cursor]))
            self.cursor += 1
        return picks

    def next(self) -> list:
        g = self.next_global()
        return g[self.rank * self.batch:(self.rank + 1) * self.batch]


def grad_scale(batch: int, world: int) -> float:
    """Per-slice gradient weight: the global step uses the mean over the
    batch*world slices (batch=1, world=1 reproduces the reference exactly)."""
    return 1.0 / (batch * world)


def pack_aos12(d_means, d_l_raw, d_intensity_raw, d_opacity_raw, d_bg,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """Raw-parameter gradients -> AoS-12 buffer (include/ugs.h layout)."""
    d_means = torch.as_tensor(d_means, dtype=torch.float32)
    n = d_means.shape[0]
    if out is None:
        out = torch.zeros(12 * n + 2, dtype=torch.float32, device=d_means.device)
    rows = out[:12 * n].view(n, 12)
    rows[:, 0:3] = d_means
    rows[:, 3:9] = torch.as_tensor(d_l_raw, dtype=torch.float32, device=out.device)
    rows[:, 9] = torch.as_tensor(d_intensity_raw, dtype=torch.float32, device=out.device)
    rows[:, 10] = torch.as_tensor(d_opacity_raw, dtype=torch.float32, device=out.device)
    out[12 * n:12 * n + 2] = torch.as_tensor(np.asarray(d_bg, np.float32), device=out.device)
    return out


def unpack_aos12(flat: torch.Tensor, n: int) -> dict:
    rows = flat[:12 * n].view(n, 12)
    return {"d_means": rows[:, 0:3], "d_l_raw": rows[:, 3:9],
            "d_intensity_raw": rows[:, 9], "d_opacity_raw": rows[:, 10],
            "d_bg": flat[12 * n:12 * n + 2]}


def allreduce_gradients(flat: torch.Tensor, touched: torch.Tensor | None = None,
                        group=None) -> None:
    """The only exchange of a step: sum the AoS-12 gradient, max the
    accepted-Gaussian mask (densify statistics count a Gaussian once per
    step if any rank's slice accepted it)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(flat, group=group)
    if touched is not None:
        dist.all_reduce(touched, op=dist.ReduceOp.MAX, group=group)
