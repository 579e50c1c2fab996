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


# ---------------------------------------------------------------------------
# Fused multi-GPU update over peer memory (ugs_peer_update, include/ugs.h)
# ---------------------------------------------------------------------------

class _CudaArray:
    """A raw device range as a __cuda_array_interface__ object, so torch can
    alias it without a copy."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _align(x: int, a: int = 256) -> int:
    return (x + a - 1) // a * a


class PeerArena:
    """One rank's arena -- parameters, AoS-12 gradient and moments, densify
    statistics and background -- in a single CUDA IPC-exportable allocation,
    plus every peer's arena mapped into this process (cudaIpcOpenMemHandle;
    over NVLink on an NVSwitch node).  ``views`` describes all of them for
    ugs_peer_update / ugs_peer_gather.  Collective: every rank constructs
    (and closes) its arena at the same point of the program."""

    # (name, floats-or-ints per row, extra entries, typestr)
    _FIELDS = (("means", 3, 0, "<f4"), ("l_raw", 6, 0, "<f4"),
               ("intensity_raw", 1, 0, "<f4"), ("opacity_raw", 1, 0, "<f4"),
               ("grad", 12, 4, "<f4"), ("m", 12, 4, "<f4"), ("v", 12, 4, "<f4"),
               ("grad_sum", 1, 0, "<f4"), ("grad_cnt", 1, 0, "<i4"),
               ("sync", 0, 64, "<u4"))   # device-side step barrier flags

    def __init__(self, n: int, world: int, rank: int, group=None):
        import ctypes
        import torch.distributed as dist
        from . import _lib
        self.n, self.world, self.rank, self.group = n, world, rank, group
        L = _lib.lib()
        off, self.offsets = 0, {}
        for name, per, extra, _ in self._FIELDS:
            self.offsets[name] = off
            off = _align(off + 4 * (per * n + extra))
        self.offsets["bg_raw"] = off
        self.nbytes = off + 16
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_ubyte * 64)()
        _lib.check(L.ugs_ipc_alloc(self.nbytes, ctypes.byref(ptr), handle), "ugs_ipc_alloc")
        self.ptr = ptr.value
        # the barrier flags start at 0 (epochs count from 1) before any peer
        # can map and signal this arena
        torch.as_tensor(_CudaArray(self.ptr + self.offsets["sync"], (64,), "<u4"),
                        device="cuda").zero_()
        torch.cuda.synchronize()
        self.epoch = 0
        handles = [None] * world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.bases = []
        for q in range(world):
            if q == rank:
                self.bases.append(self.ptr)
                continue
            h = (ctypes.c_ubyte * 64).from_buffer_copy(handles[q])
            pp = ctypes.c_void_p()
            _lib.check(L.ugs_ipc_open(h, ctypes.byref(pp)), "ugs_ipc_open")
            self.bases.append(pp.value)
        self.views = (_lib.PeerView * world)()
        for q, b in enumerate(self.bases):
            v = self.views[q]
            for name in ("means", "l_raw", "intensity_raw", "opacity_raw", "grad", "m",
                         "v", "grad_sum", "grad_cnt", "bg_raw", "sync"):
                setattr(v, name, b + self.offsets[name])
        # this rank's arena as torch tensors (aliases, no copies)
        self.t = {}
        for name, per, extra, ts in self._FIELDS:
            if name == "sync":
                continue
            shape = (n, per) if (per > 1 and extra == 0) else (per * n + extra,)
            self.t[name] = torch.as_tensor(
                _CudaArray(self.ptr + self.offsets[name], shape, ts), device="cuda")
        self.t["bg_raw"] = torch.as_tensor(
            _CudaArray(self.ptr + self.offsets["bg_raw"], (2,), "<f8"), device="cuda")

    def shard(self):
        """[lo, hi) of the Gaussians this rank updates (ugs_peer_shard:
        multiples of 32, so a warp's rows move as 16-byte vectors)."""
        import ctypes
        from . import _lib
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().ugs_peer_shard(self.n, self.world, self.rank, ctypes.byref(lo),
                                             ctypes.byref(hi)), "ugs_peer_shard")
        return lo.value, hi.value

    def close(self, barrier) -> None:
        """Unmap the peers and free this arena once every rank is done with it."""
        from . import _lib
        barrier()
        L = _lib.lib()
        for q, b in enumerate(self.bases):
            if q != self.rank:
                _lib.check(L.ugs_ipc_close(b), "ugs_ipc_close")
        self.t = {}
        torch.cuda.synchronize()
        _lib.check(L.ugs_ipc_free(self.ptr), "ugs_ipc_free")
        self.bases = []
