"""Training on the B200 (ref pkg/src/echosplat/trainer.py).

Same public surface as the reference -- TrainConfig, AdamState, init_cloud,
loss, mean_lr, general_lr, adam_step, densify_prune_resample, train,
save/load_checkpoint -- with the parameters, moments, gradients and
densify statistics resident in HBM.  One training step is

    ugs_bin -> ugs_forward -> loss (device, float64) -> ugs_backward
      [-> NCCL all-reduce of the flat gradient when world_size > 1]
      -> ugs_grad_stats -> ugs_adam_step

over a batch of ``config.batch`` slices per GPU (the reference reads one
slice per iteration and never uses ``batch``, trainer.py:60; batch=1 on one
GPU reproduces its iteration exactly).  Densify/prune keeps its selection
and RNG on the host with numpy (bit-compatible candidate order and draws)
and applies the row surgery on the device (ugs_densify_apply).
"""

from __future__ import annotations

import ctypes
import json
import math
import os
import struct
import time
from dataclasses import asdict, dataclass

import numpy as np
import torch

from . import _lib
from .dataset import SliceDataset
from .geometry import InvalidParameterError, fill_slice
from .gradients import ParamGradients, grad_buffer
from .metrics import fused_loss, ssim_batch
from .metrics import loss as _loss
from .model import GaussianCloud
from .parallel import SliceScheduler, allreduce_gradients, grad_scale
from .rasterizer import Renderer, _stream

CHECKPOINT_MAGIC = b"UGSC"
CHECKPOINT_VERSION = 1
GROUPS = ("means", "l_raw", "intensity_raw", "opacity_raw")


class TrainingDivergedError(RuntimeError):
    def __init__(self, message, snapshot_path=None):
        super().__init__(message)
        self.snapshot_path = snapshot_path


class CheckpointFormatError(ValueError):
    pass


@dataclass
class TrainConfig:
    """ref trainer.py:43-74 (same fields, defaults and validation)."""

    n_gaussians: int = 20000
    iterations: int = 3000
    lr_general: float = 0.05
    lr_general_final: float | None = None
    lr_means_start: float = 0.00016
    lr_means_final: float = 1.6e-6
    ssim_loss_weight: float = 0.2
    l2_loss: bool = False
    heuristic_interval: int = 100
    densify_grad_threshold: float | None = None
    prune_alpha_threshold: float = 0.01
    split_variance_factor: float = 1.6
    split_scale_fraction: float = 0.01
    p_mass: float = 0.95
    seed: int = 0
    batch: int = 1
    workers: int = 1
    eval_interval: int = 100
    l_init_low: float = 4.0
    l_init_high: float = 5.0
    beta: float = 0.01

    def __post_init__(self):
        if self.n_gaussians < 1:
            raise InvalidParameterError("n_gaussians must be >= 1")
        if not 0.0 <= self.ssim_loss_weight <= 1.0:
            raise InvalidParameterError("ssim_loss_weight must be in [0, 1]")
        for name in ("lr_general", "lr_means_start", "lr_means_final"):
            if not getattr(self, name) > 0:
                raise InvalidParameterError(f"{name} must be > 0")


# AoS-12 rows (include/ugs.h): column ranges of each group, plus background
_COLS = {"means": (0, 3), "l_raw": (3, 9), "intensity_raw": (9, 10),
         "opacity_raw": (10, 11)}


def aos_views(flat: torch.Tensor, n: int) -> dict:
    """Per-group (strided) views of an AoS-12 buffer of 12n+2 floats."""
    rows = flat[:12 * n].view(n, 12)
    out = {k: (rows[:, a:b] if b - a > 1 else rows[:, a]) for k, (a, b) in _COLS.items()}
    out["bg"] = flat[12 * n:12 * n + 2]
    return out


class AdamState:
    """First/second moments (ref trainer.py:77-107) as float32 device buffers
    in the AoS-12 gradient layout; ``m``/``v`` give per-group views."""

    def __init__(self, n, device, t=0, beta1=0.9, beta2=0.999, eps=1e-15,
                 m_flat=None, v_flat=None):
        self.n = n
        self.m_flat = m_flat if m_flat is not None else torch.zeros(
            12 * n + 2, dtype=torch.float32, device=device)
        self.v_flat = v_flat if v_flat is not None else torch.zeros_like(self.m_flat)
        self.t = t
        self.beta1, self.beta2, self.eps = beta1, beta2, eps

    @staticmethod
    def for_cloud(cloud: GaussianCloud) -> "AdamState":
        return AdamState(cloud.n, cloud.device)

    def _views(self, flat):
        return aos_views(flat, self.n)

    @property
    def m(self):
        return self._views(self.m_flat)

    @property
    def v(self):
        return self._views(self.v_flat)


def init_cloud(config: TrainConfig, bounds, device=None) -> GaussianCloud:
    """Uniform means in `bounds`, default raws (ref trainer.py:110-127); the
    same numpy stream as the reference, then uploaded."""
    bounds = np.asarray(bounds, dtype=np.float64)
    if bounds.shape != (2, 3) or np.any(bounds[1] <= bounds[0]):
        raise InvalidParameterError("bounds must be a non-degenerate (2,3) box")
    rng = np.random.default_rng(config.seed)
    n = config.n_gaussians
    means = rng.uniform(bounds[0], bounds[1], size=(n, 3))
    l_raw = rng.uniform(config.l_init_low, config.l_init_high, size=(n, 6))
    return GaussianCloud(means.astype(np.float32), l_raw.astype(np.float32),
                         np.zeros(n, np.float32), np.full(n, 1.0, np.float32),
                         0.0, -4.0, config.beta, device=device)


def loss(pred, target, lam: float, l2: bool = False):
    """(1-lam)*L1 + lam*(1-SSIM) or MSE, and the pixel gradient (ref :130-151)."""
    return _loss(pred, target, lam, l2)


def mean_lr(config: TrainConfig, t: int) -> float:
    frac = min(t / max(config.iterations, 1), 1.0)
    return config.lr_means_start * (config.lr_means_final / config.lr_means_start) ** frac


def general_lr(config: TrainConfig, t: int) -> float:
    if config.lr_general_final is None:
        return config.lr_general
    frac = min(t / max(config.iterations, 1), 1.0)
    return config.lr_general * (config.lr_general_final / config.lr_general) ** frac


def _lr_array(lrs: dict):
    return (ctypes.c_double * 5)(lrs["means"], lrs["l_raw"], lrs["intensity_raw"],
                                 lrs["opacity_raw"], lrs["bg"])


def _adam_flat(state: AdamState, cloud: GaussianCloud, grad_flat: torch.Tensor,
               lrs: dict, zero_grad: bool, stats=None) -> None:
    """ugs_adam_step on an AoS-12 gradient; stats = (touched, sum, cnt)."""
    state.t += 1
    touched, gsum, gcnt = stats if stats is not None else (None, None, None)
    _lib.check(_lib.lib().ugs_adam_step(
        cloud.means.data_ptr(), cloud.l_raw.data_ptr(),
        cloud.intensity_raw.data_ptr(), cloud.opacity_raw.data_ptr(),
        cloud.bg_raw.data_ptr(), grad_flat.data_ptr(), state.m_flat.data_ptr(),
        state.v_flat.data_ptr(), cloud.n, state.t, _lr_array(lrs), state.beta1,
        state.beta2, state.eps, 1 if zero_grad else 0, _lib.ptr(touched),
        _lib.ptr(gsum), _lib.ptr(gcnt), _stream()), "ugs_adam_step")
    cloud.mark_mutated()


def adam_step(state: AdamState, cloud: GaussianCloud, grads: ParamGradients,
              lrs: dict) -> GaussianCloud:
    """One in-place Adam update (ref trainer.py:170-200), bit-compatible."""
    n = cloud.n
    if state.n != n:
        raise InvalidParameterError("moment/gradient shape mismatch")
    flat = grad_buffer(n, cloud.device)
    views = aos_views(flat, n)
    shapes = {"means": (n, 3), "l_raw": (n, 6), "intensity_raw": (n,),
              "opacity_raw": (n,)}
    for k in GROUPS:
        g = getattr(grads, "d_" + k)
        g = torch.as_tensor(g if isinstance(g, torch.Tensor) else np.asarray(g))
        if tuple(g.shape) != shapes[k]:
            raise InvalidParameterError(f"moment/gradient shape mismatch for {k}")
        views[k].copy_(g.to(device=cloud.device, dtype=torch.float32))
    flat[12 * n] = float(np.float32(grads.d_bg_intensity_raw))
    flat[12 * n + 1] = float(np.float32(grads.d_bg_opacity_raw))
    _adam_flat(state, cloud, flat, lrs, zero_grad=False)
    return cloud


def _sigmoid32(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, np.float32)
    return 1.0 / (1.0 + np.exp(-x))


def densify_prune_resample(cloud: GaussianCloud, grad_norm_avg, state: AdamState,
                           config: TrainConfig, rng: np.random.Generator,
                           scene_extent: float, threshold: float, max_total: int):
    """Prune transparent, split/clone high-gradient Gaussians (ref :203-279).

    Selection and RNG draws on the host (numpy, the reference's exact order);
    the row surgery, child means and shrunk factors on the device."""
    avg = np.asarray(grad_norm_avg.cpu().numpy() if isinstance(
        grad_norm_avg, torch.Tensor) else grad_norm_avg)
    keep = _sigmoid32(cloud.opacity_raw.cpu().numpy()) >= config.prune_alpha_threshold
    idx = np.nonzero(keep)[0]
    avg = avg[idx]
    n_keep = len(idx)
    budget = max_total - n_keep
    cand = np.nonzero(avg > threshold)[0]
    if budget <= 0 or len(cand) == 0:
        cand = cand[:0]
    elif len(cand) > budget:
        cand = cand[np.argsort(avg[cand])[::-1][:budget]]
    split = np.zeros(len(cand), np.uint8)
    z = np.zeros((len(cand), 6), np.float64)
    if len(cand):
        l_kept = cloud.l_raw[torch.as_tensor(idx[cand], device=cloud.device)].cpu().numpy()
        l64 = l_kept.astype(np.float64)
        beta = cloud.beta
        L = np.zeros((len(cand), 3, 3))
        for j in range(3):
            L[:, j, j] = l64[:, j] ** 2 + beta
        L[:, 1, 0], L[:, 2, 0], L[:, 2, 1] = l64[:, 3], l64[:, 4], l64[:, 5]
        inv = np.zeros_like(L)
        for j in range(3):
            inv[:, j, j] = 1.0 / L[:, j, j]
        inv[:, 1, 0] = -L[:, 1, 0] * inv[:, 0, 0] * inv[:, 1, 1]
        inv[:, 2, 1] = -L[:, 2, 1] * inv[:, 1, 1] * inv[:, 2, 2]
        inv[:, 2, 0] = -(L[:, 2, 0] * inv[:, 0, 0] + L[:, 2, 1] * inv[:, 1, 0]) * inv[:, 2, 2]
        cov = np.swapaxes(inv, -1, -2) @ inv
        max_var = np.max(np.diagonal(cov, axis1=-2, axis2=-1), axis=-1)
        split = (np.sqrt(max_var) > config.split_scale_fraction * scene_extent).astype(np.uint8)
        for j in range(len(cand)):
            if split[j]:
                z[j, :3] = rng.standard_normal(3)
                z[j, 3:] = rng.standard_normal(3)
    n_new = len(cand)
    n_dst = n_keep + n_new
    dev = cloud.device
    out = GaussianCloud(torch.empty((n_dst, 3), device=dev), torch.empty((n_dst, 6), device=dev),
                        torch.empty(n_dst, device=dev), torch.empty(n_dst, device=dev),
                        beta=cloud.beta, bg_raw=cloud.bg_raw.clone())
    st2 = AdamState(n_dst, dev, state.t, state.beta1, state.beta2, state.eps)
    keep_t = torch.as_tensor(idx.astype(np.int32), device=dev)
    cand_t = torch.as_tensor(cand.astype(np.int32), device=dev)
    split_t = torch.as_tensor(split, device=dev)
    z_t = torch.as_tensor(z, device=dev)
    src = cloud.c_struct()
    _lib.check(_lib.lib().ugs_densify_apply(
        ctypes.byref(src), state.m_flat.data_ptr(), state.v_flat.data_ptr(),
        keep_t.data_ptr() if n_keep else None, n_keep,
        cand_t.data_ptr() if n_new else None, split_t.data_ptr() if n_new else None,
        z_t.data_ptr() if n_new else None, n_new, float(config.split_variance_factor),
        out.means.data_ptr(), out.l_raw.data_ptr(), out.intensity_raw.data_ptr(),
        out.opacity_raw.data_ptr(), st2.m_flat.data_ptr(), st2.v_flat.data_ptr(),
        _stream()), "ugs_densify_apply")
    return out, st2


def dataset_bounds(dataset: SliceDataset, margin: float = 0.0) -> np.ndarray:
    """ref trainer.py:282-292."""
    corners = []
    for img in dataset.slices:
        h, w = img.pixels.shape
        x1 = (w - 1) / 2.0 * img.spacing
        x2 = (h - 1) / 2.0 * img.spacing
        local = np.array([[sx, sy, 0.0] for sx in (-x1, x1) for sy in (-x2, x2)])
        corners.append(img.pose.apply(local))
    pts = np.concatenate(corners)
    return np.stack([pts.min(axis=0) - margin, pts.max(axis=0) + margin])


def save_checkpoint(cloud: GaussianCloud, path, config: TrainConfig | None = None,
                    iteration: int = 0) -> None:
    """'UGSC' v1 little-endian checkpoint + JSON trailer, atomic (ref :295-313)."""
    trailer = json.dumps({"config": asdict(config) if config else None,
                          "iteration": iteration}).encode()
    d = cloud.to_numpy()
    parts = [CHECKPOINT_MAGIC, struct.pack("<II", CHECKPOINT_VERSION, cloud.n)]
    for k in GROUPS:
        parts.append(np.ascontiguousarray(d[k], "<f4").tobytes())
    parts += [struct.pack("<fff", d["bg_intensity_raw"], d["bg_opacity_raw"], cloud.beta),
              struct.pack("<I", len(trailer)), trailer]
    tmp = str(path) + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(b"".join(parts))
    os.replace(tmp, path)


def load_checkpoint(path, device=None):
    """(cloud, meta) from a 'UGSC' file (ref trainer.py:316-348)."""
    blob = open(path, "rb").read()
    if blob[:4] != CHECKPOINT_MAGIC:
        raise CheckpointFormatError(f"bad magic in {path}")
    if len(blob) < 12:
        raise CheckpointFormatError(f"truncated checkpoint {path}")
    version, n = struct.unpack_from("<II", blob, 4)
    if version != CHECKPOINT_VERSION:
        raise CheckpointFormatError(f"unsupported checkpoint version {version}")
    off = 12
    need = off + 44 * n + 12 + 4
    if len(blob) < need:
        raise CheckpointFormatError(f"truncated checkpoint {path}")
    arrs = {}
    for k, cols in (("means", 3), ("l_raw", 6), ("intensity_raw", 1), ("opacity_raw", 1)):
        a = np.frombuffer(blob, "<f4", count=n * cols, offset=off).copy()
        arrs[k] = a.reshape(n, cols) if cols > 1 else a
        off += 4 * n * cols
    bg_c, bg_a, beta = struct.unpack_from("<fff", blob, off)
    off += 12
    (tlen,) = struct.unpack_from("<I", blob, off)
    off += 4
    if off + tlen != len(blob):
        raise CheckpointFormatError(
            f"trailer size mismatch in {path}: expected {off + tlen} bytes, "
            f"file has {len(blob)}")
    meta = json.loads(blob[off:off + tlen].decode())
    cloud = GaussianCloud(arrs["means"], arrs["l_raw"], arrs["intensity_raw"],
                          arrs["opacity_raw"], float(bg_c), float(bg_a), float(beta),
                          device=device)
    return cloud, meta


# ---- training-state extension (the reference has no
# resume): the UGSC checkpoint stays bit-compatible and the optimiser /
# scheduler state goes to a sidecar "<path>.adam":
#   b"UGSA" | u32 version | u32 n | u64 t |
#   f32 m[12n+2] | f32 v[12n+2]        (AoS-12 layout, include/ugs.h)
#   f32 grad_sum[n] | i32 grad_cnt[n]  (densify statistics)
#   u32 trailer length | JSON {beta1, beta2, eps, iteration, beta (exact),
#                              threshold, rng (numpy bit-generator state),
#                              order, cursor}
STATE_MAGIC = b"UGSA"
STATE_VERSION = 1


def save_training_state(path, cloud: GaussianCloud, state: "AdamState", grad_sum, grad_cnt,
                        config: TrainConfig | None, iteration: int, extra: dict) -> None:
    """UGSC checkpoint at `path` + the resume sidecar `path + '.adam'`
    (both written atomically)."""
    save_checkpoint(cloud, path, config, iteration)
    n = cloud.n
    trailer = dict(extra)
    trailer.update(beta1=state.beta1, beta2=state.beta2, eps=state.eps, iteration=iteration,
                   beta=cloud.beta)   # exact (UGSC stores beta as float32)
    tb = json.dumps(trailer).encode()
    parts = [STATE_MAGIC, struct.pack("<IIQ", STATE_VERSION, n, state.t),
             state.m_flat.detach().cpu().numpy().astype("<f4").tobytes(),
             state.v_flat.detach().cpu().numpy().astype("<f4").tobytes(),
             grad_sum.detach().cpu().numpy().astype("<f4").tobytes(),
             grad_cnt.detach().cpu().numpy().astype("<i4").tobytes(),
             struct.pack("<I", len(tb)), tb]
    tmp = str(path) + ".adam.tmp"
    with open(tmp, "wb") as fh:
        fh.write(b"".join(parts))
    os.replace(tmp, str(path) + ".adam")


def load_training_state(path, device=None):
    """(cloud, AdamState, grad_sum, grad_cnt, meta) from save_training_state;
    meta is the UGSC trailer merged with the sidecar's JSON."""
    cloud, meta = load_checkpoint(path, device)
    blob = open(str(path) + ".adam", "rb").read()
    if blob[:4] != STATE_MAGIC or len(blob) < 20:
        raise CheckpointFormatError(f"bad training-state sidecar for {path}")
    version, n, t = struct.unpack_from("<IIQ", blob, 4)
    if version != STATE_VERSION:
        raise CheckpointFormatError(f"unsupported training-state version {version}")
    if n != cloud.n:
        raise CheckpointFormatError(f"sidecar has {n} Gaussians, checkpoint {cloud.n}")
    k = 12 * n + 2
    off = 20
    need = off + 4 * (2 * k + 2 * n) + 4
    if len(blob) < need:
        raise CheckpointFormatError(f"truncated training-state sidecar for {path}")
    m = np.frombuffer(blob, "<f4", count=k, offset=off).copy()
    v = np.frombuffer(blob, "<f4", count=k, offset=off + 4 * k).copy()
    off += 8 * k
    gs = np.frombuffer(blob, "<f4", count=n, offset=off).copy()
    gc = np.frombuffer(blob, "<i4", count=n, offset=off + 4 * n).copy()
    off += 8 * n
    (tlen,) = struct.unpack_from("<I", blob, off)
    off += 4
    if off + tlen != len(blob):
        raise CheckpointFormatError(f"trailer size mismatch in {path}.adam")
    extra = json.loads(blob[off:off + tlen].decode())
    cloud.beta = float(extra.get("beta", cloud.beta))
    dev = cloud.device
    state = AdamState(n, dev, int(t), extra["beta1"], extra["beta2"], extra["eps"],
                      m_flat=torch.as_tensor(m, device=dev),
                      v_flat=torch.as_tensor(v, device=dev))
    meta = dict(meta)
    meta.update(extra)
    return (cloud, state, torch.as_tensor(gs, device=dev), torch.as_tensor(gc, device=dev),
            meta)


# ---------------------------------------------------------------------------
# the training step engine (shared by train() and bench.py)
# ---------------------------------------------------------------------------

class TrainEngine:
    """Device-resident training state and the fused per-step pipeline."""

    def __init__(self, cloud: GaussianCloud, config: TrainConfig, specs, targets,
                 world_size: int = 1, rank: int = 0, process_group=None,
                 peer_update: bool | None = None):
        self.cloud = cloud
        self.config = config
        self.state = AdamState.for_cloud(cloud)
        # world > 1: fused reduce-scatter + Adam + all-gather over peer memory
        # (ugs_peer_update) instead of the NCCL all-reduce + replicated Adam
        # (default for world > 1; UGS_PEER_UPDATE=0 selects the NCCL path)
        if peer_update is None:
            peer_update = os.environ.get("UGS_PEER_UPDATE", "1") == "1"
        self.peer = bool(peer_update) and world_size > 1
        self.arena = None
        self.renderer = Renderer()
        self.specs = list(specs)
        # (n_slices, H, W) float32 on the device, or -- slices of different
        # sizes, which the reference also trains on (trainer.py:380-390) -- a
        # list of (H_i, W_i) tensors; ugs_bin / forward / backward take
        # per-slice sizes (pix_base offsets), only the loss runs per size
        self.targets = targets
        self.sizes = [(int(s.height), int(s.width)) for s in self.specs]
        self.uniform = len(set(self.sizes)) <= 1 and isinstance(targets, torch.Tensor)
        if self.uniform:
            h, w = self.targets.shape[-2:]
            if any(sz != (h, w) for sz in self.sizes):
                raise InvalidParameterError("targets do not match the slice sizes")
        else:
            if len(targets) != len(self.specs) or any(
                    tuple(t.shape[-2:]) != sz for t, sz in zip(targets, self.sizes)):
                raise InvalidParameterError("targets do not match the slice sizes")
            h, w = self.sizes[0]
        self.h, self.w = int(h), int(w)
        self.world_size, self.rank, self.pg = world_size, rank, process_group
        # per-slice constant structs, built once (host), copied per batch
        self._consts = (_lib.Slice * len(self.specs))()
        for i, s in enumerate(self.specs):
            fill_slice(self._consts[i], s, config.p_mass, 0)
        self._alloc_stats()
        self.grad = grad_buffer(cloud.n, cloud.device)
        self.last_loss = None
        self.last_pred = None
        if self.peer:
            self._bar = torch.zeros(1, dtype=torch.float32, device=cloud.device)
            self.peer = self._try_adopt_arena()

    # ---- peer-memory update (world > 1) ----
    def barrier(self):
        """All ranks' work enqueued so far is complete everywhere.  NCCL: a
        1-element all-reduce, ordered on the stream (no host sync); gloo
        (two ranks on one GPU in the tests): host-side."""
        import torch.distributed as dist
        if dist.get_backend(self.pg) == "nccl":
            dist.all_reduce(self._bar, group=self.pg)
        else:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.pg)

    def _try_adopt_arena(self) -> bool:
        """Set up the peer arenas; every rank agrees on the outcome, and any
        failure (no CUDA IPC / peer access) falls back to the NCCL path."""
        import torch.distributed as dist
        from .parallel import PeerArena
        arena, ok = None, 1.0
        try:
            arena = PeerArena(self.cloud.n, self.world_size, self.rank, self.pg)
        except Exception as exc:  # pragma: no cover - depends on the node
            ok = 0.0
            self.peer_error = repr(exc)
        flag = torch.tensor([ok], device=self.cloud.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.pg)
        if flag.item() < 1.0:
            if arena is not None:
                try:
                    arena.close(lambda: None)
                except Exception:  # pragma: no cover
                    pass
            return False
        self._adopt_arena(arena)
        return True

    def _adopt_arena(self, a=None):
        """Move the cloud, moments and statistics into a (fresh) peer arena."""
        from .parallel import PeerArena
        old = self.arena
        if a is None:
            a = PeerArena(self.cloud.n, self.world_size, self.rank, self.pg)
        c, st = self.cloud, self.state
        a.t["means"].copy_(c.means)
        a.t["l_raw"].copy_(c.l_raw)
        a.t["intensity_raw"].copy_(c.intensity_raw)
        a.t["opacity_raw"].copy_(c.opacity_raw)
        a.t["bg_raw"].copy_(c.bg_raw)
        a.t["m"][:st.m_flat.numel()].copy_(st.m_flat)
        a.t["v"][:st.v_flat.numel()].copy_(st.v_flat)
        a.t["grad_sum"].copy_(self.grad_sum)
        a.t["grad_cnt"].copy_(self.grad_cnt)
        c.means, c.l_raw = a.t["means"], a.t["l_raw"]
        c.intensity_raw, c.opacity_raw = a.t["intensity_raw"], a.t["opacity_raw"]
        c.bg_raw = a.t["bg_raw"]
        n = c.n
        st.m_flat, st.v_flat = a.t["m"][:12 * n + 2], a.t["v"][:12 * n + 2]
        self.grad = a.t["grad"][:12 * n + 2]
        self.grad_sum, self.grad_cnt = a.t["grad_sum"], a.t["grad_cnt"]
        self.arena = a
        if old is not None:
            old.close(self.barrier)
        self.barrier()

    # the step's two barriers as device flags in the peer arenas (signal /
    # fused wait-and-signal inside ugs_peer_update / wait) instead of two
    # 1-element NCCL all-reduces; UGS_PEER_FLAGS=0 keeps the collectives
    device_barriers = os.environ.get("UGS_PEER_FLAGS", "1") == "1"

    def _peer_step(self, lrs):
        st = self.state
        st.t += 1
        lo, hi = self.arena.shard()
        L = _lib.lib()
        a, W, r = self.arena, self.world_size, self.rank
        if self.device_barriers:
            a.epoch += 1
            e = a.epoch
            # ready: this rank's gradient is in its arena (peers wait on it
            # inside their update kernels)
            _lib.check(L.ugs_peer_signal(a.views, W, r, e, _stream()), "ugs_peer_signal")
            _lib.check(L.ugs_peer_update(a.views, W, r, self.cloud.n, lo, hi, st.t,
                                         _lr_array(lrs), st.beta1, st.beta2, st.eps, 1, e,
                                         _stream()), "ugs_peer_update")
            # done: every rank stored its shard's rows here
            _lib.check(L.ugs_peer_wait(a.views, W, r, e, _stream()), "ugs_peer_wait")
        else:
            self.barrier()            # every rank's gradient is in its arena
            _lib.check(L.ugs_peer_update(a.views, W, r, self.cloud.n, lo, hi, st.t,
                                         _lr_array(lrs), st.beta1, st.beta2, st.eps, 1, 0,
                                         _stream()), "ugs_peer_update")
            self.barrier()            # every parameter row is stored everywhere
        self.cloud.mark_mutated()

    def _alloc_stats(self):
        n, dev = self.cloud.n, self.cloud.device
        self.grad_sum = torch.zeros(n, dtype=torch.float32, device=dev)
        self.grad_cnt = torch.zeros(n, dtype=torch.int32, device=dev)
        self.touched = torch.zeros(n, dtype=torch.uint8, device=dev)

    def batch_structs(self, idx):
        B = len(idx)
        arr = (_lib.Slice * B)()
        sz = ctypes.sizeof(_lib.Slice)
        off = 0
        for j, i in enumerate(idx):
            ctypes.memmove(ctypes.byref(arr, j * sz), ctypes.byref(self._consts, int(i) * sz), sz)
            arr[j].pix_base = off
            h, w = self.sizes[int(i)]
            off += h * w
        return arr

    # optional CUDA-event instrumentation of the non-library parts of a step
    profile = False
    pairs_total = 0

    def _mark(self, name):
        if self.profile:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._events.setdefault(name, []).append(ev)

    def event_times(self, reset=True):
        """{name: total ms} between paired '<name>0'/'<name>1' marks."""
        torch.cuda.synchronize()
        out = {}
        ev = getattr(self, "_events", {})
        for k in list(ev):
            if k.endswith("0"):
                a, b = ev[k], ev.get(k[:-1] + "1", [])
                out[k[:-1]] = (sum(x.elapsed_time(y) for x, y in zip(a, b)), len(b))
        if reset:
            self._events = {}
        return out

    # sync-free binning (ugs_bin_async) on one GPU: the step never waits for
    # the host; its counts are harvested at the start of the next step (or by
    # settle()), and a batch that overflowed the plan's buffers -- its
    # forward / backward / Adam were device-side no-ops -- is re-issued then
    async_bin = os.environ.get("UGS_ASYNC_BIN", "1") == "1"
    reissued = 0          # steps re-issued after a sync-free binning overflow

    def _harvest(self):
        """Counts of the last launched step; True if it must be re-issued."""
        r = self.renderer
        if not r.counts_pending:
            return False
        ovf = r.poll()
        if not ovf:
            self.pairs_total += int(r.pairs.sum())
        return ovf

    def settle(self):
        """Make the last launched step final: harvest its counts and re-issue
        it if it overflowed (every later read of the cloud, the moments or
        the statistics goes through here)."""
        pend = getattr(self, "_pending", None)
        self._pending = None
        if pend is None:
            self._harvest()
            return
        while self._harvest():
            idx, it, targets_batch, loss_t, t0 = pend
            self.reissued += 1
            self.state.t = t0
            with torch.cuda.device(self.cloud.device):
                self._step(idx, it, False, targets_batch, loss_out=loss_t)

    def forward_loss(self, idx, targets_batch=None, loss_out=None):
        """bin + forward + loss for the slices `idx` (this rank's batch)."""
        cfg = self.config
        B = len(idx)
        if B > 64:
            raise InvalidParameterError("the GPU engine takes at most 64 slices per "
                                        "step and rank (config.batch <= 64)")
        if not self.uniform and targets_batch is None:
            return self._forward_loss_mixed(idx)
        if targets_batch is None:
            # slice ids via pinned memory: an async copy (a pageable one would
            # block the host until the stream drains)
            ids = torch.tensor(np.asarray(idx, np.int64)).pin_memory()
            ids = ids.to(self.cloud.device, non_blocking=True)
        structs = self.batch_structs(idx)
        specs = [self.specs[i] for i in idx]
        if self.async_bin and self.world_size == 1:
            self.renderer.bin_async(self.cloud, specs, cfg.p_mass, structs)
        else:
            self.renderer.bin(self.cloud, specs, cfg.p_mass, structs)
            self.pairs_total += int(self.renderer.pairs.sum())
        num = torch.empty((B, self.h, self.w), dtype=torch.float32, device=self.cloud.device)
        den = torch.empty_like(num)
        self.renderer.forward(self.cloud, num, den)
        self._mark("loss0")
        self.loss_mean = loss_out if loss_out is not None else \
            torch.empty((), dtype=torch.float64, device=self.cloud.device)
        if targets_batch is None:
            # the loss kernel reads the dataset rows directly (no gather copy)
            lv, dpix, _ = fused_loss(num, den, self.targets, cfg.ssim_loss_weight,
                                     cfg.l2_loss, target_index=ids, mean_out=self.loss_mean)
            tgt = self.targets[int(idx[0]):int(idx[0]) + 1]   # slice 0's target (a view)
        else:
            tgt = targets_batch
            lv, dpix, _ = fused_loss(num, den, tgt, cfg.ssim_loss_weight, cfg.l2_loss,
                                     mean_out=self.loss_mean)
        self._mark("loss1")
        return num, den, None, tgt, lv, dpix

    def _forward_loss_mixed(self, idx):
        """A batch whose slices differ in size: one flat (num, den, d_pixels)
        buffer at the slices' pix_base offsets; the loss runs per slice."""
        cfg = self.config
        dev = self.cloud.device
        structs = self.batch_structs(idx)
        self.renderer.bin(self.cloud, [self.specs[i] for i in idx], cfg.p_mass, structs)
        self.pairs_total += int(self.renderer.pairs.sum())
        offs = [int(structs[j].pix_base) for j in range(len(idx))]
        sizes = [self.sizes[int(i)] for i in idx]
        total = offs[-1] + sizes[-1][0] * sizes[-1][1]
        num = torch.empty(total, dtype=torch.float32, device=dev)
        den = torch.empty_like(num)
        dpix = torch.empty_like(num)
        self.renderer.forward(self.cloud, num, den)
        self._mark("loss0")
        lvs = []
        for j, i in enumerate(idx):
            (h, w), o = sizes[j], offs[j]
            view = (1, h, w)
            lv, dp, _ = fused_loss(num[o:o + h * w].view(view), den[o:o + h * w].view(view),
                                   self.targets[int(i)].view(view), cfg.ssim_loss_weight,
                                   cfg.l2_loss)
            dpix[o:o + h * w].copy_(dp.view(-1))
            lvs.append(lv)
        lv = torch.cat(lvs)
        self.loss_mean = lv.mean()
        self._mark("loss1")
        h0, w0 = sizes[0]
        first = (1, h0, w0)
        return (num[:h0 * w0].view(first), den[:h0 * w0].view(first), None,
                self.targets[int(idx[0])].view(first), lv, dpix, num, den)

    def step(self, idx, it: int, check_finite: bool = True, targets_batch=None):
        """One full training step; returns the mean loss over all ranks
        (python float) when check_finite, else this rank's batch mean as a
        device tensor (no collective).  Runs on the cloud's device."""
        with torch.cuda.device(self.cloud.device):
            self.settle()                    # the previous step is final
            if check_finite:
                return self._step(idx, it, True, targets_batch)
            t0 = self.state.t
            out = self._step(idx, it, False, targets_batch)
            self._pending = (list(idx), it, targets_batch, out, t0)
            return out

    def _step(self, idx, it, check_finite, targets_batch, loss_out=None):
        cfg = self.config
        out = self.forward_loss(idx, targets_batch, loss_out)
        if check_finite:
            # the loss is read before the update (the reference aborts on a
            # non-finite loss before it, trainer.py:392-396): a sync-free
            # batch is made final first, re-binned if it overflowed
            while self._harvest():
                out = self.forward_loss(idx, targets_batch, self.loss_mean)
        num, den, pred, tgt, lv, dpix = out[:6]
        self.last_num, self.last_den, self.last_tgt = num, den, tgt
        if len(out) > 6:
            num, den = out[6], out[7]     # flat buffers of a mixed-size batch
        loss_t = self.loss_mean
        if self.world_size > 1 and check_finite:
            # every rank takes the same abort decision (a NaN anywhere
            # propagates through the sum); without the check the step returns
            # this rank's batch mean and issues no collective for it
            torch.distributed.all_reduce(loss_t, group=self.pg)
            loss_t = loss_t / self.world_size
        loss_val = None
        if check_finite:
            loss_val = float(loss_t.item())
            if not math.isfinite(loss_val):
                return loss_val
        scale = grad_scale(len(idx), self.world_size)
        lr_g = general_lr(cfg, it)
        lrs = {"means": mean_lr(cfg, it), "l_raw": lr_g, "intensity_raw": lr_g,
               "opacity_raw": lr_g, "bg": lr_g}
        dpix = dpix.to(torch.float32).contiguous()
        if self.world_size == 1:
            # single GPU: backward + ordered accumulation + stats + Adam in one
            # call; the dense gradient is never materialised
            self._mark("backward_adam0")
            st = self.state
            st.t += 1
            cs = self.cloud.c_struct()
            _lib.check(_lib.lib().ugs_backward_adam(
                self.renderer._plan, ctypes.byref(cs), num.data_ptr(), den.data_ptr(),
                dpix.data_ptr(), float(scale), st.m_flat.data_ptr(),
                st.v_flat.data_ptr(), st.t, _lr_array(lrs), st.beta1, st.beta2, st.eps,
                self.grad_sum.data_ptr(), self.grad_cnt.data_ptr(), _stream()),
                "ugs_backward_adam")
            self.cloud.mark_mutated()
            self._mark("backward_adam1")
            return loss_val if check_finite else loss_t
        if self.peer:
            # the rank's gradient rows are overwritten (no 48 B/Gaussian memset)
            self.renderer.backward_dense(self.cloud, num, den, dpix, self.grad, scale)
            self._mark("adam0")
            self._peer_step(lrs)
            self._mark("adam1")
            return loss_val if check_finite else loss_t
        self.renderer.backward(self.cloud, num, den, dpix, self.grad, self.touched, scale)
        self._mark("allreduce0")
        allreduce_gradients(self.grad, self.touched, self.pg)
        self._mark("allreduce1")
        self._mark("adam0")
        _adam_flat(self.state, self.cloud, self.grad, lrs, zero_grad=True,
                   stats=(self.touched, self.grad_sum, self.grad_cnt))
        self._mark("adam1")
        return loss_val if check_finite else loss_t

    def gather_state(self):
        """Under the peer update every rank owns a shard of m, v and the
        statistics; fetch the owners' rows so this rank holds the full state
        (before densify or a training-state save)."""
        self.settle()
        if self.peer:
            self.barrier()
            _lib.check(_lib.lib().ugs_peer_gather(self.arena.views, self.world_size,
                                                  self.rank, self.cloud.n, _stream()),
                       "ugs_peer_gather")

    def load_state(self, state: "AdamState", grad_sum, grad_cnt):
        """Resume: adopt saved moments and statistics (same n as the cloud)."""
        self.settle()
        if state.n != self.cloud.n:
            raise InvalidParameterError("training state does not match the cloud")
        self.state = state
        self.grad_sum = grad_sum.to(torch.float32).contiguous()
        self.grad_cnt = grad_cnt.to(torch.int32).contiguous()
        if self.peer:
            self._adopt_arena()

    def densify(self, rng, scene_extent, threshold, max_total):
        self.settle()
        # every rank densifies the same full state
        self.gather_state()
        avg = (self.grad_sum.double() / torch.clamp(self.grad_cnt, min=1).double()).cpu().numpy()
        if threshold is None:
            threshold = float(np.quantile(avg, 0.9))
        self.cloud, self.state = densify_prune_resample(
            self.cloud, avg, self.state, self.config, rng, scene_extent, threshold,
            max_total)
        self._alloc_stats()
        self.grad = grad_buffer(self.cloud.n, self.cloud.device)
        if self.peer:
            self._adopt_arena()
        return threshold


def train(dataset: SliceDataset, config: TrainConfig, bounds=None,
          checkpoint_path=None, log_path=None, snapshot_path=None,
          time_budget_s: float | None = None, device=None,
          state_path=None, state_interval: int = 0, resume_from=None):
    """Full optimisation run (ref trainer.py:351-434) -> (cloud, log).

    Under torch.distributed (world_size > 1) every rank draws the same slice
    order and takes its own `config.batch` slices of each global step.

    Extension (the reference has no resume): `state_path` saves the full
    training state (UGSC checkpoint + the Adam / statistics / RNG / slice-
    order sidecar, save_training_state) every `state_interval` iterations and
    at the end (a "{iter}" field in the path keeps one file per save);
    `resume_from` continues such a run -- bitwise the same trajectory as an
    uninterrupted one."""
    train_slices = dataset.subset("train")
    if not train_slices:
        raise InvalidParameterError("dataset has no training slices")
    if bounds is None:
        bounds = dataset_bounds(dataset)
    bounds = np.asarray(bounds, np.float64)
    world, rank, pg = 1, 0, None
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        world, rank = torch.distributed.get_world_size(), torch.distributed.get_rank()
    rng = np.random.default_rng(config.seed)
    start = 1
    if resume_from is not None:
        cloud, r_state, r_gs, r_gc, r_meta = load_training_state(resume_from, device)
    else:
        cloud = init_cloud(config, bounds, device)
    specs = [s.spec for s in train_slices]
    if config.batch > 64:
        raise InvalidParameterError("the GPU engine takes at most 64 slices per step "
                                    "and rank: config.batch must be <= 64")
    pix = [np.asarray(s.pixels, np.float32) for s in train_slices]
    if len({p.shape for p in pix}) == 1:
        targets = torch.as_tensor(np.stack(pix), device=cloud.device)
    else:   # slices of different sizes (the reference trains on any slice)
        targets = [torch.as_tensor(p, device=cloud.device) for p in pix]
    eng = TrainEngine(cloud, config, specs, targets, world, rank, pg)
    scene_extent = float(np.linalg.norm(bounds[1] - bounds[0]))
    max_total = 2 * config.n_gaussians
    threshold = config.densify_grad_threshold
    sched = SliceScheduler(rng, len(train_slices), config.batch, world, rank)
    if resume_from is not None:
        eng.load_state(r_state, r_gs, r_gc)
        rng.bit_generator.state = r_meta["rng"]
        sched.order = np.asarray(r_meta["order"], dtype=np.int64)
        sched.cursor = int(r_meta["cursor"])
        threshold = r_meta["threshold"]
        start = int(r_meta["iteration"]) + 1

    def save_state(it):
        eng.gather_state()
        if rank == 0:
            path = str(state_path)
            path = path.format(iter=it) if "{iter" in path else path
            save_training_state(path, eng.cloud, eng.state, eng.grad_sum, eng.grad_cnt,
                                config, it, {"threshold": threshold,
                                             "rng": rng.bit_generator.state,
                                             "order": [int(x) for x in sched.order],
                                             "cursor": sched.cursor})

    log = []
    t0 = time.perf_counter()
    it = start - 1
    for it in range(start, config.iterations + 1):
        loss_val = eng.step(sched.next(), it)
        if not math.isfinite(loss_val):
            snap = snapshot_path or (str(checkpoint_path or "echosplat") + ".diverged")
            if rank == 0:
                save_checkpoint(eng.cloud, snap, config, it)
            raise TrainingDivergedError(
                f"non-finite loss at iteration {it}; snapshot at {snap}", snap)
        if config.heuristic_interval > 0 and it % config.heuristic_interval == 0:
            threshold = eng.densify(rng, scene_extent, threshold, max_total)
        if it % config.eval_interval == 0 or it == config.iterations:
            pred = eng.last_num[:1] / eng.last_den[:1]
            s = ssim_batch(torch.clamp(pred, 0, 1), eng.last_tgt[:1])
            entry = {"iter": it, "wall_ms": (time.perf_counter() - t0) * 1000.0,
                     "loss": loss_val, "train_ssim": float(s[0])}
            log.append(entry)
            if log_path is not None and rank == 0:
                with open(log_path, "a") as fh:
                    fh.write(json.dumps(entry) + "\n")
        if state_path is not None and state_interval > 0 and it % state_interval == 0:
            save_state(it)
        if time_budget_s is not None and time.perf_counter() - t0 >= time_budget_s:
            break
    if state_path is not None:
        save_state(it)
    if checkpoint_path is not None and rank == 0:
        save_checkpoint(eng.cloud, checkpoint_path, config, config.iterations)
    return eng.cloud, log
