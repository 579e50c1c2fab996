"""Slice rendering on the B200 (ref pkg/src/echosplat/rasterizer.py).

``rasterize`` / ``render_slice`` keep the reference signatures
(rasterizer.py:140-186).  Underneath, a ``Renderer`` owns one libugs plan:

  ugs_bin      per-Gaussian factor + chi^2 box + cull + compact + windows
               (bit-exact with _prepare, rasterizer.py:109-137), plane-
               conditioned records, tile expansion and the stable radix sort
               into per-(slice, 16x16 tile) lists;
  ugs_forward  tile-resident accumulation + background blend.

The plan keeps the binning of the last batch, so the backward pass reuses it
instead of recomputing phase 1 the way the reference does
(gradients.py:49-52); a generation counter detects stale buffers.
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .geometry import (InvalidParameterError, SliceImage, SliceSpec,
                       chi2_cutoff, fill_slice, fill_slices)
from .model import GaussianCloud, ProbeFrameGaussian

DEFAULT_P_MASS = 0.95


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _device_index(device) -> int:
    """An index-less 'cuda' means the current device (torch semantics)."""
    d = torch.device(device) if device is not None else None
    if d is None or d.index is None:
        return torch.cuda.current_device()
    return d.index


class Renderer:
    """One libugs plan: the binning state of one batch of slices."""

    def __init__(self):
        L = _lib.lib()
        self._plan = ctypes.c_void_p()
        _lib.check(L.ugs_plan_create(ctypes.byref(self._plan)), "ugs_plan_create")
        self.generation = 0
        self.S = 0
        self.m = np.zeros(0, np.int64)
        self.k = np.zeros(0, np.int64)
        self.specs: list = []
        self.p_mass = DEFAULT_P_MASS
        self._cloud_key = None
        self._slices = None
        self.device_index = None
        self.counts_pending = False
        self.pairs = np.zeros(0, np.int64)

    def __del__(self):
        try:
            if self._plan:
                _lib.lib().ugs_plan_destroy(self._plan)
                self._plan = ctypes.c_void_p()
        except Exception:
            pass

    @staticmethod
    def cloud_key(cloud: GaussianCloud):
        return (cloud.means.data_ptr(), cloud.l_raw.data_ptr(), cloud.n,
                cloud.means._version, cloud.l_raw._version,
                cloud.intensity_raw._version, cloud.opacity_raw._version,
                getattr(cloud, "mutations", 0))

    def _guard(self, device):
        """Library calls run on the cloud's device (plan buffers, launches
        and the current stream all follow the current device); a plan is
        bound to the device of its first use."""
        idx = _device_index(device)
        if self.device_index is None:
            self.device_index = idx
        elif idx != self.device_index:
            raise InvalidParameterError(
                f"this Renderer's plan lives on cuda:{self.device_index}, "
                f"the cloud on cuda:{idx}")
        if idx == torch.cuda.current_device():
            return contextlib.nullcontext()   # already there: no device switch
        return torch.cuda.device(idx)

    def bin(self, cloud: GaussianCloud, specs, p: float = DEFAULT_P_MASS,
            slices=None):
        """Phase 1 + tile binning for a batch of slices (one host sync)."""
        with self._guard(cloud.device):
            return self._bin(cloud, specs, p, slices)

    def _bin(self, cloud, specs, p, slices):
        S = len(specs)
        if S < 1 or S > 64:
            raise InvalidParameterError("a batch holds 1..64 slices")
        if slices is None:
            slices = (_lib.Slice * S)()
            fill_slices(slices, specs, p)
        m = (ctypes.c_int64 * S)()
        k = (ctypes.c_int64 * S)()
        pp = (ctypes.c_int64 * S)()
        cs = cloud.c_struct()
        _lib.check(_lib.lib().ugs_bin(self._plan, ctypes.byref(cs), slices, S,
                                      _stream(), m, k, pp), "ugs_bin")
        self.pairs = np.frombuffer(pp, np.int64).copy()
        self._slices = slices
        self.S = S
        self.m = np.frombuffer(m, np.int64).copy()
        self.k = np.frombuffer(k, np.int64).copy()
        self.specs = list(specs)
        self.p_mass = p
        self._cloud_key = self.cloud_key(cloud)
        self.generation += 1
        return self.m, self.k

    def bin_async(self, cloud: GaussianCloud, specs, p: float = DEFAULT_P_MASS,
                  slices=None):
        """Phase 1 + binning without the host synchronisation
        (ugs_bin_async): the counts arrive with poll(), which also reports
        whether the batch overflowed the plan's buffers (then the forward /
        backward / update launched on it did nothing and must be re-issued)."""
        with self._guard(cloud.device):
            S = len(specs)
            if S < 1 or S > 64:
                raise InvalidParameterError("a batch holds 1..64 slices")
            if slices is None:
                slices = (_lib.Slice * S)()
                fill_slices(slices, specs, p)
            cs = cloud.c_struct()
            _lib.check(_lib.lib().ugs_bin_async(self._plan, ctypes.byref(cs), slices, S,
                                                _stream()), "ugs_bin_async")
            self._slices = slices
            self.S = S
            self.specs = list(specs)
            self.p_mass = p
            self._cloud_key = self.cloud_key(cloud)
            self.generation += 1
            self.counts_pending = True

    def render_batch(self, cloud: GaussianCloud, specs, pixels: torch.Tensor,
                     p: float = DEFAULT_P_MASS, slices=None):
        """bin_async + render in one library call (ugs_render_batch: the
        kernel chain replayed as one CUDA graph while the plan, cloud and
        batch shape repeat); poll() afterwards, as after bin_async."""
        with self._guard(cloud.device):
            S = len(specs)
            if S < 1 or S > 64:
                raise InvalidParameterError("a batch holds 1..64 slices")
            if slices is None:
                slices = (_lib.Slice * S)()
                fill_slices(slices, specs, p)
            cs = cloud.c_struct()
            _lib.check(_lib.lib().ugs_render_batch(self._plan, ctypes.byref(cs), slices, S,
                                                   pixels.data_ptr(), _stream()),
                       "ugs_render_batch")
            self._slices = slices
            self.S = S
            self.specs = list(specs)
            self.p_mass = p
            self._cloud_key = self.cloud_key(cloud)
            self.generation += 1
            self.counts_pending = True

    def poll(self) -> bool:
        """Counts of the last bin / bin_async (waits on one event); True if
        that sync-free batch overflowed (the plan has grown: retry it)."""
        S = max(self.S, 1)
        m = (ctypes.c_int64 * S)()
        k = (ctypes.c_int64 * S)()
        pp = (ctypes.c_int64 * S)()
        ovf = ctypes.c_int(0)
        _lib.check(_lib.lib().ugs_plan_poll(self._plan, ctypes.byref(ovf), m, k, pp),
                   "ugs_plan_poll")
        self.m = np.frombuffer(m, np.int64)[:self.S].copy()
        self.k = np.frombuffer(k, np.int64)[:self.S].copy()
        self.pairs = np.frombuffer(pp, np.int64)[:self.S].copy()
        self.counts_pending = False
        return bool(ovf.value)

    def forward(self, cloud: GaussianCloud, num: torch.Tensor, den: torch.Tensor):
        cs = cloud.c_struct()
        with self._guard(cloud.device):
            _lib.check(_lib.lib().ugs_forward(self._plan, ctypes.byref(cs),
                                              num.data_ptr(), den.data_ptr(),
                                              _stream()), "ugs_forward")

    def render(self, cloud: GaussianCloud, pixels: torch.Tensor):
        """clip(num / den, 0, 1) straight from the forward (ugs_render)."""
        cs = cloud.c_struct()
        with self._guard(cloud.device):
            _lib.check(_lib.lib().ugs_render(self._plan, ctypes.byref(cs), pixels.data_ptr(),
                                             _stream()), "ugs_render")

    def backward(self, cloud: GaussianCloud, num, den, dpix, grad, touched=None,
                 scale: float = 1.0):
        cs = cloud.c_struct()
        with self._guard(cloud.device):
            _lib.check(_lib.lib().ugs_backward(
                self._plan, ctypes.byref(cs), num.data_ptr(), den.data_ptr(),
                dpix.data_ptr(), grad.data_ptr(), _lib.ptr(touched), float(scale),
                _stream()), "ugs_backward")

    def backward_dense(self, cloud: GaussianCloud, num, den, dpix, grad, scale: float = 1.0):
        """ugs_backward_dense: grad (AoS-12) OVERWRITTEN with scale x the
        batch gradient, pad slot = accepted (no zeroing needed)."""
        cs = cloud.c_struct()
        with self._guard(cloud.device):
            _lib.check(_lib.lib().ugs_backward_dense(
                self._plan, ctypes.byref(cs), num.data_ptr(), den.data_ptr(),
                dpix.data_ptr(), grad.data_ptr(), float(scale), _stream()),
                "ugs_backward_dense")

    def accepted(self, device, windows: bool = False):
        """(accepted int64 per slice list, windows (M,4) int64 or None)."""
        with self._guard(device):
            return self._accepted(device, windows)

    def _settled(self):
        if self.counts_pending and self.poll():
            raise InvalidParameterError("the last sync-free batch overflowed the plan; "
                                        "re-bin it before exporting")

    def _accepted(self, device, windows):
        self._settled()
        M = int(self.m.sum())
        acc = torch.empty(max(M, 1), dtype=torch.int32, device=device)
        win = torch.empty((max(M, 1), 4), dtype=torch.int32, device=device) \
            if windows else None
        _lib.check(_lib.lib().ugs_export_accepted(
            self._plan, acc.data_ptr(), _lib.ptr(win), _stream()),
            "ugs_export_accepted")
        offs = np.concatenate([[0], np.cumsum(self.m)])
        accs = [acc[offs[s]:offs[s + 1]].long() for s in range(self.S)]
        wins = None if win is None else [win[offs[s]:offs[s + 1]].long()
                                         for s in range(self.S)]
        return accs, wins

    def bins(self, device):
        """(bin_range (n_bins,2) int32, sorted Gaussian ids (K,) int32)."""
        with self._guard(device):
            return self._bins(device)

    def _bins(self, device):
        self._settled()
        nb = ctypes.c_int32()
        kt = ctypes.c_int64()
        L = _lib.lib()
        _lib.check(L.ugs_export_bins(self._plan, None, None, ctypes.byref(nb),
                                     ctypes.byref(kt), _stream()), "ugs_export_bins")
        rng = torch.empty((max(nb.value, 1), 2), dtype=torch.int32, device=device)
        srt = torch.empty(max(kt.value, 1), dtype=torch.int32, device=device)
        _lib.check(L.ugs_export_bins(self._plan, rng.data_ptr(), srt.data_ptr(),
                                     None, None, _stream()), "ugs_export_bins")
        return rng[:nb.value], srt[:kt.value]

    def set_ordered(self, ordered: bool = True):
        """Strict per-pixel ascending-index accumulation (the reference's
        workers=1 order) instead of per-warp private buffers."""
        _lib.check(_lib.lib().ugs_plan_set_ordered(self._plan, int(ordered)),
                   "ugs_plan_set_ordered")

    def set_timing(self, enabled: bool = True):
        _lib.check(_lib.lib().ugs_plan_set_timing(self._plan, int(enabled)),
                   "ugs_plan_set_timing")

    def timings(self, reset: bool = False) -> dict:
        """{stage: (total ms, calls)} accumulated since the last reset."""
        n = len(_lib.STAGES)
        ms = (ctypes.c_double * n)()
        calls = (ctypes.c_int64 * n)()
        rc = _lib.lib().ugs_plan_timings(self._plan, ms, calls, n, int(reset))
        if rc < 0:
            _lib.check(rc, "ugs_plan_timings")
        return {name: (ms[i], calls[i]) for i, name in enumerate(_lib.STAGES)}

    def slice_info(self):
        """Per slice: (tiles_x, tiles_y, tile_base) as filled by ugs_bin."""
        return [(self._slices[s].tiles_x, self._slices[s].tiles_y,
                 self._slices[s].tile_base) for s in range(self.S)]


_DEFAULT: dict = {}


def default_renderer(device=None) -> Renderer:
    dev = _device_index(device)
    r = _DEFAULT.get(dev)
    if r is None:
        r = _DEFAULT[dev] = Renderer()
    return r


@dataclass
class RenderBuffers:
    """Accumulators plus the forward state backward needs (ref :40-52).

    ``intensity_num`` / ``opacity_sum`` are (H, W) float32 device tensors,
    ``accepted`` the ascending int64 indices of the surviving Gaussians.
    """

    intensity_num: torch.Tensor
    opacity_sum: torch.Tensor
    accepted: torch.Tensor
    spec: SliceSpec
    p_mass: float
    _renderer: Renderer = field(default=None, repr=False)
    _generation: int = field(default=-1, repr=False)
    _cloud_key: tuple = field(default=None, repr=False)

    @property
    def pixels(self) -> torch.Tensor:
        return torch.clamp(self.intensity_num / self.opacity_sum, 0.0, 1.0)


def as_cloud(cloud, device=None) -> GaussianCloud:
    """Accept our GaussianCloud or any object with the reference's fields."""
    if isinstance(cloud, GaussianCloud):
        return cloud
    return GaussianCloud(cloud.means, cloud.l_raw, cloud.intensity_raw,
                         cloud.opacity_raw, cloud.bg_intensity_raw,
                         cloud.bg_opacity_raw, cloud.beta, device=device)


def rasterize(cloud, spec: SliceSpec, p: float = DEFAULT_P_MASS,
              workers: int = 1, renderer: Renderer | None = None) -> RenderBuffers:
    """Render accumulators for one slice (ref rasterizer.py:140-179).

    ``workers`` is accepted for signature compatibility; the GPU path is
    always deterministic (fixed per-pixel accumulation order).
    """
    del workers
    chi2_cutoff(p)   # validates p like the reference
    cloud = as_cloud(cloud)
    r = renderer or default_renderer(cloud.device)
    r.bin(cloud, [spec], p)
    num = torch.empty((spec.height, spec.width), dtype=torch.float32,
                      device=cloud.device)
    den = torch.empty_like(num)
    r.forward(cloud, num, den)
    acc, _ = r.accepted(cloud.device)
    return RenderBuffers(num, den, acc[0], spec, p, r, r.generation,
                         r.cloud_key(cloud))


def render_slice(cloud, spec: SliceSpec, p: float = DEFAULT_P_MASS,
                 workers: int = 1) -> SliceImage:
    """One slice image, pixels = clip(num/den, 0, 1) (ref :182-186).
    Pixels are returned as a host float32 array, like the reference."""
    buf = rasterize(cloud, spec, p=p, workers=workers)
    return SliceImage(pixels=buf.pixels.cpu().numpy(), spacing=spec.spacing,
                      pose=spec.pose)


def render_slices(cloud, specs, p: float = DEFAULT_P_MASS,
                  renderer: Renderer | None = None) -> torch.Tensor:
    """Batched render-only path (the serving consumer of the forward, config
    C5): (S, H, W) clipped pixels on the device, written by the forward
    itself (ugs_render).  Binning is sync-free once the plan is sized: the
    host waits only for each chunk's count stage, to re-issue a chunk that
    overflowed the plan's buffers.  All specs must share width/height."""
    cloud = as_cloud(cloud)
    h, w = specs[0].height, specs[0].width
    if any(s.height != h or s.width != w for s in specs):
        raise InvalidParameterError("render_slices needs equal slice sizes")
    chi2_cutoff(p)
    r = renderer or default_renderer(cloud.device)
    out = torch.empty((len(specs), h, w), dtype=torch.float32, device=cloud.device)
    for i in range(0, len(specs), 64):
        chunk = specs[i:i + 64]
        _render_chunk(r, cloud, chunk, out[i:i + len(chunk)], p)
    return out


def _render_chunk(r, cloud, chunk, view, p):
    """One batch of render_slices; a batch whose tile instances exceed the
    library's 31-bit index budget (huge footprints) is split in halves."""
    try:
        r.render_batch(cloud, chunk, view, p)
        if r.poll():                  # overflowed: the plan has grown, retry
            r.bin(cloud, chunk, p)
            r.render(cloud, view)
    except _lib.UGSError as exc:
        if exc.status != _lib.UGS_ERR_RANGE or len(chunk) == 1:
            raise
        half = len(chunk) // 2
        _render_chunk(r, cloud, chunk[:half], view[:half], p)
        _render_chunk(r, cloud, chunk[half:], view[half:], p)


# ---- host utilities with the reference signatures (rasterizer.py:33-106) --

@dataclass(frozen=True)
class BoundingBox3:
    b_min: np.ndarray
    b_max: np.ndarray


def bounding_box(g: ProbeFrameGaussian, p: float = DEFAULT_P_MASS) -> BoundingBox3:
    cut = chi2_cutoff(p)
    half = np.sqrt(cut * np.diag(np.linalg.inv(g.precision_probe)))
    return BoundingBox3(g.mean_probe - half, g.mean_probe + half)


def cull(bboxes, spec: SliceSpec | None = None) -> np.ndarray:
    if isinstance(bboxes, tuple):
        b_min, b_max = bboxes
    else:
        b_min = np.array([b.b_min for b in bboxes]).reshape(-1, 3)
        b_max = np.array([b.b_max for b in bboxes]).reshape(-1, 3)
    mask = (b_min[:, 2] <= 0.0) & (b_max[:, 2] >= 0.0)
    if spec is not None:
        x1 = (spec.width - 1) / 2.0 * spec.spacing
        x2 = (spec.height - 1) / 2.0 * spec.spacing
        mask &= (b_max[:, 0] >= -x1) & (b_min[:, 0] <= x1)
        mask &= (b_max[:, 1] >= -x2) & (b_min[:, 1] <= x2)
    return mask


def compact(mask) -> np.ndarray:
    return np.nonzero(np.asarray(mask))[0]
