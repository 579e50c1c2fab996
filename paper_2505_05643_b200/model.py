"""Gaussian cloud on the device (ref pkg/src/echosplat/model.py).

Same parameters and raw layout as the reference's ``GaussianCloud``
(model.py:31-89): means (N,3) mm, l_raw (N,6) = (L11, L22, L33, L21, L31,
L32) with L_jj = l_jj^2 + beta, sigmoid intensity / opacity, and a uniform
background (bg_intensity_raw, bg_opacity_raw).  The arrays live in HBM as
float32 torch tensors (44 B/Gaussian, structure of arrays); the background
raws are a float64 device pair so Adam can update them without a host trip.

The small triangular-factor helpers (build_L, invert_lower_triangular, ...)
are host numpy utilities with the reference's signatures; the render path
never uses them (the kernels rebuild L in registers).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .geometry import InvalidParameterError, ProbePose


class SingularMatrixError(ValueError):
    """Triangular factor has a non-positive diagonal entry (ref model.py:23)."""


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x)))


def _dev(device):
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2505_05643_b200 needs a CUDA device "
                               "(there is no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


_F64_WARNED = False


def _warn_f64(x):
    """The reference renders a float64 cloud in float64 (a side effect of
    numba typing); this path computes in float32 (the fp32 tolerance of the
    task): say so once instead of converting silently."""
    global _F64_WARNED
    dt = getattr(x, "dtype", None)
    if not _F64_WARNED and dt in (np.float64, torch.float64):
        _F64_WARNED = True
        import warnings
        warnings.warn("GaussianCloud: float64 parameters are stored and rendered in float32 "
                      "(the CUDA path's arithmetic type); the reference would render them "
                      "in float64", stacklevel=3)


def _as_param(x, shape_tail, device):
    _warn_f64(x)
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.float32)
    else:
        t = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32),
                            device=device)
    t = t.contiguous()
    if t.shape[1:] != shape_tail:
        raise InvalidParameterError("parameter has the wrong trailing shape")
    return t


class GaussianCloud:
    """Structure-of-arrays Gaussian cloud resident on one CUDA device."""

    def __init__(self, means, l_raw, intensity_raw, opacity_raw,
                 bg_intensity_raw=0.0, bg_opacity_raw=-4.0, beta=0.01,
                 device=None, bg_raw=None):
        if not beta > 0:
            raise InvalidParameterError("beta must be > 0")
        dev = _dev(device if device is not None else
                   (means.device if isinstance(means, torch.Tensor)
                    and means.is_cuda else None))
        self.means = _as_param(means, (3,), dev)
        n = self.means.shape[0]
        self.l_raw = _as_param(l_raw, (6,), dev)
        self.intensity_raw = _as_param(intensity_raw, (), dev)
        self.opacity_raw = _as_param(opacity_raw, (), dev)
        if self.l_raw.shape[0] != n:
            raise InvalidParameterError("means must be (N,3) and l_raw (N,6)")
        if self.intensity_raw.shape != (n,) or self.opacity_raw.shape != (n,):
            raise InvalidParameterError("intensity_raw/opacity_raw must be (N,)")
        if bg_raw is not None:
            self.bg_raw = bg_raw.to(device=dev, dtype=torch.float64).contiguous()
        else:
            self.bg_raw = torch.tensor([float(bg_intensity_raw),
                                        float(bg_opacity_raw)],
                                       dtype=torch.float64, device=dev)
        self.beta = float(beta)
        # bumped by every library call that rewrites the parameters through
        # raw pointers (Adam, the fused step, the peer update): those writes
        # do not bump the tensors' torch _version, and the renderer's cached
        # binning / records must not be reused across them
        self.mutations = 0

    def mark_mutated(self) -> None:
        self.mutations += 1

    # --- reference-compatible accessors ----------------------------------
    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    @property
    def device(self):
        return self.means.device

    @property
    def intensity(self) -> torch.Tensor:
        return torch.sigmoid(self.intensity_raw)

    @property
    def opacity(self) -> torch.Tensor:
        return torch.sigmoid(self.opacity_raw)

    @property
    def bg_intensity_raw(self) -> float:
        return float(self.bg_raw[0].item())

    @bg_intensity_raw.setter
    def bg_intensity_raw(self, value):
        self.bg_raw[0] = float(value)

    @property
    def bg_opacity_raw(self) -> float:
        return float(self.bg_raw[1].item())

    @bg_opacity_raw.setter
    def bg_opacity_raw(self, value):
        self.bg_raw[1] = float(value)

    @property
    def bg_intensity(self) -> float:
        return float(sigmoid(self.bg_intensity_raw))

    @property
    def bg_opacity(self) -> float:
        return float(sigmoid(self.bg_opacity_raw))

    def copy(self) -> "GaussianCloud":
        return GaussianCloud(self.means.clone(), self.l_raw.clone(),
                             self.intensity_raw.clone(), self.opacity_raw.clone(),
                             beta=self.beta, bg_raw=self.bg_raw.clone())

    def to_numpy(self) -> dict:
        return dict(means=self.means.cpu().numpy(), l_raw=self.l_raw.cpu().numpy(),
                    intensity_raw=self.intensity_raw.cpu().numpy(),
                    opacity_raw=self.opacity_raw.cpu().numpy(),
                    bg_intensity_raw=self.bg_intensity_raw,
                    bg_opacity_raw=self.bg_opacity_raw, beta=self.beta)

    @staticmethod
    def from_numpy(d: dict, device=None) -> "GaussianCloud":
        return GaussianCloud(d["means"], d["l_raw"], d["intensity_raw"],
                             d["opacity_raw"], d["bg_intensity_raw"],
                             d["bg_opacity_raw"], d.get("beta", 0.01), device)

    def c_struct(self):
        """The ugs_cloud view of this cloud (pointers stay valid while the
        tensors live)."""
        from ._lib import Cloud
        return Cloud(self.means.data_ptr(), self.l_raw.data_ptr(),
                     self.intensity_raw.data_ptr(), self.opacity_raw.data_ptr(),
                     self.bg_raw.data_ptr(), self.n, self.beta)


# ---- host helpers with the reference signatures (model.py:101-176) -------

def build_L(l_raw: np.ndarray, beta: float) -> np.ndarray:
    if not beta > 0:
        raise InvalidParameterError("beta must be > 0")
    l = np.atleast_2d(np.asarray(l_raw))
    L = np.zeros(l.shape[:-1] + (3, 3), dtype=l.dtype)
    for j in range(3):
        L[..., j, j] = l[..., j] ** 2 + beta
    L[..., 1, 0], L[..., 2, 0], L[..., 2, 1] = l[..., 3], l[..., 4], l[..., 5]
    return L[0] if np.asarray(l_raw).ndim == 1 else L


def invert_lower_triangular(L: np.ndarray) -> np.ndarray:
    L = np.asarray(L)
    if np.any(np.stack([L[..., j, j] for j in range(3)], -1) <= 0):
        raise SingularMatrixError("non-positive diagonal in triangular factor")
    inv = np.zeros_like(L)
    for j in range(3):
        inv[..., j, j] = 1.0 / L[..., j, j]
    inv[..., 1, 0] = -L[..., 1, 0] * inv[..., 0, 0] * inv[..., 1, 1]
    inv[..., 2, 1] = -L[..., 2, 1] * inv[..., 1, 1] * inv[..., 2, 2]
    inv[..., 2, 0] = -(L[..., 2, 0] * inv[..., 0, 0]
                       + L[..., 2, 1] * inv[..., 1, 0]) * inv[..., 2, 2]
    return inv


def covariance_from_L(L: np.ndarray) -> np.ndarray:
    Li = invert_lower_triangular(L)
    return np.swapaxes(Li, -1, -2) @ Li


def sample_gaussian(mean, L, z):
    Li = invert_lower_triangular(L)
    z = np.asarray(z)
    return np.asarray(mean) + np.squeeze(np.swapaxes(Li, -1, -2) @ z[..., None], -1)


@dataclass(frozen=True)
class ProbeFrameGaussian:
    mean_probe: np.ndarray
    l_probe: np.ndarray
    precision_probe: np.ndarray


def to_probe_frame(mean, L, pose: ProbePose) -> ProbeFrameGaussian:
    inv = pose.inverse()
    mp = inv.rotation @ np.asarray(mean, np.float64) + inv.translation
    lp = inv.rotation @ np.asarray(L, np.float64)
    return ProbeFrameGaussian(mp, lp, lp @ lp.T)


def evaluate_opacity(x, g: ProbeFrameGaussian, alpha: float) -> float:
    d = np.array([x[0], x[1], 0.0]) - g.mean_probe
    return float(alpha * np.exp(-0.5 * float(d @ g.precision_probe @ d)))
