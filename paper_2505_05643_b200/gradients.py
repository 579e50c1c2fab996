"""Analytic backward pass on the B200 (ref pkg/src/echosplat/gradients.py).

``backward(cloud, spec, buffers, d_pixels)`` keeps the reference signature
(gradients.py:36-113) and returns dense raw-parameter gradients.  The GPU
reuses the binning kept by ``rasterize`` (no second phase-1 pass); if the
renderer has been reused since, it re-bins and checks that the accepted set
is unchanged, raising InvalidParameterError like the reference does.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .geometry import InvalidParameterError, SliceSpec
from .rasterizer import RenderBuffers, Renderer, as_cloud


@dataclass
class ParamGradients:
    """Raw-space gradients (ref gradients.py:24-33); device tensors, the
    background terms as python floats."""

    d_means: torch.Tensor
    d_l_raw: torch.Tensor
    d_intensity_raw: torch.Tensor
    d_opacity_raw: torch.Tensor
    d_bg_intensity_raw: float
    d_bg_opacity_raw: float

    @staticmethod
    def from_flat(flat: torch.Tensor, n: int, bg_as_float: bool = True):
        bg = flat[11 * n:11 * n + 2]
        bgv = bg.double().cpu().numpy() if bg_as_float else (bg[0], bg[1])
        return ParamGradients(flat[:3 * n].view(n, 3),
                              flat[3 * n:9 * n].view(n, 6),
                              flat[9 * n:10 * n], flat[10 * n:11 * n],
                              float(bgv[0]), float(bgv[1]))


def grad_buffer(n: int, device) -> torch.Tensor:
    """Flat float32 gradient layout [means 3n | l_raw 6n | c n | a n | bg 2]."""
    return torch.zeros(11 * n + 2, dtype=torch.float32, device=device)


def backward(cloud, spec: SliceSpec, buffers: RenderBuffers, d_pixels,
             workers: int = 1) -> ParamGradients:
    """Chain an upstream per-pixel gradient to all raw parameters."""
    del workers
    cloud = as_cloud(cloud)
    if buffers.spec is not spec and (buffers.spec.width != spec.width
                                     or buffers.spec.height != spec.height):
        raise InvalidParameterError("buffers were rendered with a different spec")
    dpix = torch.as_tensor(np.asarray(d_pixels) if not isinstance(
        d_pixels, torch.Tensor) else d_pixels)
    if tuple(dpix.shape) != (spec.height, spec.width):
        raise InvalidParameterError("d_pixels shape mismatch")
    dpix = dpix.to(device=cloud.device, dtype=torch.float32).contiguous()
    r: Renderer = buffers._renderer
    fresh = (r is not None and r.generation == buffers._generation
             and r.cloud_key(cloud) == buffers._cloud_key)
    if not fresh:
        if r is None:
            from .rasterizer import default_renderer
            r = default_renderer(cloud.device)
        r.bin(cloud, [spec], buffers.p_mass)
        acc, _ = r.accepted(cloud.device)
        if not torch.equal(acc[0].cpu(), buffers.accepted.cpu()):
            raise InvalidParameterError("buffers do not match this cloud")
    grad = grad_buffer(cloud.n, cloud.device)
    r.backward(cloud, buffers.intensity_num.contiguous(),
               buffers.opacity_sum.contiguous(), dpix, grad, None, 1.0)
    return ParamGradients.from_flat(grad, cloud.n)
