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
        """Views (made contiguous) of an AoS-12 gradient buffer."""
        rows = flat[:12 * n].view(n, 12)
        bg = flat[12 * n:12 * n + 2].double().cpu().numpy()
        return ParamGradients(rows[:, 0:3].contiguous(), rows[:, 3:9].contiguous(),
                              rows[:, 9].contiguous(), rows[:, 10].contiguous(),
                              float(bg[0]), float(bg[1]))


def grad_buffer(n: int, device) -> torch.Tensor:
    """AoS-12 float32 gradient (include/ugs.h): Gaussian g owns entries
    [12g, 12g+12) = [d_means 3 | d_l_raw 6 | d_c | d_a | pad], background
    entries at [12n, 12n+2)."""
    return torch.zeros(12 * n + 2, dtype=torch.float32, device=device)


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
