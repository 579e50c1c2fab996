"""torch.autograd.Function over the libugs forward/backward.

``rasterize_autograd(cloud_tensors..., specs)`` returns the (S, H, W)
unclipped prediction num/den and differentiates into the raw parameters, so
a user can build any torch loss on top.  Phase 1 and the tile lists are
computed once in forward and reused by backward (the reference recomputes
them, gradients.py:49).
"""

from __future__ import annotations

import torch

from .gradients import grad_buffer
from .model import GaussianCloud
from .rasterizer import DEFAULT_P_MASS, Renderer


class RasterizeSlices(torch.autograd.Function):
    @staticmethod
    def forward(ctx, means, l_raw, intensity_raw, opacity_raw, bg_raw, beta,
                specs, p, renderer):
        cloud = GaussianCloud(means.detach(), l_raw.detach(),
                              intensity_raw.detach(), opacity_raw.detach(),
                              beta=beta, bg_raw=bg_raw.detach())
        r = renderer if renderer is not None else Renderer()
        r.bin(cloud, specs, p)
        S = len(specs)
        h, w = specs[0].height, specs[0].width
        num = torch.empty((S, h, w), dtype=torch.float32, device=means.device)
        den = torch.empty_like(num)
        r.forward(cloud, num, den)
        ctx.save_for_backward(num, den)
        ctx.cloud, ctx.r, ctx.gen = cloud, r, r.generation
        ctx.specs, ctx.p = specs, p
        return num / den

    @staticmethod
    def backward(ctx, d_pred):
        num, den = ctx.saved_tensors
        cloud, r = ctx.cloud, ctx.r
        if r.generation != ctx.gen:
            r.bin(cloud, ctx.specs, ctx.p)
        n = cloud.n
        grad = grad_buffer(n, num.device)
        r.backward(cloud, num, den, d_pred.to(torch.float32).contiguous(), grad,
                   None, 1.0)
        rows = grad[:12 * n].view(n, 12)
        return (rows[:, 0:3].contiguous(), rows[:, 3:9].contiguous(),
                rows[:, 9].contiguous(), rows[:, 10].contiguous(),
                grad[12 * n:12 * n + 2].double(), None, None, None, None)


def rasterize_autograd(means, l_raw, intensity_raw, opacity_raw, bg_raw, specs,
                       beta: float = 0.01, p: float = DEFAULT_P_MASS,
                       renderer: Renderer | None = None) -> torch.Tensor:
    """Differentiable (S, H, W) prediction num/den for equal-size slices."""
    return RasterizeSlices.apply(means, l_raw, intensity_raw, opacity_raw,
                                 bg_raw, beta, list(specs), p, renderer)
