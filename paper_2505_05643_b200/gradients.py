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


def grad_check(cloud, spec: SliceSpec, seed: int = 0,
               h: float | tuple = (1e-3, 3e-3, 1e-2), p: float = 0.9999) -> dict:
    """Finite-difference check of backward() (ref gradients.py:123-177).

    Same protocol as the reference: scalar loss = sum of squared rendered
    pixels, central differences at every step in `h` with the best agreement
    kept per entry, entries with |analytic| + |numeric| <= 1e-8 skipped, and
    the worst relative error per parameter group returned.  The renders here
    are the float32 CUDA path (the loss is summed in float64), so agreement
    is ~1e-3 rather than the reference's float64 ~1e-5; the default steps are
    larger accordingly.  For small clouds (N <= 50)."""
    from .rasterizer import rasterize
    del seed   # deterministic; kept for signature parity
    steps = (h,) if np.isscalar(h) else tuple(h)
    base = as_cloud(cloud).copy()

    def render_loss(c):
        b = rasterize(c, spec, p=p)
        pix = (b.intensity_num / b.opacity_sum).double()
        return float(torch.sum(pix * pix)), b, pix

    _, buf, pix = render_loss(base)
    g = backward(base, spec, buf, (2.0 * pix).float())
    groups = {"means": g.d_means, "l_raw": g.d_l_raw, "intensity_raw": g.d_intensity_raw,
              "opacity_raw": g.d_opacity_raw}

    def perturbed(name, idx, delta):
        """(loss, parameter value actually set): float32 parameters round
        the step, so the difference quotient uses the realised values."""
        c = base.copy()
        if name in ("bg_intensity_raw", "bg_opacity_raw"):
            val = getattr(base, name) + delta
            setattr(c, name, val)
            val = getattr(c, name)
        else:
            t = getattr(c, name)
            t[idx] = t[idx] + delta
            val = float(t[idx])
        return render_loss(c)[0], val

    def entry_error(name, idx, ana):
        best = None
        for s in steps:
            (lp, vp), (lm, vm) = perturbed(name, idx, s), perturbed(name, idx, -s)
            num = (lp - lm) / (vp - vm)
            den = abs(ana) + abs(num)
            err = abs(ana - num) / den if den > 1e-8 else 0.0
            best = err if best is None else min(best, err)
        return best

    report = {}
    for name, ga in groups.items():
        ga = ga.detach().cpu().numpy()
        report[name] = max((entry_error(name, idx, float(ga[idx]))
                            for idx in np.ndindex(ga.shape)), default=0.0)
    report["bg_intensity_raw"] = entry_error("bg_intensity_raw", None,
                                             float(g.d_bg_intensity_raw))
    report["bg_opacity_raw"] = entry_error("bg_opacity_raw", None, float(g.d_bg_opacity_raw))
    return report
