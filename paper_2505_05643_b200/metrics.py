"""SSIM / PSNR and the training loss on the device (ref metrics.py:17-105,
trainer.py:130-151).

Same formulation as the reference: 11x11 Gaussian window (sigma 1.5),
C1 = 1e-4, C2 = 9e-4, valid windows only, float64 arithmetic; the analytic
gradient of mean SSIM uses the adjoint (zero-padded full correlation) of the
valid-window filter.

``ssim`` / ``ssim_with_grad`` / ``loss`` and their batched forms run on the
hand-written CUDA kernel (ugs_loss: float64 filters over float32 images, the
precision the training path feeds it).  The separable float64 conv2d
formulation (``*_torch``) is kept only as an independent cross-check for the
tests.
"""

from __future__ import annotations

import datetime
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from .geometry import InvalidParameterError

WIN = 11
PAD = WIN // 2
SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2

_KCACHE: dict = {}


def _kernels(device):
    k = _KCACHE.get(device)
    if k is None:
        x = np.arange(WIN) - PAD
        w = np.exp(-0.5 * (x / SIGMA) ** 2)
        w = torch.tensor(w / w.sum(), dtype=torch.float64, device=device)
        k = (w.view(1, 1, WIN, 1), w.view(1, 1, 1, WIN))
        _KCACHE[device] = k
    return k


def _filt(x):
    """Valid-window Gaussian mean of (B,1,H,W) -> (B,1,H-10,W-10)."""
    kv, kh = _kernels(x.device)
    return F.conv2d(F.conv2d(x, kv), kh)


def _adj(f):
    """Adjoint of _filt: (B,1,H-10,W-10) -> (B,1,H,W)."""
    kv, kh = _kernels(f.device)
    f = F.pad(f, (2 * PAD, 2 * PAD, 2 * PAD, 2 * PAD))
    return F.conv2d(F.conv2d(f, kv), kh)


def _as4d(a, device=None):
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
    if device is not None:
        t = t.to(device)
    t = t.to(torch.float64)
    if t.dim() == 2:
        t = t[None]
    return t[:, None]


def ssim_with_grad_batch_torch(x, y):
    """x, y (B,H,W) -> (mean SSIM per image (B,), d meanSSIM/dx (B,H,W))."""
    x = _as4d(x)
    y = _as4d(y, x.device)
    if x.shape != y.shape:
        raise InvalidParameterError("image dimensions differ")
    if min(x.shape[-2:]) < WIN:
        raise InvalidParameterError(f"images must be at least {WIN}x{WIN}")
    mx, my = _filt(x), _filt(y)
    sxx = _filt(x * x) - mx * mx
    syy = _filt(y * y) - my * my
    sxy = _filt(x * y) - mx * my
    a1 = 2.0 * mx * my + C1
    a2 = 2.0 * sxy + C2
    b1 = mx * mx + my * my + C1
    b2 = sxx + syy + C2
    s = (a1 * a2) / (b1 * b2)
    nv = s.shape[-1] * s.shape[-2]
    d_mu = (2.0 * my * a2) / (b1 * b2) - (2.0 * mx * a1 * a2) / (b1 * b1 * b2)
    d_sxx = -s / b2
    d_sxy = 2.0 * a1 / (b1 * b2)
    grad = (_adj(d_mu - 2.0 * mx * d_sxx - my * d_sxy) + 2.0 * x * _adj(d_sxx)
            + y * _adj(d_sxy))
    return s.mean(dim=(1, 2, 3)), (grad / nv)[:, 0]


def ssim_batch_torch(x, y):
    x = _as4d(x)
    y = _as4d(y, x.device)
    if x.shape != y.shape:
        raise InvalidParameterError("image dimensions differ")
    if min(x.shape[-2:]) < WIN:
        raise InvalidParameterError(f"images must be at least {WIN}x{WIN}")
    mx, my = _filt(x), _filt(y)
    sxx = _filt(x * x) - mx * mx
    syy = _filt(y * y) - my * my
    sxy = _filt(x * y) - mx * my
    s = ((2.0 * mx * my + C1) * (2.0 * sxy + C2)) / \
        ((mx * mx + my * my + C1) * (sxx + syy + C2))
    return s.mean(dim=(1, 2, 3))


def _dev_for(a, b):
    for t in (a, b):
        if isinstance(t, torch.Tensor) and t.is_cuda:
            return t.device
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def _images(a, b):
    """(S,H,W) float32 contiguous device tensors of two image stacks."""
    dev = _dev_for(a, b)
    if dev.type != "cuda":
        raise RuntimeError("paper_2505_05643_b200 needs a CUDA device "
                           "(there is no CPU fallback)")
    x = (a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a)))
    y = (b if isinstance(b, torch.Tensor) else torch.as_tensor(np.asarray(b)))
    x = x.to(device=dev, dtype=torch.float32)
    y = y.to(device=dev, dtype=torch.float32)
    if x.dim() == 2:
        x = x[None]
    if y.dim() == 2:
        y = y[None]
    if x.shape != y.shape:
        raise InvalidParameterError("image dimensions differ")
    return x.contiguous(), y.contiguous()


def _kernel_loss(x, y, lam: float, l2: bool):
    """ugs_loss over (S,H,W) stacks in chunks of 64: (loss (S,) float64,
    d loss/d x (S,H,W) float32, SSIM (S,) float64)."""
    if not l2 and lam > 0.0 and min(x.shape[-2:]) < WIN:
        raise InvalidParameterError(f"images must be at least {WIN}x{WIN}")
    lvs, dps, svs = [], [], []
    for i in range(0, x.shape[0], 64):
        lv, dp, sv = fused_loss(x[i:i + 64], None, y[i:i + 64], lam, l2)
        lvs.append(lv)
        dps.append(dp)
        svs.append(sv)
    return torch.cat(lvs), torch.cat(dps), torch.cat(svs)


def ssim_batch(x, y):
    """Mean SSIM per image of two (B,H,W) stacks (CUDA kernel)."""
    x, y = _images(x, y)
    return _kernel_loss(x, y, 1.0, False)[2]


def ssim_with_grad_batch(x, y):
    """(mean SSIM per image (B,), d meanSSIM/dx (B,H,W) float64): the loss
    kernel at lam = 1 gives d(1 - SSIM)/dx."""
    x, y = _images(x, y)
    _, d, s = _kernel_loss(x, y, 1.0, False)
    return s, -d.double()


def ssim(a, b) -> float:
    """Mean SSIM of two [0,1] images (ref metrics.py:68-74)."""
    return float(ssim_batch(a, b)[0])


def ssim_with_grad(a, b):
    """(SSIM, dSSIM/da) (ref metrics.py:77-98)."""
    s, g = ssim_with_grad_batch(a, b)
    return float(s[0]), g[0]


def psnr(a, b) -> float:
    """PSNR in dB for range-1 images; inf when equal (ref metrics.py:101-107)."""
    x = _as4d(a)
    y = _as4d(b, x.device)
    if x.shape != y.shape:
        raise InvalidParameterError("image dimensions differ")
    mse = float(torch.mean((x - y) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)


@dataclass
class EvalReport:
    """Per-plane-family reconstruction quality (ref metrics.py:110-120)."""

    families: dict  # family -> {ssim_mean, ssim_std, psnr_mean, psnr_std, count, psnr_inf_count}
    timestamp: str

    def to_json_dict(self) -> dict:
        return {"families": {k: dict(sorted(v.items()))
                             for k, v in sorted(self.families.items())},
                "timestamp": self.timestamp}


def family_poses(volume, family: str, n: int):
    """n linearly spaced orthogonal planes of one family through the volume
    (ref metrics.py:123-145): [(ProbePose, SliceSpec)].  axial: the stack's
    axial_pose at plane i*d/n (w x h); coronal: plane axes world x and z,
    normal -y, at y = (i*h/n - (h-1)/2)*s (w x d); sagittal: plane axes
    world y and z, normal x, at x = (i*w/n - (w-1)/2)*s (h x d)."""
    from .dataset import axial_pose
    from .geometry import ProbePose, SliceSpec
    d, h, w = volume.voxels.shape
    s = volume.spacing
    out = []
    if family == "axial":
        for i in range(n):
            out.append((axial_pose(volume, i * d / n), w, h))
    elif family == "coronal":
        rot = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]])
        for i in range(n):
            out.append((ProbePose(rot, np.array([0.0, (i * h / n - (h - 1) / 2.0) * s, 0.0])),
                        w, d))
    elif family == "sagittal":
        rot = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
        for i in range(n):
            out.append((ProbePose(rot, np.array([(i * w / n - (w - 1) / 2.0) * s, 0.0, 0.0])),
                        h, d))
    else:
        raise InvalidParameterError(f"unknown family {family!r}")
    return [(pose, SliceSpec(width=pw, height=ph, spacing=s, pose=pose))
            for pose, pw, ph in out]


def evaluate_views(cloud, volume, n_per_axis: int, p_mass: float = 0.95,
                   workers: int = 1) -> EvalReport:
    """Render linearly spaced axial / coronal / sagittal views and score them
    against trilinear ground truth, SSIM and PSNR mean and std per family
    (ref metrics.py:148-178).  Each family is ONE batched render
    (render_slices) and one GPU sampling pass (sample_slices); SSIM float64
    per view as ssim(), PSNR from the float64 per-view MSE (inf views are
    counted, not averaged).  `workers` is accepted and ignored."""
    from .rasterizer import as_cloud, render_slices
    from .volume import sample_slices
    cloud = as_cloud(cloud)
    families = {}
    for family in ("axial", "coronal", "sagittal"):
        specs = [spec for _, spec in family_poses(volume, family, n_per_axis)]
        pred = render_slices(cloud, specs, p_mass)
        truth = sample_slices(volume, specs, device=cloud.device)
        ssims = ssim_batch(pred, truth).cpu().numpy()
        mse = torch.mean((pred.to(torch.float64) - truth.to(torch.float64)) ** 2,
                         dim=(1, 2)).cpu().numpy()
        psnrs = [10.0 * math.log10(1.0 / float(m)) for m in mse if m != 0.0]
        families[family] = {
            "count": n_per_axis,
            "ssim_mean": float(np.mean(ssims)),
            "ssim_std": float(np.std(ssims)),
            "psnr_mean": float(np.mean(psnrs)) if psnrs else None,
            "psnr_std": float(np.std(psnrs)) if psnrs else None,
            "psnr_inf_count": int(np.sum(mse == 0.0)),
        }
    stamp = datetime.datetime.now(datetime.timezone.utc).isoformat()
    return EvalReport(families=families, timestamp=stamp)


_WS: dict = {}


def fused_loss(num: torch.Tensor, den: torch.Tensor, target: torch.Tensor,
               lam: float, l2: bool = False, target_index: torch.Tensor | None = None,
               mean_out: torch.Tensor | None = None):
    """Training loss straight from the render accumulators, one fused CUDA
    pass (ugs_loss_ex): pred = num/den, (1-lam)*L1 + lam*(1-SSIM) per slice.

    num, den: (S, H, W) float32 on the device; target: (S, H, W), or -- with
    target_index (S,) int64 on the device -- the whole dataset (N, H, W), slice
    s comparing against target[target_index[s]] (no gather copy).  mean_out
    (0-dim float64 on the device) receives the batch-mean loss.  Returns
    (loss (S,) float64, d_pixels (S, H, W) float32, ssim (S,) float64)."""
    import ctypes
    from . import _lib
    S, H, W = num.shape
    L = _lib.lib()
    nbytes = L.ugs_loss_workspace_bytes(S, H, W)
    ws = _WS.get(num.device)
    if ws is None or ws.numel() < nbytes:
        ws = _WS[num.device] = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8,
                                           device=num.device)
    dpix = torch.empty((S, H, W), dtype=torch.float32, device=num.device)
    lv = torch.empty(S, dtype=torch.float64, device=num.device)
    sv = torch.empty(S, dtype=torch.float64, device=num.device)
    tgt = target.to(dtype=torch.float32).contiguous()
    if target_index is not None:
        target_index = target_index.to(dtype=torch.int64).contiguous()
        if tgt.shape[-2:] != (H, W) or target_index.shape != (S,):
            raise InvalidParameterError("target / target_index shapes do not match")
    elif tgt.shape != (S, H, W):
        raise InvalidParameterError("prediction/target dimensions differ")
    _lib.check(L.ugs_loss_ex(num.data_ptr(), _lib.ptr(den), tgt.data_ptr(),
                             _lib.ptr(target_index), S, H, W, float(lam), int(bool(l2)),
                             dpix.data_ptr(), lv.data_ptr(), sv.data_ptr(),
                             _lib.ptr(mean_out), ws.data_ptr(),
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "ugs_loss_ex")
    return lv, dpix, sv


def loss_batch(pred, target, lam: float, l2: bool = False):
    """Per-image training loss and its pixel gradient (ref trainer.py:130-151)
    on the CUDA kernel.  pred, target (B,H,W); returns (loss (B,) float64,
    d_pixels (B,H,W) float64)."""
    x, y = _images(pred, target)
    lv, d, _ = _kernel_loss(x, y, lam, l2)
    return lv, d.double()


def loss_batch_torch(pred, target, lam: float, l2: bool = False):
    """The same in float64 torch ops (cross-check only)."""
    x = pred.to(torch.float64)
    y = target.to(device=x.device, dtype=torch.float64)
    if x.shape != y.shape:
        raise InvalidParameterError("prediction/target dimensions differ")
    diff = x - y
    npx = x.shape[-1] * x.shape[-2]
    if l2:
        return (diff * diff).mean(dim=(1, 2)), 2.0 * diff / npx
    val = (1.0 - lam) * diff.abs().mean(dim=(1, 2))
    d = (1.0 - lam) * torch.sign(diff) / npx
    if lam > 0.0:
        s, ds = ssim_with_grad_batch_torch(x, y)
        val = val + lam * (1.0 - s)
        d = d - lam * ds
    return val, d


def loss(pred, target, lam: float, l2: bool = False):
    """Reference signature: (float, (H,W) gradient)."""
    v, d = loss_batch(pred, target, lam, l2)
    return float(v[0]), d[0]
