"""Synthetic ground-truth volumes and slice sampling (ref volume.py).

Offline data generation is outside the hot path; this is
a compact restatement so the benchmark and the trainer can build the same
synthetic phantoms and ground-truth slices on any host.  ``sample_slices``
is the GPU trilinear sampler (torch grid gather) used for large datasets;
``sample_slice`` keeps the reference's host signature.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .geometry import InvalidParameterError, SliceImage, SliceSpec, pixel_grid_world, plane_axes


@dataclass
class Volume:
    voxels: np.ndarray   # (D, H, W) float32
    spacing: float

    def __post_init__(self):
        if not self.spacing > 0:
            raise InvalidParameterError("spacing must be > 0")

    @property
    def dims(self):
        return self.voxels.shape

    @property
    def extent_mm(self):
        d, h, w = self.voxels.shape
        return np.array([w, h, d]) * self.spacing

    def world_bounds(self):
        half = self.extent_mm / 2.0
        return np.stack([-half, half])


def save_volume(volume: Volume, path) -> None:
    base = Path(path).with_suffix("")
    base.with_suffix(".raw").write_bytes(
        np.ascontiguousarray(volume.voxels, "<f4").tobytes())
    base.with_suffix(".json").write_text(json.dumps(
        {"dims": list(volume.voxels.shape), "spacing": volume.spacing, "version": 1}))


def load_volume(path) -> Volume:
    base = Path(path).with_suffix("")
    meta = json.loads(base.with_suffix(".json").read_text())
    dims = tuple(int(x) for x in meta["dims"])
    vox = np.frombuffer(base.with_suffix(".raw").read_bytes(), "<f4").reshape(dims)
    return Volume(vox.copy(), float(meta["spacing"]))


def _centers(dims, spacing):
    d, h, w = dims
    return ((np.arange(w) - (w - 1) / 2.0) * spacing,
            (np.arange(h) - (h - 1) / 2.0) * spacing,
            (np.arange(d) - (d - 1) / 2.0) * spacing)


def blobs_params(dims, spacing, seed, k=12):
    """Random anisotropic Gaussians of the blobs phantom (ref volume.py:139-160)."""
    rng = np.random.default_rng(seed)
    d, h, w = dims
    half = np.array([w, h, d]) * spacing / 2.0
    means = rng.uniform(-0.55 * half, 0.55 * half, size=(k, 3))
    sigma = rng.uniform(2.5, 7.0, size=(k, 3))
    beta = 0.01
    l_diag = np.sqrt(np.maximum(1.0 / sigma - beta, 1e-6))
    l_off = rng.uniform(-0.03, 0.03, size=(k, 3))
    c = rng.uniform(0.3, 0.95, size=k)
    a = rng.uniform(0.4, 0.85, size=k)
    logit = lambda q: np.log(q / (1.0 - q))
    return dict(means=means.astype(np.float32),
                l_raw=np.concatenate([l_diag, l_off], 1).astype(np.float32),
                intensity_raw=logit(c).astype(np.float32),
                opacity_raw=logit(a).astype(np.float32),
                bg_intensity_raw=float(logit(0.05)), bg_opacity_raw=-4.0, beta=beta)


def evaluate_params_on_grid(cl: dict, dims, spacing) -> np.ndarray:
    """Blend equation at every voxel centre, float64, no truncation
    (ref volume.py:109-136)."""
    d, h, w = dims
    xs, ys, zs = _centers(dims, spacing)
    l = cl["l_raw"].astype(np.float64)
    beta = cl["beta"]
    L = np.zeros((len(l), 3, 3))
    for j in range(3):
        L[:, j, j] = l[:, j] ** 2 + beta
    L[:, 1, 0], L[:, 2, 0], L[:, 2, 1] = l[:, 3], l[:, 4], l[:, 5]
    sig = lambda x: 1.0 / (1.0 + np.exp(-np.asarray(x, np.float64)))
    colors = sig(cl["intensity_raw"].astype(np.float32)).astype(np.float64)
    alphas = sig(cl["opacity_raw"].astype(np.float32)).astype(np.float64)
    cbg, abg = float(sig(cl["bg_intensity_raw"])), float(sig(cl["bg_opacity_raw"]))
    grid_xy = np.stack(np.meshgrid(xs, ys, indexing="xy"), axis=-1)
    out = np.empty(dims)
    for iz in range(d):
        num = np.full((h, w), abg * cbg)
        den = np.full((h, w), abg)
        for g in range(len(l)):
            e = np.empty((h, w, 3))
            e[..., :2] = grid_xy - cl["means"][g, :2].astype(np.float64)
            e[..., 2] = zs[iz] - float(cl["means"][g, 2])
            y = e @ L[g]
            wgt = alphas[g] * np.exp(-0.5 * np.sum(y * y, -1))
            num += wgt * colors[g]
            den += wgt
        out[iz] = num / den
    return np.clip(out, 0.0, 1.0)


def _shells(dims, spacing, rng):
    from scipy.ndimage import gaussian_filter
    d, h, w = dims
    xs, ys, zs = _centers(dims, spacing)
    half = np.array([w, h, d]) * spacing / 2.0
    zz, yy, xx = np.meshgrid(zs, ys, xs, indexing="ij")
    vol = np.full(dims, 0.08)
    radii = np.array([0.85, 0.60, 0.35])[:, None] * half[None, :]
    for r, th, lvl, jit in zip(radii, [0.10, 0.09, 0.30], [0.55, 0.80, 0.40],
                               rng.uniform(0.9, 1.1, size=(3, 3))):
        rr = np.sqrt((xx / (r[0] * jit[0])) ** 2 + (yy / (r[1] * jit[1])) ** 2
                     + (zz / (r[2] * jit[2])) ** 2)
        shell = np.exp(-0.5 * ((rr - 1.0) / th) ** 2) if th < 0.2 else (rr <= 1.0) * 1.0
        vol = np.maximum(vol, lvl * shell)
    vol = gaussian_filter(vol, sigma=1.0)
    speckle = gaussian_filter(rng.standard_normal(dims), sigma=2.0)
    speckle = 1.0 + 0.45 * speckle / max(np.std(speckle), 1e-9)
    return np.clip(vol * np.clip(speckle, 0.3, 1.7), 0.0, 1.0)


def make_phantom(kind: str, dims, spacing: float, seed: int = 0) -> Volume:
    """'shells' | 'blobs' | 'checker' phantoms (ref volume.py:198-220)."""
    if isinstance(dims, int):
        dims = (dims, dims, dims)
    dims = tuple(int(x) for x in dims)
    if min(dims) < 8:
        raise InvalidParameterError("phantom dims must be >= 8 per axis")
    rng = np.random.default_rng(seed)
    if kind == "blobs":
        vox = evaluate_params_on_grid(blobs_params(dims, spacing, seed), dims, spacing)
    elif kind == "shells":
        vox = _shells(dims, spacing, rng)
    elif kind == "checker":
        d, h, w = dims
        block = max(2, min(dims) // 8)
        iz, iy, ix = np.meshgrid(np.arange(d) // block, np.arange(h) // block,
                                 np.arange(w) // block, indexing="ij")
        lo, hi = rng.uniform(0.05, 0.2), rng.uniform(0.7, 0.95)
        vox = np.where((iz + iy + ix) % 2 == 0, lo, hi)
    else:
        raise InvalidParameterError(f"unknown phantom kind {kind!r}")
    return Volume(vox.astype(np.float32), float(spacing))


def sample_volume_at(volume: Volume, points) -> np.ndarray:
    """Trilinear interpolation, outside -> 0 (ref volume.py:223-255)."""
    d, h, w = volume.voxels.shape
    s = volume.spacing
    p = np.asarray(points, np.float64)
    f = [p[..., 0] / s + (w - 1) / 2.0, p[..., 1] / s + (h - 1) / 2.0,
         p[..., 2] / s + (d - 1) / 2.0]
    i0 = [np.floor(q).astype(np.int64) for q in f]
    t = [q - i for q, i in zip(f, i0)]
    out = np.zeros(p.shape[:-1])
    vox = volume.voxels
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                xi, yi, zi = i0[0] + dx, i0[1] + dy, i0[2] + dz
                ok = (xi >= 0) & (xi < w) & (yi >= 0) & (yi < h) & (zi >= 0) & (zi < d)
                val = np.where(ok, vox[np.clip(zi, 0, d - 1), np.clip(yi, 0, h - 1),
                                       np.clip(xi, 0, w - 1)], 0.0)
                wgt = ((t[0] if dx else 1.0 - t[0]) * (t[1] if dy else 1.0 - t[1])
                       * (t[2] if dz else 1.0 - t[2]))
                out += wgt * val
    return out


def sample_slice(volume: Volume, spec: SliceSpec) -> SliceImage:
    px = sample_volume_at(volume, pixel_grid_world(spec))
    return SliceImage(px.astype(np.float32), spec.spacing, spec.pose)


def sample_slices(volume: Volume, specs, device=None) -> torch.Tensor:
    """GPU trilinear ground truth for many equal-size slices: (S, H, W) f32.

    float64 coordinates, same zero-outside convention as sample_volume_at."""
    dev = torch.device("cuda") if device is None else torch.device(device)
    vox = torch.as_tensor(volume.voxels, device=dev, dtype=torch.float64)
    d, h, w = volume.voxels.shape
    s = volume.spacing
    out = []
    for spec in specs:
        o, du, dv = plane_axes(spec, np.float64)
        uu = torch.arange(spec.width, device=dev, dtype=torch.float64)
        vv = torch.arange(spec.height, device=dev, dtype=torch.float64)
        pts = (torch.as_tensor(o, device=dev)[None, None]
               + uu[None, :, None] * torch.as_tensor(du, device=dev)[None, None]
               + vv[:, None, None] * torch.as_tensor(dv, device=dev)[None, None])
        f = [pts[..., 0] / s + (w - 1) / 2.0, pts[..., 1] / s + (h - 1) / 2.0,
             pts[..., 2] / s + (d - 1) / 2.0]
        i0 = [torch.floor(q).long() for q in f]
        t = [q - i for q, i in zip(f, i0)]
        acc = torch.zeros_like(f[0])
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    xi, yi, zi = i0[0] + dx, i0[1] + dy, i0[2] + dz
                    ok = (xi >= 0) & (xi < w) & (yi >= 0) & (yi < h) & (zi >= 0) & (zi < d)
                    val = vox[zi.clamp(0, d - 1), yi.clamp(0, h - 1), xi.clamp(0, w - 1)]
                    val = torch.where(ok, val, torch.zeros_like(val))
                    wgt = ((t[0] if dx else 1.0 - t[0]) * (t[1] if dy else 1.0 - t[1])
                           * (t[2] if dz else 1.0 - t[2]))
                    acc = acc + wgt * val
        out.append(acc.float())
    return torch.stack(out)
