"""Deterministic input generators shared by the golden-vector script and the
tests (numpy PCG64 streams are bit-reproducible across hosts).

``random_cloud`` / ``random_pose`` restate the reference test fixtures
(pkg/tests/conftest.py:8-30); ``uniform_cloud`` restates ``init_cloud``
(pkg/src/echosplat/trainer.py:110-127).  Each returns plain numpy arrays so
they feed the reference, the oracle and the CUDA path alike.
"""

from __future__ import annotations

import numpy as np


def random_cloud(rng, n, extent=8.0, sigma_range=(0.8, 3.0),
                 bg_opacity_raw=-4.0):
    sigma = rng.uniform(*sigma_range, size=(n, 3))
    beta = 0.01
    l_diag = np.sqrt(np.maximum(1.0 / sigma - beta, 1e-6))
    l_off = rng.uniform(-0.05, 0.05, size=(n, 3))
    return dict(
        means=rng.uniform(-extent, extent, size=(n, 3)).astype(np.float32),
        l_raw=np.concatenate([l_diag, l_off], axis=1).astype(np.float32),
        intensity_raw=rng.normal(0.0, 1.0, n).astype(np.float32),
        opacity_raw=rng.normal(1.0, 0.5, n).astype(np.float32),
        bg_intensity_raw=float(rng.normal(0.0, 0.5)),
        bg_opacity_raw=float(bg_opacity_raw),
        beta=beta,
    )


def random_rotation(rng):
    from scipy.spatial.transform import Rotation
    quat = rng.standard_normal(4)
    return Rotation.from_quat(quat / np.linalg.norm(quat)).as_matrix()


def random_pose(rng, translate=5.0):
    R = random_rotation(rng)
    return R, rng.uniform(-translate, translate, 3)


def uniform_cloud(seed, n, bounds, l_lo, l_hi, beta=0.01):
    """init_cloud(TrainConfig(n, seed, l_init_low, l_init_high), bounds)."""
    bounds = np.asarray(bounds, np.float64)
    rng = np.random.default_rng(seed)
    means = rng.uniform(bounds[0], bounds[1], size=(n, 3))
    l_raw = rng.uniform(l_lo, l_hi, size=(n, 6))
    return dict(
        means=means.astype(np.float32), l_raw=l_raw.astype(np.float32),
        intensity_raw=np.zeros(n, np.float32),
        opacity_raw=np.full(n, 1.0, np.float32),
        bg_intensity_raw=0.0, bg_opacity_raw=-4.0, beta=beta)


# ---- phase-1 (cull / compact / windows) cases: bit-exact targets --------
PREPARE_CASES = [
    # (name, seed, n, image px, spacing, l_lo, l_hi, half-extent, translate)
    ("c3_like_256", 101, 20000, 256, 0.375, 0.85, 1.05, 48.0, 12.0),
    ("c1_like_128", 102, 20000, 128, 0.3, 0.85, 1.05, 19.2, 5.0),
    ("wide_512", 103, 20000, 512, 0.1875, 0.3, 2.0, 48.0, 12.0),
    ("small_64", 104, 5000, 64, 1.0, 0.3, 2.0, 40.0, 10.0),
    ("tiny_sigma_256", 105, 20000, 256, 0.375, 2.0, 5.0, 48.0, 12.0),
    ("nonsquare", 106, 8000, (96, 160), 0.5, 0.5, 1.5, 40.0, 8.0),
]


def prepare_case(case):
    name, seed, n, px, spacing, lo, hi, ext, tr = case
    rng = np.random.default_rng(seed)
    R, t = random_pose(rng, translate=tr)
    w, h = (px, px) if np.isscalar(px) else px
    cloud = uniform_cloud(seed + 1000, n, [[-ext] * 3, [ext] * 3], lo, hi)
    return cloud, R, t, w, h, spacing


# ---- render / backward cases: float targets ------------------------------
RENDER_CASES = [
    # (name, seed, n, extent, w, h, spacing, translate, p)
    ("rc_small", 11, 200, 10.0, 24, 24, 1.0, 2.0, 0.95),
    ("rc_tight", 12, 150, 8.0, 20, 28, 0.8, 2.0, 0.9999),
    ("rc_mid", 13, 2000, 14.0, 64, 64, 0.45, 3.0, 0.95),
    ("rc_ragged", 14, 800, 12.0, 37, 53, 0.6, 3.0, 0.95),
]


def render_case(case):
    name, seed, n, ext, w, h, spacing, tr, p = case
    rng = np.random.default_rng(seed)
    cloud = random_cloud(rng, n, extent=ext)
    R, t = random_pose(rng, translate=tr)
    dpix = rng.standard_normal((h, w)).astype(np.float32)
    return cloud, R, t, w, h, spacing, p, dpix


def input_checksum(*arrays) -> float:
    return float(sum(float(np.sum(np.asarray(a, np.float64) *
                                  (1.0 + np.arange(np.asarray(a).size).reshape(
                                      np.asarray(a).shape) % 7)))
                     for a in arrays))


def eval_cloud(bounds):
    """The seeded 3000-Gaussian cloud of the evaluate_views fixture
    (make_golden_eval.py)."""
    c = uniform_cloud(21, 3000, bounds, 1.2, 1.6)
    c["intensity_raw"] = np.random.default_rng(3).normal(0, 1, 3000).astype(np.float32)
    return c
