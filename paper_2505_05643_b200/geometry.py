"""Probe poses, slice grids and the per-slice constants the kernels consume.

Host-side (numpy, float64) like the reference (pkg/src/echosplat/
geometry.py); the float32 casts that feed the GPU are made here, in the same
order the reference makes them, so the device sees bit-identical constants
(ref rasterizer.py:115-135, geometry.py:61-64 and :107-120).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_ORTHO_TOL = 1e-6


class InvalidParameterError(ValueError):
    """A contract precondition was violated (ref geometry.py:21-22)."""


@dataclass(frozen=True)
class ProbePose:
    """Rigid transform probe frame -> world frame (ref geometry.py:25-74)."""

    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        R = np.asarray(self.rotation, dtype=np.float64)
        t = np.asarray(self.translation, dtype=np.float64).reshape(3)
        if R.shape != (3, 3):
            raise InvalidParameterError(f"rotation must be 3x3, got {R.shape}")
        if np.max(np.abs(R.T @ R - np.eye(3))) > _ORTHO_TOL:
            raise InvalidParameterError("rotation is not orthonormal")
        if abs(np.linalg.det(R) - 1.0) > _ORTHO_TOL:
            raise InvalidParameterError("rotation must have det +1")
        object.__setattr__(self, "rotation", R)
        object.__setattr__(self, "translation", t)

    @staticmethod
    def identity() -> "ProbePose":
        return ProbePose(np.eye(3), np.zeros(3))

    @staticmethod
    def from_euler_deg(rx, ry, rz, tx=0.0, ty=0.0, tz=0.0) -> "ProbePose":
        from scipy.spatial.transform import Rotation
        R = Rotation.from_euler("ZYX", [rz, ry, rx], degrees=True).as_matrix()
        return ProbePose(R, np.array([tx, ty, tz], dtype=np.float64))

    def to_euler_deg(self):
        from scipy.spatial.transform import Rotation
        rz, ry, rx = Rotation.from_matrix(self.rotation).as_euler("ZYX", degrees=True)
        tx, ty, tz = self.translation
        return float(rx), float(ry), float(rz), float(tx), float(ty), float(tz)

    def inverse(self) -> "ProbePose":
        """World -> probe (the rendering view transform)."""
        Rinv = self.rotation.T
        return ProbePose(Rinv, -Rinv @ self.translation)

    def compose(self, other: "ProbePose") -> "ProbePose":
        return ProbePose(self.rotation @ other.rotation,
                         self.rotation @ other.translation + self.translation)

    def apply(self, points: np.ndarray) -> np.ndarray:
        p = np.asarray(points, dtype=np.float64)
        return p @ self.rotation.T + self.translation


@dataclass(frozen=True)
class SliceSpec:
    """Pixel grid of one slice (ref geometry.py:77-90)."""

    width: int
    height: int
    spacing: float
    pose: ProbePose = field(default_factory=ProbePose.identity)

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise InvalidParameterError("width and height must be >= 1")
        if not self.spacing > 0:
            raise InvalidParameterError("spacing must be > 0")


@dataclass
class SliceImage:
    """H x W intensity image with spacing and pose (ref geometry.py:133-144)."""

    pixels: np.ndarray
    spacing: float
    pose: ProbePose

    @property
    def spec(self) -> SliceSpec:
        return SliceSpec(width=self.pixels.shape[1], height=self.pixels.shape[0],
                         spacing=self.spacing, pose=self.pose)


def pixel_to_plane(u, v, spec: SliceSpec):
    """Pixel indices -> centred in-plane mm (ref geometry.py:93-104)."""
    u = np.asarray(u)
    v = np.asarray(v)
    if (np.any(u < 0) or np.any(u >= spec.width) or np.any(v < 0)
            or np.any(v >= spec.height)):
        raise InvalidParameterError("pixel index out of range")
    return ((u - (spec.width - 1) / 2.0) * spec.spacing,
            (v - (spec.height - 1) / 2.0) * spec.spacing)


def plane_axes(spec: SliceSpec, dtype=np.float64):
    """(origin, du, dv): world position of pixel (u,v) = origin + u du + v dv."""
    R = spec.pose.rotation
    t = spec.pose.translation
    du = R[:, 0] * spec.spacing
    dv = R[:, 1] * spec.spacing
    origin = t - (spec.width - 1) / 2.0 * du - (spec.height - 1) / 2.0 * dv
    return origin.astype(dtype), du.astype(dtype), dv.astype(dtype)


def pixel_grid_world(spec: SliceSpec, dtype=np.float64) -> np.ndarray:
    origin, du, dv = plane_axes(spec, dtype)
    uu = np.arange(spec.width, dtype=dtype)
    vv = np.arange(spec.height, dtype=dtype)
    return (origin[None, None, :] + uu[None, :, None] * du[None, None, :]
            + vv[:, None, None] * dv[None, None, :])


_CHI2_CACHE: dict = {}


def chi2_cutoff(p: float) -> float:
    """Squared-Mahalanobis cutoff of mass p, 3 dof (ref rasterizer.py:55-59)."""
    if not 0.0 < p < 1.0:
        raise InvalidParameterError("mass fraction p must be in (0, 1)")
    if p not in _CHI2_CACHE:
        from scipy.stats import chi2
        _CHI2_CACHE[p] = float(chi2.ppf(p, df=3))
    return _CHI2_CACHE[p]


# struct ugs_slice (include/ugs.h) as a numpy record: 27 float32, 6 int32,
# padding, int64 pix_base = 144 bytes
SLICE_DTYPE = np.dtype([("f", "<f4", (27,)), ("i", "<i4", (6,)), ("pad", "<i4"),
                        ("pix_base", "<i8")])


def fill_slices(dst, specs, p: float) -> None:
    """Fill a ctypes array of ugs_slice structs for a batch (pix_base = the
    running pixel offset) -- the same float32 constants as fill_slice
    (byte-identical), computed by the library's host helper
    ugs_fill_slices in one call (the serving path renders many small
    batches; numpy's per-op overhead was ~100 us per 16-slice batch)."""
    import ctypes
    import struct
    from . import _lib
    S = len(specs)
    # the poses are float64 (ProbePose enforces it); tobytes() is C order
    # whatever the arrays' strides, and joining bytes is ~5x cheaper than
    # np.stack for a handful of 3x3 matrices
    R = b"".join([sp.pose.rotation.tobytes() for sp in specs])
    t = b"".join([sp.pose.translation.tobytes() for sp in specs])
    sp_ = struct.pack(f"{S}d", *[float(sp.spacing) for sp in specs])
    W = struct.pack(f"{S}i", *[int(sp.width) for sp in specs])
    H = struct.pack(f"{S}i", *[int(sp.height) for sp in specs])
    _lib.check(_lib.lib().ugs_fill_slices(R, t, sp_, W, H, S, chi2_cutoff(p),
                                          ctypes.addressof(dst)),
               "ugs_fill_slices")


def fill_slices_numpy(dst, specs, p: float) -> None:
    """numpy restatement of fill_slices (vectorised over the batch, one
    memmove): the byte-identity check of the C helper in the CPU tests."""
    import ctypes
    f32 = np.float32
    S = len(specs)
    R = np.stack([sp.pose.rotation for sp in specs])            # (S,3,3) f64
    t = np.stack([sp.pose.translation for sp in specs])         # (S,3)
    sp_ = np.array([sp.spacing for sp in specs], np.float64)
    W = np.array([sp.width for sp in specs], np.int64)
    H = np.array([sp.height for sp in specs], np.int64)
    Rinv = np.transpose(R, (0, 2, 1))                           # ProbePose.inverse
    # -R^T t per pose (ref geometry.py:61-64); numpy's stacked matmul runs the
    # same inner product as the per-pose `-Rinv[j] @ t[j]` (bitwise equal
    # on 2e5 random poses; test_capi_cpu pins it against the oracle)
    tw = -(Rinv @ t[:, :, None])[:, :, 0]
    du = R[:, :, 0] * sp_[:, None]                              # plane_axes
    dv = R[:, :, 1] * sp_[:, None]
    cxw = (W - 1) / 2.0
    cyh = (H - 1) / 2.0
    origin = t - cxw[:, None] * du - cyh[:, None] * dv
    rec = np.zeros(S, SLICE_DTYPE)
    f = rec["f"]
    f[:, 0:9] = Rinv.astype(f32).reshape(S, 9)
    f[:, 9:12] = tw.astype(f32)
    f[:, 12:15] = origin.astype(f32)
    f[:, 15:18] = du.astype(f32)
    f[:, 18:21] = dv.astype(f32)
    f[:, 21] = np.sqrt(f32(chi2_cutoff(p)))
    f[:, 22] = sp_.astype(f32)
    f[:, 23] = cxw.astype(f32)
    f[:, 24] = cyh.astype(f32)
    f[:, 25] = (cxw * sp_).astype(f32)
    f[:, 26] = (cyh * sp_).astype(f32)
    rec["i"][:, 0] = W
    rec["i"][:, 1] = H
    rec["pix_base"] = np.concatenate([[0], np.cumsum(W * H)[:-1]])
    ctypes.memmove(dst, rec.ctypes.data, rec.nbytes)


def fill_slice(dst, spec: SliceSpec, p: float, pix_base: int = 0) -> None:
    """Fill one ugs_slice struct with the reference's float32 constants."""
    f32 = np.float32
    inv = spec.pose.inverse()
    rw = inv.rotation.astype(f32).reshape(9)
    tw = inv.translation.astype(f32)
    origin, du, dv = plane_axes(spec, f32)
    dst.rw[:] = [float(x) for x in rw]
    dst.tw[:] = [float(x) for x in tw]
    dst.origin[:] = [float(x) for x in origin]
    dst.du[:] = [float(x) for x in du]
    dst.dv[:] = [float(x) for x in dv]
    dst.sqrt_cut = float(np.sqrt(f32(chi2_cutoff(p))))
    dst.s = float(f32(spec.spacing))
    dst.cx = float(f32((spec.width - 1) / 2.0))
    dst.cy = float(f32((spec.height - 1) / 2.0))
    dst.x1h = float(f32((spec.width - 1) / 2.0 * spec.spacing))
    dst.x2h = float(f32((spec.height - 1) / 2.0 * spec.spacing))
    dst.width = int(spec.width)
    dst.height = int(spec.height)
    dst.pix_base = int(pix_base)
