"""CPU-only checks of the boundary: libugs.so loads, exports exactly the
entry points include/ugs.h declares, the ctypes structs match the C layout,
and the host-side constants equal the oracle's (no GPU work here)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "ugs.h")).read()
    return sorted(set(re.findall(r"UGS_API\s+[\w\s\*]*?\b(ugs_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = header_functions()
    assert "ugs_bin" in names and "ugs_forward" in names and "ugs_backward" in names
    assert len(names) >= 12


def test_library_exports_every_header_symbol():
    from paper_2505_05643_b200 import _lib
    L = _lib.load()
    for name in header_functions():
        assert hasattr(L, name), name
    assert set(header_functions()) == set(_lib.EXPORTS)
    assert L.ugs_abi_version() == 2


def test_struct_layout():
    from paper_2505_05643_b200 import _lib
    # ugs_slice: 27 floats + 6 int32 + pad + int64 = 144 bytes
    assert ctypes.sizeof(_lib.Slice) == 144
    assert _lib.Slice.pix_base.offset == 136
    assert ctypes.sizeof(_lib.Cloud) == 56
    # ugs_peer_view: 11 device pointers
    assert ctypes.sizeof(_lib.PeerView) == 88
    assert _lib.PeerView.bg_raw.offset == 72
    assert _lib.PeerView.sync.offset == 80


def test_error_path_without_gpu():
    """Invalid arguments are rejected before any CUDA call."""
    from paper_2505_05643_b200 import _lib
    L = _lib.load()
    assert L.ugs_bin(None, None, None, 0, None, None, None, None) == -1
    assert b"S" in L.ugs_last_error() or b"plan" in L.ugs_last_error()


def test_slice_constants_match_oracle():
    from paper_2505_05643_b200 import _lib
    from paper_2505_05643_b200.geometry import ProbePose, SliceSpec, fill_slice
    from oracle import oracle as O
    import cases
    rng = np.random.default_rng(4)
    for w, h, s, p in ((256, 256, 0.375, 0.95), (37, 53, 0.6, 0.9999), (512, 96, 0.1875, 0.95)):
        R, t = cases.random_pose(rng, 12.0)
        st = _lib.Slice()
        fill_slice(st, SliceSpec(w, h, s, ProbePose(R, t)), p)
        sc = O.slice_constants(R, t, w, h, s, p)
        assert np.array_equal(np.array(st.rw, np.float32), sc["rw"])
        assert np.array_equal(np.array(st.tw, np.float32), sc["tw"])
        for k in ("origin", "du", "dv"):
            assert np.array_equal(np.array(getattr(st, k), np.float32), sc[k])
        for k in ("sqrt_cut", "s", "cx", "cy", "x1h", "x2h"):
            assert np.float32(getattr(st, k)) == sc[k], k


def test_batched_slice_constants_identical():
    """fill_slices (vectorised, the serving path) writes byte-identical
    structs to per-slice fill_slice (the reference's float32 constants)."""
    from paper_2505_05643_b200 import _lib
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.geometry import fill_slice, fill_slices
    for seed in range(3):
        specs = random_pose_specs(20, 96 + seed, 80, 0.4 + 0.05 * seed, seed=seed)
        a, b = (_lib.Slice * 20)(), (_lib.Slice * 20)()
        pix = 0
        for j, sp in enumerate(specs):
            fill_slice(a[j], sp, 0.95, pix)
            pix += sp.width * sp.height
        fill_slices(b, specs, 0.95)
        assert bytes(a) == bytes(b)


def test_fill_slices_c_helper_matches_numpy():
    """ugs_fill_slices (the library's host helper) writes byte-identical
    structs to the numpy restatement over many random poses, sizes and
    spacings (the float64 operation order of ProbePose.inverse / plane_axes
    then float32)."""
    from paper_2505_05643_b200 import _lib
    from paper_2505_05643_b200.geometry import (ProbePose, SliceSpec, fill_slices,
                                                fill_slices_numpy)
    rng = np.random.default_rng(7)
    for trial in range(40):
        S = int(rng.integers(1, 65))
        specs = []
        for _ in range(S):
            q = rng.normal(size=4)
            q /= np.linalg.norm(q)
            w, x, y, z = q
            R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                          [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                          [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
            t = rng.uniform(-60, 60, size=3)
            specs.append(SliceSpec(int(rng.integers(1, 700)), int(rng.integers(1, 700)),
                                   float(rng.uniform(0.05, 2.0)), ProbePose(R, t)))
        p = float(rng.choice([0.95, 0.9999, 0.5]))
        a, b = (_lib.Slice * S)(), (_lib.Slice * S)()
        fill_slices(a, specs, p)
        fill_slices_numpy(b, specs, p)
        assert bytes(a) == bytes(b), trial


def test_render_chunk_splits_on_range_error():
    """render_slices splits a batch whose tile instances exceed the 31-bit
    budget (ugs_bin's UGS_ERR_RANGE) in halves until each part fits; other
    errors propagate (host logic, no GPU: a stand-in renderer)."""
    import pytest
    from paper_2505_05643_b200 import _lib
    from paper_2505_05643_b200.rasterizer import _render_chunk

    class Fake:
        def __init__(self, limit, status=_lib.UGS_ERR_RANGE):
            self.limit, self.status, self.done = limit, status, []

        def bin_async(self, cloud, chunk, p):
            if len(chunk) > self.limit:
                raise _lib.UGSError("too many", self.status)
            self.cur = list(chunk)

        def render(self, cloud, view):
            view[:] = self.cur
            self.done.append(list(self.cur))

        def render_batch(self, cloud, chunk, view, p):   # ugs_render_batch
            self.bin_async(cloud, chunk, p)
            self.render(cloud, view)

        def poll(self):
            return False

    specs = list(range(13))
    out = np.full(13, -1)            # slices of it are views, like the (S, H, W) tensor
    r = Fake(limit=3)
    _render_chunk(r, None, specs, out, 0.95)
    assert out.tolist() == specs and all(len(c) <= 3 for c in r.done)
    with pytest.raises(_lib.UGSError):
        _render_chunk(Fake(limit=3, status=_lib.UGS_ERR_CUDA), None, specs, np.full(13, -1),
                      0.95)
