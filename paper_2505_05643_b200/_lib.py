"""ctypes binding of libugs.so (include/ugs.h) -- the only path to the GPU.

There is deliberately no fallback: if the shared library (or a CUDA device)
is missing, ``lib()`` raises, so every caller fails loudly instead of
silently computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# UGS_LIB overrides the path (experiments: tools/build_variant.py builds
# in-tree variants with different compile-time constants)
LIB_PATH = os.environ.get("UGS_LIB") or os.path.join(HERE, "libugs.so")

_lock = threading.Lock()
_LIB = None

c_f = ctypes.c_float
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p


# status codes of include/ugs.h
UGS_OK, UGS_ERR_INVALID, UGS_ERR_CUDA, UGS_ERR_OOM, UGS_ERR_RANGE = 0, -1, -2, -3, -4


class UGSError(RuntimeError):
    """A libugs entry point returned a non-zero status (``.status``)."""

    def __init__(self, message, status=0):
        super().__init__(message)
        self.status = status


class Slice(ctypes.Structure):
    """struct ugs_slice (include/ugs.h)."""
    _fields_ = [("rw", c_f * 9), ("tw", c_f * 3), ("origin", c_f * 3),
                ("du", c_f * 3), ("dv", c_f * 3), ("sqrt_cut", c_f),
                ("s", c_f), ("cx", c_f), ("cy", c_f), ("x1h", c_f),
                ("x2h", c_f), ("width", c_i32), ("height", c_i32),
                ("tiles_x", c_i32), ("tiles_y", c_i32), ("tile_base", c_i32),
                ("reserved", c_i32), ("pix_base", c_i64)]


class Cloud(ctypes.Structure):
    """struct ugs_cloud (include/ugs.h)."""
    _fields_ = [("means", c_vp), ("l_raw", c_vp), ("intensity_raw", c_vp),
                ("opacity_raw", c_vp), ("bg_raw", c_vp), ("n", c_i64),
                ("beta", ctypes.c_double)]


class PeerView(ctypes.Structure):
    """struct ugs_peer_view (include/ugs.h): one rank's arena, as mapped here."""
    _fields_ = [("means", c_vp), ("l_raw", c_vp), ("intensity_raw", c_vp),
                ("opacity_raw", c_vp), ("grad", c_vp), ("m", c_vp), ("v", c_vp),
                ("grad_sum", c_vp), ("grad_cnt", c_vp), ("bg_raw", c_vp), ("sync", c_vp)]


EXPORTS = {
    "ugs_last_error": (ctypes.c_char_p, []),
    "ugs_abi_version": (ctypes.c_int, []),
    "ugs_plan_create": (ctypes.c_int, [ctypes.POINTER(c_vp)]),
    "ugs_plan_destroy": (ctypes.c_int, [c_vp]),
    "ugs_bin": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), ctypes.POINTER(Slice),
                               ctypes.c_int, c_vp, ctypes.POINTER(c_i64),
                               ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "ugs_bin_async": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), ctypes.POINTER(Slice),
                                     ctypes.c_int, c_vp]),
    "ugs_plan_poll": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                                     ctypes.POINTER(c_i64)]),
    "ugs_export_accepted": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "ugs_export_bins": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(c_i32),
                                       ctypes.POINTER(c_i64), c_vp]),
    "ugs_forward": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), c_vp, c_vp, c_vp]),
    "ugs_render": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), c_vp, c_vp]),
    "ugs_render_batch": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), c_vp, ctypes.c_int,
                                        c_vp, c_vp]),
    "ugs_backward": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), c_vp, c_vp, c_vp,
                                    c_vp, c_vp, c_f, c_vp]),
    "ugs_grad_stats": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ugs_adam_step": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                     c_i64, c_i64, ctypes.POINTER(ctypes.c_double),
                                     ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_int, c_vp, c_vp, c_vp,
                                     c_vp]),
    "ugs_backward_dense": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), c_vp, c_vp, c_vp,
                                          c_vp, c_f, c_vp]),
    "ugs_backward_adam": (ctypes.c_int, [c_vp, ctypes.POINTER(Cloud), c_vp, c_vp, c_vp,
                                         c_f, c_vp, c_vp, c_i64,
                                         ctypes.POINTER(ctypes.c_double),
                                         ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, c_vp, c_vp, c_vp]),
    "ugs_densify_apply": (ctypes.c_int, [ctypes.POINTER(Cloud), c_vp, c_vp, c_vp,
                                         c_i64, c_vp, c_vp, c_vp, c_i64,
                                         ctypes.c_double, c_vp, c_vp, c_vp, c_vp,
                                         c_vp, c_vp, c_vp]),
    "ugs_launch_count": (ctypes.c_longlong, []),
    "ugs_fill_slices": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int,
                                       ctypes.c_double, c_vp]),
    "ugs_fp32_peak_probe": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, c_vp]),
    "ugs_plan_set_timing": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "ugs_plan_set_ordered": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "ugs_loss_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int]),
    "ugs_loss": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ctypes.c_double, ctypes.c_int, c_vp,
                                c_vp, c_vp, c_vp, c_vp]),
    "ugs_loss_ex": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_double, ctypes.c_int, c_vp,
                                   c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ugs_plan_timings": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(c_i64), ctypes.c_int,
                                        ctypes.c_int]),
    "ugs_ipc_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(c_vp), c_vp]),
    "ugs_ipc_open": (ctypes.c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "ugs_ipc_close": (ctypes.c_int, [c_vp]),
    "ugs_ipc_free": (ctypes.c_int, [c_vp]),
    "ugs_peer_update": (ctypes.c_int, [ctypes.POINTER(PeerView), ctypes.c_int, ctypes.c_int,
                                       c_i64, c_i64, c_i64, c_i64,
                                       ctypes.POINTER(ctypes.c_double), ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                       ctypes.c_uint32, c_vp]),
    "ugs_peer_shard": (ctypes.c_int, [c_i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(c_i64),
                                      ctypes.POINTER(c_i64)]),
    "ugs_peer_signal": (ctypes.c_int, [ctypes.POINTER(PeerView), ctypes.c_int, ctypes.c_int,
                                       ctypes.c_uint32, c_vp]),
    "ugs_peer_wait": (ctypes.c_int, [ctypes.POINTER(PeerView), ctypes.c_int, ctypes.c_int,
                                     ctypes.c_uint32, c_vp]),
    "ugs_peer_gather": (ctypes.c_int, [ctypes.POINTER(PeerView), ctypes.c_int, ctypes.c_int,
                                       c_i64, c_vp]),
}

STAGES = ("prepare_count", "prepare_emit", "sort", "bin_ranges", "forward",
          "backward", "finalize", "update")


def load(path: str = LIB_PATH):
    """Load the library and bind every export (no CUDA work happens here)."""
    global _LIB
    with _lock:
        if _LIB is not None:
            return _LIB
        if not os.path.exists(path):
            raise UGSError(
                f"{path} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
        return L


def lib():
    return load()


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = lib().ugs_last_error()
        msg = msg.decode() if msg else ""
        raise UGSError(f"{what or 'libugs'} failed (status {status}): {msg}", status)


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else t.data_ptr()
