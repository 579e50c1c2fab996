"""Build libugs.so (sm_100a) in-tree with nvcc.

Used by ``__graft_entry__.build()`` and by ``python -m
paper_2505_05643_b200._build``.  The shared library lands next to this file
so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libugs.so")
BUILD = os.path.join(HERE, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
          "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include")]
# files whose float arithmetic must stay unfused (bit-compatible Adam and the
# densify float64 math follow numpy's unfused rounding)
NO_FMAD = {"ugs_adam.cu"}
SOURCES = ["ugs_api.cu", "ugs_prepare.cu", "ugs_sort.cu", "ugs_raster.cu",
           "ugs_adam.cu", "ugs_diag.cu", "ugs_loss.cu", "ugs_peer.cu"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if os.path.exists(cand) else "nvcc"


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), out: str = LIB,
          build_dir: str = BUILD) -> str:
    """Compile every source (stale ones only) and link ``out``; ``defines``
    (e.g. ["UGS_WIDE_MIN=8"]) go to every translation unit -- used by
    tools/build_variant.py for in-tree experiment variants."""
    BUILD_ = build_dir
    os.makedirs(BUILD_, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "ugs.h"))
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD_, src.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not _stale(obj, [path] + headers):
            continue
        flags = list(COMMON) + ["-D" + d for d in defines]
        if src in NO_FMAD:
            flags.append("-fmad=false")
        cmd = [nvcc()] + ARCH + flags + ["-Xptxas", "-v", "-c", path, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
    if force or _stale(out, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", out] + objs
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc link failed")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
