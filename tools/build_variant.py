#!/usr/bin/env python
"""Build an experiment variant of libugs.so with extra compile-time defines,
in-tree (so it travels to the GPU box), selected at run time by UGS_LIB:

    python tools/build_variant.py wide8 UGS_WIDE_MIN=8
    UGS_LIB=paper_2505_05643_b200/variants/libugs_wide8.so python bench.py ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_05643_b200 import _build  # noqa: E402

tag, defines = sys.argv[1], sys.argv[2:]
vdir = os.path.join(_build.HERE, "variants")
out = os.path.join(vdir, f"libugs_{tag}.so")
print(_build.build(defines=defines, out=out, build_dir=os.path.join(vdir, "build_" + tag),
                   force=True))
