"""Golden fixtures for the data formats either side of the hot path, made
with the REFERENCE (run here only; the GPU box has no /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_io.py

- ref_checkpoint.ugsc: echosplat.trainer.save_checkpoint of a seeded 50-
  Gaussian cloud with a non-default TrainConfig (ref trainer.py:295-313);
- io.npz: echosplat.volume.make_phantom("shells"/"blobs", 24^3, 0.6 mm) and
  sample_slice at three seeded poses (ref volume.py:198-263).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.environ.get("ECHOSPLAT_SRC", "/root/reference/pkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import cases  # noqa: E402
from echosplat import trainer, volume  # noqa: E402
from echosplat.geometry import ProbePose, SliceSpec  # noqa: E402
from echosplat.model import GaussianCloud  # noqa: E402


def main():
    c = cases.random_cloud(np.random.default_rng(2024), 50, extent=10.0)
    cloud = GaussianCloud(means=c["means"], l_raw=c["l_raw"],
                          intensity_raw=c["intensity_raw"], opacity_raw=c["opacity_raw"],
                          bg_intensity_raw=c["bg_intensity_raw"],
                          bg_opacity_raw=c["bg_opacity_raw"], beta=c["beta"])
    cfg = trainer.TrainConfig(n_gaussians=50, iterations=123, seed=9, batch=4,
                              lr_general_final=0.005, l_init_low=0.85, l_init_high=1.05)
    trainer.save_checkpoint(cloud, os.path.join(HERE, "ref_checkpoint.ugsc"), cfg, 77)
    out = {}
    for kind in ("shells", "blobs"):
        v = volume.make_phantom(kind, 24, 0.6, seed=1)
        out[f"{kind}/voxels"] = v.voxels
        rng = np.random.default_rng(5)
        for i in range(3):
            R, t = cases.random_pose(rng, 3.0)
            spec = SliceSpec(20, 17, 0.45, ProbePose(R, t))
            out[f"{kind}/slice{i}/R"] = R
            out[f"{kind}/slice{i}/t"] = t
            out[f"{kind}/slice{i}/pixels"] = volume.sample_slice(v, spec).pixels
    np.savez_compressed(os.path.join(HERE, "io.npz"), **out)


if __name__ == "__main__":
    main()
