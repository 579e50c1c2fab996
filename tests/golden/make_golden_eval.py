"""Golden fixture for evaluate_views, made with the
REFERENCE (run here only; the GPU box has no /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_eval.py

eval.npz holds, for a non-cubic (20, 24, 28) @0.6 mm volume cut from the
reference's shells phantom and a seeded 3000-Gaussian cloud:
- family/<name>/<i>/{R, t, wh}: echosplat.metrics._family_poses(volume, name, 5);
- report/<name>/<key>: echosplat.metrics.evaluate_views(cloud, volume, 5)
  (workers=1, p=0.95) -- ssim/psnr mean and std, count, psnr_inf_count;
- the volume (the cloud is regenerated from its seeds by cases.eval_cloud).
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
from echosplat import metrics, volume  # noqa: E402
from echosplat.model import GaussianCloud  # noqa: E402

FAMILIES = ("axial", "coronal", "sagittal")
N_PER_AXIS = 5


def main():
    big = volume.make_phantom("shells", 28, 0.6, seed=1)
    vol = volume.Volume(np.ascontiguousarray(big.voxels[4:24, 2:26, :]), 0.6)
    c = cases.eval_cloud(vol.world_bounds())
    cloud = GaussianCloud(means=c["means"], l_raw=c["l_raw"],
                          intensity_raw=c["intensity_raw"], opacity_raw=c["opacity_raw"],
                          bg_intensity_raw=0.0, bg_opacity_raw=-4.0, beta=c["beta"])
    out = {"voxels": vol.voxels, "spacing": np.float64(vol.spacing)}
    for name in FAMILIES:
        for i, (pose, spec) in enumerate(metrics._family_poses(vol, name, N_PER_AXIS)):
            out[f"family/{name}/{i}/R"] = pose.rotation
            out[f"family/{name}/{i}/t"] = pose.translation
            out[f"family/{name}/{i}/wh"] = np.array([spec.width, spec.height])
    rep = metrics.evaluate_views(cloud, vol, N_PER_AXIS)
    for name, d in rep.families.items():
        for k, v in d.items():
            out[f"report/{name}/{k}"] = np.float64(np.nan if v is None else v)
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **out)
    print({k: {kk: round(vv, 5) if isinstance(vv, float) else vv for kk, vv in d.items()}
           for k, d in rep.families.items()})


if __name__ == "__main__":
    main()
