"""Config-C1 training trajectory from the REFERENCE (north_star config 1).

Run here only (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_c1.py

C1 = ``make_phantom("shells", 64, 0.6, seed=1)``, the 64 axial 128x128
slices of ``make_axial_stack`` (0.6 mm), ``TrainConfig(n_gaussians=10000,
iterations=200, seed=0)`` with the reference's own scene-scale settings
(``scene_config``, pkg/tests/test_acceptance.py:40-46: l_init U[0.85,1.05),
lr_means 0.016 -> 1.6e-4, lr_general_final 0.005) and densification every
100 iterations, at workers=1 (the reference's deterministic sequential mode,
trainer.py:351-434).  The log is taken every 10 iterations.  Inputs are
regenerated on the GPU box by this repo's restated phantom / stack
generators; their checksum is stored so the test can prove they match.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("ECHOSPLAT_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from echosplat import trainer, volume as evol, dataset as eds  # noqa: E402

C1 = dict(n_gaussians=10000, iterations=200, seed=0, l_init_low=0.85, l_init_high=1.05,
          lr_means_start=0.016, lr_means_final=1.6e-4, lr_general_final=0.005,
          heuristic_interval=100, eval_interval=10, workers=1)


def main():
    vol = evol.make_phantom("shells", 64, 0.6, seed=1)
    ds = eds.make_axial_stack(vol, 64)
    slices = np.stack([s.pixels for s in ds.slices]).astype(np.float32)
    cfg = trainer.TrainConfig(**C1)
    # record the Gaussian count after each densify pass (the reference's
    # train() does not log it)
    counts = []
    orig = trainer.densify_prune_resample

    def densify(*a, **kw):
        cloud, state = orig(*a, **kw)
        counts.append(cloud.n)
        return cloud, state

    trainer.densify_prune_resample = densify
    t0 = time.time()
    cloud, log = trainer.train(ds, cfg, bounds=vol.world_bounds())
    took = time.time() - t0
    out = {"slices_sha256": np.frombuffer(hashlib.sha256(slices.tobytes()).digest(),
                                          np.uint8),
           "bounds": np.asarray(vol.world_bounds(), np.float64),
           "iters": np.array([e["iter"] for e in log]),
           "loss": np.array([e["loss"] for e in log]),
           "train_ssim": np.array([e["train_ssim"] for e in log]),
           "final_n": np.int64(cloud.n),
           "densify_n": np.array(counts, np.int64),
           "final_bg": np.array([cloud.bg_intensity_raw, cloud.bg_opacity_raw]),
           "ref_seconds": np.float64(took)}
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        out[f"final/{k}"] = getattr(cloud, k).astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "train_c1.npz"), **out)
    print(f"C1: final n {cloud.n}, {took:.1f} s, loss {out['loss'][0]:.4f} -> "
          f"{out['loss'][-1]:.4f}, ssim {out['train_ssim'][-1]:.4f}")


if __name__ == "__main__":
    main()
