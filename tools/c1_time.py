#!/usr/bin/env python
"""North_star config C1 timed: the reference's own CPU run (recorded when
tests/golden/make_golden_c1.py generated train_c1.npz: workers=1) next to the
GPU path's train() on the same inputs and recipe (64^3 shells phantom, 64
axial 128x128 slices, 10k Gaussians, 200 iterations, densify every 100).

    python tools/c1_time.py [--out gpurun_out/c1_time.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/c1_time.json")
    ap.add_argument("--repeats", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2505_05643_b200 as ug
    z = np.load(os.path.join(ROOT, "tests", "golden", "train_c1.npz"))
    vol = ug.make_phantom("shells", 64, 0.6, seed=1)
    ds = ug.make_axial_stack(vol, 64)
    cfg = ug.TrainConfig(n_gaussians=10000, iterations=200, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=100, eval_interval=10,
                         workers=1)
    runs = []
    for _ in range(a.repeats + 1):          # the first run warms the plans up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cloud, log = ug.train(ds, cfg, bounds=vol.world_bounds())
        torch.cuda.synchronize()
        runs.append({"seconds": time.perf_counter() - t0, "final_n": cloud.n,
                     "final_loss": log[-1]["loss"], "final_train_ssim": log[-1]["train_ssim"]})
    ref = float(z["ref_seconds"])
    best = min(r["seconds"] for r in runs[1:])
    out = {"config": "C1: 64^3 shells phantom, 64 axial 128x128 slices, 10k Gaussians, "
                     "200 iterations at batch 1, densify every 100 (scene_config)",
           "reference_seconds": ref,
           "reference_note": "echosplat train() at workers=1 on this build's container CPU, "
                             "recorded by tests/golden/make_golden_c1.py",
           "reference_final": {"n": int(z["final_n"]), "loss": float(z["loss"][-1]),
                               "train_ssim": float(z["train_ssim"][-1])},
           "gpu_seconds_best": best, "gpu_runs": runs[1:], "warmup_run": runs[0],
           "speedup": ref / best}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("reference_seconds", "gpu_seconds_best", "speedup")}))


if __name__ == "__main__":
    main()
