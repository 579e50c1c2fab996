#!/usr/bin/env python
"""Config C4: cine-sweep reconstruction.

make_axial_stack(160^3 shells phantom, 1000 frames, perturb 5 deg, seed 0)
-> seeded N(0, 0.05^2) noise clipped to [0, 1] -> 50 % subsample (every
other frame: 500) -> split_dataset(0.8, seed 0): 400 noisy training frames,
100 held-out poses scored against the CLEAN trilinear ground truth.
500k Gaussians, one GPU; reports held-out SSIM against training time and the
time to --target (the paper's cine sweeps reach 0.91-0.93 test SSIM on
clinical data).

    python tools/cine_sweep.py [--budget 300] [--target 0.99]
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
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=500_000)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--budget", type=float, default=300.0)
    ap.add_argument("--target", type=float, default=0.99)
    ap.add_argument("--eval-every", type=int, default=100)
    ap.add_argument("--densify", type=int, default=0, help="heuristic interval (0 = off)")
    ap.add_argument("--out", default="gpurun_out/cine_sweep.json")
    a = ap.parse_args()

    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import axial_pose
    from time_to_ssim import train_to_target

    t_setup = time.perf_counter()
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    d, h, w = vol.voxels.shape
    rng = np.random.default_rng(0)
    specs = []   # the draws of make_axial_stack(vol, 1000, perturb_deg=5, seed=0)
    for i in range(1000):
        tx, ty = np.deg2rad(rng.uniform(-5.0, 5.0, size=2))
        specs.append(ug.SliceSpec(w, h, vol.spacing, axial_pose(vol, i * d / 1000, tx, ty)))
    clean = ug.sample_slices(vol, specs)
    g = torch.Generator(device="cpu").manual_seed(0)
    noise = torch.randn(clean.shape, generator=g).to(clean.device) * 0.05
    noisy = torch.clamp(clean + noise, 0.0, 1.0)
    keep = list(range(0, 1000, 2))                      # 50 % subsample
    n_test = int(np.floor(len(keep) * 0.2 + 1e-9))      # split_dataset(0.8, seed 0)
    perm = np.random.default_rng(0).permutation(len(keep))
    test_set = set(perm[:n_test].tolist())
    tr = [keep[i] for i in range(len(keep)) if i not in test_set]
    te = [keep[i] for i in range(len(keep)) if i in test_set]
    train_specs = [specs[i] for i in tr]
    test_specs = [specs[i] for i in te]
    gt_train = noisy[torch.as_tensor(tr, device=noisy.device)].contiguous()
    gt_test = clean[torch.as_tensor(te, device=clean.device)].contiguous()
    setup_s = time.perf_counter() - t_setup
    out = train_to_target(vol.world_bounds(), train_specs, gt_train, test_specs, gt_test,
                          n=a.n, batch=a.batch, budget=a.budget, target=a.target,
                          eval_every=a.eval_every, densify=a.densify,
                          log=lambda m: print(m, flush=True))
    out.update({"metric": "C4 cine sweep: held-out SSIM vs clean GT against training time",
                "config": vars(a), "setup_s": setup_s, "train_frames": len(tr),
                "test_frames": len(te), "frame": [h, w], "spacing_mm": vol.spacing})
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("target", "reached_s", "best_ssim", "iterations")}))


if __name__ == "__main__":
    main()
