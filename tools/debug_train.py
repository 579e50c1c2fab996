#!/usr/bin/env python
"""Diagnose non-finite training steps: run the engine on the C2 setup and
report the first step where the loss or any parameter stops being finite."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.parallel import SliceScheduler
    from paper_2505_05643_b200.trainer import TrainEngine
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 120
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(256, 256, 256, 0.375, seed=11, translate=12.0)
    gt = ug.sample_slices(vol, specs)
    cfg = ug.TrainConfig(n_gaussians=n, iterations=20000, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=0, batch=B)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs, gt)
    sched = SliceScheduler(np.random.default_rng(0), len(specs), B)
    for it in range(1, steps + 1):
        idx = sched.next()
        c = eng.cloud
        before = {k: getattr(c, k).clone() for k in ("means", "l_raw", "intensity_raw",
                                                       "opacity_raw")}
        bg_before = c.bg_raw.clone()
        num, den, _, tgt, lv, dpix = eng.forward_loss(idx)
        bad = []
        for name, t in (("num", num), ("den", den), ("loss", lv), ("dpix", dpix)):
            if not torch.isfinite(t).all():
                bad.append(name)
        if (den <= 0).any():
            bad.append("den<=0")
        loss = eng.step(idx, it)
        for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
            if not torch.isfinite(getattr(c, k)).all():
                bad.append("param:" + k)
        if not torch.isfinite(c.bg_raw).all():
            bad.append("bg")
        pairs = int(eng.renderer.pairs.sum())
        if it % 10 == 0 or bad:
            print(f"it {it} loss {loss:.5f} pairs/slice {pairs / B:.3e} "
                  f"max|l_raw| {float(c.l_raw.abs().max()):.3f} "
                  f"bg {c.bg_raw.tolist()} bad {bad}", flush=True)
        if bad:
            for k, v in before.items():
                nowv = getattr(c, k)
                badrows = (~torch.isfinite(nowv)).reshape(nowv.shape[0], -1).any(1)
                ids = torch.nonzero(badrows).flatten()[:5]
                print(" ", k, "nonfinite rows", int(badrows.sum()), "e.g.", ids.tolist())
                for i in ids.tolist()[:2]:
                    print("    before", before["means"][i].tolist(), before["l_raw"][i].tolist(),
                          float(before["intensity_raw"][i]), float(before["opacity_raw"][i]))
            print("  bg before", bg_before.tolist())
            break


if __name__ == "__main__":
    main()
