#!/usr/bin/env python
"""Per-step wall time of the first C2 training steps (time-to-SSIM setup,
batch 48): where a slow start goes.   python tools/tts_steps.py [--steps 40]"""
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
    ap.add_argument("--steps", type=int, default=40)
    a = ap.parse_args()
    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.parallel import SliceScheduler
    from paper_2505_05643_b200.trainer import TrainEngine
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(2048 + 64, 256, 256, 0.375, seed=11, translate=12.0)
    gt = ug.sample_slices(vol, specs[:2048])
    cfg = ug.TrainConfig(n_gaussians=200_000, iterations=20000, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=0, batch=48)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs[:2048], gt)
    sched = SliceScheduler(np.random.default_rng(0), 2048, 48)
    torch.cuda.synchronize()
    out = []
    for it in range(1, a.steps + 1):
        t0 = time.perf_counter()
        r0 = eng.reissued
        eng.step(sched.next(), it)
        torch.cuda.synchronize()
        out.append((it, round((time.perf_counter() - t0) * 1e3, 2), eng.reissued - r0,
                    int(eng.renderer.k.sum()) if hasattr(eng.renderer, "k") else -1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
