#!/usr/bin/env python
"""Where a C2 training step's time goes while the cloud trains (the
time-to-SSIM loop): per window of steps, the host wall time, the GPU stage
times (CUDA events) and the (Gaussian, pixel) pairs per slice.

    python tools/tts_profile.py [--batch 48] [--steps 200] [--window 20]
"""
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
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--batch", type=int, default=48)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--window", type=int, default=20)
    ap.add_argument("--check-finite", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.parallel import SliceScheduler
    from paper_2505_05643_b200.trainer import TrainEngine
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(2048, 256, 256, 0.375, seed=11, translate=12.0)
    gt = ug.sample_slices(vol, specs)
    cfg = ug.TrainConfig(n_gaussians=a.n, iterations=20000, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=0, batch=a.batch)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs, gt)
    sched = SliceScheduler(np.random.default_rng(0), len(specs), a.batch)
    eng.renderer.set_timing(True)
    eng.renderer.timings(reset=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pairs = 0
    for it in range(1, a.steps + 1):
        eng.pairs_total = 0
        eng.step(sched.next(), it, check_finite=bool(a.check_finite))
        pairs += eng.pairs_total
        if it % a.window == 0:
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            st = eng.renderer.timings(reset=True)
            gpu = {k: round(v[0] / a.window, 3) for k, v in st.items() if v[0] > 0}
            print(json.dumps({"steps": f"{it - a.window + 1}-{it}",
                              "wall_ms_per_step": round((t1 - t0) * 1e3 / a.window, 3),
                              "gpu_stage_ms_per_step": gpu,
                              "gpu_sum": round(sum(gpu.values()), 3),
                              "pairs_per_slice": pairs / (a.window * a.batch)}))
            pairs = 0
            t0 = time.perf_counter()


if __name__ == "__main__":
    main()
