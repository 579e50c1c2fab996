#!/usr/bin/env python
"""Where a batch-1 step of the reference recipe goes (C2, densify every 100):
train N iterations, then time M steps -- wall per step, GPU time per step
(CUDA events), and the library's per-stage times.
    python tools/batch1_profile.py [--warm 3000 --steps 200]"""
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
    ap.add_argument("--warm", type=int, default=3000)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.parallel import SliceScheduler
    from paper_2505_05643_b200.trainer import TrainEngine
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(2048, 256, 256, 0.375, seed=11, translate=12.0)
    gt = ug.sample_slices(vol, specs)
    cfg = ug.TrainConfig(n_gaussians=200_000, iterations=20000, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=100, batch=1)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs, gt)
    rng = np.random.default_rng(0)
    sched = SliceScheduler(rng, len(specs), 1)
    b = np.asarray(vol.world_bounds(), np.float64)
    extent = float(np.linalg.norm(b[1] - b[0]))
    thr = cfg.densify_grad_threshold
    it = 0
    for _ in range(a.warm):
        it += 1
        eng.step(sched.next(), it)
        if it % 100 == 0:
            thr = eng.densify(rng, extent, thr, 2 * cfg.n_gaussians)
    torch.cuda.synchronize()
    eng.renderer.set_timing(True)
    eng.renderer.timings(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        it += 1
        eng.step(sched.next(), it)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / a.steps
    gpu = e0.elapsed_time(e1) / a.steps
    st = {k: v[0] / a.steps for k, v in eng.renderer.timings().items()}
    print(json.dumps({"n": eng.cloud.n, "pairs_per_slice": float(np.mean(eng.renderer.pairs)),
                      "wall_ms_per_step": wall, "gpu_ms_per_step": gpu,
                      "stage_ms": {k: round(v, 4) for k, v in st.items()}}))


if __name__ == "__main__":
    main()
