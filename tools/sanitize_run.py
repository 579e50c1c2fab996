#!/usr/bin/env python
"""Workload for compute-sanitizer (tools/sanitize.sh): smoke() plus two
fused training steps (ugs_bin_async -> forward -> loss -> backward + Adam)
on a reduced C3-like batch, the render-only path and the multi-slice
ugs_backward, so memcheck / racecheck / synccheck see every kernel of the
hot path."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import __graft_entry__
    __graft_entry__.smoke()
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.trainer import TrainEngine
    vol = ug.make_phantom("shells", 64, 1.5, seed=1)
    specs = random_pose_specs(8, 128, 128, 0.75, seed=3, translate=12.0)
    tg = ug.sample_slices(vol, specs)
    cfg = ug.TrainConfig(n_gaussians=50_000, iterations=10, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         heuristic_interval=0, batch=4)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs, tg)
    eng.step([0, 1, 2, 3], 1)
    eng.step([4, 5, 6, 7], 2, check_finite=False)
    eng.settle()
    px = ug.render_slices(eng.cloud, specs[:4])
    px2 = ug.render_slices(eng.cloud, specs[4:8])        # the replayed bin graph
    # a dense cloud: tiles of several 512-instance backward batches (the
    # staging pipeline's id prefetch across batches) and multi-batch forwards
    cfg2 = ug.TrainConfig(n_gaussians=400_000, iterations=10, seed=1, l_init_low=0.85,
                          l_init_high=1.05, heuristic_interval=0, batch=2)
    dense = ug.init_cloud(cfg2, vol.world_bounds(), device="cuda")
    specs2 = random_pose_specs(2, 64, 64, 1.5, seed=5, translate=4.0)
    eng2 = TrainEngine(dense, cfg2, specs2, ug.sample_slices(vol, specs2))
    eng2.step([0, 1], 1, check_finite=False)
    eng2.settle()
    r2 = eng2.renderer
    print("dense: max instances per slice", int(np.max(r2.k)), "tiles", 16)
    r = ug.Renderer()
    r.bin(eng.cloud, specs[:3], 0.95)
    num = torch.empty((3, 128, 128), device="cuda")
    den = torch.empty_like(num)
    r.forward(eng.cloud, num, den)
    from paper_2505_05643_b200.gradients import grad_buffer
    g = grad_buffer(eng.cloud.n, "cuda")
    r.backward(eng.cloud, num, den, torch.ones_like(num), g, None, 1.0 / 3)
    torch.cuda.synchronize()
    print("sanitize workload OK", float(px.mean()), float(px2.mean()), float(g.abs().sum()))


if __name__ == "__main__":
    main()
