#!/usr/bin/env python
"""cProfile of the host side of C3 training steps (what the Python / ctypes
layer spends per step).  python tools/host_profile.py [--steps 40]"""

from __future__ import annotations

import cProfile
import io
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import numpy as np
    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.trainer import TrainEngine
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 40
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(256, 256, 256, 0.375, seed=0, translate=12.0)
    targets = ug.sample_slices(vol, specs)
    cfg = ug.TrainConfig(n_gaussians=1_000_000, iterations=10000, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=0, batch=16)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs, targets)
    order = np.random.default_rng(1234).permutation(len(specs))

    def step(i):
        idx = [int(order[(i * 16 + j) % len(order)]) for j in range(16)]
        return eng.step(idx, i + 1, check_finite=False)

    for i in range(5):
        step(i)
    eng.settle()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for i in range(5, 5 + steps):
        step(i)
    eng.settle()
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(30)
    print(s.getvalue())


if __name__ == "__main__":
    main()
