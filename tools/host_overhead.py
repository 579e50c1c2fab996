#!/usr/bin/env python
"""Host cost of one C3 training step versus its device time: whether the
GPU ever waits for the Python / ctypes side.

    python tools/host_overhead.py [--steps 30]
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
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--n-gaussians", type=int, default=1_000_000)
    ap.add_argument("--sync-bin", action="store_true")
    a = ap.parse_args()

    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.trainer import TrainEngine

    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(256, 256, 256, 0.375, seed=0, translate=12.0)
    targets = ug.sample_slices(vol, specs)
    cfg = ug.TrainConfig(n_gaussians=a.n_gaussians, iterations=10000, seed=0,
                         l_init_low=0.85, l_init_high=1.05, lr_means_start=0.016,
                         lr_means_final=1.6e-4, lr_general_final=0.005,
                         heuristic_interval=0, batch=a.batch)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs, targets)
    eng.async_bin = not a.sync_bin
    init = [t.clone() for t in (cloud.means, cloud.l_raw, cloud.intensity_raw,
                                cloud.opacity_raw, cloud.bg_raw)]
    order = np.random.default_rng(1234).permutation(len(specs))

    def step(i):
        c = eng.cloud
        torch._foreach_copy_([c.means, c.l_raw, c.intensity_raw, c.opacity_raw, c.bg_raw],
                             init)
        idx = [int(order[(i * a.batch + j) % len(order)]) for j in range(a.batch)]
        return eng.step(idx, i + 1, check_finite=False)

    for i in range(5):
        step(i)
    eng.settle()
    torch.cuda.synchronize()
    host = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for i in range(5, 5 + a.steps):
        h0 = time.perf_counter()
        step(i)
        host.append(time.perf_counter() - h0)
    t_launch = time.perf_counter() - t0
    eng.settle()
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / a.steps
    out = {"host_ms_per_step_call": 1e3 * float(np.median(host)),
           "host_ms_per_step_mean": 1e3 * t_launch / a.steps,
           "gpu_ms_per_step_paced": gpu_ms,
           "async_bin": eng.async_bin, "reissued": eng.reissued}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
