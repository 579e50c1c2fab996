#!/usr/bin/env python
"""Host side of the C5 render-only path at a small configuration: per-batch
wall time, the host's own time per call, and a cProfile of the Python /
ctypes layer.   python tools/render_host_profile.py [--n 100000 --size 128]
"""

from __future__ import annotations

import argparse
import cProfile
import io
import json
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--out", default="gpurun_out/render_host_profile.json")
    a = ap.parse_args()
    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    import numpy as np
    bounds = np.array([[-48.0] * 3, [48.0] * 3])     # as tools/render_sweep.py
    cfg = ug.TrainConfig(n_gaussians=a.n, seed=0, l_init_low=0.85, l_init_high=1.05)
    cloud = ug.init_cloud(cfg, bounds, device="cuda")
    specs = random_pose_specs(a.batch * 8, a.size, a.size, 96.0 / a.size, seed=a.size,
                              translate=12.0)
    batches = [specs[i:i + a.batch] for i in range(0, len(specs), a.batch)]
    for b in batches[:3]:
        ug.render_slices(cloud, b)
    torch.cuda.synchronize()
    # 1) device-timed batches back to back (what the sweep reports)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for i in range(a.iters):
        ug.render_slices(cloud, batches[i % len(batches)])
    t_host = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    t_dev = e0.elapsed_time(e1) / a.iters
    # 2) one batch at a time, GPU drained in between: the GPU's own time
    solo = []
    for i in range(20):
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        ug.render_slices(cloud, batches[i % len(batches)])
        s1.record()
        torch.cuda.synchronize()
        solo.append(s0.elapsed_time(s1))
    # 3) cProfile of the host layer
    pr = cProfile.Profile()
    pr.enable()
    for i in range(a.iters):
        ug.render_slices(cloud, batches[i % len(batches)])
    pr.disable()
    torch.cuda.synchronize()
    buf = io.StringIO()
    pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(25)
    res = {"config": f"{a.n} Gaussians, {a.size}^2, batch {a.batch}",
           "ms_per_batch_back_to_back": t_dev,
           "host_ms_per_call": t_host * 1e3 / a.iters,
           "ms_per_batch_solo_median": sorted(solo)[len(solo) // 2],
           "slices_per_s": a.batch / (t_dev * 1e-3)}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps(res))
    print(buf.getvalue()[:6000])


if __name__ == "__main__":
    main()
