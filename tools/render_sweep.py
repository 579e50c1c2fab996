#!/usr/bin/env python
"""Config C5: render-only (forward) throughput sweep on
one GPU -- N in {100k, 250k, 500k, 1M, 2M, 4M} Gaussians (init_cloud
distribution over the 96 mm cube, l_init U[0.85,1.05)) x H = W in {128, 256,
512} at 96/H mm, batches of 16 random-pose slices (seeded), inputs resident.
Reports slices/s of the whole render path (ugs_bin + forward + clip), the
forward kernel's share, and (Gaussian, pixel) pairs per slice.

    python tools/render_sweep.py [--out gpurun_out/render_sweep.json] [--quick]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/render_sweep.json")
    ap.add_argument("--quick", action="store_true", help="N <= 1M, H <= 256")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--batch", type=int, default=16)
    a = ap.parse_args()

    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs

    ns = [100_000, 250_000, 500_000, 1_000_000, 2_000_000, 4_000_000]
    sizes = [128, 256, 512]
    if a.quick:
        ns, sizes = ns[:4], sizes[:2]
    bounds = np.array([[-48.0] * 3, [48.0] * 3])
    res = []
    for n in ns:
        cfg = ug.TrainConfig(n_gaussians=n, seed=0, l_init_low=0.85, l_init_high=1.05)
        cloud = ug.init_cloud(cfg, bounds, device="cuda")
        for hw in sizes:
            specs = random_pose_specs(a.batch, hw, hw, 96.0 / hw, seed=hw, translate=12.0)
            r = ug.Renderer()
            for _ in range(2):
                ug.render_slices(cloud, specs, renderer=r)
            # throughput uninstrumented; stage times in a second pass
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                ug.render_slices(cloud, specs, renderer=r)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            r.set_timing(True)
            r.timings(reset=True)
            for _ in range(a.iters):
                ug.render_slices(cloud, specs, renderer=r)
            torch.cuda.synchronize()
            st = {k: v[0] / max(v[1], 1) for k, v in r.timings().items()}
            r.set_timing(False)
            pairs = float(np.sum(r.pairs)) / a.batch
            ent = {"n_gaussians": n, "size": hw, "spacing_mm": 96.0 / hw,
                   "slices_per_s": a.batch / (ms * 1e-3), "ms_per_batch": ms,
                   "pairs_per_slice": pairs,
                   "gpairs_per_s": pairs * a.batch / (ms * 1e-3) / 1e9,
                   "forward_ms": st.get("forward"), "stage_ms": st}
            res.append(ent)
            print(json.dumps({k: ent[k] for k in ("n_gaussians", "size", "slices_per_s",
                                                 "pairs_per_slice", "forward_ms")}),
                  flush=True)
            del r
            torch.cuda.empty_cache()
        del cloud
        torch.cuda.empty_cache()
    out = {"config": "C5 render-only sweep, 1 GPU, batch %d random-pose slices, fixed "
                     "init-distribution clouds, inputs resident, CUDA-event timing, mean of "
                     "%d batches after 2 warm-up" % (a.batch, a.iters),
           "gpu": torch.cuda.get_device_name(0), "results": res}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
