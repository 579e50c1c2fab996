#!/usr/bin/env python
"""GPU timeline of C3 training steps (torch.profiler / CUPTI; nsys is not in
the image): per-kernel device time, and the idle gaps between consecutive
device activities -- where a step loses time to host synchronisation or
launch latency.

    python tools/gpu_timeline.py [--steps 6] [--out gpurun_out/timeline.json]
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
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--n-gaussians", type=int, default=1_000_000)
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    a = ap.parse_args()

    import torch
    from torch.profiler import ProfilerActivity, profile
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
    init = [t.clone() for t in (cloud.means, cloud.l_raw, cloud.intensity_raw,
                                cloud.opacity_raw, cloud.bg_raw)]
    order = np.random.default_rng(1234).permutation(len(specs))

    def step(i):
        c = eng.cloud
        torch._foreach_copy_([c.means, c.l_raw, c.intensity_raw, c.opacity_raw, c.bg_raw],
                             init)
        idx = [int(order[(i * a.batch + j) % len(order)]) for j in range(a.batch)]
        return eng.step(idx, i + 1, check_finite=False)

    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(3, 3 + a.steps):
            step(i)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    # device activities (kernels, memcpy, memset) in time order
    acts = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs),
                  key=lambda x: x[0])
    per = {}
    for s, e, n in acts:
        d = per.setdefault(n, [0, 0.0])
        d[0] += 1
        d[1] += (e - s)
    span = acts[-1][1] - acts[0][0]
    busy = 0.0
    cur_s, cur_e = acts[0][0], acts[0][1]
    gaps = []
    for s, e, n in acts[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, n))
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy += cur_e - cur_s
    gaps.sort(reverse=True)
    gap_by_next = {}
    for g, n in gaps:
        d = gap_by_next.setdefault(n, [0, 0.0])
        d[0] += 1
        d[1] += g
    out = {"steps": a.steps, "span_us_per_step": span / a.steps,
           "busy_us_per_step": busy / a.steps,
           "idle_us_per_step": (span - busy) / a.steps,
           "idle_before": {k: {"count": v[0] / a.steps, "us_per_step": v[1] / a.steps}
                           for k, v in sorted(gap_by_next.items(), key=lambda kv: -kv[1][1])[:15]},
           "activities": {k: {"count": v[0] / a.steps, "us_per_step": v[1] / a.steps}
                          for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("span_us_per_step", "busy_us_per_step",
                                         "idle_us_per_step")}))
    for k, v in list(out["idle_before"].items())[:10]:
        print(f"  idle before {k[:60]:60s} {v['us_per_step']:8.1f} us/step ({v['count']:.1f}x)")


if __name__ == "__main__":
    main()
