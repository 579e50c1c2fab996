#!/usr/bin/env python
"""Time-to-SSIM on held-out synthetic slices (BASELINE.json metric, part 2;
SURVEY section 8d config C2).

160^3 shells phantom (0.6 mm voxels), N Gaussians from init_cloud, 256x256
@0.375 mm slices at random poses: a training set and a disjoint held-out set,
ground truth by trilinear sampling.  Trains with the GPU engine and logs the
mean held-out SSIM against wall-clock time; stops at --target or --budget.

    python tools/time_to_ssim.py --n 200000 --budget 600 --target 0.99
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
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--train-slices", type=int, default=2048)
    ap.add_argument("--test-slices", type=int, default=64)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--budget", type=float, default=600.0, help="seconds of training")
    ap.add_argument("--target", type=float, default=0.99)
    ap.add_argument("--eval-every", type=int, default=100)
    ap.add_argument("--iterations", type=int, default=20000,
                    help="schedule length (learning-rate decay horizon)")
    ap.add_argument("--densify", type=int, default=0, help="heuristic interval (0=off)")
    ap.add_argument("--l-lo", type=float, default=0.85)
    ap.add_argument("--l-hi", type=float, default=1.05)
    ap.add_argument("--out", default="gpurun_out/time_to_ssim.json")
    a = ap.parse_args()

    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    from paper_2505_05643_b200.metrics import ssim_batch
    from paper_2505_05643_b200.parallel import SliceScheduler
    from paper_2505_05643_b200.trainer import TrainEngine

    t_setup = time.perf_counter()
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(a.train_slices + a.test_slices, 256, 256, 0.375, seed=11,
                              translate=12.0)
    train_specs, test_specs = specs[:a.train_slices], specs[a.train_slices:]
    gt_train = ug.sample_slices(vol, train_specs)
    gt_test = ug.sample_slices(vol, test_specs)
    cfg = ug.TrainConfig(n_gaussians=a.n, iterations=a.iterations, seed=0,
                         l_init_low=a.l_lo, l_init_high=a.l_hi, lr_means_start=0.016,
                         lr_means_final=1.6e-4, lr_general_final=0.005,
                         heuristic_interval=a.densify, batch=a.batch)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, train_specs, gt_train)
    renderer = ug.Renderer()
    bounds = vol.world_bounds()
    scene_extent = float(np.linalg.norm(bounds[1] - bounds[0]))
    rng = np.random.default_rng(cfg.seed)
    sched = SliceScheduler(rng, len(train_specs), a.batch)
    threshold = cfg.densify_grad_threshold
    setup_s = time.perf_counter() - t_setup

    def heldout():
        preds = ug.render_slices(eng.cloud, test_specs, cfg.p_mass, renderer)
        return float(ssim_batch(preds, gt_test).mean())

    log = [{"iter": 0, "train_s": 0.0, "ssim": heldout(), "n": eng.cloud.n}]
    print(json.dumps(log[-1]), flush=True)
    t0 = time.perf_counter()
    eval_s = 0.0
    reached = None
    it = 0
    while True:
        it += 1
        loss = eng.step(sched.next(), it)
        if not np.isfinite(loss):
            print("diverged", flush=True)
            break
        if a.densify and it % a.densify == 0:
            threshold = eng.densify(rng, scene_extent, threshold, 2 * a.n)
        if it % a.eval_every == 0:
            torch.cuda.synchronize()
            te = time.perf_counter()
            el = te - t0 - eval_s
            s = heldout()
            eval_s += time.perf_counter() - te
            log.append({"iter": it, "train_s": el, "ssim": s, "loss": loss,
                        "n": eng.cloud.n, "slices": it * a.batch})
            print(json.dumps(log[-1]), flush=True)
            if reached is None and s >= a.target:
                reached = el
            if reached is not None or el >= a.budget:
                break
    out = {"metric": "time to held-out SSIM target", "target": a.target,
           "reached_s": reached, "best_ssim": max(e["ssim"] for e in log),
           "config": vars(a), "setup_s": setup_s, "log": log,
           "note": "train_s is wall-clock training time; held-out evaluations "
                   "are excluded"}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("target", "reached_s", "best_ssim")}))


if __name__ == "__main__":
    main()
