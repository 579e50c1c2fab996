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


def train_to_target(bounds, train_specs, gt_train, test_specs, gt_test, n=200_000,
                    batch=16, budget=600.0, target=0.99, eval_every=100, iterations=20000,
                    densify=0, l_lo=0.85, l_hi=1.05, log=print):
    """Train on (train_specs, gt_train) until the mean SSIM of the renders at
    test_specs against gt_test reaches `target` or the budget runs out."""
    import torch
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.metrics import ssim_batch
    from paper_2505_05643_b200.parallel import SliceScheduler
    from paper_2505_05643_b200.trainer import TrainEngine

    cfg = ug.TrainConfig(n_gaussians=n, iterations=iterations, seed=0,
                         l_init_low=l_lo, l_init_high=l_hi, lr_means_start=0.016,
                         lr_means_final=1.6e-4, lr_general_final=0.005,
                         heuristic_interval=densify, batch=batch)
    cloud = ug.init_cloud(cfg, bounds, device="cuda")
    eng = TrainEngine(cloud, cfg, train_specs, gt_train)
    renderer = ug.Renderer()
    bounds = np.asarray(bounds, np.float64)
    scene_extent = float(np.linalg.norm(bounds[1] - bounds[0]))
    rng = np.random.default_rng(cfg.seed)
    sched = SliceScheduler(rng, len(train_specs), batch)
    threshold = cfg.densify_grad_threshold

    def heldout():
        preds = ug.render_slices(eng.cloud, test_specs, cfg.p_mass, renderer)
        return float(ssim_batch(preds, gt_test).mean())

    entries = [{"iter": 0, "train_s": 0.0, "ssim": heldout(), "n": eng.cloud.n}]
    log(json.dumps(entries[-1]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eval_s = 0.0
    reached = None
    it = 0
    while True:
        it += 1
        loss = eng.step(sched.next(), it)
        if not np.isfinite(loss):
            log("diverged")
            break
        if densify and it % densify == 0:
            threshold = eng.densify(rng, scene_extent, threshold, 2 * n)
        if it % eval_every == 0:
            torch.cuda.synchronize()
            te = time.perf_counter()
            el = te - t0 - eval_s
            s = heldout()
            eval_s += time.perf_counter() - te
            entries.append({"iter": it, "train_s": el, "ssim": s, "loss": loss,
                            "n": eng.cloud.n, "slices": it * batch})
            log(json.dumps(entries[-1]))
            if reached is None and s >= target:
                reached = el
            if reached is not None or el >= budget:
                break
    return {"target": target, "reached_s": reached,
            "best_ssim": max(e["ssim"] for e in entries), "iterations": it,
            "slices_trained": it * batch, "log": entries}


def run(n=200_000, train_slices=2048, test_slices=64, batch=16, budget=600.0, target=0.99,
        eval_every=100, iterations=20000, densify=0, l_lo=0.85, l_hi=1.05, log=print):
    """Config C2: random-pose train / held-out slices of the 160^3 phantom."""
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs

    cfg_in = dict(n=n, train_slices=train_slices, test_slices=test_slices, batch=batch,
                  budget=budget, target=target, eval_every=eval_every,
                  iterations=iterations, densify=densify, l_lo=l_lo, l_hi=l_hi)
    t_setup = time.perf_counter()
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(train_slices + test_slices, 256, 256, 0.375, seed=11,
                              translate=12.0)
    train_specs, test_specs = specs[:train_slices], specs[train_slices:]
    gt_train = ug.sample_slices(vol, train_specs)
    gt_test = ug.sample_slices(vol, test_specs)
    setup_s = time.perf_counter() - t_setup
    out = train_to_target(vol.world_bounds(), train_specs, gt_train, test_specs, gt_test, n,
                          batch, budget, target, eval_every, iterations, densify, l_lo,
                          l_hi, log)
    out.update({"metric": "time to held-out SSIM target", "config": cfg_in,
                "setup_s": setup_s,
                "note": "C2: 160^3 shells phantom, init_cloud over its bounds, 256x256 "
                        "@0.375 mm random-pose slices (train set + disjoint held-out "
                        "set, trilinear GT); train_s is wall-clock training time on one "
                        "GPU, held-out evaluations excluded"})
    return out


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
    out = run(a.n, a.train_slices, a.test_slices, a.batch, a.budget, a.target, a.eval_every,
              a.iterations, a.densify, a.l_lo, a.l_hi, log=lambda m: print(m, flush=True))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("target", "reached_s", "best_ssim")}))


if __name__ == "__main__":
    main()
