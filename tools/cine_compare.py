#!/usr/bin/env python
"""Reduced config C4 (cine sweep) run by BOTH implementations on the same
recipe, to tell whether the held-out SSIM decay seen at full C4
(profiles/cine_sweep_r01.json) is the training recipe's or the GPU path's.

Data (identical on both sides, each built with its own package):
  make_phantom("shells", 64, 0.6, seed=1); make_axial_stack(vol, 200,
  perturb_deg=5, seed=0); seeded N(0, 0.05^2) pixel noise clipped to [0, 1]
  (numpy default_rng(0), one draw per frame in order); 50 % subsample (every
  other frame -> 100); split_dataset(0.8, seed=0) -> 80 noisy training
  frames, 20 held-out poses scored against the CLEAN trilinear slice.
Recipe: the reference's train() loop (trainer.py:351-434) at batch 1:
  TrainConfig(n_gaussians=20000, iterations=3000, seed=0, l_init 0.85-1.05,
  lr_means 0.016 -> 1.6e-4, lr_general_final 0.005, heuristic_interval=100)
  -- scene_config of tests/test_acceptance.py:40-46 with densification on.
Every --eval-every iterations: mean SSIM of the held-out renders.

    # reference, CPU (this container; imports /root/reference/pkg/src):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tools/cine_compare.py --impl reference --out profiles/cine_compare_ref_r02.json
    # ours, GPU:
    python tools/cine_compare.py --impl gpu --out gpurun_out/cine_compare_gpu.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_data(mod_volume, mod_dataset, frames, size):
    vol = mod_volume.make_phantom("shells", size, 0.6, seed=1)
    stack = mod_dataset.make_axial_stack(vol, frames, perturb_deg=5.0, seed=0)
    rng = np.random.default_rng(0)
    clean = [s.pixels for s in stack.slices]
    noisy = [np.clip(p + rng.normal(0.0, 0.05, p.shape), 0.0, 1.0).astype(np.float32)
             for p in clean]
    keep = list(range(0, frames, 2))
    sub = mod_dataset.SliceDataset([type(stack.slices[i])(noisy[i], stack.slices[i].spacing,
                                                          stack.slices[i].pose)
                                    for i in keep])
    split = mod_dataset.split_dataset(sub, 0.8, seed=0)
    test_idx = [keep[k] for k, lab in enumerate(split.split) if lab == "test"]
    test_specs = [stack.slices[i].spec for i in test_idx]
    test_gt = [np.asarray(clean[i], np.float32) for i in test_idx]
    return vol, split, test_specs, test_gt


def run_reference(a):
    from echosplat import dataset as D, volume as V
    from echosplat.metrics import ssim
    from echosplat.rasterizer import rasterize, render_slice
    from echosplat.gradients import backward
    from echosplat.trainer import (AdamState, TrainConfig, adam_step, dataset_bounds,
                                   densify_prune_resample, general_lr, init_cloud, loss,
                                   mean_lr)
    vol, ds, test_specs, test_gt = build_data(V, D, a.frames, a.size)
    cfg = TrainConfig(**config_kw(a))
    train_slices = ds.subset("train")
    bounds = dataset_bounds(ds)
    rng = np.random.default_rng(cfg.seed)
    cloud = init_cloud(cfg, bounds)
    state = AdamState.for_cloud(cloud)
    scene_extent = float(np.linalg.norm(bounds[1] - bounds[0]))
    threshold = cfg.densify_grad_threshold
    grad_sum = np.zeros(cloud.n, np.float32)
    grad_cnt = np.zeros(cloud.n, np.int64)
    order = rng.permutation(len(train_slices))
    cursor = 0

    def heldout(c):
        return float(np.mean([ssim(render_slice(c, s, p=cfg.p_mass).pixels, g)
                              for s, g in zip(test_specs, test_gt)]))

    log = [{"iter": 0, "train_s": 0.0, "heldout_ssim": heldout(cloud), "n": cloud.n}]
    print(json.dumps(log[-1]), flush=True)
    t_train = 0.0
    for it in range(1, cfg.iterations + 1):
        t0 = time.perf_counter()
        if cursor >= len(order):
            order = rng.permutation(len(train_slices))
            cursor = 0
        img = train_slices[order[cursor]]
        cursor += 1
        buffers = rasterize(cloud, img.spec, p=cfg.p_mass, workers=cfg.workers)
        pred = buffers.intensity_num / buffers.opacity_sum
        loss_val, dpix = loss(pred, img.pixels, cfg.ssim_loss_weight, l2=cfg.l2_loss)
        grads = backward(cloud, img.spec, buffers, dpix, workers=cfg.workers)
        norms = np.linalg.norm(grads.d_means, axis=1)
        grad_sum[buffers.accepted] += norms[buffers.accepted]
        grad_cnt[buffers.accepted] += 1
        lr_g = general_lr(cfg, it)
        lrs = {"means": mean_lr(cfg, it), "l_raw": lr_g, "intensity_raw": lr_g,
               "opacity_raw": lr_g, "bg": lr_g}
        cloud = adam_step(state, cloud, grads, lrs)
        if cfg.heuristic_interval > 0 and it % cfg.heuristic_interval == 0:
            avg = grad_sum / np.maximum(grad_cnt, 1)
            if threshold is None:
                threshold = float(np.quantile(avg, 0.9))
            cloud, state = densify_prune_resample(cloud, avg, state, cfg, rng, scene_extent,
                                                  threshold, 2 * cfg.n_gaussians)
            grad_sum = np.zeros(cloud.n, np.float32)
            grad_cnt = np.zeros(cloud.n, np.int64)
        t_train += time.perf_counter() - t0
        if it % a.eval_every == 0:
            log.append({"iter": it, "train_s": t_train, "heldout_ssim": heldout(cloud),
                        "loss": float(loss_val), "n": cloud.n})
            print(json.dumps(log[-1]), flush=True)
    return log


def run_gpu(a):
    import torch
    sys.path.insert(0, ROOT)
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200 import dataset as D, volume as V
    from paper_2505_05643_b200.metrics import ssim_batch
    from paper_2505_05643_b200.parallel import SliceScheduler
    from paper_2505_05643_b200.trainer import TrainEngine, dataset_bounds
    vol, ds, test_specs, test_gt = build_data(V, D, a.frames, a.size)
    cfg = ug.TrainConfig(**config_kw(a))
    train_slices = ds.subset("train")
    bounds = np.asarray(dataset_bounds(ds), np.float64)
    rng = np.random.default_rng(cfg.seed)
    cloud = ug.init_cloud(cfg, bounds, device="cuda")
    targets = torch.as_tensor(np.stack([s.pixels for s in train_slices]), device="cuda")
    eng = TrainEngine(cloud, cfg, [s.spec for s in train_slices], targets)
    scene_extent = float(np.linalg.norm(bounds[1] - bounds[0]))
    threshold = cfg.densify_grad_threshold
    sched = SliceScheduler(rng, len(train_slices), cfg.batch)
    gt = torch.as_tensor(np.stack(test_gt), device="cuda")
    renderer = ug.Renderer()

    def heldout():
        preds = ug.render_slices(eng.cloud, test_specs, cfg.p_mass, renderer)
        return float(ssim_batch(preds, gt).mean())

    log = [{"iter": 0, "train_s": 0.0, "heldout_ssim": heldout(), "n": eng.cloud.n}]
    print(json.dumps(log[-1]), flush=True)
    torch.cuda.synchronize()
    t_train = 0.0
    t0 = time.perf_counter()
    for it in range(1, cfg.iterations + 1):
        loss_val = eng.step(sched.next(), it)
        if cfg.heuristic_interval > 0 and it % cfg.heuristic_interval == 0:
            threshold = eng.densify(rng, scene_extent, threshold, 2 * cfg.n_gaussians)
        if it % a.eval_every == 0:
            torch.cuda.synchronize()
            t_train += time.perf_counter() - t0
            log.append({"iter": it, "train_s": t_train, "heldout_ssim": heldout(),
                        "loss": float(loss_val), "n": eng.cloud.n})
            print(json.dumps(log[-1]), flush=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
    return log


def config_kw(a):
    return dict(n_gaussians=a.n, iterations=a.iterations, seed=0, l_init_low=0.85,
                l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                lr_general_final=0.005, heuristic_interval=a.densify, batch=1, workers=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=("reference", "gpu"), required=True)
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--iterations", type=int, default=3000)
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--densify", type=int, default=100)
    ap.add_argument("--eval-every", type=int, default=100)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    t0 = time.perf_counter()
    log = run_reference(a) if a.impl == "reference" else run_gpu(a)
    best = max(log, key=lambda e: e["heldout_ssim"])
    out = {"impl": a.impl, "config": vars(a), "wall_s": time.perf_counter() - t0,
           "best": best, "final": log[-1], "log": log,
           "recipe": "reference train() loop at batch 1 (trainer.py:351-434), "
                     "scene_config (test_acceptance.py:40-46) + heuristic_interval"}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({"best": best, "final": log[-1]}))


if __name__ == "__main__":
    main()
