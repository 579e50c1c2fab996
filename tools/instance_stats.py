#!/usr/bin/env python
"""Clipped-rectangle statistics of the tile instances at C3 (what the raster
kernels' lane layouts see): histogram of (width, height) per instance and
the lane use of the forward's narrow layout (16-lane groups, pow2 columns x
rows sweeps) and wide layout (32 lanes x 8 rows).

    python tools/instance_stats.py [--out gpurun_out/instance_stats.json]
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
    ap.add_argument("--out", default="gpurun_out/instance_stats.json")
    ap.add_argument("--slices", type=int, default=4)
    a = ap.parse_args()
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200.dataset import random_pose_specs
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)
    cfg = ug.TrainConfig(n_gaussians=1_000_000, seed=0, l_init_low=0.85, l_init_high=1.05)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    specs = random_pose_specs(a.slices, 256, 256, 0.375, seed=0, translate=12.0)
    r = ug.Renderer()
    r.bin(cloud, specs, 0.95)
    _, wins = r.accepted("cuda", windows=True)      # per slice (M_s, 4): iu0 iu1 iv0 iv1
    win = np.concatenate([w.cpu().numpy() for w in wins])
    iu0, iu1, iv0, iv1 = win[:, 0], win[:, 1], win[:, 2], win[:, 3]
    ws, hs = [], []
    for tx0 in range(0, 256, 16):
        x0 = np.maximum(iu0, tx0)
        x1 = np.minimum(iu1, tx0 + 15)
        okx = x1 >= x0
        for ty0 in range(0, 256, 16):
            y0 = np.maximum(iv0, ty0)
            y1 = np.minimum(iv1, ty0 + 15)
            ok = okx & (y1 >= y0)
            ws.append((x1 - x0 + 1)[ok])
            hs.append((y1 - y0 + 1)[ok])
    w = np.concatenate(ws)
    h = np.concatenate(hs)
    hist = np.zeros((17, 17), np.int64)
    np.add.at(hist, (w, h), 1)
    narrow = w < 9
    # narrow layout: cw = pow2 >= w lanes x R = 16 / cw rows per sweep
    cw = np.where(w <= 1, 1, 1 << np.ceil(np.log2(np.maximum(w, 1))).astype(int))
    R = 16 // cw
    sweeps = (h + R - 1) // R
    useful = (w * h)[narrow].sum()
    issued = (16 * sweeps)[narrow].sum()
    wide_pix = (w * h)[~narrow].sum()
    out = {"instances": int(w.size), "narrow_frac": float(narrow.mean()),
           "pixel_updates": int((w * h).sum()),
           "narrow_pixel_frac": float(useful / (w * h).sum()),
           "narrow_lane_use": float(useful / issued),
           "wide_lane_use_rows8": float(wide_pix / (256 * (~narrow).sum())),
           "mean_w_h_narrow": [float(w[narrow].mean()), float(h[narrow].mean())],
           "mean_w_h_wide": [float(w[~narrow].mean()), float(h[~narrow].mean())],
           "top_shapes": sorted(((int(hist[i, j]), i, j) for i in range(17) for j in range(17)
                                 if hist[i, j]), reverse=True)[:25]}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
