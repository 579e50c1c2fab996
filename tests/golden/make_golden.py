"""Generate golden vectors from the REFERENCE implementation (echosplat).

Run here only (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference read-only from /root/reference/pkg/src and writes
small ``.npz`` fixtures next to this script.  Inputs are regenerated from the
seeded recipes in ``cases.py`` (checksums stored), outputs are what the
reference computes at workers=1 (its deterministic sequential mode).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
REF = os.environ.get("ECHOSPLAT_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import cases  # noqa: E402
from echosplat import geometry, rasterizer, gradients, trainer, metrics  # noqa: E402
from echosplat import volume as evol, dataset as eds  # noqa: E402
from echosplat.model import GaussianCloud  # noqa: E402


def to_cloud(c):
    return GaussianCloud(means=c["means"].copy(), l_raw=c["l_raw"].copy(),
                         intensity_raw=c["intensity_raw"].copy(),
                         opacity_raw=c["opacity_raw"].copy(),
                         bg_intensity_raw=c["bg_intensity_raw"],
                         bg_opacity_raw=c["bg_opacity_raw"], beta=c["beta"])


def ref_constants(spec, p):
    """The f32 constants the reference's _prepare/plane_axes actually use."""
    inv = spec.pose.inverse()
    o, du, dv = geometry.plane_axes(spec, np.float32)
    return dict(rw=inv.rotation.astype(np.float32).reshape(9),
                tw=inv.translation.astype(np.float32),
                origin=o, du=du, dv=dv,
                cut=np.float32(rasterizer.chi2_cutoff(p)))


def gen_prepare():
    out = {}
    for case in cases.PREPARE_CASES:
        cloud, R, t, w, h, s = cases.prepare_case(case)
        spec = geometry.SliceSpec(width=w, height=h, spacing=s,
                                  pose=geometry.ProbePose(R, t))
        acc, L, win, _ = rasterizer._prepare(to_cloud(cloud), spec, 0.95)
        name = case[0]
        out[f"{name}/accepted"] = acc
        out[f"{name}/windows"] = np.stack(win, axis=1)
        out[f"{name}/checksum"] = np.float64(
            cases.input_checksum(cloud["means"], cloud["l_raw"]))
        for k, v in ref_constants(spec, 0.95).items():
            out[f"{name}/{k}"] = v
        P, K = _counts(np.stack(win, axis=1))
        print(f"prepare {name}: n={len(cloud['means'])} M={len(acc)} P={P} K={K}")
    np.savez_compressed(os.path.join(HERE, "prepare.npz"), **out)


def _counts(win):
    P = int(np.sum((win[:, 1] - win[:, 0] + 1) * (win[:, 3] - win[:, 2] + 1)))
    K = int(np.sum(((win[:, 1] >> 4) - (win[:, 0] >> 4) + 1)
                   * ((win[:, 3] >> 4) - (win[:, 2] >> 4) + 1)))
    return P, K


def gen_render():
    out = {}
    for case in cases.RENDER_CASES:
        cloud, R, t, w, h, s, p, dpix = cases.render_case(case)
        name = case[0]
        spec = geometry.SliceSpec(width=w, height=h, spacing=s,
                                  pose=geometry.ProbePose(R, t))
        c = to_cloud(cloud)
        buf = rasterizer.rasterize(c, spec, p=p, workers=1)
        g = gradients.backward(c, spec, buf, dpix, workers=1)
        out[f"{name}/num"] = buf.intensity_num
        out[f"{name}/den"] = buf.opacity_sum
        out[f"{name}/accepted"] = buf.accepted
        out[f"{name}/d_means"] = g.d_means
        out[f"{name}/d_l_raw"] = g.d_l_raw
        out[f"{name}/d_intensity_raw"] = g.d_intensity_raw
        out[f"{name}/d_opacity_raw"] = g.d_opacity_raw
        out[f"{name}/d_bg"] = np.array([g.d_bg_intensity_raw,
                                        g.d_bg_opacity_raw])
        out[f"{name}/checksum"] = np.float64(
            cases.input_checksum(cloud["means"], cloud["l_raw"], dpix))
        # loss on the rendered prediction against a smooth target
        pred = buf.intensity_num / buf.opacity_sum
        tgt = np.clip(pred + 0.05 * np.sin(np.arange(pred.size)).reshape(
            pred.shape), 0, 1).astype(np.float32)
        if min(pred.shape) >= 11:
            lv, lg = trainer.loss(pred, tgt, 0.2)
            out[f"{name}/target"] = tgt
            out[f"{name}/loss"] = np.float64(lv)
            out[f"{name}/dloss"] = lg
            out[f"{name}/ssim"] = np.float64(metrics.ssim(np.clip(pred, 0, 1), tgt))
        print(f"render {name}: M={len(buf.accepted)}")
    # known-answer tests (pkg/tests/test_rasterizer.py:118-135)
    logit = lambda q: np.log(q / (1 - q))
    empty = GaussianCloud(means=np.zeros((0, 3), np.float32),
                          l_raw=np.zeros((0, 6), np.float32),
                          intensity_raw=np.zeros(0, np.float32),
                          opacity_raw=np.zeros(0, np.float32),
                          bg_intensity_raw=float(logit(0.37)),
                          bg_opacity_raw=-4.0)
    img = rasterizer.render_slice(empty, geometry.SliceSpec(8, 8, 1.0))
    out["kat_empty/pixels"] = img.pixels
    ld = np.sqrt(1.0 / 2.0 - 0.01)
    single = GaussianCloud(means=np.zeros((1, 3), np.float32),
                           l_raw=np.array([[ld] * 3 + [0, 0, 0]], np.float32),
                           intensity_raw=np.array([logit(1 - 1e-7)], np.float32),
                           opacity_raw=np.array([logit(0.8)], np.float32),
                           bg_intensity_raw=-30.0, bg_opacity_raw=-4.0,
                           beta=0.01)
    img = rasterizer.render_slice(single, geometry.SliceSpec(17, 17, 1.0),
                                  p=0.9999)
    out["kat_single/pixels"] = img.pixels
    np.savez_compressed(os.path.join(HERE, "render.npz"), **out)


def gen_adam_densify():
    out = {}
    rng = np.random.default_rng(21)
    cloud = cases.random_cloud(rng, 64)
    c = to_cloud(cloud)
    st = trainer.AdamState.for_cloud(c)
    lrs = {"means": 0.016, "l_raw": 0.05, "intensity_raw": 0.05,
           "opacity_raw": 0.05, "bg": 0.05}
    for step in range(5):
        g = gradients.ParamGradients(
            d_means=rng.standard_normal((64, 3)).astype(np.float32) * 1e-3,
            d_l_raw=rng.standard_normal((64, 6)).astype(np.float32),
            d_intensity_raw=rng.standard_normal(64).astype(np.float32) * 1e-5,
            d_opacity_raw=np.where(np.arange(64) % 3 == 0, 0.0,
                                   rng.standard_normal(64)).astype(np.float32),
            d_bg_intensity_raw=float(rng.standard_normal()),
            d_bg_opacity_raw=float(rng.standard_normal() * 1e-3))
        for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
            out[f"adam/step{step}/d_{k}"] = getattr(g, "d_" + k)
        out[f"adam/step{step}/d_bg"] = np.array([g.d_bg_intensity_raw,
                                                 g.d_bg_opacity_raw])
        trainer.adam_step(st, c, g, lrs)
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        out[f"adam/init/{k}"] = cloud[k]
        out[f"adam/final/{k}"] = getattr(c, k)
        out[f"adam/final/m_{k}"] = st.m[k]
        out[f"adam/final/v_{k}"] = st.v[k]
    out["adam/init/bg"] = np.array([cloud["bg_intensity_raw"],
                                    cloud["bg_opacity_raw"]])
    out["adam/final/bg"] = np.array([c.bg_intensity_raw, c.bg_opacity_raw])

    # densify: prune + clone + split with a seeded rng
    rng = np.random.default_rng(22)
    cloud = cases.random_cloud(rng, 40)
    cloud["opacity_raw"][:4] = -10.0
    c = to_cloud(cloud)
    st = trainer.AdamState.for_cloud(c)
    for k in st.m:
        st.m[k][:] = 0.5
        st.v[k][:] = 0.25
    avg = np.abs(rng.standard_normal(40)).astype(np.float32)
    cfg = trainer.TrainConfig()
    c2, st2 = trainer.densify_prune_resample(
        c, avg, st, cfg, np.random.default_rng(99), scene_extent=60.0,
        threshold=0.8, max_total=48)
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        out[f"densify/init/{k}"] = cloud[k]
        out[f"densify/final/{k}"] = getattr(c2, k)
        out[f"densify/final/m_{k}"] = st2.m[k]
    out["densify/avg"] = avg
    np.savez_compressed(os.path.join(HERE, "adam_densify.npz"), **out)
    print("adam/densify: n_out", c2.n)


def gen_train():
    """Short seeded training run: pins loss, Adam, densify and the loop."""
    vol = evol.make_phantom("blobs", 16, 1.0, seed=0)
    ds = eds.make_axial_stack(vol, 8)
    cfg = trainer.TrainConfig(n_gaussians=300, iterations=40, seed=7,
                              heuristic_interval=20, eval_interval=10,
                              workers=1)
    cloud, log = trainer.train(ds, cfg)
    out = {"slices": np.stack([s.pixels for s in ds.slices]),
           "rot": np.stack([s.pose.rotation for s in ds.slices]),
           "trans": np.stack([s.pose.translation for s in ds.slices]),
           "spacing": np.float64(ds.slices[0].spacing),
           "bounds": trainer.dataset_bounds(ds),
           "loss": np.array([e["loss"] for e in log]),
           "train_ssim": np.array([e["train_ssim"] for e in log]),
           "iters": np.array([e["iter"] for e in log])}
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        out[f"final/{k}"] = getattr(cloud, k)
    out["final/bg"] = np.array([cloud.bg_intensity_raw, cloud.bg_opacity_raw])
    np.savez_compressed(os.path.join(HERE, "train.npz"), **out)
    print("train: final n", cloud.n, "losses", out["loss"])


if __name__ == "__main__":
    gen_prepare()
    gen_render()
    gen_adam_densify()
    gen_train()
