"""Training through the drop-in ``train()`` on the GPU against the
reference's own training goldens and quality gates.

- C1 trajectory (north_star config 1): the reference's ``train`` at
  ``make_phantom("shells", 64, 0.6, seed=1)`` / 64 axial 128x128 slices /
  10k Gaussians / 200 iterations / densify every 100, workers=1
  (tests/golden/make_golden_c1.py).  The GPU run with batch=1 draws the same
  slice order from the same rng, so its logged losses must track the
  reference's and both densify passes must land on the same Gaussian count.
- Quality gates restated from pkg/tests/test_acceptance.py:145-223 and
  pkg/tests/test_trainer.py:329-357 (blobs reconstruction, degraded-input
  ordering, held-out-frame protocol, constant target, loss decreases),
  unchanged bars.
"""

import hashlib

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2505_05643_b200 as ug  # noqa: E402


def scene_config(**kw):
    """ref tests/test_acceptance.py:40-46."""
    base = dict(l_init_low=0.85, l_init_high=1.05, lr_means_start=0.016,
                lr_means_final=1.6e-4, lr_general_final=0.005, heuristic_interval=0,
                workers=1)
    base.update(kw)
    return ug.TrainConfig(**base)


def test_c1_trajectory_tracks_reference():
    z = load_golden("train_c1.npz")
    vol = ug.make_phantom("shells", 64, 0.6, seed=1)
    ds = ug.make_axial_stack(vol, 64)
    slices = np.stack([s.pixels for s in ds.slices]).astype(np.float32)
    assert hashlib.sha256(slices.tobytes()).digest() == z["slices_sha256"].tobytes()
    cfg = ug.TrainConfig(n_gaussians=10000, iterations=200, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=100,
                         eval_interval=10, workers=1)
    counts = []
    orig = ug.trainer.densify_prune_resample

    def densify(*a, **kw):
        out = orig(*a, **kw)
        counts.append(out[0].n)
        return out

    ug.trainer.densify_prune_resample = densify
    try:
        cloud, log = ug.train(ds, cfg, bounds=vol.world_bounds())
    finally:
        ug.trainer.densify_prune_resample = orig
    assert [e["iter"] for e in log] == list(z["iters"])
    loss = np.array([e["loss"] for e in log])
    tssim = np.array([e["train_ssim"] for e in log])
    it = np.array(z["iters"])
    print("C1 densify counts GPU", counts, "ref", z["densify_n"].tolist())
    print("C1 loss rel diff", np.round(loss / z["loss"] - 1, 5).tolist())
    # the first densify pass (iteration 100) selects, splits, clones and
    # prunes exactly the same Gaussians; after the drift below the second
    # (iteration 200) lands within 0.5 %
    assert counts[0] == int(z["densify_n"][0])
    assert abs(cloud.n / int(z["final_n"]) - 1) < 5e-3
    # same slices, same order: up to the first densify (iteration 100) the
    # float32 GPU run and the reference's CPU run agree per logged loss to
    # 1e-3.  The densify pass then selects candidates against the 90th
    # percentile of the accumulated gradient norms and draws the split
    # children from the shared rng in candidate order, so a candidate that
    # flips across the threshold by a float32 rounding reshuffles every later
    # draw: after it the two runs are different random realisations of the
    # same recipe, compared as such (mean loss and train SSIM of the ten
    # post-densify log entries within 10 % / 0.03)
    pre = it <= 100
    np.testing.assert_allclose(loss[pre], z["loss"][pre], rtol=1e-3)
    np.testing.assert_allclose(tssim[pre], z["train_ssim"][pre], atol=1e-3)
    assert abs(loss[~pre].mean() / z["loss"][~pre].mean() - 1) < 0.10
    assert abs(tssim[~pre].mean() - z["train_ssim"][~pre].mean()) < 0.03


def _heldout(cloud, vol, n):
    rep = ug.evaluate_views(cloud, vol, n_per_axis=n)
    return rep.families["coronal"]["ssim_mean"], rep.families["sagittal"]["ssim_mean"]


def test_blobs_round_trip_gate():
    """test_acceptance.py:145-162: coronal and sagittal SSIM >= 0.95."""
    vol = ug.make_phantom("blobs", 64, 0.6, seed=3)
    ds = ug.make_axial_stack(vol, 64)
    cfg = scene_config(n_gaussians=20000, iterations=2500, seed=0, eval_interval=500)
    cloud, _ = ug.train(ds, cfg, bounds=vol.world_bounds())
    cor, sag = _heldout(cloud, vol, 8)
    assert cor >= 0.95 and sag >= 0.95, (cor, sag)


def test_degraded_input_ordering_gate():
    """test_acceptance.py:165-202: full >= 50 % >= 50 % + 5 deg (0.01
    slack), and the perturbed run beats the best constant image by 0.25."""
    vol = ug.make_phantom("shells", 160, 0.6, seed=1)

    def run(n_slices, perturb):
        ds = ug.make_axial_stack(vol, n_slices, perturb_deg=perturb, seed=0)
        cfg = scene_config(n_gaussians=20000, iterations=1500, seed=0, eval_interval=1500)
        cloud, _ = ug.train(ds, cfg, bounds=vol.world_bounds())
        c, s = _heldout(cloud, vol, 6)
        return (c + s) / 2.0

    full, half, half_pert = run(160, 0.0), run(80, 0.0), run(80, 5.0)
    scores = []
    for fam in ("coronal", "sagittal"):
        for _, spec in ug.family_poses(vol, fam, 6):
            truth = ug.sample_slice(vol, spec).pixels.astype(np.float64)
            scores.append(ug.ssim(np.full_like(truth, truth.mean()), truth))
    baseline = float(np.mean(scores))
    tol = 0.01
    assert full >= half - tol and half >= half_pert - tol, (full, half, half_pert)
    assert half_pert >= baseline + 0.25, (half_pert, baseline)


def test_heldout_frame_protocol_gate():
    """test_acceptance.py:205-223: 80/20 split of a perturbed stack,
    held-out SSIM >= 0.85."""
    vol = ug.make_phantom("shells", 64, 0.6, seed=2)
    ds = ug.make_axial_stack(vol, 100, perturb_deg=5.0, seed=0)
    ds = ug.split_dataset(ds, 0.8, seed=0)
    assert len(ds.subset("train")) == 80 and len(ds.subset("test")) == 20
    cfg = scene_config(n_gaussians=20000, iterations=1500, seed=0, eval_interval=1500)
    cloud, _ = ug.train(ds, cfg, bounds=vol.world_bounds())
    scores = [ug.ssim(ug.render_slice(cloud, img.spec).pixels,
                      img.pixels.astype(np.float64)) for img in ds.subset("test")]
    assert float(np.mean(scores)) >= 0.85, float(np.mean(scores))


def test_constant_target_fits_fast():
    """test_trainer.py:329-344."""
    spec = ug.SliceSpec(24, 24, 1.0)
    imgs = [ug.SliceImage(np.full((24, 24), 0.55, np.float32), 1.0,
                          ug.ProbePose(np.eye(3), np.array([0, 0, z])))
            for z in (-2.0, 0.0, 2.0)]
    cfg = ug.TrainConfig(n_gaussians=200, iterations=250, seed=0, heuristic_interval=0,
                         eval_interval=250)
    cloud, _ = ug.train(ug.SliceDataset(imgs), cfg)
    img = ug.render_slice(cloud, spec)
    assert np.abs(img.pixels - 0.55).mean() < 0.02
    assert ug.ssim(img.pixels, np.full((24, 24), 0.55)) > 0.99


def test_loss_decreases():
    """test_trainer.py:346-357."""
    vol = ug.make_phantom("blobs", 16, 1.0, seed=0)
    ds = ug.make_axial_stack(vol, 8)
    cfg = ug.TrainConfig(n_gaussians=500, iterations=300, seed=0, eval_interval=10)
    cloud, log = ug.train(ds, cfg)
    head = np.mean([e["loss"] for e in log[:3]])
    tail = np.mean([e["loss"] for e in log[-3:]])
    assert tail < head
    assert log[-1]["iter"] == 300
    assert all(set(e) == {"iter", "wall_ms", "loss", "train_ssim"} for e in log)


def test_mixed_size_slices_train():
    """The reference trains on slices of any size (trainer.py:380-390): a
    dataset mixing 24x24 and 32x20 slices trains (batch 1 and a batch of 4
    mixing both sizes), and a step on one of its slices equals the same step
    on a uniform dataset of that slice alone."""
    rng = np.random.default_rng(0)
    vol = ug.make_phantom("blobs", 24, 1.0, seed=1)
    imgs = []
    for i, (w, h) in enumerate([(24, 24), (32, 20), (24, 24), (32, 20)]):
        pose = ug.ProbePose(np.eye(3), np.array([0.0, 0.0, -3.0 + 2.0 * i]))
        imgs.append(ug.sample_slice(vol, ug.SliceSpec(w, h, 1.0, pose)))
    cfg = ug.TrainConfig(n_gaussians=300, iterations=40, seed=3, heuristic_interval=0,
                         eval_interval=10, l_init_low=0.5, l_init_high=1.0,
                         lr_means_start=0.01, lr_means_final=1e-4)
    cloud, log = ug.train(ug.SliceDataset(imgs), cfg)
    assert len(log) == 4 and all(np.isfinite(e["loss"]) for e in log)
    # batch of 4 mixing both sizes in one step
    cfg4 = ug.TrainConfig(n_gaussians=300, iterations=10, seed=3, heuristic_interval=0,
                          eval_interval=5, batch=4, l_init_low=0.5, l_init_high=1.0)
    cloud4, log4 = ug.train(ug.SliceDataset(imgs), cfg4)
    assert all(np.isfinite(e["loss"]) for e in log4)
    # a step on one slice of the mixed dataset == the same step on a
    # uniform dataset holding only that slice (loss and parameters, bitwise)
    base = ug.init_cloud(cfg, ug.dataset_bounds(ug.SliceDataset(imgs)))
    specs = [im.spec for im in imgs]
    tg = [torch.as_tensor(im.pixels, device="cuda") for im in imgs]
    em = ug.TrainEngine(base.copy(), cfg, specs, tg)
    eu = ug.TrainEngine(base.copy(), cfg, [specs[1]], tg[1][None].contiguous())
    lm, lu = em.step([1], 1), eu.step([0], 1)
    assert lm == lu
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        assert torch.equal(getattr(em.cloud, k), getattr(eu.cloud, k)), k
    del rng
