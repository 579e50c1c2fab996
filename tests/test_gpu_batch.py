"""GPU parity of the exact path the headline bench measures: a 16-slice
batch at config C3 (1M Gaussians, 256x256 @0.375 mm, init cloud seed 0),
through ugs_bin -> ugs_forward -> ugs_backward / ugs_backward_adam.

- batched gradient: ugs_backward(scale=1/16) over the 16-slice batch equals
  the sum of the oracle's per-slice gradients / 16 (ref gradients.py:36-113),
  per group rtol 1e-4 / atol 1e-5*max|group|;
- fused step: one TrainEngine.step (ugs_backward_adam: ordered multi-slice
  accumulation + densify statistics + Adam in one kernel) gives parameters and
  moments BIT-identical to oracle.adam_step (ref trainer.py:170-200) applied
  to that batch's device gradient, and grad_sum / grad_cnt follow the
  reference rule (trainer.py:399-401) for the batch;
- the LSD-radix bin-sort fallback (slices of more than 1024 tiles) gives
  bit-exact tile lists and an oracle-equal render;
- a config-C5 forward sample (4M Gaussians, 512x512) against the oracle.
"""

import ctypes
import os

import numpy as np
import pytest

import cases
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2505_05643_b200 as ug  # noqa: E402
from paper_2505_05643_b200 import _lib  # noqa: E402
from paper_2505_05643_b200.gradients import ParamGradients, grad_buffer  # noqa: E402
from paper_2505_05643_b200.metrics import fused_loss  # noqa: E402
from paper_2505_05643_b200 import trainer as T  # noqa: E402

RTOL, ATOL = 1e-4, 1e-5
WORKERS = max(1, min(16, os.cpu_count() or 1))
S = 16
GROUPS = ("d_means", "d_l_raw", "d_intensity_raw", "d_opacity_raw")


def _oargs(c, sc):
    return (c["means"], c["l_raw"], c["intensity_raw"], c["opacity_raw"],
            c["bg_intensity_raw"], c["bg_opacity_raw"], c["beta"], sc)


@pytest.fixture(scope="module")
def c3():
    cloud_np = cases.uniform_cloud(0, 1_000_000, [[-48] * 3, [48] * 3], 0.85, 1.05)
    rng = np.random.default_rng(2024)
    poses = [cases.random_pose(rng, 12.0) for _ in range(S)]
    specs = [ug.SliceSpec(256, 256, 0.375, ug.ProbePose(R, t)) for R, t in poses]
    scs = [O.slice_constants(R, t, 256, 256, 0.375, 0.95) for R, t in poses]
    return cloud_np, specs, scs


def test_batched_gradient_c3_s16(c3):
    cloud_np, specs, scs = c3
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    r = ug.Renderer()
    r.bin(cloud, specs, 0.95)
    num = torch.empty((S, 256, 256), device="cuda")
    den = torch.empty_like(num)
    r.forward(cloud, num, den)
    dpix = torch.as_tensor(np.random.default_rng(7).standard_normal((S, 256, 256))
                           .astype(np.float32), device="cuda")
    grad = grad_buffer(cloud.n, cloud.device)
    r.backward(cloud, num, den, dpix, grad, None, 1.0 / S)
    g = ParamGradients.from_flat(grad, cloud.n)
    torch.cuda.synchronize()

    n = cloud.n
    ref = {k: np.zeros((n, 3) if k == "d_means" else (n, 6) if k == "d_l_raw" else n)
           for k in GROUPS}
    ref_bg = np.zeros(2)
    num_h, den_h, dp_h = num.cpu().numpy(), den.cpu().numpy(), dpix.cpu().numpy()
    for s in range(S):
        on, od, acc, G = O.rasterize(*_oargs(cloud_np, scs[s]), workers=WORKERS)
        np.testing.assert_allclose(num_h[s], on, rtol=RTOL, atol=ATOL, err_msg=f"num {s}")
        np.testing.assert_allclose(den_h[s], od, rtol=RTOL, atol=ATOL, err_msg=f"den {s}")
        o = O.backward(*_oargs(cloud_np, scs[s]), on, od, dp_h[s], workers=WORKERS,
                       gathered=G)
        for k in GROUPS:
            ref[k] += o[k].astype(np.float64)
        ref_bg += [o["d_bg_intensity_raw"], o["d_bg_opacity_raw"]]
    for k in GROUPS:
        want = ref[k] / S
        np.testing.assert_allclose(getattr(g, k).cpu().numpy(), want, rtol=RTOL,
                                   atol=ATOL * np.abs(want).max(), err_msg=k)
    want_bg = ref_bg / S
    np.testing.assert_allclose([g.d_bg_intensity_raw, g.d_bg_opacity_raw], want_bg,
                               rtol=RTOL, atol=ATOL * np.abs(want_bg).max())


def _host_groups(flat, n):
    rows = flat[:12 * n].reshape(n, 12)
    return {"means": np.ascontiguousarray(rows[:, 0:3]),
            "l_raw": np.ascontiguousarray(rows[:, 3:9]),
            "intensity_raw": np.ascontiguousarray(rows[:, 9]),
            "opacity_raw": np.ascontiguousarray(rows[:, 10]),
            "bg": np.ascontiguousarray(flat[12 * n:12 * n + 2])}


def test_fused_step_bit_exact_vs_oracle_adam(c3):
    cloud_np, specs, scs = c3
    n = len(cloud_np["means"])
    cfg = ug.TrainConfig(n_gaussians=n, iterations=1000, seed=0, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4,
                         lr_general_final=0.005, heuristic_interval=100)
    # targets: GT-like images in [0, 1]
    tg = torch.as_tensor(np.random.default_rng(3).random((S, 256, 256), np.float32),
                         device="cuda")
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    eng = T.TrainEngine(cloud, cfg, specs, tg)
    # non-trivial moments (a mid-training state), a step > 1 and stats > 0
    rs = np.random.default_rng(11)
    m0 = (rs.standard_normal(12 * n + 2) * 1e-3).astype(np.float32)
    v0 = (rs.random(12 * n + 2) * 1e-4).astype(np.float32)
    eng.state.m_flat.copy_(torch.as_tensor(m0))
    eng.state.v_flat.copy_(torch.as_tensor(v0))
    eng.state.t = 4
    gs0 = (rs.random(n) * 0.1).astype(np.float32)
    gc0 = rs.integers(0, 5, n).astype(np.int32)
    eng.grad_sum.copy_(torch.as_tensor(gs0))
    eng.grad_cnt.copy_(torch.as_tensor(gc0))
    it = 37
    idx = np.arange(S)
    eng.step(idx, it)
    torch.cuda.synchronize()

    # the same batch's device gradient through ugs_backward on the input cloud
    ref_cloud = ug.GaussianCloud.from_numpy(cloud_np)
    r = ug.Renderer()
    r.bin(ref_cloud, specs, cfg.p_mass)
    num = torch.empty((S, 256, 256), device="cuda")
    den = torch.empty_like(num)
    r.forward(ref_cloud, num, den)
    assert torch.equal(num, eng.last_num) and torch.equal(den, eng.last_den)
    _, dpix, _ = fused_loss(num, den, tg, cfg.ssim_loss_weight, cfg.l2_loss)
    grad = grad_buffer(n, ref_cloud.device)
    r.backward(ref_cloud, num, den, dpix.float().contiguous(), grad, None, 1.0 / S)
    gflat = grad.cpu().numpy()
    gg = _host_groups(gflat, n)
    accs, _ = r.accepted(ref_cloud.device)
    hit = np.zeros(n, bool)
    for a in accs:
        hit[a.cpu().numpy()] = True

    params = {k: np.array(cloud_np[k], np.float32, copy=True)
              for k in ("means", "l_raw", "intensity_raw", "opacity_raw")}
    params["bg_intensity_raw"] = cloud_np["bg_intensity_raw"]
    params["bg_opacity_raw"] = cloud_np["bg_opacity_raw"]
    m, v = _host_groups(m0.copy(), n), _host_groups(v0.copy(), n)
    grads = {"d_" + k: gg[k] for k in ("means", "l_raw", "intensity_raw", "opacity_raw")}
    grads["d_bg_intensity_raw"], grads["d_bg_opacity_raw"] = float(gg["bg"][0]), float(gg["bg"][1])
    lr_g = T.general_lr(cfg, it)
    lrs = {"means": T.mean_lr(cfg, it), "l_raw": lr_g, "intensity_raw": lr_g,
           "opacity_raw": lr_g, "bg": lr_g}
    O.adam_step(params, grads, m, v, 5, lrs)

    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        got = getattr(eng.cloud, k).cpu().numpy()
        assert np.array_equal(got, params[k]), k
    mg, vg = _host_groups(eng.state.m_flat.cpu().numpy(), n), \
        _host_groups(eng.state.v_flat.cpu().numpy(), n)
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw", "bg"):
        assert np.array_equal(mg[k], m[k]), "m " + k
        assert np.array_equal(vg[k], v[k]), "v " + k
    assert eng.cloud.bg_intensity_raw == params["bg_intensity_raw"]
    assert eng.cloud.bg_opacity_raw == params["bg_opacity_raw"]
    # densify statistics: accepted by any slice of the batch -> += |d_means|
    dm = gg["means"]
    nrm = np.sqrt((dm[:, 0] * dm[:, 0] + dm[:, 1] * dm[:, 1]) + dm[:, 2] * dm[:, 2])
    want_gs = gs0.copy()
    want_gs[hit] = (gs0[hit] + nrm[hit]).astype(np.float32)
    want_gc = gc0.copy()
    want_gc[hit] += 1
    assert np.array_equal(eng.grad_sum.cpu().numpy(), want_gs)
    assert np.array_equal(eng.grad_cnt.cpu().numpy(), want_gc)


def _expected_tiles(win, acc, w, h):
    tx, ty = (w + 15) // 16, (h + 15) // 16
    lists = [[] for _ in range(tx * ty)]
    for (iu0, iu1, iv0, iv1), g in zip(win, acc):
        for y in range(iv0 >> 4, (iv1 >> 4) + 1):
            for x in range(iu0 >> 4, (iu1 >> 4) + 1):
                lists[y * tx + x].append(int(g))
    return lists


def test_radix_fallback_large_slices():
    """Slices of more than 1024 tiles take the two-pass LSD radix sort
    (ugs_api.cu); the tile lists must still be bit-exact and the render must
    match the oracle."""
    cloud_np = cases.uniform_cloud(5, 200_000, [[-48] * 3, [48] * 3], 0.5, 1.2)
    rng = np.random.default_rng(77)
    poses = [cases.random_pose(rng, 12.0) for _ in range(2)]
    W = H = 768
    sp = 96.0 / W
    specs = [ug.SliceSpec(W, H, sp, ug.ProbePose(R, t)) for R, t in poses]
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    r = ug.Renderer()
    r.set_timing(True)
    r.timings(reset=True)
    r.bin(cloud, specs, 0.95)
    num = torch.empty((2, H, W), device="cuda")
    den = torch.empty_like(num)
    r.forward(cloud, num, den)
    torch.cuda.synchronize()
    assert r.timings()["bin_ranges"][1] >= 1, "the radix fallback did not run"
    accs, wins = r.accepted(cloud.device, windows=True)
    rng_, srt = r.bins(cloud.device)
    rng_, srt = rng_.cpu().numpy(), srt.cpu().numpy()
    ntile = ((W + 15) // 16) * ((H + 15) // 16)
    for s, (R, t) in enumerate(poses):
        sc = O.slice_constants(R, t, W, H, sp, 0.95)
        acc, win, _ = O.prepare(cloud_np["means"], cloud_np["l_raw"], 0.01, sc)
        assert np.array_equal(accs[s].cpu().numpy(), acc)
        assert np.array_equal(wins[s].cpu().numpy(), win)
        lists = _expected_tiles(win, acc, W, H)
        for b, lst in enumerate(lists):
            lo, hi = rng_[s * ntile + b]
            got = srt[lo:hi].tolist() if hi > lo else []
            assert got == lst, f"slice {s} tile {b}"
        on, od, _, _ = O.rasterize(*_oargs(cloud_np, sc), workers=WORKERS)
        np.testing.assert_allclose(num[s].cpu().numpy(), on, rtol=RTOL, atol=ATOL)
        np.testing.assert_allclose(den[s].cpu().numpy(), od, rtol=RTOL, atol=ATOL)


def test_c5_forward_4m_512():
    """Config C5's largest cell: 4M Gaussians x 512x512 @96/512 mm."""
    cloud_np = cases.uniform_cloud(0, 4_000_000, [[-48] * 3, [48] * 3], 0.85, 1.05)
    rng = np.random.default_rng(55)
    R, t = cases.random_pose(rng, 12.0)
    sp = 96.0 / 512
    spec = ug.SliceSpec(512, 512, sp, ug.ProbePose(R, t))
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    buf = ug.rasterize(cloud, spec)
    sc = O.slice_constants(R, t, 512, 512, sp, 0.95)
    on, od, acc, _ = O.rasterize(*_oargs(cloud_np, sc), workers=WORKERS)
    assert np.array_equal(buf.accepted.cpu().numpy(), acc)
    np.testing.assert_allclose(buf.intensity_num.cpu().numpy(), on, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(buf.opacity_sum.cpu().numpy(), od, rtol=RTOL, atol=ATOL)
    # the batched render-only path gives the same pixels
    pix = ug.render_slices(cloud, [spec, spec])
    assert torch.equal(pix[0], buf.pixels) and torch.equal(pix[1], buf.pixels)


def test_async_bin_overflow_reissue():
    """Sync-free binning (ugs_bin_async): a batch that overflows the plan's
    capacities turns its forward / backward / Adam into device-side no-ops,
    ugs_plan_poll reports it and the engine re-issues the step -- the
    trajectory is bitwise the one of synchronous binning."""
    cloud_np = cases.uniform_cloud(3, 200_000, [[-48] * 3, [48] * 3], 0.85, 1.05)
    rng = np.random.default_rng(8)
    poses = [cases.random_pose(rng, 12.0) for _ in range(8)]
    specs = [ug.SliceSpec(256, 256, 0.375, ug.ProbePose(R, t)) for R, t in poses]
    tg = torch.as_tensor(np.random.default_rng(1).random((8, 256, 256), np.float32),
                         device="cuda")
    cfg = ug.TrainConfig(n_gaussians=200_000, iterations=100, l_init_low=0.85,
                         l_init_high=1.05, lr_means_start=0.016, lr_means_final=1.6e-4)
    runs = []
    for async_bin in (True, False):
        eng = T.TrainEngine(ug.GaussianCloud.from_numpy(cloud_np), cfg, specs, tg)
        eng.async_bin = async_bin
        # size the plan on a tiny batch so the next batches overflow it
        tiny = ug.SliceSpec(16, 16, 0.375, ug.ProbePose(np.eye(3), np.array([0, 0, 47.0])))
        eng.renderer.bin(eng.cloud, [tiny], cfg.p_mass)
        losses = []
        for it, idx in enumerate(([0, 1, 2, 3], [4, 5, 6, 7], [0, 2, 4, 6]), start=1):
            losses.append(eng.step(idx, it, check_finite=False))
        eng.settle()
        losses = [float(x) for x in losses]
        runs.append((eng, losses))
    (ea, la), (eb, lb) = runs
    assert ea.reissued >= 1
    assert la == lb
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw", "bg_raw"):
        assert torch.equal(getattr(ea.cloud, k), getattr(eb.cloud, k)), k
    assert torch.equal(ea.state.m_flat, eb.state.m_flat)
    assert torch.equal(ea.grad_sum, eb.grad_sum) and torch.equal(ea.grad_cnt, eb.grad_cnt)
    assert ea.pairs_total == eb.pairs_total


def test_render_mode_and_overflow_retry():
    """ugs_render writes clip(num/den) bitwise equal to the two-output
    forward; render_slices re-issues a chunk that overflowed a small plan."""
    cloud_np = cases.uniform_cloud(9, 300_000, [[-48] * 3, [48] * 3], 0.85, 1.05)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    rng = np.random.default_rng(21)
    specs = [ug.SliceSpec(128, 128, 0.75, ug.ProbePose(*cases.random_pose(rng, 12.0)))
             for _ in range(24)]
    r = ug.Renderer()
    # size the plan on a tiny batch: the 24-slice chunk must overflow it
    r.bin(cloud, [ug.SliceSpec(16, 16, 0.75, ug.ProbePose(np.eye(3), np.array([0, 0, 47.0])))])
    pix = ug.render_slices(cloud, specs, renderer=r)
    r2 = ug.Renderer()
    r2.bin(cloud, specs, 0.95)
    num = torch.empty((24, 128, 128), device="cuda")
    den = torch.empty_like(num)
    r2.forward(cloud, num, den)
    assert torch.equal(pix, torch.clamp(num / den, 0.0, 1.0))
    # sized now: a second call is sync-free and identical
    assert torch.equal(ug.render_slices(cloud, specs, renderer=r), pix)


def test_render_batch_graph_replay():
    """ugs_render_batch replays its captured kernel chain: repeated batches
    (new poses, same shape) equal the plain bin + render bitwise, and a new
    cloud, a new batch shape or a plan that grew re-capture correctly."""
    rng = np.random.default_rng(33)
    clouds = [ug.GaussianCloud.from_numpy(
        cases.uniform_cloud(seed, 150_000, [[-48] * 3, [48] * 3], 0.85, 1.05))
        for seed in (4, 5)]

    def batch(n, hw):
        return [ug.SliceSpec(hw, hw, 96.0 / hw, ug.ProbePose(*cases.random_pose(rng, 12.0)))
                for _ in range(n)]

    def plain(cloud, specs):
        r2 = ug.Renderer()
        r2.bin(cloud, specs, 0.95)
        out = torch.empty((len(specs), specs[0].height, specs[0].width), device="cuda")
        r2.render(cloud, out)
        return out

    r = ug.Renderer()
    r.bin(clouds[0], batch(16, 128))          # sizes the plan
    for cloud, n, hw in ((clouds[0], 16, 128), (clouds[0], 16, 128), (clouds[0], 16, 128),
                         (clouds[1], 16, 128), (clouds[1], 8, 128), (clouds[1], 8, 96),
                         (clouds[0], 64, 128), (clouds[0], 64, 128)):
        specs = batch(n, hw)
        out = torch.empty((n, hw, hw), device="cuda")
        r.render_batch(cloud, specs, out)
        if r.poll():                           # the 64-slice batch outgrows the plan
            r.bin(cloud, specs)
            r.render(cloud, out)
        assert torch.equal(out, plain(cloud, specs)), (n, hw)


def test_huge_footprints_recursive_scan():
    """Gaussians whose footprints cover whole slices (the reference recipe at
    batch 1 grows them): a 64-slice render_slices batch of ~330M tile
    instances takes the LSD radix path with a sort table beyond one scan
    block (the recursive exclusive scan) and must equal the per-slice
    renders bitwise."""
    cloud_np = cases.uniform_cloud(3, 20_000, [[-40] * 3, [40] * 3], 0.05, 0.1)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    rng = np.random.default_rng(5)
    specs = [ug.SliceSpec(256, 256, 0.375, ug.ProbePose(*cases.random_pose(rng, 4.0)))
             for _ in range(64)]
    r = ug.Renderer()
    pix = ug.render_slices(cloud, specs, renderer=r)
    assert int(np.sum(r.k)) > (1 << 24) * 16, "the batch must need a two-level scan"
    for s in (0, 37, 63):
        one = ug.render_slice(cloud, specs[s]).pixels
        assert np.array_equal(pix[s].cpu().numpy(), one)
