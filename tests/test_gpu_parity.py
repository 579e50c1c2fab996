"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors.  Bit-exact for the accepted set, windows and
tile lists; rtol 1e-4 / atol 1e-5 for renders (north_star tolerance);
per-group rtol 1e-4 / atol 1e-5 * max|group| for gradients."""

import numpy as np
import pytest

import cases
from conftest import load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2505_05643_b200 as ug  # noqa: E402

RTOL, ATOL = 1e-4, 1e-5


def spec_of(R, t, w, h, s):
    return ug.SliceSpec(w, h, s, ug.ProbePose(R, t))


def expected_tiles(win, acc, w, h):
    """Per-16x16-tile ascending Gaussian lists from (oracle) windows."""
    tx, ty = (w + 15) // 16, (h + 15) // 16
    lists = [[] for _ in range(tx * ty)]
    for (iu0, iu1, iv0, iv1), g in zip(win, acc):
        for y in range(iv0 >> 4, (iv1 >> 4) + 1):
            for x in range(iu0 >> 4, (iu1 >> 4) + 1):
                lists[y * tx + x].append(int(g))
    return lists


def oracle_args(cloud, sc):
    return (cloud["means"], cloud["l_raw"], cloud["intensity_raw"],
            cloud["opacity_raw"], cloud["bg_intensity_raw"],
            cloud["bg_opacity_raw"], cloud["beta"], sc)


@pytest.fixture(scope="module")
def prep():
    return load_golden("prepare.npz")


@pytest.fixture(scope="module")
def rend():
    return load_golden("render.npz")


@pytest.mark.parametrize("case", cases.PREPARE_CASES, ids=lambda c: c[0])
def test_prepare_and_tiles_bit_exact(case, prep):
    cloud_np, R, t, w, h, s = cases.prepare_case(case)
    name = case[0]
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    r = ug.Renderer()
    r.bin(cloud, [spec_of(R, t, w, h, s)], 0.95)
    accs, wins = r.accepted(cloud.device, windows=True)
    acc = accs[0].cpu().numpy()
    win = wins[0].cpu().numpy()
    assert np.array_equal(acc, prep[f"{name}/accepted"])
    assert np.array_equal(win, prep[f"{name}/windows"])
    rng_, srt = r.bins(cloud.device)
    rng_, srt = rng_.cpu().numpy(), srt.cpu().numpy()
    lists = expected_tiles(win, acc, w, h)
    assert len(rng_) == len(lists)
    for b, lst in enumerate(lists):
        got = srt[rng_[b, 0]:rng_[b, 1]].tolist() if rng_[b, 1] > rng_[b, 0] else []
        assert got == lst, f"tile {b}"


def test_batch_binning_matches_single(prep):
    """S slices binned together == each slice binned alone (bit-exact)."""
    cloud_np = cases.uniform_cloud(7, 30000, [[-40] * 3, [40] * 3], 0.5, 1.5)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    rng = np.random.default_rng(3)
    specs = [spec_of(*cases.random_pose(rng, 10.0), 96, 96, 0.5) for _ in range(7)]
    r = ug.Renderer()
    r.bin(cloud, specs, 0.95)
    accs, wins = r.accepted(cloud.device, windows=True)
    num = torch.empty((7, 96, 96), device="cuda")
    den = torch.empty_like(num)
    r.forward(cloud, num, den)
    for s, spec in enumerate(specs):
        sc = O.slice_constants(spec.pose.rotation, spec.pose.translation, 96, 96, 0.5, 0.95)
        a, wv, _ = O.prepare(cloud_np["means"], cloud_np["l_raw"], 0.01, sc)
        assert np.array_equal(accs[s].cpu().numpy(), a)
        assert np.array_equal(wins[s].cpu().numpy(), wv)
        n1 = ug.rasterize(cloud, spec).intensity_num
        assert torch.equal(n1, num[s])


@pytest.mark.parametrize("case", cases.RENDER_CASES, ids=lambda c: c[0])
def test_render_backward_vs_reference(case, rend):
    cloud_np, R, t, w, h, s, p, dpix = cases.render_case(case)
    name = case[0]
    spec = spec_of(R, t, w, h, s)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    buf = ug.rasterize(cloud, spec, p=p)
    assert np.array_equal(buf.accepted.cpu().numpy(), rend[f"{name}/accepted"])
    np.testing.assert_allclose(buf.intensity_num.cpu().numpy(), rend[f"{name}/num"],
                               rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(buf.opacity_sum.cpu().numpy(), rend[f"{name}/den"],
                               rtol=RTOL, atol=ATOL)
    g = ug.backward(cloud, spec, buf, dpix)
    for k in ("d_means", "d_l_raw", "d_intensity_raw", "d_opacity_raw"):
        ref = rend[f"{name}/{k}"]
        np.testing.assert_allclose(getattr(g, k).cpu().numpy(), ref, rtol=RTOL,
                                   atol=ATOL * np.abs(ref).max(), err_msg=k)
    ref_bg = rend[f"{name}/d_bg"]    # the background group (2 entries)
    np.testing.assert_allclose([g.d_bg_intensity_raw, g.d_bg_opacity_raw],
                               ref_bg, rtol=RTOL, atol=ATOL * np.abs(ref_bg).max())
    if f"{name}/loss" in rend:
        pred = buf.intensity_num / buf.opacity_sum
        lv, lg = ug.loss(pred, rend[f"{name}/target"], 0.2)
        assert lv == pytest.approx(float(rend[f"{name}/loss"]), rel=1e-4, abs=1e-6)
        s_gpu = ug.ssim(torch.clamp(pred, 0, 1), rend[f"{name}/target"])
        assert round(s_gpu, 4) == round(float(rend[f"{name}/ssim"]), 4)


def test_kats(rend):
    logit = lambda q: float(np.log(q / (1 - q)))
    empty = ug.GaussianCloud(np.zeros((0, 3)), np.zeros((0, 6)), np.zeros(0),
                             np.zeros(0), logit(0.37), -4.0)
    img = ug.render_slice(empty, ug.SliceSpec(8, 8, 1.0))
    assert np.allclose(img.pixels, 0.37, atol=1e-6)
    ld = np.sqrt(1.0 / 2.0 - 0.01)
    single = ug.GaussianCloud(np.zeros((1, 3)), np.array([[ld] * 3 + [0, 0, 0]]),
                              np.array([logit(1 - 1e-7)]), np.array([logit(0.8)]),
                              -30.0, -4.0)
    img = ug.render_slice(single, ug.SliceSpec(17, 17, 1.0), p=0.9999)
    assert img.pixels[8, 8] == pytest.approx(0.8 / 0.818, abs=1e-4)
    np.testing.assert_allclose(img.pixels, rend["kat_single/pixels"], rtol=RTOL, atol=ATOL)
    # the batched render path (ugs_render_batch) on the same KATs: an empty
    # cloud (plain launches) and, on a sized plan, the graph replay -- twice,
    # with per-stage timing toggled in between (graph path vs timed path)
    r = ug.Renderer()
    px = ug.render_slices(empty, [ug.SliceSpec(8, 8, 1.0)] * 3, renderer=r)
    assert torch.allclose(px, torch.full_like(px, 0.37), atol=1e-6)
    r2 = ug.Renderer()
    specs = [ug.SliceSpec(17, 17, 1.0)] * 2
    a = ug.render_slices(single, specs, 0.9999, renderer=r2)    # sizes the plan
    b = ug.render_slices(single, specs, 0.9999, renderer=r2)    # graph capture
    r2.set_timing(True)
    c = ug.render_slices(single, specs, 0.9999, renderer=r2)    # timed: plain launches
    r2.set_timing(False)
    d = ug.render_slices(single, specs, 0.9999, renderer=r2)    # graph replay
    for x in (a, b, c, d):
        np.testing.assert_array_equal(x[0].cpu().numpy(), img.pixels)


def test_zero_upstream_and_culled(rng):
    cloud_np = cases.random_cloud(rng, 100, extent=30.0)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    spec = ug.SliceSpec(12, 12, 1.0)
    buf = ug.rasterize(cloud, spec)
    g0 = ug.backward(cloud, spec, buf, np.zeros((12, 12), np.float32))
    assert not g0.d_means.any() and not g0.d_l_raw.any()
    assert g0.d_bg_intensity_raw == 0.0
    g1 = ug.backward(cloud, spec, buf, np.ones((12, 12), np.float32))
    rejected = np.setdiff1d(np.arange(cloud.n), buf.accepted.cpu().numpy())
    assert len(rejected) > 0
    assert not g1.d_means.cpu().numpy()[rejected].any()
    assert not g1.d_opacity_raw.cpu().numpy()[rejected].any()
    with pytest.raises(ug.InvalidParameterError):
        ug.backward(cloud, spec, buf, np.zeros((4, 4), np.float32))


def test_full_size_c3_parity():
    """BASELINE config C3: 1M Gaussians, 256x256 @0.375 mm, random pose --
    accepted set and windows bit-exact; render and gradients vs oracle."""
    cloud_np = cases.uniform_cloud(0, 1_000_000, [[-48] * 3, [48] * 3], 0.85, 1.05)
    rng = np.random.default_rng(5)
    R, t = cases.random_pose(rng, 12.0)
    spec = spec_of(R, t, 256, 256, 0.375)
    sc = O.slice_constants(R, t, 256, 256, 0.375, 0.95)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    buf = ug.rasterize(cloud, spec)
    num, den, acc, G = O.rasterize(*oracle_args(cloud_np, sc), workers=8)
    assert np.array_equal(buf.accepted.cpu().numpy(), acc)
    np.testing.assert_allclose(buf.intensity_num.cpu().numpy(), num, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(buf.opacity_sum.cpu().numpy(), den, rtol=RTOL, atol=ATOL)
    dpix = np.random.default_rng(1).standard_normal((256, 256)).astype(np.float32)
    g = ug.backward(cloud, spec, buf, dpix)
    ref = O.backward(*oracle_args(cloud_np, sc), num, den, dpix, workers=8, gathered=G)
    for k in ("d_means", "d_l_raw", "d_intensity_raw", "d_opacity_raw"):
        np.testing.assert_allclose(getattr(g, k).cpu().numpy(), ref[k], rtol=RTOL,
                                   atol=ATOL * np.abs(ref[k]).max(), err_msg=k)


def test_forward_deterministic():
    cloud_np = cases.uniform_cloud(1, 200_000, [[-48] * 3, [48] * 3], 0.85, 1.05)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    spec = spec_of(*cases.random_pose(np.random.default_rng(9), 12.0), 256, 256, 0.375)
    b1 = ug.rasterize(cloud, spec)
    n1 = b1.intensity_num.clone()
    dp = np.random.default_rng(2).standard_normal((256, 256)).astype(np.float32)
    g1 = ug.backward(cloud, spec, b1, dp)
    b2 = ug.rasterize(cloud, spec)
    g2 = ug.backward(cloud, spec, b2, dp)
    assert torch.equal(n1, b2.intensity_num)
    assert torch.equal(g1.d_means, g2.d_means) and torch.equal(g1.d_l_raw, g2.d_l_raw)


def test_adam_bit_exact():
    z = load_golden("adam_densify.npz")
    cloud = ug.GaussianCloud(z["adam/init/means"], z["adam/init/l_raw"],
                             z["adam/init/intensity_raw"], z["adam/init/opacity_raw"],
                             float(z["adam/init/bg"][0]), float(z["adam/init/bg"][1]))
    st = ug.AdamState.for_cloud(cloud)
    lrs = {"means": 0.016, "l_raw": 0.05, "intensity_raw": 0.05,
           "opacity_raw": 0.05, "bg": 0.05}
    for step in range(5):
        d = z[f"adam/step{step}/d_bg"]
        g = ug.ParamGradients(*(torch.as_tensor(z[f"adam/step{step}/d_{k}"])
                                for k in ("means", "l_raw", "intensity_raw", "opacity_raw")),
                              float(d[0]), float(d[1]))
        ug.adam_step(st, cloud, g, lrs)
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        assert np.array_equal(getattr(cloud, k).cpu().numpy(), z[f"adam/final/{k}"]), k
        assert np.array_equal(st.m[k].cpu().numpy(), z[f"adam/final/m_{k}"]), k
        assert np.array_equal(st.v[k].cpu().numpy(), z[f"adam/final/v_{k}"]), k
    assert [cloud.bg_intensity_raw, cloud.bg_opacity_raw] == list(z["adam/final/bg"])


def test_densify_matches_reference():
    z = load_golden("adam_densify.npz")
    cloud = ug.GaussianCloud(z["densify/init/means"], z["densify/init/l_raw"],
                             z["densify/init/intensity_raw"],
                             z["densify/init/opacity_raw"], 0.0, -4.0)
    st = ug.AdamState.for_cloud(cloud)
    st.m_flat[:] = 0.5
    st.v_flat[:] = 0.25
    out, st2 = ug.densify_prune_resample(cloud, z["densify/avg"], st, ug.TrainConfig(),
                                         np.random.default_rng(99), 60.0, 0.8, 48)
    for k in ("l_raw", "intensity_raw", "opacity_raw"):
        assert np.array_equal(getattr(out, k).cpu().numpy(), z[f"densify/final/{k}"]), k
    np.testing.assert_allclose(out.means.cpu().numpy(), z["densify/final/means"],
                               rtol=1e-6, atol=1e-6)
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        assert np.array_equal(st2.m[k].cpu().numpy(), z[f"densify/final/m_{k}"]), k


def _train_golden():
    z = load_golden("train.npz")
    slices = [ug.SliceImage(z["slices"][i], float(z["spacing"]),
                            ug.ProbePose(z["rot"][i], z["trans"][i]))
              for i in range(len(z["slices"]))]
    return z, ug.SliceDataset(slices)


def test_train_short_run_tracks_reference():
    z, ds = _train_golden()
    cfg = ug.TrainConfig(n_gaussians=300, iterations=40, seed=7, heuristic_interval=20,
                         eval_interval=10, workers=1)
    cloud, log = ug.train(ds, cfg)
    assert [e["iter"] for e in log] == list(z["iters"])
    np.testing.assert_allclose([e["loss"] for e in log], z["loss"], rtol=2e-3)
    assert cloud.n == len(z["final/means"])
    np.testing.assert_allclose(cloud.means.cpu().numpy(), z["final/means"], atol=2e-3)


def test_train_bitwise_deterministic():
    _, ds = _train_golden()
    cfg = ug.TrainConfig(n_gaussians=300, iterations=60, seed=7, heuristic_interval=20)
    a, _ = ug.train(ds, cfg)
    b, _ = ug.train(ds, cfg)
    assert torch.equal(a.means, b.means) and torch.equal(a.l_raw, b.l_raw)
    assert a.bg_opacity_raw == b.bg_opacity_raw


def test_autograd_matches_backward():
    cloud_np, R, t, w, h, s, p, dpix = cases.render_case(cases.RENDER_CASES[3])
    spec = spec_of(R, t, w, h, s)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    params = [x.clone().requires_grad_(True) for x in
              (cloud.means, cloud.l_raw, cloud.intensity_raw, cloud.opacity_raw)]
    bg = cloud.bg_raw.clone().requires_grad_(True)
    pred = ug.rasterize_autograd(*params, bg, [spec], p=p)
    (pred[0] * torch.as_tensor(dpix, device="cuda")).sum().backward()
    g = ug.backward(cloud, spec, ug.rasterize(cloud, spec, p=p), dpix)
    assert torch.allclose(params[0].grad, g.d_means)
    assert torch.allclose(params[1].grad, g.d_l_raw)


@pytest.mark.parametrize("case", cases.RENDER_CASES, ids=lambda c: c[0])
def test_ordered_forward(case, rend):
    """Strict ascending-order accumulation (the reference's workers=1 order)
    also meets the tolerance, and agrees with the default mode."""
    cloud_np, R, t, w, h, s, p, dpix = cases.render_case(case)
    name = case[0]
    spec = spec_of(R, t, w, h, s)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    r = ug.Renderer()
    r.set_ordered(True)
    b1 = ug.rasterize(cloud, spec, p=p, renderer=r)
    np.testing.assert_allclose(b1.intensity_num.cpu().numpy(), rend[f"{name}/num"],
                               rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(b1.opacity_sum.cpu().numpy(), rend[f"{name}/den"],
                               rtol=RTOL, atol=ATOL)
    b0 = ug.rasterize(cloud, spec, p=p)
    np.testing.assert_allclose(b0.intensity_num.cpu().numpy(),
                               b1.intensity_num.cpu().numpy(), rtol=1e-5, atol=1e-6)


def _needle_cloud(rng, n, R, t, beta=1e-6):
    """Needles (sigma 60 mm x 0.4 x 0.4) whose long axis lies within ~1e-4 rad
    of the slice plane, 1-3 mm off it: their in-plane conditional centre is
    far outside the image while the ridge crosses it."""
    means, l_raw = [], []
    for _ in range(n):
        phi = rng.uniform(0, np.pi)
        eps = rng.uniform(-1e-4, 1e-4)
        d_local = np.array([np.cos(phi) * np.cos(eps), np.sin(phi) * np.cos(eps), np.sin(eps)])
        d = R @ d_local
        q, _ = np.linalg.qr(np.column_stack([d, rng.standard_normal((3, 2))]))
        sig = np.array([60.0, rng.uniform(0.3, 0.6), rng.uniform(0.3, 0.6)])
        prec = q @ np.diag(1.0 / sig ** 2) @ q.T
        # lower-triangular L with L L^T = prec: reverse-order Cholesky
        J = np.eye(3)[::-1]
        C = np.linalg.cholesky(J @ np.linalg.inv(prec) @ J)
        L = np.linalg.inv(J @ C @ J).T
        L = L * np.sign(np.diag(L))[None, :]
        assert np.allclose(L @ L.T, prec, rtol=1e-8, atol=1e-10)
        ld = np.sqrt(np.diag(L) - beta)
        l_raw.append([ld[0], ld[1], ld[2], L[1, 0], L[2, 0], L[2, 1]])
        off = R @ np.array([rng.uniform(-15, 15), rng.uniform(-15, 15), rng.uniform(-3, 3)])
        means.append(t + off)
    return dict(means=np.asarray(means, np.float32), l_raw=np.asarray(l_raw, np.float32),
                intensity_raw=rng.normal(0, 1, n).astype(np.float32),
                opacity_raw=rng.normal(0, 1, n).astype(np.float32),
                bg_intensity_raw=0.3, bg_opacity_raw=-4.0, beta=beta)


@pytest.mark.parametrize("kind", ["broad_lraw", "needles"])
def test_degenerate_clouds_vs_oracle(kind):
    """Training-state stress: l_raw components crossing zero (huge, strongly
    anisotropic footprints) and near-in-plane needles (conditional centre far
    outside the image).  Renders stay finite and within tolerance."""
    rng = np.random.default_rng(17)
    R, t = cases.random_pose(rng, 5.0)
    if kind == "broad_lraw":
        cloud_np = cases.uniform_cloud(3, 1500, [[-20] * 3, [20] * 3], -3.0, 3.0)
    else:
        cloud_np = _needle_cloud(rng, 300, R, t)
    w = h = 128
    spec = spec_of(R, t, w, h, 0.375)
    sc = O.slice_constants(R, t, w, h, 0.375, 0.95)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    buf = ug.rasterize(cloud, spec)
    num, den, acc, G = O.rasterize(*oracle_args(cloud_np, sc), workers=8)
    assert np.array_equal(buf.accepted.cpu().numpy(), acc)
    gn, gd = buf.intensity_num.cpu().numpy(), buf.opacity_sum.cpu().numpy()
    assert np.isfinite(gn).all() and np.isfinite(gd).all()
    np.testing.assert_allclose(gn, num, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(gd, den, rtol=RTOL, atol=ATOL)
    dpix = np.random.default_rng(4).standard_normal((h, w)).astype(np.float32)
    g = ug.backward(cloud, spec, buf, dpix)
    ref = O.backward(*oracle_args(cloud_np, sc), num, den, dpix, workers=8, gathered=G)
    for k in ("d_means", "d_l_raw", "d_intensity_raw", "d_opacity_raw"):
        got = getattr(g, k).cpu().numpy()
        assert np.isfinite(got).all(), k
        np.testing.assert_allclose(got, ref[k], rtol=RTOL,
                                   atol=ATOL * np.abs(ref[k]).max(), err_msg=k)


@pytest.mark.parametrize("kind", ["shells", "blobs"])
def test_gpu_sampler_matches_reference(kind):
    """sample_slices (GPU trilinear ground truth) vs the reference's
    sample_slice (ref volume.py:223-263) on its own fixtures."""
    z = load_golden("io.npz")
    v = ug.make_phantom(kind, 24, 0.6, seed=1)
    specs = [ug.SliceSpec(20, 17, 0.45, ug.ProbePose(z[f"{kind}/slice{i}/R"],
                                                     z[f"{kind}/slice{i}/t"]))
             for i in range(3)]
    got = ug.sample_slices(v, specs).cpu().numpy()
    for i in range(3):
        np.testing.assert_allclose(got[i], z[f"{kind}/slice{i}/pixels"], rtol=1e-5, atol=1e-6)


def test_render_slices_matches_render_slice():
    """The batched render-only path (C5, the /slice consumer) equals the
    single-slice API on every slice."""
    cloud_np = cases.uniform_cloud(4, 20000, [[-20] * 3, [20] * 3], 0.85, 1.05)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    specs = [spec_of(*cases.random_pose(np.random.default_rng(40 + i), 5.0), 64, 64, 0.5)
             for i in range(5)]
    batch = ug.render_slices(cloud, specs).cpu().numpy()
    for i, sp in enumerate(specs):
        one = ug.render_slice(cloud, sp).pixels
        np.testing.assert_allclose(batch[i], one, rtol=0, atol=0)


def test_sparse_acceptance_vs_oracle():
    """Small Gaussians, few accepted per 32-Gaussian warp: a build warp's 32
    records span more than 32 Gaussian warps, so build_records takes its
    per-lane search path (the dense configs use the register search).
    Accepted set bit-exact; render and gradients vs the oracle."""
    cloud_np = cases.uniform_cloud(11, 300_000, [[-40] * 3, [40] * 3], 2.0, 3.0)
    rng = np.random.default_rng(12)
    R, t = cases.random_pose(rng, 8.0)
    spec = spec_of(R, t, 128, 128, 0.6)
    sc = O.slice_constants(R, t, 128, 128, 0.6, 0.95)
    cloud = ug.GaussianCloud.from_numpy(cloud_np)
    buf = ug.rasterize(cloud, spec)
    num, den, acc, G = O.rasterize(*oracle_args(cloud_np, sc), workers=8)
    assert 0 < len(acc) < 300_000 // 64        # < one record per two warps
    assert np.array_equal(buf.accepted.cpu().numpy(), acc)
    np.testing.assert_allclose(buf.intensity_num.cpu().numpy(), num, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(buf.opacity_sum.cpu().numpy(), den, rtol=RTOL, atol=ATOL)
    dpix = np.random.default_rng(3).standard_normal((128, 128)).astype(np.float32)
    g = ug.backward(cloud, spec, buf, dpix)
    ref = O.backward(*oracle_args(cloud_np, sc), num, den, dpix, workers=8, gathered=G)
    for k in ("d_means", "d_l_raw", "d_intensity_raw", "d_opacity_raw"):
        np.testing.assert_allclose(getattr(g, k).cpu().numpy(), ref[k], rtol=RTOL,
                                   atol=ATOL * np.abs(ref[k]).max(), err_msg=k)


def test_fused_step_misaligned_parameters_bitwise():
    """The fused backward + Adam moves parameter rows as float4 streams when
    the arrays are 16-byte aligned and falls back to per-Gaussian rows
    otherwise: both give bitwise the same training trajectory."""
    from paper_2505_05643_b200.trainer import TrainEngine
    cloud_np = cases.uniform_cloud(13, 5000, [[-20] * 3, [20] * 3], 0.85, 1.05)
    rng = np.random.default_rng(14)
    specs = [spec_of(*cases.random_pose(rng, 6.0), 64, 64, 0.5) for _ in range(6)]
    targets = torch.rand((6, 64, 64), generator=torch.Generator().manual_seed(1)).cuda()
    cfg = ug.TrainConfig(n_gaussians=5000, iterations=100, seed=0, batch=3,
                         heuristic_interval=0)

    def run(misaligned):
        n = 5000
        arrs = {}
        for k, w in (("means", 3), ("l_raw", 6)):
            base = torch.empty(n * w + 1, device="cuda")
            view = base[1:] if misaligned else base[:-1]
            view.copy_(torch.as_tensor(cloud_np[k]).reshape(-1))
            arrs[k] = view.view(n, w)
        cloud = ug.GaussianCloud(arrs["means"], arrs["l_raw"], cloud_np["intensity_raw"],
                                 cloud_np["opacity_raw"], device="cuda")
        assert (cloud.means.data_ptr() % 16 != 0) == misaligned
        eng = TrainEngine(cloud, cfg, specs, targets)
        for it in range(1, 5):
            eng.step([(2 * it) % 6, (2 * it + 1) % 6, (2 * it + 3) % 6], it)
        return [getattr(eng.cloud, k).cpu().numpy() for k in
                ("means", "l_raw", "intensity_raw", "opacity_raw")]

    for a, b in zip(run(False), run(True)):
        assert np.array_equal(a, b)


def test_resume_reproduces_uninterrupted_run(tmp_path):
    """Training-state extension: a run resumed from its iteration-7 state
    (Adam moments, densify statistics and threshold, RNG, slice order) ends
    bitwise where the uninterrupted run ends, densify included."""
    from conftest import load_golden as _lg
    z = _lg("train.npz")
    ds = ug.SliceDataset([ug.SliceImage(z["slices"][i], float(z["spacing"]),
                                        ug.ProbePose(z["rot"][i], z["trans"][i]))
                          for i in range(len(z["slices"]))])
    cfg = ug.TrainConfig(n_gaussians=400, iterations=12, seed=3, batch=2,
                         heuristic_interval=5, eval_interval=12)
    full, _ = ug.train(ds, cfg, device="cuda:0",
                       state_path=str(tmp_path / "s{iter}.ugsc"), state_interval=7)
    assert (tmp_path / "s7.ugsc.adam").exists() and (tmp_path / "s12.ugsc.adam").exists()
    resumed, _ = ug.train(ds, cfg, device="cuda:0", resume_from=str(tmp_path / "s7.ugsc"))
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        assert torch.equal(getattr(full, k), getattr(resumed, k)), k
    assert (full.bg_intensity_raw, full.bg_opacity_raw) == \
        (resumed.bg_intensity_raw, resumed.bg_opacity_raw)


def test_grad_check_small_cloud():
    """ref gradients.py grad_check protocol on the float32 CUDA path: every
    group agrees with central finite differences (float64 loss) to 2e-2
    relative in its worst entry (measured: means 1.1e-2, l_raw 1.4e-3, the
    rest <= 5e-4; the reference's float64 path reaches 1e-5)."""
    rng = np.random.default_rng(31)
    c = cases.random_cloud(rng, 12, extent=3.0)
    cloud = ug.GaussianCloud.from_numpy(c)
    R, t = cases.random_pose(rng, 1.0)
    spec = spec_of(R, t, 24, 20, 0.4)
    rep = ug.grad_check(cloud, spec)
    assert set(rep) == {"means", "l_raw", "intensity_raw", "opacity_raw",
                        "bg_intensity_raw", "bg_opacity_raw"}
    for k, v in rep.items():
        assert v < 2e-2, (k, v)


def test_float64_cloud_warns_and_matches_float32():
    """A float64 cloud (the reference would render it in float64) is
    converted to the float32 path with a one-time UserWarning; the render
    equals the float32 cloud's bitwise."""
    import warnings
    from paper_2505_05643_b200 import model as M
    cloud_np, R, t, w, h, s, p, _ = cases.render_case(cases.RENDER_CASES[2])
    spec = ug.SliceSpec(w, h, s, ug.ProbePose(R, t))
    c64 = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) else v)
           for k, v in cloud_np.items()}
    M._F64_WARNED = False
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        a = ug.GaussianCloud.from_numpy(c64)
    assert any("float64" in str(x.message) for x in rec)
    b = ug.GaussianCloud.from_numpy(cloud_np)
    pa = ug.render_slice(a, spec, p=p).pixels
    pb = ug.render_slice(b, spec, p=p).pixels
    assert np.array_equal(pa, pb)
