"""Pin the oracle against vectors produced by the reference itself.

These run on CPU (no GPU) and gate every GPU parity claim: the GPU path is
compared with the oracle, and the oracle is compared here with the reference
(tests/golden/make_golden.py).
"""

import numpy as np
import pytest

import cases
from conftest import load_golden
from oracle import oracle as O


@pytest.fixture(scope="module")
def prep():
    return load_golden("prepare.npz")


@pytest.fixture(scope="module")
def rend():
    return load_golden("render.npz")


@pytest.mark.parametrize("case", cases.PREPARE_CASES, ids=lambda c: c[0])
def test_prepare_bit_exact(case, prep):
    cloud, R, t, w, h, s = cases.prepare_case(case)
    name = case[0]
    assert cases.input_checksum(cloud["means"], cloud["l_raw"]) == \
        prep[f"{name}/checksum"]
    sc = O.slice_constants(R, t, w, h, s, 0.95)
    for k in ("rw", "tw", "origin", "du", "dv"):
        assert np.array_equal(sc[k], prep[f"{name}/{k}"]), k
    assert np.sqrt(prep[f"{name}/cut"]) == sc["sqrt_cut"]
    acc, win, _ = O.prepare(cloud["means"], cloud["l_raw"], cloud["beta"], sc)
    assert np.array_equal(acc, prep[f"{name}/accepted"])
    assert np.array_equal(win, prep[f"{name}/windows"])


@pytest.mark.parametrize("case", cases.RENDER_CASES, ids=lambda c: c[0])
def test_render_backward_loss(case, rend):
    cloud, R, t, w, h, s, p, dpix = cases.render_case(case)
    name = case[0]
    sc = O.slice_constants(R, t, w, h, s, p)
    args = (cloud["means"], cloud["l_raw"], cloud["intensity_raw"],
            cloud["opacity_raw"], cloud["bg_intensity_raw"],
            cloud["bg_opacity_raw"], cloud["beta"], sc)
    num, den, acc, G = O.rasterize(*args)
    assert np.array_equal(acc, rend[f"{name}/accepted"])
    # numba (fastmath=False) and the C restatement share types and op order
    assert np.array_equal(num, rend[f"{name}/num"])
    assert np.array_equal(den, rend[f"{name}/den"])
    g = O.backward(*args, num, den, dpix, gathered=G)
    for k in ("d_means", "d_l_raw", "d_intensity_raw", "d_opacity_raw"):
        ref = rend[f"{name}/{k}"]
        assert np.array_equal(g[k], ref), k
    np.testing.assert_allclose([g["d_bg_intensity_raw"], g["d_bg_opacity_raw"]],
                               rend[f"{name}/d_bg"], rtol=1e-5)
    if f"{name}/loss" in rend:
        pred = num / den
        lv, lg = O.loss(pred, rend[f"{name}/target"], 0.2)
        assert lv == pytest.approx(float(rend[f"{name}/loss"]), abs=1e-12)
        np.testing.assert_allclose(lg, rend[f"{name}/dloss"], rtol=1e-9,
                                   atol=1e-15)
        assert round(O.ssim(np.clip(pred, 0, 1), rend[f"{name}/target"]), 4) \
            == round(float(rend[f"{name}/ssim"]), 4)


def test_workers_match_sequential():
    cloud, R, t, w, h, s, p, dpix = cases.render_case(cases.RENDER_CASES[2])
    sc = O.slice_constants(R, t, w, h, s, p)
    args = (cloud["means"], cloud["l_raw"], cloud["intensity_raw"],
            cloud["opacity_raw"], cloud["bg_intensity_raw"],
            cloud["bg_opacity_raw"], cloud["beta"], sc)
    n1, d1, _, _ = O.rasterize(*args, workers=1)
    n4, d4, _, _ = O.rasterize(*args, workers=4)
    assert np.abs(n1 / d1 - n4 / d4).max() <= 1e-5


def test_kats(rend):
    assert np.allclose(rend["kat_empty/pixels"], 0.37, atol=1e-6)
    assert rend["kat_single/pixels"][8, 8] == pytest.approx(0.8 / 0.818, abs=1e-4)
    # oracle reproduces the single-Gaussian KAT
    ld = np.sqrt(1.0 / 2.0 - 0.01)
    logit = lambda q: np.log(q / (1 - q))
    sc = O.slice_constants(np.eye(3), np.zeros(3), 17, 17, 1.0, 0.9999)
    num, den, _, _ = O.rasterize(
        np.zeros((1, 3), np.float32),
        np.array([[ld] * 3 + [0, 0, 0]], np.float32),
        np.array([logit(1 - 1e-7)], np.float32),
        np.array([logit(0.8)], np.float32), -30.0, -4.0, 0.01, sc)
    np.testing.assert_array_equal(np.clip(num / den, 0, 1),
                                  rend["kat_single/pixels"])


def test_adam_bit_exact():
    z = load_golden("adam_densify.npz")
    params = {k: z[f"adam/init/{k}"].copy() for k in O.GROUPS}
    params["bg_intensity_raw"], params["bg_opacity_raw"] = map(
        float, z["adam/init/bg"])
    m = {k: np.zeros_like(params[k]) for k in O.GROUPS}
    v = {k: np.zeros_like(params[k]) for k in O.GROUPS}
    m["bg"] = np.zeros(2, np.float32)
    v["bg"] = np.zeros(2, np.float32)
    lrs = {"means": 0.016, "l_raw": 0.05, "intensity_raw": 0.05,
           "opacity_raw": 0.05, "bg": 0.05}
    for step in range(5):
        g = {f"d_{k}": z[f"adam/step{step}/d_{k}"] for k in O.GROUPS}
        g["d_bg_intensity_raw"], g["d_bg_opacity_raw"] = map(
            float, z[f"adam/step{step}/d_bg"])
        O.adam_step(params, g, m, v, step + 1, lrs)
    for k in O.GROUPS:
        assert np.array_equal(params[k], z[f"adam/final/{k}"]), k
        assert np.array_equal(m[k], z[f"adam/final/m_{k}"]), k
        assert np.array_equal(v[k], z[f"adam/final/v_{k}"]), k
    assert [params["bg_intensity_raw"], params["bg_opacity_raw"]] == \
        list(z["adam/final/bg"])


def test_densify_exact():
    z = load_golden("adam_densify.npz")
    params = {k: z[f"densify/init/{k}"].copy() for k in O.GROUPS}
    params["beta"] = 0.01
    m = {k: np.full_like(params[k], 0.5) for k in O.GROUPS}
    v = {k: np.full_like(params[k], 0.25) for k in O.GROUPS}
    out, m2, _ = O.densify_prune_resample(
        params, m, v, z["densify/avg"], np.random.default_rng(99), 60.0, 0.8, 48)
    for k in O.GROUPS:
        assert np.array_equal(out[k], z[f"densify/final/{k}"]), k
        assert np.array_equal(m2[k], z[f"densify/final/m_{k}"]), k
