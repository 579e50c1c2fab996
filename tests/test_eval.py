"""evaluate_views (GPU ground truth + evaluation) against
the reference's own output (tests/golden/eval.npz, make_golden_eval.py)."""

import numpy as np
import pytest

import cases
from conftest import load_golden

import paper_2505_05643_b200 as ug

FAMILIES = ("axial", "coronal", "sagittal")


@pytest.fixture(scope="module")
def gold():
    return load_golden("eval.npz")


def _volume(z):
    return ug.Volume(z["voxels"], float(z["spacing"]))


def test_family_poses_match_reference(gold):
    vol = _volume(gold)
    for name in FAMILIES:
        poses = ug.family_poses(vol, name, 5)
        assert len(poses) == 5
        for i, (pose, spec) in enumerate(poses):
            np.testing.assert_array_equal(pose.rotation, gold[f"family/{name}/{i}/R"])
            np.testing.assert_array_equal(pose.translation, gold[f"family/{name}/{i}/t"])
            assert [spec.width, spec.height] == list(gold[f"family/{name}/{i}/wh"])
            assert spec.spacing == vol.spacing and spec.pose is pose
    with pytest.raises(ug.InvalidParameterError):
        ug.family_poses(vol, "oblique", 3)


def test_eval_report_json_schema():
    rep = ug.EvalReport(families={"b": {"z": 1, "a": 2}, "a": {"count": 3}},
                        timestamp="t")
    d = rep.to_json_dict()
    assert list(d["families"]) == ["a", "b"] and list(d["families"]["b"]) == ["a", "z"]
    assert d["timestamp"] == "t"


@pytest.mark.gpu
def test_evaluate_views_matches_reference(gold):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs CUDA")
    vol = _volume(gold)
    c = cases.eval_cloud(vol.world_bounds())
    cloud = ug.GaussianCloud(c["means"], c["l_raw"], c["intensity_raw"], c["opacity_raw"],
                             device="cuda")
    rep = ug.evaluate_views(cloud, vol, 5)
    for name in FAMILIES:
        got = rep.families[name]
        assert got["count"] == 5
        assert got["psnr_inf_count"] == int(gold[f"report/{name}/psnr_inf_count"])
        for k in ("ssim_mean", "ssim_std"):
            assert got[k] == pytest.approx(float(gold[f"report/{name}/{k}"]), abs=1e-4), k
        for k in ("psnr_mean", "psnr_std"):
            assert got[k] == pytest.approx(float(gold[f"report/{name}/{k}"]), rel=1e-4,
                                           abs=1e-4), k
