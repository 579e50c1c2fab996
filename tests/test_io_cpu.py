"""Data formats either side of the hot path, against fixtures made with the
reference (tests/golden/make_golden_io.py): the UGSC checkpoint (ref
trainer.py:295-348) byte for byte, the synthetic phantoms and the trilinear
slice sampler (ref volume.py:198-263)."""

import os

import numpy as np
import pytest

import cases
from conftest import ROOT, load_golden

torch = pytest.importorskip("torch")

import paper_2505_05643_b200 as ug  # noqa: E402
from paper_2505_05643_b200 import trainer as T  # noqa: E402

CKPT = os.path.join(ROOT, "tests", "golden", "ref_checkpoint.ugsc")


def _ref_inputs():
    c = cases.random_cloud(np.random.default_rng(2024), 50, extent=10.0)
    cfg = ug.TrainConfig(n_gaussians=50, iterations=123, seed=9, batch=4,
                         lr_general_final=0.005, l_init_low=0.85, l_init_high=1.05)
    return c, cfg


def test_load_reference_checkpoint():
    c, cfg = _ref_inputs()
    cloud, meta = ug.load_checkpoint(CKPT, device="cpu")
    for k in ("means", "l_raw", "intensity_raw", "opacity_raw"):
        assert np.array_equal(getattr(cloud, k).numpy(), c[k]), k
    assert cloud.bg_intensity_raw == float(np.float32(c["bg_intensity_raw"]))
    assert cloud.bg_opacity_raw == float(np.float32(c["bg_opacity_raw"]))
    assert meta["iteration"] == 77 and meta["config"]["iterations"] == 123


def test_save_checkpoint_bytes_match_reference(tmp_path):
    c, cfg = _ref_inputs()
    cloud = ug.GaussianCloud.from_numpy(c, device="cpu")
    out = tmp_path / "ours.ugsc"
    ug.save_checkpoint(cloud, out, cfg, 77)
    assert out.read_bytes() == open(CKPT, "rb").read()


def test_checkpoint_errors(tmp_path):
    blob = open(CKPT, "rb").read()
    bad = tmp_path / "bad.ugsc"
    bad.write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(T.CheckpointFormatError):
        ug.load_checkpoint(bad, device="cpu")
    bad.write_bytes(blob[:-3])
    with pytest.raises(T.CheckpointFormatError):
        ug.load_checkpoint(bad, device="cpu")


@pytest.mark.parametrize("kind", ["shells", "blobs"])
def test_phantom_and_sampler_match_reference(kind):
    z = load_golden("io.npz")
    v = ug.make_phantom(kind, 24, 0.6, seed=1)
    # offline data generation: float32 summation order may differ by 1 ulp
    np.testing.assert_allclose(v.voxels, z[f"{kind}/voxels"], rtol=1e-6, atol=1e-7)
    for i in range(3):
        spec = ug.SliceSpec(20, 17, 0.45, ug.ProbePose(z[f"{kind}/slice{i}/R"],
                                                       z[f"{kind}/slice{i}/t"]))
        px = ug.sample_slice(v, spec).pixels
        np.testing.assert_allclose(px, z[f"{kind}/slice{i}/pixels"], rtol=1e-6, atol=1e-7)


def test_training_state_roundtrip(tmp_path):
    """The resume sidecar (extension): the UGSC file stays byte-identical to
    the reference's format and the moments / statistics / JSON state come
    back exactly."""
    c, cfg = _ref_inputs()
    cloud = ug.GaussianCloud.from_numpy(c, device="cpu")
    n = cloud.n
    g = torch.Generator().manual_seed(5)
    st = T.AdamState(n, "cpu", t=41, m_flat=torch.randn(12 * n + 2, generator=g),
                     v_flat=torch.rand(12 * n + 2, generator=g))
    gs = torch.rand(n, generator=g)
    gc = torch.randint(0, 9, (n,), generator=g, dtype=torch.int32)
    rng = np.random.default_rng(17)
    rng.standard_normal(7)
    extra = {"threshold": 0.125, "rng": rng.bit_generator.state, "order": [3, 1, 2],
             "cursor": 2}
    path = tmp_path / "run.ugsc"
    ug.save_training_state(path, cloud, st, gs, gc, cfg, 77, extra)
    assert path.read_bytes() == open(CKPT, "rb").read()      # UGSC unchanged
    cloud2, st2, gs2, gc2, meta = ug.load_training_state(path, device="cpu")
    assert st2.t == 41 and (st2.beta1, st2.beta2, st2.eps) == (0.9, 0.999, 1e-15)
    assert torch.equal(st2.m_flat, st.m_flat) and torch.equal(st2.v_flat, st.v_flat)
    assert torch.equal(gs2, gs) and torch.equal(gc2, gc)
    assert meta["iteration"] == 77 and meta["threshold"] == 0.125
    assert meta["order"] == [3, 1, 2] and meta["cursor"] == 2
    r2 = np.random.default_rng()
    r2.bit_generator.state = meta["rng"]
    assert np.array_equal(r2.standard_normal(4), rng.standard_normal(4))
    side = tmp_path / "run.ugsc.adam"
    blob = side.read_bytes()
    side.write_bytes(blob[:-5])
    with pytest.raises(T.CheckpointFormatError):
        ug.load_training_state(path, device="cpu")
    side.write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(T.CheckpointFormatError):
        ug.load_training_state(path, device="cpu")
