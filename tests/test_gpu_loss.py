"""Fused loss kernel (ugs_loss) against the oracle (numpy/scipy restatement
of trainer.loss / metrics.ssim_with_grad, pinned to the reference)."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2505_05643_b200.metrics import fused_loss  # noqa: E402


@pytest.mark.parametrize("shape", [(3, 64, 64), (2, 37, 53), (1, 256, 256), (2, 11, 40)])
@pytest.mark.parametrize("lam,l2", [(0.2, False), (0.0, False), (0.2, True), (1.0, False)])
def test_fused_loss_matches_oracle(shape, lam, l2):
    rng = np.random.default_rng(sum(shape))
    S, H, W = shape
    num = rng.uniform(0.05, 1.0, shape).astype(np.float32)
    den = rng.uniform(0.5, 1.5, shape).astype(np.float32)
    tgt = np.clip(num / den + rng.normal(0, 0.1, shape), 0, 1).astype(np.float32)
    t = lambda a: torch.as_tensor(a, device="cuda")
    lv, dpix, sv = fused_loss(t(num), t(den), t(tgt), lam, l2)
    for s in range(S):
        pred = num[s] / den[s]
        ref_v, ref_d = O.loss(pred, tgt[s], lam, l2)
        assert float(lv[s]) == pytest.approx(ref_v, rel=1e-12, abs=1e-14)
        np.testing.assert_allclose(dpix[s].cpu().numpy(), ref_d.astype(np.float32),
                                   rtol=1e-6, atol=1e-12)
        if not l2 and lam > 0:
            assert float(sv[s]) == pytest.approx(O.ssim(pred, tgt[s]), abs=1e-12)


@pytest.mark.parametrize("shape", [(64, 64), (37, 53), (256, 256), (11, 40)])
def test_public_api_on_kernel(shape):
    """ssim / ssim_with_grad / loss (the reference's public metrics API,
    metrics.py:68-98, trainer.py:130-151) run on ugs_loss and match the
    oracle; the float64 torch formulation agrees as an independent check."""
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200 import metrics as M
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    a = rng.uniform(0, 1, shape).astype(np.float32)
    b = np.clip(a + rng.normal(0, 0.15, shape), 0, 1).astype(np.float32)
    n0 = _lib_launches()
    s = ug.ssim(a, b)
    assert _lib_launches() > n0, "ssim() must run the CUDA kernel"
    assert s == pytest.approx(O.ssim(a, b), abs=1e-12)
    assert round(s, 4) == round(O.ssim(a, b), 4)
    s2, g = ug.ssim_with_grad(a, b)
    ref_s, ref_g = O.ssim_with_grad(a.astype(np.float64), b.astype(np.float64))
    assert s2 == pytest.approx(ref_s, abs=1e-12)
    np.testing.assert_allclose(g.cpu().numpy(), ref_g, rtol=1e-6,
                               atol=1e-6 * np.abs(ref_g).max())
    for lam, l2 in ((0.2, False), (0.0, False), (0.5, True)):
        v, d = ug.loss(a, b, lam, l2)
        rv, rd = O.loss(a, b, lam, l2)
        assert v == pytest.approx(rv, rel=1e-12, abs=1e-14)
        np.testing.assert_allclose(d.cpu().numpy(), rd, rtol=1e-6, atol=1e-6 * np.abs(rd).max())
    # independent float64 torch formulation of the same SSIM
    st, gt = M.ssim_with_grad_batch_torch(torch.as_tensor(a[None], device="cuda"),
                                         torch.as_tensor(b[None], device="cuda"))
    assert float(st[0]) == pytest.approx(s, abs=1e-12)
    np.testing.assert_allclose(gt[0].cpu().numpy(), g.cpu().numpy(), rtol=1e-6,
                               atol=1e-6 * float(gt.abs().max()))


def _lib_launches():
    from paper_2505_05643_b200 import _lib
    return _lib.lib().ugs_launch_count()
