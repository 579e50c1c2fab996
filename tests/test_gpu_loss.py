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
