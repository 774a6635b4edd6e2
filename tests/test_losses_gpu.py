"""The fused training losses (csrc/loss.cu via paper_2006_10004_b200.losses)
against the oracle restatement of the reference's compute_loss
(oracle/train_oracle.py, pinned to fixtures made by executing
/root/reference's losses.py:54-129): values, d total / d pred, the skipped-band
accounting and the error behaviour, for all four selectors."""
import numpy as np
import pytest
import torch

from oracle.train_oracle import compute_loss as ref_loss
from oracle.train_oracle import train_batch
from oracle.tvspecnet_oracle import build_seeded_state
from paper_2006_10004_b200 import TVSpecNet
from paper_2006_10004_b200.losses import HUBER_DELTA, SELECTORS, LossValue, compute_loss

pytestmark = pytest.mark.gpu


def _case(seed, B, K, H, W, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    gt = torch.randn(B, K, H, W, generator=g) * scale
    pred = gt + 0.3 * scale * torch.randn(B, K, H, W, generator=g)
    # gradients on both sides of the Huber knee (delta = 0.01)
    pred[:, :, : H // 2] = gt[:, :, : H // 2] + 0.004 * torch.randn(B, K, H // 2, W, generator=g)
    res = 0.1 * torch.randn(B, 1, H, W, generator=g)
    img = gt.sum(1, keepdim=True) + res + 0.05 * torch.randn(B, 1, H, W, generator=g)
    return pred, gt, img, res


@pytest.mark.parametrize("sel", SELECTORS)
@pytest.mark.parametrize("shape", [(2, 5, 32, 32), (3, 3, 17, 41), (1, 1, 1, 1), (2, 5, 1, 9)])
def test_values_and_gradient_match_reference(sel, shape):
    pred, gt, img, res = _case(11, *shape)
    p_ref = pred.clone().double().requires_grad_(True)
    v_ref = ref_loss(p_ref, gt.double(), img.double(), res.double(), sel)
    v_ref.total.backward()
    p = pred.clone().cuda().requires_grad_(True)
    v = compute_loss(p, gt.cuda(), img.cuda(), res.cuda(), sel)
    assert isinstance(v, LossValue) and v.skipped_bands == v_ref.skipped_bands
    (3.0 * v.total).backward()  # a non-unit upstream gradient
    for name in ("total", "mse", "sum_constraint", "gradient_huber"):
        a, b = getattr(v, name), getattr(v_ref, name)
        assert (a is None) == (b is None), name
        if a is not None:
            assert abs(a.item() - b.item()) <= 2e-6 * max(abs(b.item()), 1e-12), (name, a.item(), b.item())
    gref = 3.0 * p_ref.grad
    err = torch.linalg.vector_norm(p.grad.double().cpu() - gref) / torch.linalg.vector_norm(gref).clamp_min(1e-300)
    assert err <= 1e-5, err


def test_zero_energy_bands_are_skipped_and_all_zero_raises():
    pred, gt, img, res = _case(5, 2, 5, 16, 16)
    gt[0, 2] = 0.0  # zero energy (and zero gradient) band
    for sel in SELECTORS:
        v_ref = ref_loss(pred, gt, img, res, sel)
        v = compute_loss(pred.cuda(), gt.cuda(), img.cuda(), res.cuda(), sel)
        assert v.skipped_bands == v_ref.skipped_bands > 0
        assert abs(v.total.item() - v_ref.total.item()) <= 1e-5 * abs(v_ref.total.item())
    with pytest.raises(ValueError, match="zero energy"):
        compute_loss(pred.cuda(), torch.zeros_like(gt).cuda(), img.cuda(), res.cuda(), "L")


def test_errors_and_cpu_tensors():
    pred, gt, img, res = _case(6, 2, 5, 8, 8)
    with pytest.raises(ValueError, match="unknown loss selector"):
        compute_loss(pred.cuda(), gt.cuda(), img.cuda(), res.cuda(), "L9")
    with pytest.raises(ValueError, match="shape mismatch"):
        compute_loss(pred.cuda(), gt[:, :4].cuda(), img.cuda(), res.cuda(), "L")
    p = pred.clone().requires_grad_(True)  # CPU in, CPU out (the reference's convention)
    v = compute_loss(p, gt, img, res, "L3")
    v.total.backward()
    assert not v.total.is_cuda and not p.grad.is_cuda
    assert abs(v.total.item() - ref_loss(pred, gt, img, res, "L3").total.item()) <= 1e-5 * abs(v.total.item())
    assert HUBER_DELTA == 0.01


def test_training_step_with_fused_loss_matches_reference_step():
    """_epoch_pass's inner step (training.py:51-54) with both drop-ins: the
    model's train() mode and the fused loss, against the reference fixtures."""
    from pathlib import Path

    gold = dict(np.load(Path(__file__).resolve().parent / "golden" / "golden_train.npz"))
    m = TVSpecNet()
    m.load_state_dict(build_seeded_state())
    m = m.cuda().train()
    img, gt, res = (t.cuda() for t in train_batch())
    v = compute_loss(m(img), gt, img, res, "L3")
    v.total.backward()
    assert abs(v.total.item() - gold["loss_L3"]) <= 1e-5 * abs(gold["loss_L3"])
    worst = 0.0
    for n, p in m.named_parameters():
        g, ref = p.grad.detach().cpu().numpy(), gold[f"grad64_{n}"]
        worst = max(worst, float(np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)))
    assert worst <= 2e-2, worst


# ---- the reference's own loss tests (pkg/trainer/tests/test_losses.py), run
# ---- against the drop-in with the reference's CPU-tensor calling convention
def _ref_case(b=2, k=3, size=8, seed=0):  # test_losses.py:8-13
    gen = torch.Generator().manual_seed(seed)
    gt = torch.randn(b, k, size, size, generator=gen)
    res = torch.randn(b, 1, size, size, generator=gen)
    img = gt.sum(dim=1, keepdim=True) + res
    return gt, res, img


def test_reference_perfect_prediction_is_zero():  # test_losses.py:15-20
    gt, res, img = _ref_case()
    for selector in SELECTORS:
        value = compute_loss(gt.clone(), gt, img, res, selector)
        assert float(value.total) == pytest.approx(0.0, abs=1e-10)
        assert value.skipped_bands == 0


def test_reference_zero_prediction_is_unit_loss():  # test_losses.py:23-32
    gt, res, img = _ref_case()
    assert float(compute_loss(torch.zeros_like(gt), gt, img, res, "L").total) == 1.0
    value = compute_loss(torch.zeros_like(gt), gt, img, res, "L2")
    assert float(value.gradient_huber) == pytest.approx(1.0, rel=1e-6)


def test_reference_scale_invariance_and_selector_composition():  # test_losses.py:35-55
    gt, res, img = _ref_case()
    pred = gt + 0.1 * torch.randn_like(gt)
    a = compute_loss(pred, gt, img, res, "L")
    b = compute_loss(3.0 * pred, 3.0 * gt, img, res, "L")
    assert float(a.mse) == pytest.approx(float(b.mse), rel=1e-5)
    pred = gt + 0.05 * torch.randn_like(gt)
    parts = {s: compute_loss(pred, gt, img, res, s) for s in SELECTORS}
    assert float(parts["L1"].total) == pytest.approx(float(parts["L"].mse) + float(parts["L1"].sum_constraint), rel=1e-6)
    assert float(parts["L3"].total) == pytest.approx(
        float(parts["L"].mse) + float(parts["L3"].sum_constraint) + float(parts["L3"].gradient_huber), rel=1e-6)


def test_reference_band_sum_skips_and_gradients():  # test_losses.py:58-97
    gt, res, img = _ref_case()
    assert float(compute_loss(gt.clone(), gt, img, res, "L1").sum_constraint) == pytest.approx(0.0, abs=1e-10)
    gt0 = gt.clone()
    gt0[0, 1] = 0.0
    value = compute_loss(gt0 + 0.1, gt0, img, res, "L")
    assert value.skipped_bands == 1 and torch.isfinite(value.total)
    pred = (gt + 0.1 * torch.randn_like(gt)).requires_grad_(True)
    compute_loss(pred, gt, img, res, "L3").total.backward()
    assert pred.grad is not None and torch.isfinite(pred.grad).all()
