"""CPU oracle of one training step — TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import it (the product's training step is csrc/train.cu
behind paper_2006_10004_b200.train_step).  It restates in plain PyTorch:

* ``compute_loss`` — /root/reference/pkg/trainer/src/tvsurrogate/losses.py:54-129:
  per-band energy-normalised squared error (zero-energy ground-truth bands
  skipped and counted), the sum-constraint term (selectors L1/L3,
  :101-107) and the gradient-Huber term (L2/L3, delta 0.01, forward
  differences with Neumann boundary, :109-124).
* ``train_step`` — one iteration of ``_epoch_pass`` (training.py:45-61):
  zero_grad, loss = compute_loss(model(img), ...), backward, optimizer.step().

Pinned against the reference executed in this container:
tests/golden/make_golden_train.py -> golden_train.npz (losses of all four
selectors, the L3 gradients and the running statistics after one step).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

SELECTORS = ("L", "L1", "L2", "L3")
HUBER_DELTA = 0.01


@dataclass(frozen=True)
class LossValue:
    total: torch.Tensor
    mse: torch.Tensor
    sum_constraint: torch.Tensor | None
    gradient_huber: torch.Tensor | None
    skipped_bands: int


def _fwd_diff(t):
    gx = torch.zeros_like(t)
    gy = torch.zeros_like(t)
    gx[..., :, :-1] = t[..., :, 1:] - t[..., :, :-1]
    gy[..., :-1, :] = t[..., 1:, :] - t[..., :-1, :]
    return gx, gy


def compute_loss(pred, gt_bands, image, residual_band, selector="L") -> LossValue:
    if selector not in SELECTORS:
        raise ValueError(f"unknown loss selector {selector!r}")
    if pred.shape != gt_bands.shape:
        raise ValueError("shape mismatch")
    b, k = pred.shape[:2]
    energy = gt_bands.pow(2).sum(dim=(-2, -1))
    keep = energy > 0.0
    skipped = int((~keep).sum().item())
    resid = (pred - gt_bands).pow(2).sum(dim=(-2, -1))
    r = resid[keep] / energy[keep]
    if r.numel() == 0:
        raise ValueError("every ground-truth band has zero energy")
    mse = r.sum() / (b * k)
    total = mse
    sum_term = None
    if selector in ("L1", "L3"):
        recon = pred.sum(dim=1, keepdim=True) + residual_band
        den = image.pow(2).sum(dim=(-2, -1)).clamp_min(1e-30)
        sum_term = ((recon - image).pow(2).sum(dim=(-2, -1)) / den).mean()
        total = total + sum_term
    grad_term = None
    if selector in ("L2", "L3"):
        pgx, pgy = _fwd_diff(pred)
        ggx, ggy = _fwd_diff(gt_bands)
        num = (F.huber_loss(pgx, ggx, delta=HUBER_DELTA, reduction="none").sum(dim=(-2, -1))
               + F.huber_loss(pgy, ggy, delta=HUBER_DELTA, reduction="none").sum(dim=(-2, -1)))
        den = (F.huber_loss(torch.zeros_like(ggx), ggx, delta=HUBER_DELTA, reduction="none").sum(dim=(-2, -1))
               + F.huber_loss(torch.zeros_like(ggy), ggy, delta=HUBER_DELTA, reduction="none").sum(dim=(-2, -1)))
        gk = den > 0.0
        skipped += int((~gk).sum().item())
        gr = num[gk] / den[gk]
        grad_term = gr.sum() / (b * k) if gr.numel() else pred.new_zeros(())
        total = total + grad_term
    return LossValue(total, mse, sum_term, grad_term, skipped)


def train_step(model, img, gt, res, selector="L", optimizer=None):
    """One _epoch_pass iteration; returns the loss value (float)."""
    if optimizer is not None:
        optimizer.zero_grad(set_to_none=True)
    value = compute_loss(model(img), gt, img, res, selector)
    value.total.backward()
    if optimizer is not None:
        optimizer.step()
    return float(value.total.detach())


def train_batch(seed: int = 1, B: int = 2, H: int = 32, W: int = 32, K: int = 5):
    """Seeded synthetic training batch in the reference dataset's convention
    (standardised input; ground-truth bands + residual that sum to it)."""
    g = torch.Generator().manual_seed(seed)
    img = torch.randn(B, 1, H, W, generator=g)
    frac = torch.rand(B, K + 1, 1, 1, generator=g)
    frac = frac / frac.sum(1, keepdim=True)
    noise = torch.randn(B, K + 1, H, W, generator=g) * 0.05
    noise = noise - noise.mean(1, keepdim=True)
    planes = frac * img + noise
    return img, planes[:, :K].contiguous(), planes[:, K:].contiguous()
