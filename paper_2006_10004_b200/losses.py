"""Drop-in for the reference's training losses on B200.

Mirrors /root/reference/pkg/trainer/src/tvsurrogate/losses.py:54-129
(``compute_loss``, ``LossValue``, ``SELECTORS``, ``HUBER_DELTA``): same
arguments, same selectors, same errors, same skipped-band accounting.  The
reference evaluates the loss with ~100 small torch ops and backpropagates
through their autograd graph; here the value is two kernel launches
(``tvs_loss_sums``: one pass of fp64 sums, then the scalars) and the backward
one (``tvs_loss_grad``: the closed-form d total / d pred from the same sums),
csrc/loss.cu.  ``LossValue.total`` carries the gradient; the component terms
are reported detached (training.py:51-56 backpropagates ``total`` only).

CPU tensors follow the model's convention: they are moved to the current CUDA
device and the results come back on the CPU.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass

import torch

from . import _native

__all__ = ["LossValue", "compute_loss", "SELECTORS", "HUBER_DELTA"]

log = logging.getLogger(__name__)

SELECTORS = ("L", "L1", "L2", "L3")
HUBER_DELTA = 0.01
_TERMS = {"L": 0, "L1": 1, "L2": 2, "L3": 3}  # bit 0 = sum constraint, bit 1 = gradient Huber


@dataclass(frozen=True)
class LossValue:
    total: torch.Tensor
    mse: torch.Tensor
    sum_constraint: torch.Tensor | None
    gradient_huber: torch.Tensor | None
    skipped_bands: int


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


class _FusedLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, pred, gt, image, residual, terms):
        lib = _native.load()
        B, K, H, W = pred.shape
        with torch.cuda.device(pred.device):
            st = torch.cuda.current_stream(pred.device).cuda_stream
            sums = torch.empty(B * K * 4 + B * 2, device=pred.device, dtype=torch.float64)
            values = torch.empty(8, device=pred.device, dtype=torch.float32)
            _native.check(lib.tvs_loss_sums(_ptr(pred), _ptr(gt), _ptr(image), _ptr(residual), B, K, H, W, terms,
                                            ctypes.c_float(HUBER_DELTA), _ptr(sums), _ptr(values),
                                            ctypes.c_void_p(st)))
        ctx.save_for_backward(pred, gt, image, residual, sums)
        ctx.terms = terms
        ctx.mark_non_differentiable(values)
        return values[0].clone(), values

    @staticmethod
    def backward(ctx, g_total, _g_values):
        pred, gt, image, residual, sums = ctx.saved_tensors
        lib = _native.load()
        B, K, H, W = pred.shape
        with torch.cuda.device(pred.device):
            st = torch.cuda.current_stream(pred.device).cuda_stream
            g = g_total.detach().to(pred.device, torch.float32).contiguous()
            grad = torch.empty_like(pred)
            _native.check(lib.tvs_loss_grad(_ptr(pred), _ptr(gt), _ptr(image), _ptr(residual), B, K, H, W, ctx.terms,
                                            ctypes.c_float(HUBER_DELTA), _ptr(sums), _ptr(g), _ptr(grad),
                                            ctypes.c_void_p(st)))
        return grad, None, None, None, None


def compute_loss(pred: torch.Tensor, gt_bands: torch.Tensor, image: torch.Tensor, residual_band: torch.Tensor,
                 selector: str = "L") -> LossValue:
    """Evaluate the selected loss for a batch (losses.py:54-129): pred and
    gt_bands (b, k, h, w), image and residual_band (b, 1, h, w)."""
    if selector not in SELECTORS:
        raise ValueError(f"unknown loss selector {selector!r}; choose from {SELECTORS}")
    if pred.shape != gt_bands.shape:
        raise ValueError(f"shape mismatch: pred {tuple(pred.shape)} vs gt {tuple(gt_bands.shape)}")
    if pred.ndim != 4:
        raise ValueError(f"expected (b, k, h, w) bands, got {tuple(pred.shape)}")
    if not torch.cuda.is_available():
        raise RuntimeError("compute_loss (B200) needs a CUDA device; there is no CPU fallback")
    home = pred.device
    dev = home if pred.is_cuda else torch.device("cuda", torch.cuda.current_device())
    terms = _TERMS[selector]
    b, k, h, w = pred.shape
    if terms & 1 and (tuple(image.shape) != (b, 1, h, w) or tuple(residual_band.shape) != (b, 1, h, w)):
        raise ValueError(f"image / residual_band must be {(b, 1, h, w)}, got {tuple(image.shape)} / "
                         f"{tuple(residual_band.shape)}")

    def prep(t):
        return t.to(dev, torch.float32).contiguous()

    p = prep(pred)  # (differentiable: .to / .contiguous keep the graph back to the model)
    total, values = _FusedLoss.apply(p, prep(gt_bands.detach()), prep(image.detach()) if terms & 1 else None,
                                     prep(residual_band.detach()) if terms & 1 else None, terms)
    v = values.tolist()  # one synchronisation (the reference's .item() on the skipped count does the same)
    skipped = int(v[4])
    if skipped:
        log.warning("skipping %d zero-energy ground-truth band terms", skipped)
    if int(v[6]) == 0:
        raise ValueError("every ground-truth band has zero energy")
    g_skipped = int(v[5]) if terms & 2 else 0
    if g_skipped:
        log.warning("skipping %d zero-gradient ground-truth band terms", g_skipped)
    values = values.to(home)
    return LossValue(total=total.to(home), mse=values[1], sum_constraint=values[2] if terms & 1 else None,
                     gradient_huber=values[3] if terms & 2 else None, skipped_bands=skipped + g_skipped)
