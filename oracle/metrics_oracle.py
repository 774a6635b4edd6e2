"""CPU oracle for band scoring — TEST INFRASTRUCTURE ONLY (tests/ and the
scoring bench import it as the checker; the product path is
paper_2006_10004_b200/scoring.py on the GPU).

Numpy restatement of /root/reference/pkg/src/spectv/metrics.py:
  psnr           metrics.py:28-37
  _gaussian      metrics.py:40-44   (11 taps, sigma 1.5, normalised)
  _separable     metrics.py:47-58   (symmetric padding, row then column pass)
  ssim           metrics.py:61-112  (windowed: interior mean; global variant)
  _patch_starts  metrics.py:115-123 (stride 8 + clipped tail patch)
  slmse          metrics.py:126-150
  band_metrics   metrics.py:211-237 (per band: range = gt max-min floored 1e-9)
Pinned against outputs of the reference module (tests/golden/make_golden.py).
"""
from __future__ import annotations

import math

import numpy as np

SIGMA, RADIUS, PATCH, STRIDE = 1.5, 5, 16, 8


def psnr(b, bhat, max_i):
    if b.shape != bhat.shape:
        raise ValueError("shape mismatch")
    if max_i <= 0:
        raise ValueError("max_i must be positive")
    mse = float(np.mean((b - bhat) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(max_i * max_i / mse)


def _gaussian():
    x = np.arange(-RADIUS, RADIUS + 1, dtype=np.float64)
    k = np.exp(-(x * x) / (2.0 * SIGMA * SIGMA))
    return k / k.sum()


def _separable(a, k):
    r = len(k) // 2
    p = np.pad(a, ((0, 0), (r, r)), mode="symmetric")
    out = np.zeros_like(a)
    for i, wk in enumerate(k):
        out += wk * p[:, i : i + a.shape[1]]
    p = np.pad(out, ((r, r), (0, 0)), mode="symmetric")
    out = np.zeros_like(a)
    for i, wk in enumerate(k):
        out += wk * p[i : i + a.shape[0], :]
    return out


def ssim(b, bhat, data_range, windowed=True):
    if b.shape != bhat.shape:
        raise ValueError("shape mismatch")
    if data_range <= 0:
        raise ValueError("data_range must be positive")
    c1, c2 = (0.01 * data_range) ** 2, (0.03 * data_range) ** 2
    if not windowed:
        mu_b, mu_h = b.mean(), bhat.mean()
        vb, vh = b.var(), bhat.var()
        cov = float(np.mean((b - mu_b) * (bhat - mu_h)))
        cov = float(np.clip(cov, -math.sqrt(vb * vh), math.sqrt(vb * vh)))
        return float((2 * mu_b * mu_h + c1) * (2 * cov + c2) / ((mu_b**2 + mu_h**2 + c1) * (vb + vh + c2)))
    k = _gaussian()
    ux, uy = _separable(b, k), _separable(bhat, k)
    uxx, uyy, uxy = _separable(b * b, k), _separable(bhat * bhat, k), _separable(b * bhat, k)
    vx = np.maximum(uxx - ux * ux, 0.0)
    vy = np.maximum(uyy - uy * uy, 0.0)
    cap = np.sqrt(vx * vy)
    vxy = np.clip(uxy - ux * uy, -cap, cap)
    s = ((2 * ux * uy + c1) * (2 * vxy + c2)) / ((ux * ux + uy * uy + c1) * (vx + vy + c2))
    interior = s[RADIUS:-RADIUS, RADIUS:-RADIUS]
    if interior.size == 0:
        raise ValueError("image too small for the 11x11 SSIM window")
    return float(interior.mean())


def _patch_starts(dim):
    if dim < PATCH:
        raise ValueError("dimension smaller than the patch")
    starts = list(range(0, dim - PATCH + 1, STRIDE))
    if starts[-1] != dim - PATCH:
        starts.append(dim - PATCH)
    return starts


def slmse(b, bhat):
    if b.shape != bhat.shape:
        raise ValueError("shape mismatch")
    diff, ref = (b - bhat) ** 2, bhat * bhat
    num = den = 0.0
    for sy in _patch_starts(b.shape[0]):
        for sx in _patch_starts(b.shape[1]):
            num += float(diff[sy : sy + PATCH, sx : sx + PATCH].sum())
            den += float(ref[sy : sy + PATCH, sx : sx + PATCH].sum())
    if den == 0.0:
        return 1.0 if num == 0.0 else 0.0
    return 1.0 - num / den


def band_metrics(gt_bands, pred_bands):
    """-> (per_band [(ssim, psnr, slmse)], averages, ranges)"""
    gt = np.asarray(gt_bands, dtype=np.float64)
    pred = np.asarray(pred_bands, dtype=np.float64)
    per_band, ranges = [], []
    for k in range(gt.shape[0]):
        rng = max(float(gt[k].max() - gt[k].min()), 1e-9)
        ranges.append(rng)
        per_band.append((ssim(gt[k], pred[k], data_range=rng), psnr(gt[k], pred[k], max_i=rng), slmse(gt[k], pred[k])))
    averages = tuple(sum(v[j] for v in per_band) / len(per_band) for j in range(3))
    return per_band, averages, ranges
