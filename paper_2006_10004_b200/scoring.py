"""Batched band scoring on the GPU.

Mirrors /root/reference/pkg/src/spectv/metrics.py: ``psnr``, ``ssim``,
``slmse``, ``MetricsReport`` and ``band_metrics`` keep the reference's
signatures, constants (11x11 Gaussian window, sigma 1.5; c1 = (0.01 L)^2,
c2 = (0.03 L)^2; 16x16 sLMSE patches at stride 8 plus a clipped tail patch;
data range = gt max-min floored at 1e-9) and error behaviour.  The per-plane
statistics are computed in fp64 by libtvsb200's ``tvs_band_stats``
(csrc/metrics.cu); ``band_metrics_batched`` scores a whole (N, K, H, W)
prediction set in two kernel launches instead of N*K numpy passes.

Planes are scored as float32 (the BTF exchange type); the statistics are
accumulated in fp64.  The unwindowed SSIM variant (``windowed=False``) is a global-moment formula
with no spatial work; it is evaluated on the host exactly as the reference does.
"""

from __future__ import annotations

import csv
import io
import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native

__all__ = ["psnr", "ssim", "slmse", "MetricsReport", "band_metrics", "band_metrics_batched", "plane_stats"]

_R = 5
_PATCH = 16


def plane_stats(gt: torch.Tensor, pred: torch.Tensor, data_range=None) -> torch.Tensor:
    """(P, H, W) float32 planes -> (P, 8) float64 statistics (include/tvs_b200.h,
    tvs_band_stats).  ``data_range``: optional per-plane SSIM range (default:
    each gt plane's own floored range)."""
    if gt.shape != pred.shape or gt.ndim != 3:
        raise ValueError(f"shape mismatch: {tuple(gt.shape)} vs {tuple(pred.shape)}")
    dev = gt.device if gt.is_cuda else torch.device("cuda", torch.cuda.current_device())
    g = gt.to(dev, torch.float32).contiguous()
    p = pred.to(dev, torch.float32).contiguous()
    P, H, W = g.shape
    out = torch.empty((P, 8), dtype=torch.float64, device=dev)
    rng = None
    if data_range is not None:
        rng = torch.as_tensor(data_range, dtype=torch.float64).reshape(-1).expand(P).contiguous().to(dev)
    with torch.cuda.device(dev):
        _native.check(_native.load().tvs_band_stats(g.data_ptr(), p.data_ptr(), P, H, W,
                                                    rng.data_ptr() if rng is not None else None, out.data_ptr(),
                                                    torch.cuda.current_stream(dev).cuda_stream))
    return out


def _scores(stats: np.ndarray, H: int, W: int, need_ssim=True, need_slmse=True):
    """stats row -> (ssim, psnr, slmse, range) exactly as metrics.py combines them."""
    mse_sum, num, den, mx, mn, ssum, scnt = (float(v) for v in stats[:7])
    rng = max(mx - mn, 1e-9)
    mse = mse_sum / (H * W)
    ps = math.inf if mse == 0.0 else 10.0 * math.log10(rng * rng / mse)
    ss = ssum / scnt if need_ssim else float("nan")
    if need_slmse:
        sl = (1.0 if num == 0.0 else 0.0) if den == 0.0 else 1.0 - num / den
    else:
        sl = float("nan")
    return ss, ps, sl, rng


def _check_plane_sizes(H, W):
    if H - 2 * _R <= 0 or W - 2 * _R <= 0:
        raise ValueError("image too small for the 11x11 SSIM window")
    for dim in (H, W):
        if dim < _PATCH:
            raise ValueError(f"dimension {dim} smaller than the {_PATCH}-pixel patch")


def _as_plane_pair(b, bhat):
    b = np.asarray(b)
    bhat = np.asarray(bhat)
    if b.shape != bhat.shape:
        raise ValueError(f"shape mismatch: {b.shape} vs {bhat.shape}")
    return b, bhat


def psnr(b, bhat, max_i: float) -> float:
    """metrics.py:28-37: 10*log10(MAX_I^2 / MSE); +inf for identical inputs."""
    b, bhat = _as_plane_pair(b, bhat)
    if max_i <= 0:
        raise ValueError("max_i must be positive")
    st = plane_stats(torch.as_tensor(b, dtype=torch.float32)[None], torch.as_tensor(bhat, dtype=torch.float32)[None])
    mse = float(st[0, 0].item()) / b.size
    return math.inf if mse == 0.0 else 10.0 * math.log10(max_i * max_i / mse)


def ssim(b, bhat, data_range: float, windowed: bool = True) -> float:
    """metrics.py:61-112 with the given data range."""
    b, bhat = _as_plane_pair(b, bhat)
    if data_range <= 0:
        raise ValueError("data_range must be positive")
    if not windowed:  # global moments (metrics.py:80-91), host arithmetic as in the reference
        b64, h64 = b.astype(np.float64), bhat.astype(np.float64)
        c1, c2 = (0.01 * data_range) ** 2, (0.03 * data_range) ** 2
        mu_b, mu_h = b64.mean(), h64.mean()
        vb, vh = b64.var(), h64.var()
        cov = float(np.mean((b64 - mu_b) * (h64 - mu_h)))
        cov = float(np.clip(cov, -math.sqrt(vb * vh), math.sqrt(vb * vh)))
        return float((2 * mu_b * mu_h + c1) * (2 * cov + c2) / ((mu_b**2 + mu_h**2 + c1) * (vb + vh + c2)))
    H, W = b.shape
    if H - 2 * _R <= 0 or W - 2 * _R <= 0:
        raise ValueError("image too small for the 11x11 SSIM window")
    st = plane_stats(torch.as_tensor(b, dtype=torch.float32)[None], torch.as_tensor(bhat, dtype=torch.float32)[None],
                     data_range=float(data_range))
    return float(st[0, 5].item() / st[0, 6].item())


def slmse(b, bhat) -> float:
    """metrics.py:126-150: 1 - LMSE(b, bhat) / LMSE(0, bhat) over 16x16 patches, stride 8."""
    b, bhat = _as_plane_pair(b, bhat)
    for dim in b.shape:
        if dim < _PATCH:
            raise ValueError(f"dimension {dim} smaller than the {_PATCH}-pixel patch")
    st = plane_stats(torch.as_tensor(b, dtype=torch.float32)[None], torch.as_tensor(bhat, dtype=torch.float32)[None])
    num, den = float(st[0, 1]), float(st[0, 2])
    if den == 0.0:
        return 1.0 if num == 0.0 else 0.0
    return 1.0 - num / den


@dataclass
class MetricsReport:
    """metrics.py:153-208: per-band and averaged (ssim, psnr, slmse)."""

    per_band: list
    averages: tuple
    max_i: list

    def to_json(self) -> str:
        return json.dumps({"per_band": [{"ssim": s, "psnr": p, "slmse": l} for s, p, l in self.per_band],
                           "averages": {"ssim": self.averages[0], "psnr": self.averages[1],
                                        "slmse": self.averages[2]},
                           "max_i": self.max_i}, indent=2)

    @classmethod
    def average(cls, reports: "list[MetricsReport]") -> "MetricsReport":
        if not reports:
            raise ValueError("no reports to average")
        n = len(reports[0].per_band)
        if any(len(r.per_band) != n for r in reports):
            raise ValueError("reports have differing band counts")
        m = len(reports)
        per_band = [tuple(sum(r.per_band[k][j] for r in reports) / m for j in range(3)) for k in range(n)]
        averages = tuple(sum(v[j] for v in per_band) / n for j in range(3))
        max_i = [sum(r.max_i[k] for r in reports) / m for k in range(n)]
        return cls(per_band=per_band, averages=averages, max_i=max_i)

    def to_csv(self) -> str:
        n = len(self.per_band)
        header = ["metric"] + [f"band{k+1}" for k in range(n - 1)] + ["residual_band", "average"]
        buf = io.StringIO()
        writer = csv.writer(buf)
        writer.writerow(header)
        for j, name in enumerate(("ssim", "psnr", "slmse")):
            row = [name] + [f"{self.per_band[k][j]:.4f}" for k in range(n)]
            row.append(f"{self.averages[j]:.4f}")
            writer.writerow(row)
        return buf.getvalue()


def band_metrics_batched(gt_bands, pred_bands) -> list[MetricsReport]:
    """(N, K, H, W) ground truth and predictions -> N MetricsReports (metrics.py:211-237
    applied to every image), two GPU launches for the whole set."""
    gt = torch.as_tensor(np.asarray(gt_bands) if not torch.is_tensor(gt_bands) else gt_bands)
    pr = torch.as_tensor(np.asarray(pred_bands) if not torch.is_tensor(pred_bands) else pred_bands)
    if gt.shape != pr.shape or gt.ndim != 4:
        raise ValueError(f"band stacks differ in shape: {tuple(gt.shape)} vs {tuple(pr.shape)}")
    N, K, H, W = gt.shape
    _check_plane_sizes(H, W)
    st = plane_stats(gt.reshape(N * K, H, W), pr.reshape(N * K, H, W)).cpu().numpy().reshape(N, K, 8)
    reports = []
    for n in range(N):
        per_band, ranges = [], []
        for k in range(K):
            ss, ps, sl, rng = _scores(st[n, k], H, W)
            per_band.append((ss, ps, sl))
            ranges.append(rng)
        averages = tuple(sum(v[j] for v in per_band) / len(per_band) for j in range(3))
        reports.append(MetricsReport(per_band=per_band, averages=averages, max_i=ranges))
    return reports


def band_metrics(gt_bands, pred_bands) -> MetricsReport:
    """metrics.py:211-237 for one (K, H, W) stack."""
    gt = np.asarray(gt_bands)
    pred = np.asarray(pred_bands)
    if gt.shape != pred.shape:
        raise ValueError(f"band stacks differ in shape: {gt.shape} vs {pred.shape}")
    return band_metrics_batched(gt[None], pred[None])[0]
