"""Band scoring: oracle pinned to the reference
spectv.metrics outputs (CPU), and the GPU kernels vs the same fixtures."""
import math

import numpy as np
import pytest

from oracle.metrics_oracle import band_metrics as oracle_band_metrics

CASES = ["noisy", "exact", "zero_pred", "const_gt", "square_aligned"]


def _close(a, b, rtol):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    fin = ~both_inf
    np.testing.assert_allclose(a[fin], b[fin], rtol=rtol, atol=1e-12)


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference_metrics(golden, case):
    per_band, _, ranges = oracle_band_metrics(golden[f"metrics_{case}_gt"], golden[f"metrics_{case}_pred"])
    _close(per_band, golden[f"metrics_{case}_per_band"], 1e-13)
    _close(ranges, golden[f"metrics_{case}_max_i"], 0)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_band_metrics_match_reference(golden, case):
    from paper_2006_10004_b200.scoring import band_metrics

    rep = band_metrics(golden[f"metrics_{case}_gt"], golden[f"metrics_{case}_pred"])
    _close(rep.per_band, golden[f"metrics_{case}_per_band"], 1e-10)
    _close(rep.max_i, golden[f"metrics_{case}_max_i"], 0)


@pytest.mark.gpu
def test_gpu_batched_equals_single_and_api_edges(golden):
    from paper_2006_10004_b200.scoring import MetricsReport, band_metrics, band_metrics_batched, psnr, slmse, ssim

    g, p = golden["metrics_noisy_gt"], golden["metrics_noisy_pred"]
    reps = band_metrics_batched(np.stack([g, p]), np.stack([p, g]))
    one = band_metrics(g, p)
    assert reps[0].per_band == one.per_band
    avg = MetricsReport.average(reps)
    assert len(avg.per_band) == 5 and "residual_band" in avg.to_csv() and '"averages"' in avg.to_json()
    b, h = g[0].astype(np.float64), p[0].astype(np.float64)
    from oracle import metrics_oracle as o

    assert math.isclose(ssim(b, h, 3.0), o.ssim(b, h, 3.0), rel_tol=1e-10)
    assert math.isclose(ssim(b, h, 3.0, windowed=False), o.ssim(b, h, 3.0, windowed=False), rel_tol=1e-12)
    assert math.isclose(psnr(b, h, 2.0), o.psnr(b, h, 2.0), rel_tol=1e-12)
    assert math.isclose(slmse(b, h), o.slmse(b, h), rel_tol=1e-10)
    assert psnr(b, b, 1.0) == math.inf and slmse(b, b) == 1.0
    with pytest.raises(ValueError):
        ssim(np.zeros((10, 40)), np.zeros((10, 40)), 1.0)  # too small for the 11x11 window interior
    with pytest.raises(ValueError):
        slmse(np.zeros((15, 40)), np.zeros((15, 40)))
    with pytest.raises(ValueError):
        psnr(b, h, 0.0)
