"""Band-scoring throughput: band_metrics over N images x
K bands on the GPU (two launches) vs the reference per-plane numpy loop
(oracle restatement of spectv/metrics.py) on a bounded subset."""
import json, os, sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.metrics_oracle import band_metrics as ref_band_metrics  # noqa
from paper_2006_10004_b200.scoring import band_metrics_batched  # noqa

N, K, H, W = 64, 5, 256, 256
rng = np.random.default_rng(0)
gt = torch.from_numpy(rng.standard_normal((N, K, H, W)).astype(np.float32)).cuda()
pred = gt + 0.05 * torch.randn_like(gt)
for _ in range(2):
    band_metrics_batched(gt, pred)
torch.cuda.synchronize()
t0 = time.perf_counter()
reps = band_metrics_batched(gt, pred)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
g, p = gt.cpu().numpy(), pred.cpu().numpy()
t1 = time.perf_counter(); k = 0
while k < N and time.perf_counter() - t1 < 10.0:
    ref_band_metrics(g[k], p[k]); k += 1
rdt = time.perf_counter() - t1
print(json.dumps({"metric": "band_metrics megapixels/sec (images x bands scored)", "value": round(N * K * H * W / 1e6 / dt, 2),
                  "unit": "MP/s", "images": N, "bands": K, "size": [H, W], "seconds": round(dt, 4),
                  "reference_flow": {"value": round(k * K * H * W / 1e6 / rdt, 4), "unit": "MP/s", "images_timed": k,
                                     "cores": 1, "note": "numpy per-plane loop (single-threaded)"}}))
