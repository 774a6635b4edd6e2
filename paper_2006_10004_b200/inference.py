"""Frozen-model prediction helpers, mirroring
/root/reference/pkg/trainer/src/tvsurrogate/inference.py.

``predict_bands`` / ``complete_planes`` / ``bench_forward`` keep the
reference signatures and semantics (inference.py:25-42, 80-93); the forward
they call is the B200 drop-in.  ``predict_planes`` is the batched GPU
variant: it returns the 7-plane ``[input, b1..b5, closure]`` stack with the
closure computed in the head kernel's epilogue instead of on the host.
"""

from __future__ import annotations

import time

import numpy as np
import torch

__all__ = ["predict_bands", "complete_planes", "predict_planes", "bench_forward"]


def predict_bands(model, image: np.ndarray) -> np.ndarray:
    """Run one (h, w) image through the frozen model, returning (k, h, w)."""
    if image.ndim != 2:
        raise ValueError(f"expected a 2-D image, got shape {image.shape}")
    with torch.no_grad():
        x = torch.from_numpy(np.ascontiguousarray(image, dtype=np.float32))
        out = model(x[None, None])[0]
    return out.numpy()


def complete_planes(image: np.ndarray, bands: np.ndarray) -> np.ndarray:
    """Stack input, predicted bands and the closure band (input - sum bands)."""
    closure = image[None] - bands.sum(axis=0, keepdims=True)
    return np.concatenate([image[None], bands, closure]).astype("<f4")


def predict_planes(model, images: torch.Tensor) -> torch.Tensor:
    """(B,1,H,W) float32 -> (B, 2+K, H, W) planes [input, bands, closure],
    closure fused into the head kernel (no host-side band sum)."""
    with torch.no_grad():
        bands, clos = model.forward_planes(images, closure=True)
    return torch.cat([images.to(bands.device), bands, clos], dim=1)


def bench_forward(model, sizes, repeats: int = 3, seed: int = 0) -> list[dict]:
    """Time the forward pass on standardized noise at each grid size
    (best of ``repeats`` perf_counter runs of predict_bands, inference.py:80-93)."""
    rng = np.random.default_rng(seed)
    rows = []
    for size in sizes:
        field = rng.standard_normal((size, size))
        field = (field - field.mean()) / max(field.std(), 1e-12)
        best = np.inf
        for _ in range(repeats):
            t0 = time.perf_counter()
            predict_bands(model, field)
            best = min(best, time.perf_counter() - t0)
        rows.append({"size": size, "pixels": size * size, "seconds": best})
    return rows
