"""Prediction helpers around the B200 drop-in, with the calling contract of
/root/reference/pkg/trainer/src/tvsurrogate/inference.py.

* ``predict_bands`` (reference inference.py:25-32): one 2-D numpy image in,
  ``(K, h, w)`` numpy bands out, batch 1, CPU in and out.
* ``complete_planes`` (inference.py:34-42): the 7-plane
  ``[input, b1..bK, closure]`` little-endian float32 stack, closure =
  image - sum(bands), computed on the host.
* ``bench_forward`` (inference.py:80-93): the reference's timing protocol.
* ``predict_planes`` (new): the batched GPU form of the two above; the
  closure comes from the head kernel's epilogue, which also evaluates the
  band-sum reconstruction check (tvs_forward_checked).
"""

from __future__ import annotations

import time

import numpy as np
import torch

__all__ = ["predict_bands", "complete_planes", "predict_planes", "bench_forward"]


def predict_bands(model, image: np.ndarray) -> np.ndarray:
    """(h, w) array -> (K, h, w) float32 bands through ``model`` (no grad).
    Anything but a 2-D array is a ValueError, as in the reference."""
    if image.ndim != 2:
        raise ValueError(f"expected a 2-D image, got shape {image.shape}")
    plane = torch.from_numpy(np.ascontiguousarray(image, dtype=np.float32))[None, None]
    with torch.no_grad():
        bands = model(plane)
    return bands[0].numpy()


def complete_planes(image: np.ndarray, bands: np.ndarray) -> np.ndarray:
    """[image, bands..., image - sum(bands)] as one ``<f4`` array."""
    rest = image[None] - bands.sum(axis=0, keepdims=True)
    return np.concatenate([image[None], bands, rest]).astype("<f4")


def predict_planes(model, images: torch.Tensor, check_tol: float | None = 1e-5) -> torch.Tensor:
    """(B,1,H,W) float32 -> (B, 2+K, H, W) planes [input, bands, closure].

    The closure plane is written by the head kernel.  For CUDA inputs the same
    epilogue also sums ||x - sum(bands) - closure||^2 and ||x||^2 per image from
    the stored values; a relative residual above ``check_tol`` (the 1e-5 of the
    reference's closure test, test_inference.py:31-38) raises ArithmeticError.
    ``check_tol=None`` skips the check."""
    with torch.no_grad():
        if images.is_cuda and check_tol is not None:
            bands, clos, rel = model.forward_planes(images, check_reconstruction=True)
            worst = float(rel.max())
            if not worst <= check_tol:
                raise ArithmeticError(f"band-sum reconstruction check failed: relative residual {worst:.3e} "
                                      f"> {check_tol:g}")
        else:
            bands, clos = model.forward_planes(images, closure=True)
    return torch.cat([images.to(bands.device), bands, clos], dim=1)


def bench_forward(model, sizes, repeats: int = 3, seed: int = 0) -> list[dict]:
    """Reference timing protocol: for each size, a standardized N(0,1)
    size x size field (numpy seed ``seed``), the best of ``repeats``
    perf_counter timings of ``predict_bands``."""
    rng = np.random.default_rng(seed)
    out = []
    for n in sizes:
        field = rng.standard_normal((n, n))
        field = (field - field.mean()) / max(field.std(), 1e-12)
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            predict_bands(model, field)
            times.append(time.perf_counter() - t0)
        out.append({"size": n, "pixels": n * n, "seconds": min(times)})
    return out
