"""CPU oracle for the TVSpecNET forward — TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it.  The product path (``paper_2006_10004_b200``) runs on the
sm_100a kernels and raises when the CUDA extension is missing.

It restates, in plain PyTorch CPU ops, the reference path:

* ``TVSpecNetOracle``  — /root/reference/pkg/trainer/src/tvsurrogate/model.py:29-52
  (Conv2d(1,C)+ReLU, (depth-2) x [Conv2d(C,C,no bias)+BatchNorm2d+ReLU],
  Conv2d(C,K,bias); zero padding 1; ValueError on depth < 3 and on a
  non-(B,1,H,W) input).  Module order is identical, so ``state_dict`` keys,
  shapes and the torch RNG draw order at construction match the reference.
* ``receptive_field`` — model.py:55-56.
* ``predict_bands``   — /root/reference/pkg/trainer/src/tvsurrogate/inference.py:25-32
* ``complete_planes`` — inference.py:34-42 (closure = image - sum of bands).
* ``bench_forward``   — inference.py:80-93 (best-of-``repeats`` perf_counter).
* ``build_seeded_state`` — the BASELINE.json weight recipe ("Kaiming-normal
  weights from seed 0, BN running stats mean=0 var=1"): torch.manual_seed,
  construct, kaiming_normal_(fan_in, relu) on every conv weight; conv biases
  keep their default (seeded) init; BN stays gamma=1, beta=0, mu=0, var=1.

The arithmetic itself is PyTorch's CPU ATen/oneDNN convolution and eval-mode
batch norm (third-party dependency pinned by the reference as ``torch>=2.0``,
/root/reference/pkg/trainer/pyproject.toml:11-14).  The restatement is
pinned against the reference module executed in this container: see
``tests/golden/make_golden.py`` (fixtures) and ``tests/test_oracle.py``.
"""

from __future__ import annotations

import time

import numpy as np
import torch
from torch import nn

__all__ = [
    "ARCH_SPEC",
    "TVSpecNetOracle",
    "receptive_field",
    "build_seeded_state",
    "predict_bands",
    "complete_planes",
    "bench_forward",
    "band_rel_l2",
]

ARCH_SPEC = {
    "depth": 17,
    "channels": 64,
    "kernel": 3,
    "out_bands": 5,
    "batch_norm": True,
    "receptive_field": 35,
}


class TVSpecNetOracle(nn.Module):
    """model.py:29-52 restated; same module list, same parameter names."""

    def __init__(self, depth: int = 17, channels: int = 64, out_bands: int = 5):
        super().__init__()
        if depth < 3:
            raise ValueError("depth must be at least 3 (first, hidden, last)")
        layers: list[nn.Module] = [nn.Conv2d(1, channels, 3, padding=1, bias=True), nn.ReLU(inplace=True)]
        for _ in range(depth - 2):
            layers += [
                nn.Conv2d(channels, channels, 3, padding=1, bias=False),
                nn.BatchNorm2d(channels),
                nn.ReLU(inplace=True),
            ]
        layers.append(nn.Conv2d(channels, out_bands, 3, padding=1, bias=True))
        self.body = nn.Sequential(*layers)
        self.depth = depth
        self.out_bands = out_bands

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.ndim != 4 or x.shape[1] != 1:
            raise ValueError(f"expected (batch, 1, h, w) input, got {tuple(x.shape)}")
        return self.body(x)


class UnshuffledOracle(nn.Module):
    """The opt-in unshuffle = 2 variant as a plain torch composition (SURVEY F2:
    not in the reference, so this oracle is unpinned by it):
    F.pixel_unshuffle(x, 2) -> Conv2d(4, C)+ReLU -> (depth-2) x [Conv2d(C,C)+BN+ReLU]
    -> Conv2d(C, 4K) -> F.pixel_shuffle(., 2).  Module order matches
    TVSpecNet(..., unshuffle=2), so state_dicts are interchangeable."""

    def __init__(self, depth: int = 17, channels: int = 64, out_bands: int = 5):
        super().__init__()
        layers: list[nn.Module] = [nn.Conv2d(4, channels, 3, padding=1, bias=True), nn.ReLU(inplace=True)]
        for _ in range(depth - 2):
            layers += [nn.Conv2d(channels, channels, 3, padding=1, bias=False), nn.BatchNorm2d(channels),
                       nn.ReLU(inplace=True)]
        layers.append(nn.Conv2d(channels, 4 * out_bands, 3, padding=1, bias=True))
        self.body = nn.Sequential(*layers)
        self.depth, self.out_bands = depth, out_bands

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        import torch.nn.functional as F

        return F.pixel_shuffle(self.body(F.pixel_unshuffle(x, 2)), 2)


def receptive_field(depth: int = 17, kernel: int = 3) -> int:
    return depth * (kernel - 1) + 1


def build_seeded_state(depth: int = 17, channels: int = 64, out_bands: int = 5, seed: int = 0,
                       unshuffle: int = 1) -> dict:
    """The seeded weights every parity case and benchmark uses."""
    torch.manual_seed(seed)
    m = TVSpecNetOracle(depth, channels, out_bands) if unshuffle == 1 else UnshuffledOracle(depth, channels, out_bands)
    for mod in m.modules():
        if isinstance(mod, nn.Conv2d):
            nn.init.kaiming_normal_(mod.weight, mode="fan_in", nonlinearity="relu")
    return {k: v.detach().clone() for k, v in m.state_dict().items()}


def oracle_from_state(state: dict, depth: int = 17, channels: int = 64, out_bands: int = 5) -> TVSpecNetOracle:
    m = TVSpecNetOracle(depth, channels, out_bands)
    m.load_state_dict(state)
    return m.eval()


@torch.no_grad()
def forward_batched(model: nn.Module, x: np.ndarray | torch.Tensor, chunk: int = 1) -> np.ndarray:
    """Oracle forward over a (B,1,H,W) batch, ``chunk`` images at a time."""
    xt = torch.as_tensor(x, dtype=torch.float32)
    outs = [model(xt[i : i + chunk]) for i in range(0, xt.shape[0], chunk)]
    return torch.cat(outs).numpy()


def predict_bands(model, image: np.ndarray) -> np.ndarray:
    """inference.py:25-32: one (h, w) image -> (k, h, w)."""
    if image.ndim != 2:
        raise ValueError(f"expected a 2-D image, got shape {image.shape}")
    with torch.no_grad():
        x = torch.from_numpy(np.ascontiguousarray(image, dtype=np.float32))
        out = model(x[None, None])[0]
    return out.numpy()


def complete_planes(image: np.ndarray, bands: np.ndarray) -> np.ndarray:
    """inference.py:34-42: [input, bands..., input - sum(bands)] as <f4."""
    closure = image[None] - bands.sum(axis=0, keepdims=True)
    return np.concatenate([image[None], bands, closure]).astype("<f4")


def bench_forward(model, sizes, repeats: int = 3, seed: int = 0) -> list[dict]:
    """inference.py:80-93: best of ``repeats`` perf_counter runs per size."""
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


def band_rel_l2(pred: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Relative L2 per (image, band): ||pred - ref|| / ||ref|| over H, W."""
    pred = np.asarray(pred, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    num = np.sqrt(((pred - ref) ** 2).sum(axis=(-2, -1)))
    den = np.sqrt((ref**2).sum(axis=(-2, -1)))
    return num / np.maximum(den, 1e-300)
