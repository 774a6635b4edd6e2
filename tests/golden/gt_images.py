"""Deterministic source images for the ground-truth dataset fixtures (shared by
make_golden_tvflow.py and the tests; PNG is lossless so pixels are exact)."""

from pathlib import Path

import numpy as np


def make_images(d) -> list:
    from PIL import Image

    d = Path(d)
    d.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(77)
    yy, xx = np.mgrid[0:40, 0:50]
    rgb = np.stack([(xx * 5) % 256, (yy * 6) % 256, rng.integers(0, 256, (40, 50))], axis=-1).astype(np.uint8)
    gray = (128 + 60 * np.sin(np.mgrid[0:36, 0:33][1] / 3.0) + rng.normal(0, 10, (36, 33))).clip(0, 255)
    paths = [d / "a.png", d / "b.png"]
    Image.fromarray(rgb, "RGB").save(paths[0])
    Image.fromarray(gray.astype(np.uint8), "L").save(paths[1])
    return paths


GT_KW = dict(count=5, seed=3, crop_size=16, augment_fraction=0.5)
GT_CFG = dict(dt=0.2, n_steps=12, schedule=(2, 5, 11))
