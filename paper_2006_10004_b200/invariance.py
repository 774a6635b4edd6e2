"""Batched GPU scoring of the invariance protocols (
/root/reference/pkg/src/spectv/invariance.py and the ``spectv invariance
--pred`` path, pkg/src/spectv/cli.py:245-339).

The reference scores every (reference band, test band) pair of every probe
image with three numpy metric calls (``_score_pairs``, invariance.py:57-72).
Here the pairs of ALL images and all three properties are built on the host
exactly as the reference builds them (same pair names, crops, merges and
per-report data range), grouped by plane shape, and scored by one
``tvs_band_stats`` launch per shape group (csrc/metrics.cu, fp64 statistics).

* ``evaluate_probe_sets``: the three protocols for a batch of images given
  their decompositions (base, 2x contrast, shifted, rotated);
* ``score_prediction_dir``: the batched ``spectv invariance --pred DIR``
  (reads ``probes.json`` and every ``<stem>[__variant].btf`` prediction);
* ``invariance_table``: the reference CSV (invariance.py:167-181).

Pair planes are formed in float64 as in the reference (``read_tensor``
followed by ``astype(np.float64)``, cli.py:214-216) and scored as float32
planes with fp64 accumulation, like ``scoring.band_metrics``.
"""

from __future__ import annotations

import csv
import io
import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .scoring import plane_stats

__all__ = ["InvarianceReport", "translate", "homogeneity_pairs", "translation_pairs", "rotation_pairs",
           "score_reports", "evaluate_probe_sets", "score_prediction_dir", "invariance_table"]

PROBE_VARIANTS = ("x2", "shift8_0", "rot90")  # cli.py:242
_R, _PATCH = 5, 16


@dataclass
class InvarianceReport:
    """One property on one image (invariance.py:44-54): ``pairs`` maps a
    comparison label to (ssim, psnr, slmse); ``averages`` is their mean."""

    property: str
    params: dict
    pairs: dict
    averages: tuple


def translate(f: np.ndarray, dx: int, dy: int) -> np.ndarray:
    """Integer shift; the entering strip repeats the edge (invariance.py:107-113)."""
    h, w = f.shape
    py, px = (max(dy, 0), max(-dy, 0)), (max(dx, 0), max(-dx, 0))
    padded = np.pad(f, (py, px), mode="edge")
    return padded[py[1]:py[1] + h, px[1]:px[1] + w]


def homogeneity_pairs(b1: np.ndarray, b2: np.ndarray) -> list:
    """Dyadic shift (invariance.py:91-104): band k of 2f against 2 x band k-1
    of f, with the low end (bands 1+2 of 2f) and the top end merged."""
    k = b1.shape[0]
    if k < 3:
        raise ValueError("dyadic shift test needs at least 3 bands")
    pairs = [("bands1+2", 2.0 * b1[0], b2[0] + b2[1])]
    pairs += [(f"band{j + 1}", 2.0 * b1[j - 1], b2[j]) for j in range(2, k - 1)]
    pairs.append((f"band{k}+res", 2.0 * (b1[k - 2] + b1[k - 1]), b2[k - 1]))
    return pairs


def translation_pairs(bands: np.ndarray, shifted: np.ndarray, shift=(8, 0)) -> list:
    """translate(decompose(f)) vs decompose(translate(f)) on the common region:
    the shift-wide strips and a one-pixel ring cropped (invariance.py:116-145)."""
    dx, dy = shift
    h, w = bands.shape[1:]
    if abs(dx) > w // 4 or abs(dy) > h // 4:
        raise ValueError("shift magnitude must stay within a quarter of the image")
    my, mx = abs(dy) + 1, abs(dx) + 1
    return [(f"band{k + 1}", translate(bands[k], dx, dy)[my:h - my, mx:w - mx], shifted[k][my:h - my, mx:w - mx])
            for k in range(bands.shape[0])]


def rotation_pairs(bands: np.ndarray, rotated: np.ndarray, angle: int = 90) -> list:
    """rot(decompose(f)) vs decompose(rot(f)) for right angles (invariance.py:148-164)."""
    if angle not in (90, 180, 270):
        raise ValueError("angle must be one of 90, 180, 270 degrees")
    turns = angle // 90
    if bands.shape[1] != bands.shape[2] and turns % 2 == 1:
        raise ValueError("90/270 degree rotation needs a square image")
    return [(f"band{k + 1}", np.rot90(bands[k], turns), rotated[k]) for k in range(bands.shape[0])]


def _pair_scores(refs: list, tests: list, ranges: list) -> list:
    """(ssim, psnr, slmse) of every (ref, test) plane pair with its data range:
    plane statistics on the GPU, one launch per distinct plane shape."""
    out = [None] * len(refs)
    groups: dict = {}
    for i, r in enumerate(refs):
        groups.setdefault(r.shape, []).append(i)
    for (H, W), idx in groups.items():
        if H - 2 * _R <= 0 or W - 2 * _R <= 0:
            raise ValueError("image too small for the 11x11 SSIM window")
        if min(H, W) < _PATCH:
            raise ValueError(f"dimension {min(H, W)} smaller than the {_PATCH}-pixel patch")
        g = torch.from_numpy(np.stack([refs[i] for i in idx]).astype(np.float32))
        p = torch.from_numpy(np.stack([tests[i] for i in idx]).astype(np.float32))
        st = plane_stats(g, p, data_range=[ranges[i] for i in idx]).cpu().numpy()
        for row, i in zip(st, idx):
            mse_sum, num, den, ssum, scnt = float(row[0]), float(row[1]), float(row[2]), float(row[5]), float(row[6])
            mse = mse_sum / (H * W)
            rng = ranges[i]
            ps = math.inf if mse == 0.0 else 10.0 * math.log10(rng * rng / mse)
            sl = (1.0 if num == 0.0 else 0.0) if den == 0.0 else 1.0 - num / den
            out[i] = (ssum / scnt, ps, sl)
    return out


def score_reports(jobs: list) -> list:
    """[(property, params, pairs)] -> [InvarianceReport], all pairs scored in
    one batch.  A report's pairs share one data range, the largest reference
    spread among them (floored at 1e-9), as in _score_pairs
    (invariance.py:57-72)."""
    refs, tests, ranges, owner = [], [], [], []
    for j, (_, _, pairs) in enumerate(jobs):
        pairs = list(pairs)
        rng = max(max((float(r.max() - r.min()) for _, r, _ in pairs), default=0.0), 1e-9)
        for name, r, t in pairs:
            if r.shape != t.shape:
                raise ValueError(f"shape mismatch: {r.shape} vs {t.shape}")
            refs.append(r)
            tests.append(t)
            ranges.append(rng)
            owner.append((j, name))
    scores = _pair_scores(refs, tests, ranges) if refs else []
    reports = [InvarianceReport(prop, params, {}, (math.nan,) * 3) for prop, params, _ in jobs]
    for (j, name), sc in zip(owner, scores):
        reports[j].pairs[name] = sc
    for rep in reports:
        vals = list(rep.pairs.values())
        rep.averages = tuple(sum(v[i] for v in vals) / len(vals) for i in range(3))
    return reports


def evaluate_probe_sets(base: list, x2: list, shifted: list, rotated: list, shift=(8, 0), angle: int = 90) -> dict:
    """The three protocols for N images at once.  Each argument is a list of
    (K, H, W) band stacks: the decompositions of f, 2f, translate(f, shift)
    and rot(f, angle).  Returns {property: [InvarianceReport per image]}."""
    if not (len(base) == len(x2) == len(shifted) == len(rotated)):
        raise ValueError("probe lists differ in length")
    jobs = []
    for b, b2, bs, br in zip(base, x2, shifted, rotated):
        jobs.append(("one-homogeneity", {"factor": 2.0}, homogeneity_pairs(b, b2)))
        jobs.append(("translation", {"shift": [shift[0], shift[1]]}, translation_pairs(b, bs, shift)))
        jobs.append(("rotation", {"angle": angle}, rotation_pairs(b, br, angle)))
    reps = score_reports(jobs)
    out = {"one-homogeneity": [], "translation": [], "rotation": []}
    for r in reps:
        out[r.property].append(r)
    return out


def score_prediction_dir(pred_dir) -> dict:
    """Batched ``spectv invariance --pred DIR`` (cli.py:314-339): every probe
    id's base / x2 / shift8_0 / rot90 prediction (BTF, planes [input, bands...])."""
    from .export import read_tensor

    pred_dir = Path(pred_dir)
    probes = json.loads((pred_dir / "probes.json").read_text())
    sets = {v: [] for v in ("",) + PROBE_VARIANTS}
    for stem in probes["ids"]:
        for v in sets:
            path = pred_dir / (f"{stem}__{v}.btf" if v else f"{stem}.btf")
            sets[v].append(read_tensor(path).astype(np.float64)[1:])
    return evaluate_probe_sets(sets[""], sets["x2"], sets["shift8_0"], sets["rot90"], shift=(8, 0), angle=90)


def invariance_table(reports: dict) -> str:
    """One column per property, each metric averaged over its reports
    (invariance.py:167-181)."""
    props = [p for p in ("one-homogeneity", "translation", "rotation") if p in reports]
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(["metric"] + props)
    for j, name in enumerate(("ssim", "psnr", "slmse")):
        w.writerow([name] + [f"{sum(r.averages[j] for r in reports[p]) / len(reports[p]):.4f}" for p in props])
    return buf.getvalue()
