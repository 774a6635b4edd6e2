"""Emulate per-layer activation formats for the wide variant (128 feature maps,
depth 26) in fast mode, against the fp32 oracle.

A hidden layer whose INPUT is stored as an fp16 hi/lo pair sees fp32-exact
activations (the kernel runs A_hi*W + A_lo*W); a single-fp16 input costs half
the MMA work but rounds the activations.  Weights are the tap-sum compensated
fp16 pack (conv_tc.cu dc_round9); conv0 and the head are exact.

Usage: python tools/emulate_wide.py [--images 2] [--size 512]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402
from tools.emulate_precision import dc_round_fp16, fold  # noqa: E402


def e4m3(t):
    """Round to float8 e4m3 (saturating), back to float32."""
    return t.clamp(-448.0, 448.0).to(torch.float8_e4m3fn).float()


def run(layers, x, pair_in, lo_fp8=False):
    """pair_in[j] (j = 0..n_hidden-1): hidden layer j reads its input as an
    fp16 hi/lo pair (A_hi W + A_lo W, fp32-exact activations).  lo_fp8: the
    lo half is stored as e4m3(lo 2^11) and its product runs on e4m3 weights
    (W 2^10), the kind::f8f6f4 candidate for the pair layers."""
    a = torch.from_numpy(x).float()
    n = len(layers)
    wq = [None] + [dc_round_fp16(w).float() for (w, _) in layers[1:-1]] + [None]
    w8 = [None] + [e4m3(w.float() * 1024.0) / 1024.0 for (w, _) in layers[1:-1]] + [None]
    for i, (w, b) in enumerate(layers):
        if i == 0 or i == n - 1:
            y = F.conv2d(a, w.float(), None, padding=1)
        elif pair_in[i - 1] and lo_fp8:
            hi = a.half().float()
            lo = e4m3((a - hi) * 2048.0) / 2048.0
            y = F.conv2d(hi, wq[i], None, padding=1) + F.conv2d(lo, w8[i], None, padding=1)
        else:
            ain = a if pair_in[i - 1] else a.half().float()
            y = F.conv2d(ain, wq[i], None, padding=1)
        y = y + b.float()[None, :, None, None]
        if i < n - 1:
            y = torch.relu(y)
        a = y
    return a.numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=2)
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--fp8", action="store_true", help="compare fp16-lo and e4m3-lo pair layers")
    args = ap.parse_args()
    torch.set_num_threads(8)
    depth, ch = 26, 128
    nh = depth - 2
    state = build_seeded_state(depth, ch, 5)
    model = oracle_from_state(state, depth, ch, 5)
    layers = fold(state, depth)
    schemes = {
        "all pair": [True] * nh,
        "all f16": [False] * nh,
        "alternate": [j % 2 == 0 for j in range(nh)],
        "pair first 12": [j < 12 for j in range(nh)],
        "pair last 12": [j >= 12 for j in range(nh)],
        "pair 1 in 3": [j % 3 == 0 for j in range(nh)],
        "pair 2 in 3": [j % 3 != 2 for j in range(nh)],
        "pair first 6": [j < 6 for j in range(nh)],
        "pair last 6": [j >= nh - 6 for j in range(nh)],
    }
    if args.fp8:
        schemes = {"pair first 12": [j < 12 for j in range(nh)], "pair first 16": [j < 16 for j in range(nh)],
                   "all pair": [True] * nh}
    for idx in range(args.images):
        img = make_image(CONFIGS["5w"], idx)[None, None][..., : args.size, : args.size].copy()
        with torch.no_grad():
            ref = model(torch.from_numpy(img)).numpy()
            cref = img[:, 0] - ref.sum(1)
            line = [f"img{idx}"]
            for name, sch in schemes.items():
                for lo8 in ((False, True) if args.fp8 else (False,)):
                    out = run(layers, img, sch, lo8)
                    e = band_rel_l2(out, ref).max()
                    c = band_rel_l2((img[:, 0] - out.sum(1))[:, None], cref[:, None]).max()
                    line.append(f"{name} ({sum(sch)}/{nh}){' e4m3-lo' if lo8 else ''}: {e:.3e}/{c:.2e}")
                    print(line[0], line[-1], flush=True)


if __name__ == "__main__":
    main()
