"""Wide variant (128 channels, depth 26), fp32-accurate mode: the tcgen05 block
path against the CUDA-core fp32 kernels (plan option wide_cuda=1), the fp32
oracle and an fp64 reference; timing of both on config 5-wide images.

    python tools/wide_fp32_probe.py [--images 4]
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=4)
    args = ap.parse_args()
    state = build_seeded_state(26, 128, 5)
    o32 = oracle_from_state(state, 26, 128, 5)
    o64 = oracle_from_state(state, 26, 128, 5).double()
    models = {}
    for name, opts in (("tcgen05", {}), ("cuda", {"wide_cuda": 1})):
        m = TVSpecNet(26, 128, 5, precision="fp32", options=opts).eval()
        m.load_state_dict(state)
        models[name] = m
    for shape in ((128, 128), (37, 300), (2, 130), (200, 64)):
        x = make_image(CONFIGS["5w"], 1)[None, None, : shape[0], : shape[1]].copy()
        if x.shape[-1] < shape[1]:
            x = np.tile(x, (1, 1, 1, 2))[..., : shape[1]].copy()
        with torch.no_grad():
            y32 = o32(torch.from_numpy(x)).numpy()
            y64 = o64(torch.from_numpy(x).double()).numpy()
        for name, m in models.items():
            with torch.no_grad():
                out = m(torch.from_numpy(x).cuda()).cpu().numpy()
            print(f"{shape} {name}: vs fp64 {band_rel_l2(out, y64).max():.3e}  vs fp32 oracle "
                  f"{band_rel_l2(out, y32).max():.3e}  (oracle vs fp64 {band_rel_l2(y32, y64).max():.3e}) "
                  f"launches {m.last_launch_count()}", flush=True)
    xs = np.stack([make_image(CONFIGS["5w"], i) for i in range(args.images)])[:, None]
    xd = torch.from_numpy(xs).cuda()
    for name, m in models.items():
        n = 1 if name == "cuda" else 5
        with torch.no_grad():
            m(xd)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(n):
                m(xd)
            torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        print(f"{name}: {args.images} x 512^2 in {dt * 1e3:.2f} ms = {xs.size / dt / 1e6:.1f} MP/s", flush=True)


if __name__ == "__main__":
    main()
