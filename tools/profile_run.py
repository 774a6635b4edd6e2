"""Small driver for ncu: a few fast-mode forwards of one config (default 2).

    python tools/profile_run.py [--config 2] [--iters 3] [--precision fast] [--batch N]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--precision", default="fast")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--unshuffle", type=int, default=1)
a = ap.parse_args()
spec = CONFIGS[a.config if a.config == "5w" else int(a.config)]
B = a.batch or spec.batch
m = TVSpecNet(spec.depth, spec.channels, 5, precision=a.precision, unshuffle=a.unshuffle).eval()
m.load_state_dict(build_seeded_state(spec.depth, spec.channels, 5, unshuffle=a.unshuffle))
x = torch.rand(B, 1, spec.height, spec.width, device="cuda")
for _ in range(a.iters):
    y = m(x)
torch.cuda.synchronize()
print("ok", tuple(y.shape), "launches/forward", m.last_launch_count())
