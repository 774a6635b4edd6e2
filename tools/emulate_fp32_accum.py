"""Emulate fp32-mode accumulation schemes vs the fp32 oracle (worst band rel-L2).
  A: fp64 everything (current CUDA-core path, activations rounded to fp32)
  B: fp32 partial sums per 16-input-channel block (144 terms), blocks summed in fp64
  C: plain fp32 (one conv2d in fp32)"""
import sys
from pathlib import Path
import numpy as np
import torch
import torch.nn.functional as F
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state  # noqa
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa

torch.set_num_threads(8)
state = build_seeded_state()
model = oracle_from_state(state)
layers = []
for w, s, b in __import__("paper_2006_10004_b200").TVSpecNet().eval().__class__.layer_params(
        (lambda m: (m.load_state_dict(state), m)[1])(__import__("paper_2006_10004_b200").TVSpecNet().eval())):
    layers.append((w, s, b))


def run(x, scheme):
    a = torch.from_numpy(x).float()
    n = len(layers)
    for i, (w, s, b) in enumerate(layers):
        cin = w.shape[1]
        if scheme == "A":
            y = F.conv2d(a.double(), w.double(), padding=1)
        elif scheme == "C":
            y = F.conv2d(a, w.float(), padding=1).double()
        else:
            blk = 16 if cin >= 16 else cin
            y = sum(F.conv2d(a[:, c:c + blk], w[:, c:c + blk].float(), padding=1).double() for c in range(0, cin, blk))
        if s is not None:
            y = y * s[None, :, None, None]
        y = y + b[None, :, None, None]
        if i < n - 1:
            y = torch.relu(y)
        a = y.float()
    return a.numpy()


for name, spec, idx in [("cfg1", CONFIGS[1], 0), ("cfg3", CONFIGS[3], 0)]:
    x = make_image(spec, idx)[None, None]
    with torch.no_grad():
        ref = model(torch.from_numpy(x)).numpy()
        out = {k: run(x, k) for k in "ABC"}
    print(name, {k: f"{band_rel_l2(v, ref).max():.2e}" for k, v in out.items()}, flush=True)
