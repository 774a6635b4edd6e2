"""Worst-band error of the wide variant's fast mode per pair schedule
(plan option wide_pair_layers) on config 5 images 0-1 against the fp32 oracle (GPU)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402

torch.set_num_threads(max(1, os.cpu_count() or 1))
state = build_seeded_state(26, 128, 5)
o = oracle_from_state(state, 26, 128, 5)
x = np.stack([make_image(CONFIGS["5w"], i) for i in range(2)])[:, None]
with torch.no_grad():
    ref = o(torch.from_numpy(x)).numpy()
for pairs in (24, 16, 12, 8, 6, 0):
    m = TVSpecNet(26, 128, 5, options={"wide_pair_layers": pairs}).eval()
    m.load_state_dict(state)
    with torch.no_grad():
        out = m(torch.from_numpy(x).cuda()).cpu().numpy()
    e = band_rel_l2(out, ref)
    print(f"pairs={pairs:2d}: worst band per image {[f'{v:.3e}' for v in e.max(axis=1)]}", flush=True)
