"""fp32-accurate mode error per golden case on the GPU (band rel-L2 vs the
reference outputs), for comparing against tools/emulate_split_accum.py."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402

g = dict(np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "golden.npz"))
state = build_seeded_state()
xc = g["cfg1_x"][:, :, 96:160, 96:160].copy()
with torch.no_grad():
    g["crop_x"], g["crop_y"] = xc, oracle_from_state(state)(torch.from_numpy(xc)).numpy()
m = TVSpecNet(precision="fp32")
m.load_state_dict(state)
m = m.cuda().eval()
for case in ("small", "nonsq", "crop", "cfg1"):
    with torch.no_grad():
        out = m(torch.from_numpy(g[f"{case}_x"]).cuda()).cpu().numpy()
    e = band_rel_l2(out, g[f"{case}_y"])
    print(f"{case:6s} worst {e.max():.3e} mean {e.mean():.3e}", flush=True)
