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
if "--configs" in sys.argv:
    from paper_2006_10004_b200.workloads import CONFIGS, make_batch

    ora = oracle_from_state(state)
    for cfg, n, crop in ((3, 1, None), (5, 2, None), (4, 1, (0, 0, 512, 1024))):
        x = make_batch(CONFIGS[cfg], 0, n)
        if crop:
            y0, x0, h, w = crop
            x = np.ascontiguousarray(x[:, :, y0:y0 + h, x0:x0 + w])
        with torch.no_grad():
            ref = ora(torch.from_numpy(x)).numpy()
            out = m(torch.from_numpy(x).cuda()).cpu().numpy()
        e = band_rel_l2(out, ref)
        print(f"cfg{cfg}{'crop' if crop else ''} worst {e.max():.3e} mean {e.mean():.3e}", flush=True)
