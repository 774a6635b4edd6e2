"""Quick GPU bring-up check: parity of both modes vs the CPU oracle on a few
shapes, then a rough timing of the fast mode on config 2.  Prints one line
per case; not part of the test suite."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402

torch.set_num_threads(8)
state = build_seeded_state()
oracle = oracle_from_state(state)
cases = [("rand 2x16x20", np.random.default_rng(0).standard_normal((2, 1, 16, 20)).astype(np.float32)),
         ("rand 1x32x40", np.random.default_rng(1).standard_normal((1, 1, 32, 40)).astype(np.float32)),
         ("rand 1x5x300", np.random.default_rng(2).random((1, 1, 5, 300)).astype(np.float32)),
         ("cfg1", make_image(CONFIGS[1], 0)[None, None]),
         ("cfg2[0:2]", np.stack([make_image(CONFIGS[2], i) for i in range(2)])[:, None])]
for prec in ("fast", "fp32"):
    m = TVSpecNet(precision=prec).eval()
    m.load_state_dict(state)
    for name, x in cases:
        with torch.no_grad():
            ref = oracle(torch.from_numpy(x)).numpy()
            xd = torch.from_numpy(x).cuda()
            bands, clos = m.forward_planes(xd, closure=True)
            torch.cuda.synchronize()
        out = bands.cpu().numpy()
        e = band_rel_l2(out, ref)
        cref = x[:, 0] - ref.sum(1)
        ce = band_rel_l2(clos.cpu().numpy()[:, 0:1], cref[:, None]).max()
        finite = np.isfinite(out).all()
        print(f"PARITY {prec:4s} {name:14s} worst_band={e.max():.3e} closure={ce:.3e} finite={finite}", flush=True)

# rough timing, fast mode, config 2 (64 x 256^2)
m = TVSpecNet(precision="fast").eval()
m.load_state_dict(state)
x = torch.rand(64, 1, 256, 256, device="cuda")
for _ in range(3):
    m(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
n = 10
for _ in range(n):
    m(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
mp = 64 * 256 * 256 / 1e6 / (ms / 1e3)
print(f"TIMING fast cfg2 {ms:.3f} ms/forward  {mp:.1f} MP/s  {mp*1e6*1112832/1e12:.1f} TFLOP/s  launches={m.last_launch_count()}")
