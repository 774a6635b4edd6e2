"""Fused layer pairs (TVS_PAIR=1, csrc/conv_pair.cu) vs the per-layer kernels:
bitwise comparison and timing on config-2 style inputs."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402


def model(pair):
    os.environ["TVS_PAIR"] = "1" if pair else "0"
    m = TVSpecNet().eval()
    m.load_state_dict(build_seeded_state())
    m = m.cuda()
    m._plan_for(torch.device("cuda", 0))
    os.environ.pop("TVS_PAIR")
    return m


n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
hw = int(sys.argv[2]) if len(sys.argv) > 2 else 256
x = torch.from_numpy(make_batch(CONFIGS[2], 0, n)).cuda()
if hw != 256:
    x = torch.nn.functional.interpolate(x, size=(hw, hw), mode="bilinear").contiguous()
m0, m1 = model(False), model(True)
import ctypes  # noqa: E402

from paper_2006_10004_b200 import _native  # noqa: E402

dbg = (ctypes.c_int * 8)()
with torch.no_grad():
    y0 = m0(x)
    torch.cuda.synchronize()
    y1 = m1(x)
    torch.cuda.synchronize()
_native.load().tvs_debug_pair(dbg, 1)
print("pair watchdog:", list(dbg), "(abort, cta, warp, barrier id, parity, row)")
print("launches", m0.last_launch_count(), m1.last_launch_count())
print("bitwise equal:", torch.equal(y0, y1), "max abs diff", (y0 - y1).abs().max().item())
for name, m in (("per-layer", m0), ("pairs", m1)):
    with torch.no_grad():
        for _ in range(3):
            m(x)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(10):
            m(x)
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(f"{name}: {dt*1e3:.3f} ms  {x.numel()/dt/1e6:.1f} MP/s")
