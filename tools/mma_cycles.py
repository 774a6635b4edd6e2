"""MMA-issuer cycle accounting (plan option debug, bit 15): where the single MMA
thread of each CTA spends its time, summed over CTAs, for one forward."""
import ctypes
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet, _native  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

lib = _native.load()
lib.tvs_debug_cycles.restype = ctypes.c_int
lib.tvs_debug_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
extra = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # more debug bits (ablations)
for stack in ("1",):  # the accounting is compiled into the layer-stack kernel only
    m = TVSpecNet(options={"stack": int(stack)}).eval()
    m.load_state_dict(build_seeded_state())
    m = m.cuda()
    plan = m._plan_for(torch.device("cuda", 0))
    x = torch.from_numpy(make_batch(CONFIGS[cfg], 0, n)).cuda()
    with torch.no_grad():
        m(x)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8)()
    lib.tvs_debug_cycles(buf, 1)
    plan.set_option("debug", 32768 | extra)
    with torch.no_grad():
        m(x)
    torch.cuda.synchronize()
    plan.set_option("debug", 0)
    lib.tvs_debug_cycles(buf, 1)
    tot = buf[0] or 1
    print(f"stack={stack} dbg+{extra} config {cfg} x{n}: total {tot / 1e9:.3f} Gcyc (sum over CTAs); "
          f"slot wait {buf[1] / tot * 100:.1f}%, input-row wait {buf[2] / tot * 100:.1f}%, "
          f"weights wait {buf[3] / tot * 100:.1f}%, rows general {buf[4]}, fast {buf[5]}, "
          f"SM clock {buf[0] / max(1, buf[6]):.3f} GHz", flush=True)
