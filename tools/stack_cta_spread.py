"""Per-CTA start / end of the layer-stack kernel (kDbgTrace stamps) on a
BASELINE config: how long SMs idle at the launch's tail.

    python tools/stack_cta_spread.py --config 2 [--imgs 64]
"""
import ctypes
import os
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_10004_b200 import build as _build  # noqa: E402

os.environ["TVS_LIB"] = str(_build.build(trace=True))  # the row timeline is compiled in only here
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet, _native  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

flags = {sys.argv[i]: sys.argv[i + 1] for i in range(1, len(sys.argv) - 1) if sys.argv[i].startswith("--")}
cfg = int(flags.get("--config", "2"))
nimg = int(flags.get("--imgs", CONFIGS[cfg].batch))
lib = _native.load()
lib.tvs_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * (5 * 32 * 1024))()
m = TVSpecNet(options={"stack": 1}).eval()
m.load_state_dict(build_seeded_state())
x = torch.from_numpy(make_batch(CONFIGS[cfg], 0, nimg)).cuda()
with torch.no_grad():
    m(x)
    torch.cuda.synchronize()
    lib.tvs_debug_trace(buf, 1)
    m.set_plan_option("debug", 1 << 19)
    m(x)
    torch.cuda.synchronize()
lib.tvs_debug_trace(buf, 1)
t = np.frombuffer(buf, dtype=np.uint64).reshape(5, 32, 1024)
st, en = t[0, 31].astype(np.float64), t[1, 31].astype(np.float64)
n = int((en > 0).sum())
st, en = st[:n], en[:n]
t0 = st.min()
st, en = (st - t0) / 1e3, (en - t0) / 1e3
print(json.dumps({"config": cfg, "imgs": nimg, "ctas": n, "start_us": [round(float(st.min()), 2), round(float(st.max()), 2)],
                  "end_us_min": round(float(en.min()), 2), "end_us_median": round(float(np.median(en)), 2),
                  "end_us_max": round(float(en.max()), 2),
                  "idle_tail_frac": round(float((en.max() - en).sum() / (n * en.max())), 4),
                  "end_us_deciles": [round(float(v), 1) for v in np.percentile(en, np.arange(0, 101, 10))]}))
