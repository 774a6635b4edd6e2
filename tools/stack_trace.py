"""Row timeline of the layer-stack kernel (plan debug bit kDbgTrace = 1<<19):
for image 0, strip 0, per hidden layer, the globaltimer stamps of
  gate passed (producer) / input row landed (MMA issuer) / output row published.

    python tools/stack_trace.py --config 1 --rows 64 [--skew 2]
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
cfg = int(flags.get("--config", "1"))
rows = int(flags.get("--rows", "0"))
skew = int(flags.get("--skew", "1"))
nimg = int(flags.get("--imgs", "1"))
lib = _native.load()
lib.tvs_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * (5 * 32 * 1024))()
m = TVSpecNet(options={"stack": 1, "stack_band_rows": rows, "stack_skew": skew}).eval()
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
t = np.frombuffer(buf, dtype=np.uint64).reshape(5, 32, 1024).astype(np.float64)
H = x.shape[2]
t = t[:, :, :H]
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us since the first stamp
out = []
for j in range(m.depth - 2):
    gate, land, pub = t[0, j], t[1, j], t[2, j]
    rec = {"layer": j, "gate_first": np.nanmin(gate), "land_first": np.nanmin(land), "pub_first": np.nanmin(pub),
           "pub_last": np.nanmax(pub),
           "pub_rate_us_per_row": float(np.nanmedian(np.diff(pub))) if np.isfinite(pub).sum() > 2 else None,
           "land_to_pub_us": float(np.nanmedian(pub[:-1] - land[1:])) if np.isfinite(pub).sum() > 2 else None,
           "gate_to_land_us": float(np.nanmedian(land - gate)),
           "land_to_acc_us": float(np.nanmedian(t[3, j][:-1] - land[1:])),
           "acc_to_store_us": float(np.nanmedian(t[4, j] - t[3, j])),
           "store_to_pub_us": float(np.nanmedian(pub - t[4, j])),
           "prev_pub_to_gate_us": (float(np.nanmedian(gate[:-1] - t[2, j - 1][:-1])) if j > 0 else None)}
    out.append({k: (round(v, 2) if isinstance(v, float) else v) for k, v in rec.items()})
    print(json.dumps(out[-1]), flush=True)
np.save("gpurun_out/stack_trace.npy", t)
