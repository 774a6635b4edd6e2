"""Sweep the layer-stack item shape (plan options stack / stack_band_rows /
stack_skew) on BASELINE configs: median CUDA-event forward time over `reps`
forwards of device-resident input, L2 flushed between forwards, each variant
checked bitwise against the per-layer path.

    python tools/stack_sweep.py --config 1 --imgs 1 --reps 30 --rows 0,8,12,16,24,32,64 [--skews 0,2]

Prints one JSON line per variant (rows 0 = the auto choice).
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

flags = {sys.argv[i]: sys.argv[i + 1] for i in range(1, len(sys.argv) - 1) if sys.argv[i].startswith("--")}
cfg = int(flags.get("--config", "1"))
nimg = int(flags.get("--imgs", CONFIGS[cfg].batch))
reps = int(flags.get("--reps", 30))
rows = [int(r) for r in flags.get("--rows", "0,8,16,32").split(",")]
skews = [int(o) for o in flags.get("--skews", "1").split(",")]
chunk = int(flags.get("--chunk-mb", "0"))
state = build_seeded_state()
x = torch.from_numpy(make_batch(CONFIGS[cfg], 0, nimg)).cuda()
flush = torch.empty(256 << 20 >> 2, device="cuda")


def timed(m):
    """Forwards through the C-ABI plan (as bench.py: deferred status checks,
    no Python in the timed region); returns the bands and the times (ms)."""
    dev = x.device
    B, _, H, W = x.shape
    bands = torch.empty((B, 5, H, W), device=dev)
    plan = m._plan_for(dev)
    plan.set_option("check", 2)
    st = torch.cuda.current_stream().cuda_stream

    def step():
        plan.forward(x.data_ptr(), bands.data_ptr(), 0, B, H, W, 0, H, st)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    plan.sync(st)
    plan.set_option("check", 1)
    return bands.clone(), ts


def model(opts):
    if chunk:
        opts = dict(opts, chunk_mb=chunk)
    m = TVSpecNet(options=opts).eval()
    m.load_state_dict(state)
    return m.cuda()


m0 = model({"stack": 0})
y0, t0 = timed(m0)
px = x.shape[0] * x.shape[2] * x.shape[3]
print(json.dumps({"config": cfg, "imgs": nimg, "variant": "per-layer", "median_ms": round(statistics.median(t0), 4),
                  "min_ms": round(min(t0), 4), "mp_s": round(px / 1e3 / statistics.median(t0), 2)}), flush=True)
for _ in [0]:
  for o in skews:
    for r in rows:
        m = model({"stack": 1, "stack_band_rows": r, "stack_skew": o})
        y, t = timed(m)
        print(json.dumps({"config": cfg, "imgs": nimg, "variant": f"stack rows={r} skew={o}",
                          "median_ms": round(statistics.median(t), 4), "min_ms": round(min(t), 4),
                          "mp_s": round(px / 1e3 / statistics.median(t), 2), "bitwise": bool(torch.equal(y, y0)),
                          "used_stack": bool(m.last_used_stack())}), flush=True)
mauto = model({})
y, t = timed(mauto)
print(json.dumps({"config": cfg, "imgs": nimg, "variant": "default (auto)", "median_ms": round(statistics.median(t), 4),
                  "mp_s": round(px / 1e3 / statistics.median(t), 2), "bitwise": bool(torch.equal(y, y0)),
                  "used_stack": bool(mauto.last_used_stack())}), flush=True)
