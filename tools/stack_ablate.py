"""Stack timing under ablation debug bits (results of some bits are invalid;
timing only): median plan-level forward time per variant.

    python tools/stack_ablate.py --config 1 --imgs 1 --rows 6 --bits 0,1048576,2097152
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
nimg = int(flags.get("--imgs", "1"))
rows = int(flags.get("--rows", "0"))
reps = int(flags.get("--reps", "20"))
bits = [int(b) for b in flags.get("--bits", "0").split(",")]
x = torch.from_numpy(make_batch(CONFIGS[cfg], 0, nimg)).cuda()
flush = torch.empty(256 << 20 >> 2, device="cuda")
B, _, H, W = x.shape
m = TVSpecNet(options={"stack": 1, "stack_band_rows": rows}).eval()
m.load_state_dict(build_seeded_state())
plan = m._plan_for(x.device)
plan.set_option("check", 0)
bands = torch.empty((B, 5, H, W), device="cuda")
st = torch.cuda.current_stream().cuda_stream
for b in bits:
    plan.set_option("debug", b)
    ts = []
    for i in range(reps + 3):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.forward(x.data_ptr(), bands.data_ptr(), 0, B, H, W, 0, H, st)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    print(json.dumps({"config": cfg, "imgs": nimg, "rows": rows, "debug": b,
                      "median_ms": round(statistics.median(ts), 4), "min_ms": round(min(ts), 4)}), flush=True)
