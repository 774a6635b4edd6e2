"""End-to-end (CPU tensors in and out) forward time of config 2 under several
host sub-batch schedules (TVSpecNet.host_chunks), interleaved, L2 flushed:
calibrates model._host_schedule.

    python tools/host_sched_sweep.py [--reps 8]
"""
import json
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

flags = {sys.argv[i]: sys.argv[i + 1] for i in range(1, len(sys.argv) - 1) if sys.argv[i].startswith("--")}
reps = int(flags.get("--reps", "8"))
x = torch.from_numpy(make_batch(CONFIGS[2], 0, 64)).pin_memory()
m = TVSpecNet().eval()
m.load_state_dict(build_seeded_state())
flush = torch.empty(256 << 20 >> 2, device="cuda")
scheds = [None, [4, 39, 17, 4], [2, 46, 12, 4], [4, 44, 12, 4], [4, 48, 12], [4, 52, 8], [2, 50, 8, 4],
          [8, 44, 8, 4], [64], [1, 51, 8, 4], [4, 42, 10, 6, 2]]
times = {str(s): [] for s in scheds}
with torch.no_grad():
    for s in scheds:  # warm-up: plans, staging buffers, item tables per sub-batch shape
        m.host_chunks = s
        for _ in range(2):
            m.forward_planes(x)
    torch.cuda.synchronize()
    for _ in range(reps):
        for s in scheds:
            m.host_chunks = s
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m.forward_planes(x)
            torch.cuda.synchronize()
            times[str(s)].append(time.perf_counter() - t0)
auto = m._sched_cache if hasattr(m, "_sched_cache") else {}
for s in scheds:
    v = times[str(s)]
    print(json.dumps({"schedule": s if s is not None else f"auto {list(auto.values())}",
                      "median_ms": round(1e3 * statistics.median(v), 3), "min_ms": round(1e3 * min(v), 3),
                      "mp_s": round(64 * 65536 / 1e3 / statistics.median(v) / 1e3, 1)}), flush=True)
