"""Sweep the host-tensor (e2e) forward's sub-batch schedule on config 2:
pinned input -> CPU result, timed like bench.py's e2e leg (L2 flush between
steps, perf_counter around synchronized steps)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

x_host = torch.from_numpy(make_batch(CONFIGS[2], 0, 64)).pin_memory()
m = TVSpecNet().eval()
m.load_state_dict(build_seeded_state())
flush = torch.empty(256 << 20 >> 2, dtype=torch.float32, device="cuda")
xd = x_host.cuda()


def timeit(f, n=8):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        flush.add_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e3, ts[0] * 1e3


px = x_host.numel() / 1e6
med, mn = timeit(lambda: m(xd))
print(f"device forward: median {med:.3f} ms ({px / med * 1e3:.0f} MP/s)", flush=True)
for sched in [None, 4, (2, 1, 1), (4, 39, 17, 4), (3, 38, 14, 6, 2, 1), (2, 38, 16, 6, 2), None]:
    m.host_chunks = sched
    med, mn = timeit(lambda: m(x_host))
    print(f"host_chunks={sched}: median {med:.3f} ms ({px / med * 1e3:.0f} MP/s), min {mn:.3f}", flush=True)
