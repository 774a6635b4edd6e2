"""Time the pieces of the host-tensor (e2e) forward path on the GPU box."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state
from paper_2006_10004_b200 import TVSpecNet

def t(f, n=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3

x_host = torch.rand(64, 1, 256, 256).pin_memory()
xd = x_host.cuda()
out_dev = torch.empty(64, 5, 256, 256, device="cuda")
out_pin = torch.empty(64, 5, 256, 256, pin_memory=True)
print("pinned alloc 80MB  ms", t(lambda: torch.empty(64, 5, 256, 256, pin_memory=True)))
print("H2D 16MB pinned    ms", t(lambda: xd.copy_(x_host, non_blocking=True)))
print("D2H 80MB pinned    ms", t(lambda: out_pin.copy_(out_dev, non_blocking=True)))
print("D2H 80MB pageable  ms", t(lambda: out_dev.cpu()))
m = TVSpecNet().eval(); m.load_state_dict(build_seeded_state())
print("device forward     ms", t(lambda: m(xd)))
for c in (1, 2, 4, 8):
    m.host_chunks = c
    print(f"host forward c={c}  ms", t(lambda: m(x_host)))
flush = torch.empty(256 << 20 >> 2, dtype=torch.float32, device="cuda")
m.host_chunks = 4
for _ in range(2):
    m(x_host)
torch.cuda.synchronize()
for i in range(5):
    t0 = time.perf_counter()
    flush.add_(1.0)
    o = m(x_host)
    torch.cuda.synchronize()
    print("bench-like iter ms", (time.perf_counter() - t0) * 1e3)
