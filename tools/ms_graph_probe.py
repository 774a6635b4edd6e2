"""GPU-side time of the multi-stream chunked forward with host launch overhead
removed (CUDA-graph capture of one plan.forward)."""
import os, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state
from paper_2006_10004_b200 import TVSpecNet

B = 64
x = torch.rand(B, 1, 256, 256, device="cuda")
bands = torch.empty(B, 5, 256, 256, device="cuda")
clos = torch.empty(B, 1, 256, 256, device="cuda")
m = TVSpecNet().eval()
m.load_state_dict(build_seeded_state())
plan = m._plan_for(torch.device("cuda", 0))
s = torch.cuda.Stream()

def step():
    plan.forward(x.data_ptr(), bands.data_ptr(), clos.data_ptr(), B, 256, 256, 0, 256, torch.cuda.current_stream().cuda_stream)

with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
torch.cuda.synchronize()
for name, fn in (("eager", step), ("graph", g.replay)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{os.environ.get('TVS_STREAMS')} {os.environ.get('TVS_L2_CHUNK_MB')} {name}: {ms:.3f} ms  {B*65536/ms/1e3:.1f} MP/s  host {(time.perf_counter()-t0)/10*1e3:.3f} ms")
