"""Host-side cost of the reference's batch-1 calling pattern (predict_bands:
CPU numpy image in, CPU bands out) against the device forward alone.

    python tools/batch1_probe.py
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet, predict_bands  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402

m = TVSpecNet().eval()
m.load_state_dict(build_seeded_state())
img = make_image(CONFIGS[1], 0)
x_cpu = torch.from_numpy(img)[None, None]
x_gpu = x_cpu.cuda()


def t(f, n=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


with torch.no_grad():
    print(f"predict_bands (numpy in/out)        {t(lambda: predict_bands(m, img)):.3f} ms")
    print(f"model(cpu tensor) -> cpu            {t(lambda: m(x_cpu)):.3f} ms")
    print(f"model(gpu tensor), no sync per call {t(lambda: m(x_gpu)):.3f} ms")
    plan = m._plan_for(x_gpu.device)
    bands = torch.empty((1, 5, 256, 256), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    plan.set_option("check", 2)
    print(f"plan.forward (C ABI, deferred check) {t(lambda: plan.forward(x_gpu.data_ptr(), bands.data_ptr(), 0, 1, 256, 256, 0, 256, st)):.3f} ms")
    plan.sync(st)
    plan.set_option("check", 1)

# host-side CPU time per call (no device wait inside the timed region)
def cpu_time(f, n=200):
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        tot += time.perf_counter() - t0
        torch.cuda.synchronize()
    return tot / n * 1e3


with torch.no_grad():
    plan.set_option("check", 2)
    print(f"CPU: plan.forward                    {cpu_time(lambda: plan.forward(x_gpu.data_ptr(), bands.data_ptr(), 0, 1, 256, 256, 0, 256, st)):.3f} ms")
    plan.sync(st)
    plan.set_option("check", 1)
    print(f"CPU: m._plan_for + weight key        {cpu_time(lambda: m._plan_for(x_gpu.device)):.3f} ms")
