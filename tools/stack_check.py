"""Layer-stack kernel (TVS_STACK, conv_tc.cu mode 8) vs the per-layer kernels:
bitwise comparison on several shapes, the row-flag watchdog, and timing."""
import ctypes
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet, _native  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402


def model(stack, **env):
    env = {"TVS_STACK": str(stack), **env}
    os.environ.update(env)
    m = TVSpecNet().eval()
    m.load_state_dict(build_seeded_state())
    m = m.cuda()
    m._plan_for(torch.device("cuda", 0))
    for k in env:
        os.environ.pop(k)
    return m


lib = _native.load()
lib.tvs_debug_stack.restype = ctypes.c_int
lib.tvs_debug_stack.argtypes = [ctypes.c_int]
m0, m1 = model(0), model(1)
shapes = [(2, 48, 160), (1, 37, 300), (3, 64, 128), (4, 256, 256), (1, 5, 7)]
ok = True
for (n, h, w) in shapes:
    x = torch.rand(n, 1, h, w, generator=torch.Generator().manual_seed(h * w)).cuda()
    with torch.no_grad():
        y0 = m0(x)
        y1 = m1(x)
    torch.cuda.synchronize()
    err = lib.tvs_debug_stack(1)
    eq = torch.equal(y0, y1)
    ok &= eq and err == 0
    print(f"{n}x{h}x{w}: launches {m0.last_launch_count()} vs {m1.last_launch_count()}, bitwise {eq}, "
          f"max diff {(y0 - y1).abs().max().item():.3e}, watchdog {err}", flush=True)
nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x = torch.from_numpy(make_batch(CONFIGS[2], 0, nimg)).cuda()
with torch.no_grad():
    y0 = m0(x)
    y1 = m1(x)
torch.cuda.synchronize()
err = lib.tvs_debug_stack(1)
print(f"cfg2 {nimg} imgs: bitwise {torch.equal(y0, y1)}, watchdog {err}, launches {m1.last_launch_count()}", flush=True)
import subprocess  # noqa: E402


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception as e:  # noqa: BLE001
        return f"n/a ({e})"


def timed(m, reps=10):
    with torch.no_grad():
        m(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            m(x)
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


variants = [("per-layer", m0, None), ("stack", m1, None)]
for arg in sys.argv[2:]:
    if arg.startswith("skew"):
        ms = model(1, TVS_STACK_SKEW=arg[4:])
        with torch.no_grad():
            eq = torch.equal(ms(x), y0)
        print(f"{arg}: bitwise {eq}, watchdog {lib.tvs_debug_stack(1)}", flush=True)
        variants.append((f"stack {arg}", ms, None))
    else:
        variants.append((f"stack dbg={arg}", m1, arg))
res = {n: [] for n, _, _ in variants}
for rnd in range(3):
    for name, m, dbg in variants:
        if dbg is not None:
            os.environ["TVS_CONV_DBG"] = dbg
        res[name].append(timed(m))
        os.environ.pop("TVS_CONV_DBG", None)
    print(f"round {rnd}: clocks/power {clocks()}", flush=True)
for name, ts in res.items():
    ms = sorted(ts)[len(ts) // 2]
    print(f"{name}: median {ms:.3f} ms ({', '.join(f'{t:.3f}' for t in ts)})  {x.numel()/ms/1e3:.1f} MP/s", flush=True)
print("watchdog after timing", lib.tvs_debug_stack(1))
print("ALL OK" if ok else "MISMATCH")
