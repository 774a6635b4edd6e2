"""A/B of plan knobs (env vars read at plan creation): bitwise comparison of the
outputs against the default plan on several shapes and on config 2, then
interleaved CUDA-event timing of config 2 forwards (device-resident input).

    python tools/ab_env.py TVS_DIRECT=1 [TVS_STACK=0 ...] [--imgs 64] [--reps 20]
"""
import ctypes
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet, _native  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402


PREC = "fast"


def model(env, wide=False):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    arch = dict(depth=26, channels=128) if wide else {}
    m = TVSpecNet(**arch, precision=PREC).eval()
    m.load_state_dict(build_seeded_state(**arch) if wide else build_seeded_state())
    m = m.cuda()
    m._plan_for(torch.device("cuda", 0))
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    return m


args = [a for a in sys.argv[1:] if "=" in a and not a.startswith("--")]
env = dict(a.split("=", 1) for a in args)
opt = {sys.argv[i]: sys.argv[i + 1] for i in range(1, len(sys.argv) - 1) if sys.argv[i].startswith("--")}
nimg = int(opt.get("--imgs", 64))
reps = int(opt.get("--reps", 20))
cfg = int(opt.get("--config", 2))
PREC = opt.get("--precision", "fast")
lib = _native.load()
lib.tvs_debug_stack.restype = ctypes.c_int
lib.tvs_debug_stack.argtypes = [ctypes.c_int]
WIDE = opt.get("--wide", "0") == "1"
m0, m1 = model({}, WIDE), model(env, WIDE)
RUNTIME = ("TVS_CONV_DBG", "TVS_PAIR_DBG")  # read at every launch, not at plan creation


class Rt:
    """Forward wrapper that sets the launch-time knobs around m1's calls."""

    def __init__(self, m, env):
        self.m, self.env = m, {k: v for k, v in env.items() if k in RUNTIME}

    def __call__(self, x):
        os.environ.update(self.env)
        try:
            return self.m(x)
        finally:
            for k in self.env:
                os.environ.pop(k)

    def last_launch_count(self):
        return self.m.last_launch_count()


m1 = Rt(m1, env)
ok = True
for (n, h, w) in [(2, 48, 160), (1, 37, 300), (3, 64, 128), (1, 5, 7), (2, 1, 130)]:
    x = torch.rand(n, 1, h, w, generator=torch.Generator().manual_seed(h * w)).cuda()
    with torch.no_grad():
        y0, y1 = m0(x), m1(x)
    torch.cuda.synchronize()
    eq = torch.equal(y0, y1)
    ok &= eq
    print(f"{n}x{h}x{w}: bitwise {eq} max diff {(y0 - y1).abs().max().item():.3e}", flush=True)
x = torch.from_numpy(make_batch(CONFIGS[cfg], 0, nimg)).cuda()
with torch.no_grad():
    y0, y1 = m0(x), m1(x)
torch.cuda.synchronize()
wd = lib.tvs_debug_stack(1)
eq = torch.equal(y0, y1)
ok &= eq and wd == 0
print(f"config {cfg} x{nimg}: bitwise {eq}, watchdog {wd}, launches {m0.last_launch_count()} / {m1.last_launch_count()}",
      flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
t = {0: [], 1: []}
px = x.numel() / 1e6
for r in range(reps + 3):
    for i, m in ((0, m0), (1, m1)):
        flush.fill_(r & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.no_grad():
            a.record()
            m(x)
            b.record()
        torch.cuda.synchronize()
        if r >= 3:
            t[i].append(a.elapsed_time(b))
for i in (0, 1):
    v = sorted(t[i])
    print(f"{'default' if i == 0 else env}: median {v[len(v)//2]:.3f} ms ({px / v[len(v)//2] * 1e3:.1f} MP/s), "
          f"min {v[0]:.3f} ms", flush=True)
print("AB_OK" if ok else "AB_MISMATCH")
