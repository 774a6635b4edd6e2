"""A/B driver for plan options (include/tvs_b200.h tvs_plan_set_option).

Builds the default model and one with the given options, checks their outputs
for bitwise equality on ragged shapes and on a BASELINE config batch, then
times interleaved CUDA-event forwards of that batch (device-resident input,
L2 flushed between forwards).

    python tools/ab.py stack=0 [conv0_tc=0 ...] [--config 2] [--imgs 64] [--reps 20]
                       [--precision fast|fp32] [--wide 1]

Options that change numerics on purpose (e.g. wide_pair_layers) report
AB_MISMATCH; everything else must print AB_OK.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

opts = {k: int(v) for k, v in (a.split("=", 1) for a in sys.argv[1:] if "=" in a and not a.startswith("--"))}
flags = {sys.argv[i]: sys.argv[i + 1] for i in range(1, len(sys.argv) - 1) if sys.argv[i].startswith("--")}
nimg = int(flags.get("--imgs", 64))
reps = int(flags.get("--reps", 20))
cfg = flags.get("--config", "2")
cfg = cfg if cfg == "5w" else int(cfg)
prec = flags.get("--precision", "fast")
wide = flags.get("--wide", "0") == "1"


def model(options):
    arch = dict(depth=26, channels=128) if wide else {}
    m = TVSpecNet(**arch, precision=prec, options=options).eval()
    m.load_state_dict(build_seeded_state(**arch))
    return m.cuda()


m0, m1 = model({}), model(opts)
ok = True
for (n, h, w) in [(2, 48, 160), (1, 37, 300), (3, 64, 128), (1, 5, 7), (2, 1, 130)]:
    x = torch.rand(n, 1, h, w, generator=torch.Generator().manual_seed(h * w)).cuda()
    with torch.no_grad():
        y0, y1 = m0(x), m1(x)
    eq = torch.equal(y0, y1)
    ok &= eq
    print(f"{n}x{h}x{w}: bitwise {eq} max diff {(y0 - y1).abs().max().item():.3e}", flush=True)
x = torch.from_numpy(make_batch(CONFIGS[cfg], 0, nimg)).cuda()
with torch.no_grad():
    y0, y1 = m0(x), m1(x)
eq = torch.equal(y0, y1)
ok &= eq
print(f"config {cfg} x{nimg}: bitwise {eq}, stack {m0.last_used_stack()} / {m1.last_used_stack()}, "
      f"launches {m0.last_launch_count()} / {m1.last_launch_count()}", flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
t = {0: [], 1: []}
px = x.numel() / 1e6
# forwards through the C-ABI plans with deferred status checks (as bench.py):
# no host synchronisation or Python inside the timed region
st = torch.cuda.current_stream().cuda_stream
B, _, H, W = x.shape
outs = {}
for i, m in ((0, m0), (1, m1)):
    plan = m._plan_for(x.device)
    plan.set_option("check", 2)
    outs[i] = (plan, torch.empty((B, 5, H, W), device=x.device), torch.empty((B, 1, H, W), device=x.device))
for r in range(reps + 3):
    for i in (0, 1):
        plan, bands, clos = outs[i]
        flush.fill_(r & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.forward(x.data_ptr(), bands.data_ptr(), clos.data_ptr(), B, H, W, 0, H, st)
        b.record()
        torch.cuda.synchronize()
        if r >= 3:
            t[i].append(a.elapsed_time(b))
for i in (0, 1):
    outs[i][0].sync(st)
    outs[i][0].set_option("check", 1)
for i in (0, 1):
    v = sorted(t[i])
    print(f"{'default' if i == 0 else opts}: median {v[len(v)//2]:.3f} ms ({px / v[len(v)//2] * 1e3:.1f} MP/s), "
          f"min {v[0]:.3f} ms", flush=True)
print("AB_OK" if ok else "AB_MISMATCH")
