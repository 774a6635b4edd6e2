"""Event timeline of the host-tensor forward's sub-batch pipeline (config 2):
H2D / forward / D2H start+end per sub-batch, in ms from the first H2D."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

x_pin = torch.from_numpy(make_batch(CONFIGS[2], 0, 64)).pin_memory()
m = TVSpecNet().eval()
m.load_state_dict(build_seeded_state())
m = m.cuda()
plan = m._plan_for(torch.device("cuda", 0))
B, K, H, W = 64, 5, 256, 256
out = torch.empty((B, K, H, W), pin_memory=True)


def run(sched, rec=True):
    w = [float(v) for v in sched]
    cuts = [0] + [round(B * sum(w[:i + 1]) / sum(w)) for i in range(len(w))]
    bounds = [(cuts[i], cuts[i + 1]) for i in range(len(w)) if cuts[i + 1] > cuts[i]]
    per = max(e - s for s, e in bounds)
    comp = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    xbuf = [torch.empty((per, 1, H, W), device="cuda") for _ in range(2)]
    bbuf = [torch.empty((per, K, H, W), device="cuda") for _ in range(2)]
    x_free = [torch.cuda.Event() for _ in range(2)]
    b_free = [torch.cuda.Event() for _ in range(2)]
    for ev in x_free + b_free:
        ev.record(comp)
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = E()
    t0.record(comp)
    marks = []
    for i, (s, e) in enumerate(bounds):
        j, nb = i % 2, e - s
        h2d.wait_event(x_free[j])
        a1, a2, c1, c2, d1, d2 = E(), E(), E(), E(), E(), E()
        with torch.cuda.stream(h2d):
            a1.record(h2d)
            xbuf[j][:nb].copy_(x_pin[s:e], non_blocking=True)
            a2.record(h2d)
        comp.wait_event(a2)
        comp.wait_event(b_free[j])
        c1.record(comp)
        plan.forward(xbuf[j].data_ptr(), bbuf[j].data_ptr(), 0, nb, H, W, 0, H, comp.cuda_stream)
        c2.record(comp)
        x_free[j].record(comp)
        d2h.wait_event(c2)
        with torch.cuda.stream(d2h):
            d1.record(d2h)
            out[s:e].copy_(bbuf[j][:nb], non_blocking=True)
            d2.record(d2h)
        b_free[j].record(d2h)
        marks.append((nb, a1, a2, c1, c2, d1, d2))
    torch.cuda.synchronize()
    if rec:
        print(f"schedule {sched}: total {t0.elapsed_time(marks[-1][6]):.3f} ms")
        for nb, *ev in marks:
            print("   %2d imgs  H2D %.3f-%.3f  fwd %.3f-%.3f  D2H %.3f-%.3f" % ((nb,) + tuple(t0.elapsed_time(x) for x in ev)))


for sched in [(1,), (3, 1), (2, 1, 1), (1, 1, 1, 1), (6, 3, 2, 1)]:
    run(sched, False)
    run(sched)
