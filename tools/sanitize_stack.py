"""Small forwards for compute-sanitizer (memcheck / racecheck / synccheck):
the layer-stack kernel (row flags between CTAs, cooperative launch) on a
ragged two-strip shape, then the per-layer kernels, each compared bitwise.

    compute-sanitizer --tool synccheck python tools/sanitize_stack.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402

state = build_seeded_state()
x = torch.rand(2, 1, 12, 200, generator=torch.Generator().manual_seed(1)).cuda()
outs = []
for stack in (1, 0):
    m = TVSpecNet(options={"stack": stack}).eval()
    m.load_state_dict(state)
    with torch.no_grad():
        outs.append(m(x))
    print(f"stack={stack}: used_stack={m.last_used_stack()} launches={m.last_launch_count()}", flush=True)
torch.cuda.synchronize()
print("bitwise", torch.equal(outs[0], outs[1]), flush=True)
