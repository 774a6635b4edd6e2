"""Determinism soak of the layer-stack paths: repeated forwards of config 2
(whole-column items) and config 1 (row-band items) must reproduce the first
output bitwise (the row-flag protocol has no benign races to hide).

    python tools/soak.py [--reps2 300] [--reps1 3000]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_batch  # noqa: E402

flags = {sys.argv[i]: sys.argv[i + 1] for i in range(1, len(sys.argv) - 1) if sys.argv[i].startswith("--")}
m = TVSpecNet().eval()
m.load_state_dict(build_seeded_state())
bad = 0
with torch.no_grad():
    for cfg, reps in ((2, int(flags.get("--reps2", 300))), (1, int(flags.get("--reps1", 3000)))):
        x = torch.from_numpy(make_batch(CONFIGS[cfg], 0, CONFIGS[cfg].batch)).cuda()
        ref = m(x).clone()
        assert m.last_used_stack()
        n_bad = 0
        for i in range(reps):
            if not torch.equal(m(x), ref):
                n_bad += 1
        torch.cuda.synchronize()
        print(f"config {cfg}: {reps} forwards, {n_bad} differing from the first")
        bad += n_bad
print("SOAK_OK" if bad == 0 else "SOAK_MISMATCH")
sys.exit(0 if bad == 0 else 1)
