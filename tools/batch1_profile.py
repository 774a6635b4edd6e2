"""cProfile of the batch-1 host path (predict_bands and model(gpu tensor)).

    python tools/batch1_profile.py
"""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet, predict_bands  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402

m = TVSpecNet().eval()
m.load_state_dict(build_seeded_state())
img = make_image(CONFIGS[1], 0)
x_gpu = torch.from_numpy(img)[None, None].cuda()
with torch.no_grad():
    for name, f in (("predict_bands", lambda: predict_bands(m, img)), ("model(gpu)", lambda: m(x_gpu))):
        for _ in range(20):
            f()
        torch.cuda.synchronize()
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(500):
            f()
        pr.disable()
        torch.cuda.synchronize()
        print("=====", name, "(500 calls)")
        pstats.Stats(pr).sort_stats("tottime").print_stats(18)
