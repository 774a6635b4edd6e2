"""Golden fixtures of one reference training step.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden_train.py

Executes the REFERENCE TVSpecNet (model.py:29-56) in train() mode and the
REFERENCE compute_loss (losses.py:54-129) on oracle.train_oracle.train_batch
(seed 1, 2 x 32 x 32, 5 bands) with the seeded weights of
oracle.build_seeded_state, and stores:
  * loss_<sel>          the total loss for each selector L, L1, L2, L3
  * grad_<name>         every parameter gradient of the L3 loss (float32)
  * rmean_<j>, rvar_<j> BatchNorm running statistics after that step
  * loss64_L3, grad64_* the same step in float64 (the conditioning floor)
"""

import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/trainer/src")

from tvsurrogate.losses import compute_loss  # noqa: E402  (reference)
from tvsurrogate.model import TVSpecNet  # noqa: E402  (reference)

from oracle.train_oracle import train_batch  # noqa: E402
from oracle.tvspecnet_oracle import build_seeded_state  # noqa: E402


def main():
    torch.set_num_threads(8)
    state = build_seeded_state()
    img, gt, res = train_batch()
    out = {"img": img.numpy(), "gt": gt.numpy(), "res": res.numpy()}
    for sel in ("L", "L1", "L2", "L3"):
        m = TVSpecNet()
        m.load_state_dict(state)
        m.train()
        v = compute_loss(m(img), gt, img, res, sel)
        v.total.backward()
        out[f"loss_{sel}"] = np.float64(v.total.item())
        if sel == "L3":
            for n, p in m.named_parameters():
                out[f"grad_{n}"] = p.grad.numpy().astype(np.float32)
            bns = [mod for mod in m.modules() if isinstance(mod, torch.nn.BatchNorm2d)]
            for j, bn in enumerate(bns):
                out[f"rmean_{j}"] = bn.running_mean.numpy().copy()
                out[f"rvar_{j}"] = bn.running_var.numpy().copy()
    m = TVSpecNet().double()
    m.load_state_dict({k: v.double() if v.is_floating_point() else v for k, v in state.items()})
    m.train()
    v = compute_loss(m(img.double()), gt.double(), img.double(), res.double(), "L3")
    v.total.backward()
    out["loss64_L3"] = np.float64(v.total.item())
    for n, p in m.named_parameters():
        out[f"grad64_{n}"] = p.grad.numpy().astype(np.float32)
    np.savez_compressed(HERE / "golden_train.npz", **out)
    print("wrote", HERE / "golden_train.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
