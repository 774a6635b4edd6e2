"""Training-step throughput: one `_epoch_pass` iteration
of the reference loop (training.py:45-61: zero_grad, model(img), compute_loss,
backward, Adam step; TrainConfig batch_size 8) through the drop-in's train()
mode on B200, against the same step of the CPU oracle module (torch autograd,
all host threads) on the same batch.

    python tools/bench_train.py [--size 128] [--batch 8] [--steps 20] [--cpu-steps 2] [--loss fused|torch]
                                [--train-opts bn_fused=0,...]

--loss torch runs the GPU arm with the reference's own torch-op loss on CUDA
tensors instead of the fused drop-in (paper_2006_10004_b200.losses).

Prints one JSON line: steps/s and MP/s (pixels trained per second) for both.
"""
import json
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.train_oracle import compute_loss as oracle_loss, train_batch  # noqa: E402
from oracle.tvspecnet_oracle import build_seeded_state, oracle_from_state  # noqa: E402
from paper_2006_10004_b200 import TVSpecNet  # noqa: E402
from paper_2006_10004_b200.losses import compute_loss as fused_loss  # noqa: E402

flags = {sys.argv[i]: sys.argv[i + 1] for i in range(1, len(sys.argv) - 1) if sys.argv[i].startswith("--")}
S = int(flags.get("--size", 128))
B = int(flags.get("--batch", 8))
steps = int(flags.get("--steps", 20))
cpu_steps = int(flags.get("--cpu-steps", 2))
state = build_seeded_state()


loss_kind = flags.get("--loss", "fused")


def run(model, dev, n, warm, compute_loss):
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    img, gt, res = (t.to(dev) for t in train_batch(seed=3, B=B, H=S, W=S))
    loss = None
    for it in range(warm + n):
        if it == warm:
            if dev == "cuda":
                torch.cuda.synchronize()
            t0 = time.perf_counter()
        opt.zero_grad(set_to_none=True)
        v = compute_loss(model(img), gt, img, res, "L")
        v.total.backward()
        opt.step()
        loss = float(v.total.detach())  # the loop reads the loss every step (training.py:56)
    if dev == "cuda":
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n, loss


m = TVSpecNet()
m.load_state_dict(state)
for kv in filter(None, flags.get("--train-opts", "").split(",")):  # e.g. --train-opts bn_fused=0,wgrad_tc=0
    name, val = kv.split("=")
    m._train_plan(0).set_option(name, int(val))
t_gpu, loss_gpu = run(m.cuda().train(), "cuda", steps, 3, fused_loss if loss_kind == "fused" else oracle_loss)
torch.set_num_threads(os.cpu_count() or 1)
px = B * S * S / 1e6
ref = None
if cpu_steps > 0:  # --cpu-steps 0: GPU arm only
    t_cpu, loss_cpu = run(oracle_from_state(state).train(), "cpu", cpu_steps, 1, oracle_loss)
    ref = {"value": round(1.0 / t_cpu, 4), "unit": "steps/s", "ms_per_step": round(t_cpu * 1e3, 1),
           "mp_per_s": round(px / t_cpu, 4), "steps": cpu_steps, "cores": torch.get_num_threads(),
           "last_loss": loss_cpu, "note": "CPU oracle module (torch autograd fp32), same batch, same loop"}
print(json.dumps({
    "metric": "TVSpecNET training step (forward + compute_loss + backward + Adam)", "unit": "steps/s",
    "value": round(1.0 / t_gpu, 2), "ms_per_step": round(t_gpu * 1e3, 3), "mp_per_s": round(px / t_gpu, 2),
    "batch": B, "size": [S, S], "steps": steps, "selector": "L", "loss": loss_kind, "last_loss": loss_gpu,
    "reference_flow": ref,
}))
