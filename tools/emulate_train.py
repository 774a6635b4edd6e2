"""CPU emulation behind the training step's precision split (DESIGN §12,
csrc/train.cu header): which roundings to fp16 the gradients of one
reference training step (training.py:45-61, compute_loss L3) tolerate.

For the seeded 17-layer model on the fixture batch it reports the worst
per-tensor relative L2 distance of the parameter gradients from the float64
step, for
  * the float32 step (the reference itself: the conditioning floor),
  * activations rounded to fp16 in the FORWARD (every conv input),
  * hidden conv weights rounded to fp16 in the forward,
  * the BACKWARD operands rounded to fp16 (the gradient w.r.t. every hidden
    conv output, as the dgrad/wgrad kernels consume it).

    python tools/emulate_train.py
"""
import sys
from pathlib import Path

import torch
from torch import nn

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.train_oracle import compute_loss, train_batch  # noqa: E402
from oracle.tvspecnet_oracle import build_seeded_state, oracle_from_state  # noqa: E402


class _RoundFwd(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return x.half().to(x.dtype)

    @staticmethod
    def backward(ctx, g):
        return g


class _RoundBwd(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        return g.half().to(g.dtype)


def grads(dtype, act16=False, w16=False, bwd16=False):
    state = build_seeded_state()
    m = oracle_from_state(state).to(dtype).train()
    convs = [mod for mod in m.modules() if isinstance(mod, nn.Conv2d)]
    hidden = convs[1:-1]
    if w16:
        with torch.no_grad():
            for c in hidden:
                c.weight.copy_(c.weight.half().to(dtype))
    hooks = []
    for c in hidden + [convs[-1]]:
        if act16:
            hooks.append(c.register_forward_pre_hook(lambda mod, inp: (_RoundFwd.apply(inp[0]),)))
    for c in hidden:
        if bwd16:
            hooks.append(c.register_forward_hook(lambda mod, inp, out: _RoundBwd.apply(out)))
    img, gt, res = (t.to(dtype) for t in train_batch())
    v = compute_loss(m(img), gt, img, res, "L3")
    v.total.backward()
    for h in hooks:
        h.remove()
    return {n: p.grad.double().clone() for n, p in m.named_parameters()}


def worst(g, ref):
    return max(float(torch.linalg.vector_norm(g[n] - ref[n]) / torch.linalg.vector_norm(ref[n]).clamp_min(1e-300))
               for n in ref)


if __name__ == "__main__":
    torch.set_num_threads(8)
    g64 = grads(torch.float64)
    for name, kw in (("fp32 step (reference)", dict(dtype=torch.float32)),
                     ("fp16 forward activations", dict(dtype=torch.float64, act16=True)),
                     ("fp16 forward hidden weights", dict(dtype=torch.float64, w16=True)),
                     ("fp16 backward operands", dict(dtype=torch.float64, bwd16=True))):
        print(f"{name:30s} worst gradient rel-L2 vs fp64: {worst(grads(**kw), g64):.3e}", flush=True)
