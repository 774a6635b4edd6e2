"""Train-mode forward and backward of the drop-in TVSpecNet on B200.

The reference trains the module with torch autograd on the CPU
(/root/reference/pkg/trainer/src/tvsurrogate/training.py:45-61,
``_epoch_pass``: ``model.train()``, ``compute_loss(model(img), ...)``,
``value.total.backward()``, ``optimizer.step()``).  The drop-in keeps that
calling contract: in ``train()`` mode ``TVSpecNet.forward`` runs
``TrainForward``, an autograd Function whose forward and backward are the
C-ABI training step (``tvs_train_forward`` / ``tvs_train_backward``,
csrc/train.cu), so the reference loop, its losses and its Adam optimizer work
unchanged on the module's parameters (CPU or CUDA).

BatchNorm2d semantics (model.py:41, train mode): normalisation by the batch
mean and biased variance; running_mean / running_var move towards the batch
mean and unbiased variance with the layer's momentum; num_batches_tracked
counts steps.  Those buffer updates happen here, from the statistics the
kernels return.
"""

from __future__ import annotations

import torch
from torch import nn

from . import _native


def _layers(model):
    """(conv0, [(conv_j, bn_j)], head) of the reference body layout (cached per
    module list: the walk is ~50 us and a step asks three times)."""
    mods = tuple(model.body._modules.values())
    cache = model.__dict__.get("_train_layers")
    if cache is None or cache[0] != mods:
        convs = [m for m in mods if isinstance(m, nn.Conv2d)]
        bns = [m for m in mods if isinstance(m, nn.BatchNorm2d)]
        cache = (mods, (convs[0], list(zip(convs[1:-1], bns)), convs[-1]))
        model.__dict__["_train_layers"] = cache
    return cache[1]


def train_params(model) -> list[torch.Tensor]:
    """The parameters the step differentiates, in a fixed order:
    conv0.weight, conv0.bias, (conv_j.weight, bn_j.weight, bn_j.bias)*, head.weight, head.bias."""
    c0, hidden, head = _layers(model)
    out = [c0.weight, c0.bias]
    for conv, bn in hidden:
        out += [conv.weight, bn.weight, bn.bias]
    return out + [head.weight, head.bias]


def _stage_params(model, params, dev) -> list[torch.Tensor]:
    """fp32 contiguous device copies of the parameters.  Parameters already on
    the device are used in place.  CPU parameters (the reference's convention:
    training.py builds the model on the CPU) are gathered into one pinned buffer
    and cross PCIe in ONE copy; one copy per tensor cost ~2.5 ms per step."""
    if all(p.device == dev for p in params):
        return [p.detach().to(torch.float32).contiguous() for p in params]
    if not all(p.device.type == "cpu" and p.dtype == torch.float32 for p in params):
        return [p.detach().to(dev, torch.float32).contiguous() for p in params]
    sizes = [p.numel() for p in params]
    total = sum(sizes)
    cache = model.__dict__.setdefault("_train_stage", {})
    key = (dev.index, total)
    if cache.get("key") != key:
        cache.clear()
        cache.update(key=key, pin=torch.empty(total, dtype=torch.float32, pin_memory=True),
                     dev=torch.empty(total, dtype=torch.float32, device=dev), landed=torch.cuda.Event())
    else:
        cache["landed"].synchronize()  # the previous step's copy has left the pinned buffer
    torch.cat([p.detach().reshape(-1) for p in params], out=cache["pin"])
    # (the device buffer is reused every step: the previous step's kernels that read it are
    # ordered before this copy on the same stream)
    cache["dev"].copy_(cache["pin"], non_blocking=True)
    cache["landed"].record(torch.cuda.current_stream(dev))
    return [t.view(p.shape) for t, p in zip(cache["dev"].split(sizes), params)]


class TrainForward(torch.autograd.Function):
    @staticmethod
    def forward(ctx, model, x, *params):
        dev = model._exec_device(x)
        idx = dev.index
        plan = model._train_plan(idx)
        nh = model.depth - 2
        with torch.cuda.device(idx):
            stream = torch.cuda.current_stream(idx)
            staged = _stage_params(model, params, dev)
            xd = x.detach().to(dev, torch.float32).contiguous()
            w = [staged[0]] + [staged[2 + 3 * j] for j in range(nh)] + [staged[-2]]
            bias = [staged[1]] + [None] * nh + [staged[-1]]
            gamma = [staged[3 + 3 * j] for j in range(nh)]
            beta = [staged[4 + 3 * j] for j in range(nh)]
            B, _, H, W = xd.shape
            out = torch.empty((B, model.out_bands, H, W), device=dev)
            mean = torch.empty((max(nh, 1), 64), device=dev)
            var = torch.empty((max(nh, 1), 64), device=dev)
            _, hidden, _ = _layers(model)
            eps = hidden[0][1].eps if hidden else 1e-5
            plan.forward([t.data_ptr() for t in w], [0 if t is None else t.data_ptr() for t in bias],
                         [t.data_ptr() for t in gamma], [t.data_ptr() for t in beta], eps, xd.data_ptr(),
                         out.data_ptr(), mean.data_ptr(), var.data_ptr(), B, H, W, stream.cuda_stream)
            model._train_step_id = getattr(model, "_train_step_id", 0) + 1
            ctx.step_id = model._train_step_id
        _update_running_stats(model, mean, var)
        ctx.model, ctx.plan, ctx.dev = model, plan, dev
        ctx.keep = (staged, xd, w, gamma, beta)  # the plan reads these device pointers in backward
        ctx.param_devices = [(p.device, p.dtype) for p in params]
        ctx.shapes = [p.shape for p in params]
        return out if x.is_cuda else out.to(x.device)

    @staticmethod
    def backward(ctx, g_out):
        model, plan, dev = ctx.model, ctx.plan, ctx.dev
        if getattr(model, "_train_step_id", None) != ctx.step_id:
            raise RuntimeError("TVSpecNet (B200) training: backward of an older forward; the train plan keeps "
                               "one step's activations (run forward and backward in pairs)")
        nh = model.depth - 2
        idx = dev.index
        with torch.cuda.device(idx):
            stream = torch.cuda.current_stream(idx)
            g = g_out.detach().to(dev, torch.float32).contiguous()
            # one allocation for all gradients (49 torch.empty calls cost 0.35 ms of a host-bound step)
            sizes = [s.numel() for s in ctx.shapes]
            flat = torch.empty(sum(sizes), device=dev, dtype=torch.float32)
            grads = [g_.view(s) for g_, s in zip(flat.split(sizes), ctx.shapes)]
            dw = [grads[0]] + [grads[2 + 3 * j] for j in range(nh)] + [grads[-2]]
            dbias = [grads[1]] + [None] * nh + [grads[-1]]
            dgamma = [grads[3 + 3 * j] for j in range(nh)]
            dbeta = [grads[4 + 3 * j] for j in range(nh)]
            plan.backward(g.data_ptr(), [t.data_ptr() for t in dw], [0 if t is None else t.data_ptr() for t in dbias],
                          [t.data_ptr() for t in dgamma], [t.data_ptr() for t in dbeta], stream.cuda_stream)
        homes = set(ctx.param_devices)
        if len(homes) == 1 and next(iter(homes)) == (torch.device("cpu"), torch.float32):
            # the reference keeps its parameters on the CPU: one D2H of the flat gradient
            # buffer instead of one per tensor (49 small copies cost ~2 ms per step)
            out = [g_.view(s) for g_, s in zip(flat.cpu().split(sizes), ctx.shapes)]
        else:
            out = [gr.to(d, dt) for gr, (d, dt) in zip(grads, ctx.param_devices)]
        ctx.keep = None
        return (None, None, *out)


@torch.no_grad()
def _update_running_stats(model, mean: torch.Tensor, var: torch.Tensor) -> None:
    """BatchNorm2d train-mode buffer updates (torch semantics: momentum, or the
    cumulative average when momentum is None).  Layers sharing one momentum
    (the usual case) are updated with multi-tensor ops: five launches per step
    instead of five per layer (the step is host-bound at the reference's batch
    size, tools/bench_train.py)."""
    _, hidden, _ = _layers(model)
    tracked = [(j, bn) for j, (_, bn) in enumerate(hidden) if bn.track_running_stats]
    if not tracked:
        return
    torch._foreach_add_([bn.num_batches_tracked for _, bn in tracked], 1)
    groups: dict = {}
    for j, bn in tracked:
        if bn.momentum is None:  # cumulative moving average: 1 / num_batches_tracked
            m = 1.0 / float(bn.num_batches_tracked.item())
        else:
            m = float(bn.momentum)
        groups.setdefault((m, bn.running_mean.device, bn.running_mean.dtype), []).append((j, bn))
    for (m, dev, dt), items in groups.items():
        mean_d, var_d = mean.to(dev, dt), var.to(dev, dt)
        rms = [bn.running_mean for _, bn in items]
        rvs = [bn.running_var for _, bn in items]
        torch._foreach_mul_(rms, 1.0 - m)
        torch._foreach_add_(rms, [mean_d[j] for j, _ in items], alpha=m)
        torch._foreach_mul_(rvs, 1.0 - m)
        torch._foreach_add_(rvs, [var_d[j] for j, _ in items], alpha=m)


def new_train_plan(model, idx: int) -> _native.TrainPlan:
    if model.channels != 64 or model.unshuffle != 1:
        raise NotImplementedError("the B200 training step is built for the reference architecture (64 channels)")
    return _native.TrainPlan(idx, model.depth, model.out_bands)
