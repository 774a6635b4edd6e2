"""The B200 training step (csrc/train.cu via the drop-in's train() mode)
against the reference step fixtures (tests/golden/golden_train.npz, made by
executing /root/reference's TVSpecNet + compute_loss).

Tolerances: the gradients of this seeded 17-layer BN network
are ill-conditioned - the reference's own fp32 gradients are 5.3e-3 (rel-L2,
worst tensor) from its fp64 step.  The B200 step (fp32-accurate split
forward, fp16 backward operands) must land within 2e-2 of the fp64 step for
every parameter tensor; losses within 1e-5 and running statistics within
1e-5 of the reference.
"""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.train_oracle import compute_loss, train_batch
from oracle.tvspecnet_oracle import build_seeded_state, oracle_from_state
from paper_2006_10004_b200 import TVSpecNet

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "golden_train.npz"
GRAD_TOL = 2e-2


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _step(m, sel, device):
    img, gt, res = (t.to(device) for t in train_batch())
    v = compute_loss(m(img), gt, img, res, sel)
    v.total.backward()
    return v


@pytest.mark.parametrize("device", ["cuda", "cpu"])  # cpu: the reference's calling convention (CPU params/tensors)
def test_train_step_matches_reference(gold, device):
    m = TVSpecNet()
    m.load_state_dict(build_seeded_state())
    m = m.to(device).train()
    v = _step(m, "L3", device)
    assert abs(v.total.item() - gold["loss_L3"]) <= 1e-5 * abs(gold["loss_L3"])
    worst, worst32 = 0.0, 0.0
    for n, p in m.named_parameters():
        g = p.grad.detach().cpu().numpy()
        worst = max(worst, _rel(g, gold[f"grad64_{n}"]))
        worst32 = max(worst32, _rel(g, gold[f"grad_{n}"]))
    print(f"[{device}] worst gradient rel-L2 vs fp64 {worst:.3e}, vs reference fp32 {worst32:.3e}")
    assert worst <= GRAD_TOL, worst
    bns = [mod for mod in m.modules() if isinstance(mod, torch.nn.BatchNorm2d)]
    for j, bn in enumerate(bns):
        np.testing.assert_allclose(bn.running_mean.cpu().numpy(), gold[f"rmean_{j}"], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(bn.running_var.cpu().numpy(), gold[f"rvar_{j}"], rtol=1e-5, atol=1e-6)
        assert int(bn.num_batches_tracked) == 1


@pytest.mark.parametrize("sel", ["L", "L1", "L2"])
def test_train_step_selectors(gold, sel):
    m = TVSpecNet()
    m.load_state_dict(build_seeded_state())
    m = m.cuda().train()
    v = _step(m, sel, "cuda")
    assert abs(v.total.item() - gold[f"loss_{sel}"]) <= 1e-5 * abs(gold[f"loss_{sel}"])
    for _, p in m.named_parameters():
        assert torch.isfinite(p.grad).all()


def _adam_run(model, dev, dtype, steps=3):
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    losses = []
    for it in range(steps):
        img, gt, res = (t.to(dev, dtype) for t in train_batch(seed=10 + it, B=2, H=40, W=36))
        opt.zero_grad(set_to_none=True)
        v = compute_loss(model(img), gt, img, res, "L")
        v.total.backward()
        opt.step()
        losses.append(v.total.item())
    model.eval()
    img, _, _ = train_batch(seed=99, B=1, H=48, W=48)
    with torch.no_grad():
        y = model(img.to(dev, dtype)).double().cpu()
    return losses, y


def test_epoch_pass_with_adam_tracks_reference_within_its_own_fp32_floor():
    """Three _epoch_pass iterations (training.py:45-61) with Adam(lr=1e-3).
    Adam's normalised steps amplify the gradients' conditioning: the oracle's
    own fp32 run drifts from its fp64 run by 2e-3 in the third loss and 30% in
    the eval output afterwards.  The drop-in must stay within 4x that floor
    of the fp64 run."""
    state = build_seeded_state()
    ours = TVSpecNet()
    ours.load_state_dict(state)
    lo, yo = _adam_run(ours.cuda().train(), "cuda", torch.float32)
    l32, y32 = _adam_run(oracle_from_state(state).train(), "cpu", torch.float32)
    l64, y64 = _adam_run(oracle_from_state(state).double().train(), "cpu", torch.float64)
    print("losses ours", lo, "fp32", l32, "fp64", l64)
    assert abs(lo[0] - l64[0]) <= 1e-5 * abs(l64[0])
    for i in range(1, 3):
        assert abs(lo[i] - l64[i]) <= 4 * abs(l32[i] - l64[i]) + 1e-4 * abs(l64[i]), i
    floor = torch.linalg.vector_norm(y32 - y64).item()
    assert torch.linalg.vector_norm(yo - y64).item() <= 4 * floor + 1e-3 * torch.linalg.vector_norm(y64).item()


def test_ragged_shapes_and_forward_backward_pairing():
    m = TVSpecNet(depth=5, out_bands=3)
    m.load_state_dict(build_seeded_state(5, 64, 3))
    m = m.cuda().train()
    ref = oracle_from_state(build_seeded_state(5, 64, 3), 5, 64, 3).train()
    g = torch.Generator().manual_seed(5)
    for shape in ((1, 1, 7, 300), (3, 1, 130, 9), (2, 1, 1, 1)):
        x = torch.randn(*shape, generator=g)
        m.zero_grad()
        ref.zero_grad()
        (m(x.cuda()) ** 2).mean().backward()
        (ref(x) ** 2).mean().backward()
        for (n, p), (_, q) in zip(m.named_parameters(), ref.named_parameters()):
            if q.grad.abs().max() == 0:
                continue
            assert _rel(p.grad.cpu().numpy(), q.grad.numpy()) < 3e-2, (shape, n)
    out1 = m(torch.randn(1, 1, 8, 8, device="cuda"))
    m(torch.randn(1, 1, 8, 8, device="cuda"))  # a second forward replaces the plan's saved activations
    with pytest.raises(RuntimeError, match="older forward"):
        out1.sum().backward()


@pytest.mark.parametrize("shape", [(2, 32, 32), (3, 37, 150), (1, 5, 7)])
def test_wgrad_tcgen05_matches_cublas(shape):
    """The tcgen05 weight-gradient kernel (csrc/wgrad_tc.cu, MN-major operands
    straight from the pixel-major buffers) against one cuBLAS split-K GEMM per
    tap (train option wgrad_tc=0): same fp16 operands and fp32 accumulation,
    only the summation order differs (and tcgen05 truncates its fp32 accumulator
    once per MMA, tools/probe_mma_rounding.cu): measured <= 2.2e-5, gated at 1e-4."""
    B, H, W = shape
    grads = {}
    for tc in (1, 0):
        m = TVSpecNet()
        m.load_state_dict(build_seeded_state())
        m = m.cuda().train()
        m._train_plan(0).set_option("wgrad_tc", tc)
        m._train_plan(0).set_option("head_dgrad_tc", 0)  # same fp32 head dgrad in both arms
        img, gt, res = (t.cuda() for t in train_batch(seed=7, B=B, H=H, W=W))
        compute_loss(m(img), gt, img, res, "L").total.backward()
        grads[tc] = {n: p.grad.detach().cpu().numpy() for n, p in m.named_parameters()}
    for n, g in grads[1].items():
        assert np.isfinite(g).all(), n
        assert _rel(g, grads[0][n]) <= 1e-4, (n, _rel(g, grads[0][n]))


def test_head_dgrad_on_tcgen05_stays_inside_the_fp16_backward_budget(gold):
    """The head's input gradient on the hidden layers' tcgen05 dgrad kernel
    (fp16 operands, train option head_dgrad_tc, default) against the fp32
    CUDA-core kernel: both within the gradient gate of the fp64 step, and the
    two apart by no more than the fp16-backward budget (9.7e-4
    emulated for fp16 backward operands)."""
    worst = {}
    grads = {}
    for tc in (1, 0):
        m = TVSpecNet()
        m.load_state_dict(build_seeded_state())
        m = m.cuda().train()
        m._train_plan(0).set_option("head_dgrad_tc", tc)
        _step(m, "L3", "cuda")
        grads[tc] = {n: p.grad.detach().cpu().numpy() for n, p in m.named_parameters()}
        worst[tc] = max(_rel(g, gold[f"grad64_{n}"]) for n, g in grads[tc].items())
    print(f"worst gradient rel-L2 vs fp64: tcgen05 head dgrad {worst[1]:.3e}, CUDA-core {worst[0]:.3e}")
    assert worst[1] <= GRAD_TOL and worst[0] <= GRAD_TOL
    assert max(_rel(g, grads[0][n]) for n, g in grads[1].items()) <= 5e-3


@pytest.mark.parametrize("shape", [(2, 32, 32), (3, 37, 150), (1, 5, 7), (2, 1, 1)])
def test_fused_batch_statistics_match_the_separate_pass(shape):
    """BatchNorm's batch sums from the forward conv's epilogue (train option
    bn_fused, default) against the separate pass over the conv output: same
    values summed in a different order (fp32 over a warp's 32 pixels, then
    fp64), so outputs, running statistics and gradients agree closely."""
    B, H, W = shape
    res = {}
    for fused in (1, 0):
        m = TVSpecNet()
        m.load_state_dict(build_seeded_state())
        m = m.cuda().train()
        m._train_plan(0).set_option("bn_fused", fused)
        img, gt, r = (t.cuda() for t in train_batch(seed=8, B=B, H=H, W=W))
        out = m(img)
        compute_loss(out, gt, img, r, "L").total.backward()
        bns = [mod for mod in m.modules() if isinstance(mod, torch.nn.BatchNorm2d)]
        res[fused] = (out.detach().cpu().numpy(), [bn.running_var.cpu().numpy() for bn in bns],
                      {n: p.grad.detach().cpu().numpy() for n, p in m.named_parameters()})
    np.testing.assert_allclose(res[1][1][0], res[0][1][0], rtol=1e-5, atol=1e-7)  # first layer: same input
    if B * H * W <= 2:
        # two samples per channel: the normalised values are +-1 whatever the data and the
        # variance is rounding noise, so later layers amplify last-bit differences
        assert np.isfinite(res[1][0]).all()
        return
    assert _rel(res[1][0], res[0][0]) <= 1e-5  # measured 1.5-2.1e-6
    for a, b in zip(res[1][1], res[0][1]):
        np.testing.assert_allclose(a, b, rtol=1e-4, atol=1e-6)
    # last-bit differences of the statistics move these ill-conditioned gradients by ~1.3e-3
    # (measured, deterministic run to run); the reference's own fp32-vs-fp64 distance is 5.3e-3
    for n, g in res[1][2].items():
        assert _rel(g, res[0][2][n]) <= 5e-3, (n, _rel(g, res[0][2][n]))


@pytest.mark.parametrize("shape", [(2, 32, 32), (3, 37, 150), (1, 5, 7)])
def test_bn_backward_cooperative_launch_matches_two_kernels(shape):
    """BatchNorm backward's reduction and apply passes in one cooperative launch
    (train option bn_bwd_fused, default) against the two-kernel path: the same
    code on either side of a grid barrier instead of a kernel boundary; only the
    order of the fp64 atomics differs."""
    B, H, W = shape
    grads = {}
    for fused in (1, 0):
        m = TVSpecNet()
        m.load_state_dict(build_seeded_state())
        m = m.cuda().train()
        m._train_plan(0).set_option("bn_bwd_fused", fused)
        img, gt, res = (t.cuda() for t in train_batch(seed=12, B=B, H=H, W=W))
        compute_loss(m(img), gt, img, res, "L3").total.backward()
        grads[fused] = {n: p.grad.detach().cpu().numpy() for n, p in m.named_parameters()}
    for n, g in grads[1].items():
        assert np.isfinite(g).all(), n
        assert _rel(g, grads[0][n]) <= 1e-5, (n, _rel(g, grads[0][n]))
