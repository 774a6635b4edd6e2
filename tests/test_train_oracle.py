"""The training-step oracle (oracle/train_oracle.py) against the reference's
own training step, executed in the build container into
tests/golden/golden_train.npz (make_golden_train.py): losses of every
selector, the L3 gradients and the BatchNorm running statistics."""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.train_oracle import compute_loss, train_batch
from oracle.tvspecnet_oracle import build_seeded_state, oracle_from_state

GOLD = Path(__file__).resolve().parent / "golden" / "golden_train.npz"


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def test_batch_is_the_fixture_batch(gold):
    img, gt, res = train_batch()
    assert np.array_equal(img.numpy(), gold["img"]) and np.array_equal(gt.numpy(), gold["gt"])
    assert np.array_equal(res.numpy(), gold["res"])


@pytest.mark.parametrize("sel", ["L", "L1", "L2", "L3"])
def test_oracle_step_matches_reference(gold, sel):
    torch.set_num_threads(8)
    m = oracle_from_state(build_seeded_state()).train()
    img, gt, res = train_batch()
    v = compute_loss(m(img), gt, img, res, sel)
    assert abs(v.total.item() - gold[f"loss_{sel}"]) <= 1e-6 * abs(gold[f"loss_{sel}"])
    if sel != "L3":
        return
    v.total.backward()
    for n, p in m.named_parameters():
        ref = gold[f"grad_{n}"]
        np.testing.assert_allclose(p.grad.numpy(), ref, rtol=1e-4, atol=1e-6 * np.abs(ref).max())
    bns = [mod for mod in m.modules() if isinstance(mod, torch.nn.BatchNorm2d)]
    for j, bn in enumerate(bns):
        np.testing.assert_allclose(bn.running_mean.numpy(), gold[f"rmean_{j}"], rtol=1e-5, atol=1e-7)
        np.testing.assert_allclose(bn.running_var.numpy(), gold[f"rvar_{j}"], rtol=1e-5, atol=1e-7)


def test_reference_fp32_gradient_conditioning(gold):
    """The reference's own fp32 gradients vs its fp64 step: the floor any
    implementation is compared against."""
    worst = max(np.linalg.norm(gold[k] - gold[k.replace("grad_", "grad64_")]) / np.linalg.norm(gold[k.replace("grad_", "grad64_")])
                for k in gold if k.startswith("grad_"))
    assert worst < 2e-2
    print(f"reference fp32 vs fp64 worst gradient rel-L2: {worst:.2e}")
