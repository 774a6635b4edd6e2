"""Host-side contract of the losses drop-in (no GPU): the reference's names,
selectors, argument checks (losses.py:54-82) and the no-CPU-fallback rule."""
import dataclasses

import pytest
import torch

from paper_2006_10004_b200 import losses


def test_names_and_selectors_mirror_the_reference():
    assert losses.SELECTORS == ("L", "L1", "L2", "L3")
    assert losses.HUBER_DELTA == 0.01
    assert [f.name for f in dataclasses.fields(losses.LossValue)] == [
        "total", "mse", "sum_constraint", "gradient_huber", "skipped_bands"]
    assert set(losses.__all__) == {"LossValue", "compute_loss", "SELECTORS", "HUBER_DELTA"}


def test_argument_errors_come_before_any_device_work():
    p = torch.zeros(2, 5, 8, 8)
    with pytest.raises(ValueError, match="unknown loss selector"):
        losses.compute_loss(p, p, p[:, :1], p[:, :1], "L4")
    with pytest.raises(ValueError, match="shape mismatch"):
        losses.compute_loss(p, p[:, :3], p[:, :1], p[:, :1], "L")


@pytest.mark.skipif(torch.cuda.is_available(), reason="needs a box without a GPU")
def test_no_cpu_fallback():
    p = torch.ones(1, 2, 4, 4)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        losses.compute_loss(p, p, p[:, :1], p[:, :1], "L")
