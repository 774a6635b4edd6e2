"""Failure detection and numeric range of the B200 forward.

Contract (reference model.py:49-52): a forward either returns the right
values or raises.  Covered here, all through the C ABI:
  * the layer-stack watchdog: a withheld row flag (debug bit) makes the
    forward raise, and the next forward on the same plan is correct;
  * deferred status checks (plan option check=2) surface at tvs_plan_sync;
  * input magnitudes from 1e-4 to 1e4 stay within the mode's tolerance (the
    per-image power-of-two activation scale), in both precisions and on both
    the per-layer and the layer-stack paths;
  * without the scale an overflowing fast-mode forward raises
    FloatingPointError instead of returning inf; non-finite inputs propagate
    like the reference's fp32 forward.
"""
import numpy as np
import pytest
import torch

from oracle.tvspecnet_oracle import band_rel_l2, oracle_from_state
from paper_2006_10004_b200 import TVSpecNet, _native

pytestmark = pytest.mark.gpu

TOL = {"fast": 1e-2, "fp32": 1e-5}
WITHHOLD = 1 << 17  # common.cuh kDbgWithholdFlag: row 1 of (image 0, strip 0, layer 2) is never published


@pytest.fixture(scope="module")
def oracle(seeded_state):
    return oracle_from_state(seeded_state)


def _model(state, precision="fast", **opts):
    m = TVSpecNet(precision=precision, options=opts).eval()
    m.load_state_dict(state)
    return m


def test_stack_watchdog_raises_then_next_forward_is_correct(seeded_state):
    x = torch.rand(2, 1, 48, 160, generator=torch.Generator().manual_seed(5)).cuda()
    ref = _model(seeded_state, stack=0)(x)
    m = _model(seeded_state, stack=1, watchdog_ms=50)
    plan = m._plan_for(torch.device("cuda", 0))
    plan.set_option("debug", WITHHOLD)
    with pytest.raises(_native.TVSError, match="watchdog"):
        m(x)
    assert m.last_used_stack()
    plan.set_option("debug", 0)  # same plan: the status word is per forward, not sticky
    y = m(x)
    assert m.last_used_stack()
    assert torch.equal(y, ref)


def test_deferred_check_reports_at_sync(seeded_state):
    x = torch.rand(2, 1, 48, 160, generator=torch.Generator().manual_seed(6)).cuda()
    m = _model(seeded_state, stack=1, watchdog_ms=50, check=2)
    plan = m._plan_for(torch.device("cuda", 0))
    plan.set_option("debug", WITHHOLD)
    m(x)  # returns without waiting
    with pytest.raises(_native.TVSError, match="watchdog"):
        plan.sync(torch.cuda.current_stream().cuda_stream)
    plan.set_option("debug", 0)
    m(x)
    plan.sync(torch.cuda.current_stream().cuda_stream)  # nothing outstanding


@pytest.mark.parametrize("precision", ["fast", "fp32"])
@pytest.mark.parametrize("stack", [0, 1])
def test_input_scale_sweep(seeded_state, oracle, precision, stack):
    """Inputs scaled by 1e-4 .. 1e6 against the fp32 oracle on the same input."""
    if precision == "fp32" and stack == 1:
        pytest.skip("the layer stack is the fast path")
    m = _model(seeded_state, precision, stack=stack)
    base = np.random.default_rng(11).random((2, 1, 40, 150)).astype(np.float32)
    for scale in (1e-4, 1e-3, 1e-2, 1e-1, 1.0, 1e1, 1e2, 1e3, 1e4, 1e6):
        x = (base * np.float32(scale)).astype(np.float32)
        with torch.no_grad():
            ref = oracle(torch.from_numpy(x)).numpy()
        bands, clos = m.forward_planes(torch.from_numpy(x).cuda(), closure=True)
        out = bands.cpu().numpy()
        assert np.isfinite(out).all(), scale
        err = band_rel_l2(out, ref).max()
        assert err <= TOL[precision], f"scale {scale:g}: worst band rel-L2 {err:.3e}"
        cref = x - ref.sum(1, keepdims=True)
        cerr = band_rel_l2(clos.cpu().numpy(), cref).max()
        assert cerr <= TOL[precision], f"scale {scale:g}: closure rel-L2 {cerr:.3e}"


def test_in_range_inputs_are_not_rescaled(seeded_state):
    """Inputs whose conv0 bound lies in [2^-6, 2^6] (every BASELINE workload)
    keep exponent 0: the scaled and unscaled plans agree bitwise."""
    x = torch.rand(2, 1, 40, 150, generator=torch.Generator().manual_seed(2)).cuda()
    a = _model(seeded_state)(x)
    b = _model(seeded_state, input_scale=0)(x)
    assert torch.equal(a, b)


def test_overflow_raises_without_input_scale(seeded_state):
    x = (torch.rand(1, 1, 32, 64, generator=torch.Generator().manual_seed(3)) * 1e5).cuda()
    m = _model(seeded_state, input_scale=0)
    with pytest.raises(FloatingPointError):
        m(x)
    y = _model(seeded_state)(x)  # with the scale the same input is finite
    assert torch.isfinite(y).all()


def test_nonfinite_input_propagates(seeded_state):
    x = torch.rand(1, 1, 32, 64, generator=torch.Generator().manual_seed(4))
    x[0, 0, 10, 20] = float("nan")
    y = _model(seeded_state)(x.cuda()).cpu()
    assert torch.isnan(y[0, :, 10, 20]).all()
    assert torch.isfinite(y[0, :, :, :2]).all()  # far from the NaN the receptive field is clean


def test_stack_stress_bitwise(seeded_state):
    """compute-sanitizer is not available on this pool (DESIGN §3 K4), so the
    row-flag protocol is stressed instead: 40 random shapes (ragged strips,
    short columns, 1-4 images) through the layer stack, each bitwise equal to
    the per-layer kernels and raising nothing (the watchdog is armed)."""
    m0 = _model(seeded_state, stack=0)
    m1 = _model(seeded_state, stack=1, watchdog_ms=500)
    rng = np.random.default_rng(123)
    for i in range(40):
        b, h, w = int(rng.integers(1, 5)), int(rng.integers(1, 70)), int(rng.integers(1, 420))
        x = torch.from_numpy(rng.random((b, 1, h, w), dtype=np.float32)).cuda()
        if i % 2:  # row-band items of a random height and skew
            m1.set_plan_option("stack_band_rows", int(rng.integers(1, max(2, h))))
            m1.set_plan_option("stack_skew", int(rng.integers(0, 4)))
        else:
            m1.set_plan_option("stack_band_rows", 0)
        y0, y1 = m0(x), m1(x)
        assert m1.last_used_stack()
        assert torch.equal(y0, y1), (b, h, w, m1.plan_options)
