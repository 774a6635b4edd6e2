"""GPU parity of the B200 path against the CPU oracle / reference fixtures.

Tolerances (BASELINE.json north_star), relative L2 per image per band:
  * precision="fp32": <= 1e-5
  * precision="fast": <= 1e-2, closure (band-sum reconstruction) <= 1e-2
All calls go through the C ABI (libtvsb200.so) via the drop-in module.
"""
import numpy as np
import pytest
import torch

from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state
from paper_2006_10004_b200 import TVSpecNet, predict_bands, predict_planes
from paper_2006_10004_b200 import _native
from paper_2006_10004_b200.shard import forward_shard
from paper_2006_10004_b200.workloads import CONFIGS, make_image

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "fast": 1e-2}
CLOSURE_TOL = {"fp32": 1e-5, "fast": 1e-2}


@pytest.fixture(scope="module")
def oracle(seeded_state):
    torch.set_num_threads(max(1, min(32, torch.get_num_threads())))
    return oracle_from_state(seeded_state)


@pytest.fixture(scope="module", params=["fast", "fp32"])
def model(request, seeded_state):
    assert torch.cuda.is_available(), "GPU tests need a B200"
    m = TVSpecNet(precision=request.param).eval()
    m.load_state_dict(seeded_state)
    return m


def _run(m, x):
    bands, clos = m.forward_planes(torch.from_numpy(x).cuda(), closure=True)
    torch.cuda.synchronize()
    return bands.cpu().numpy(), clos.cpu().numpy()


def _check(m, x, ref):
    out, clos = _run(m, x)
    assert out.shape == ref.shape
    assert np.isfinite(out).all()
    err = band_rel_l2(out, ref)
    assert err.max() <= TOL[m.precision], f"worst band rel-L2 {err.max():.3e}"
    cref = x[:, 0:1] - ref.sum(1, keepdims=True)
    cerr = band_rel_l2(clos, cref)
    assert cerr.max() <= CLOSURE_TOL[m.precision], f"closure rel-L2 {cerr.max():.3e}"
    # the closure plane closes the decomposition exactly (inference.py:34-42)
    np.testing.assert_allclose(out.sum(1, keepdims=True) + clos, x[:, 0:1], atol=1e-5)
    return err.max()


@pytest.mark.parametrize("case", ["small", "nonsq", "tiny", "tiny2", "cfg1"])
def test_golden_fixtures(model, golden, case):
    _check(model, golden[f"{case}_x"], golden[f"{case}_y"])


def test_depth3_fixture(golden):
    for prec in ("fast", "fp32"):
        m = TVSpecNet(depth=3, precision=prec).eval()
        m.load_state_dict(build_seeded_state(3, 64, 5))
        _check(m, golden["d3_x"], golden["d3_y"])


@pytest.fixture(scope="module")
def wide_case():
    """Config 5's width/depth variant (128 feature maps, depth 26):
    image 0 of config 5, its fp32 oracle output and an fp64 reference."""
    state = build_seeded_state(26, 128, 5)
    x = make_image(CONFIGS["5w"], 0)[None, None]
    o32 = oracle_from_state(state, 26, 128, 5)
    o64 = oracle_from_state(state, 26, 128, 5).double()
    with torch.no_grad():
        y32 = o32(torch.from_numpy(x)).numpy()
        y64 = o64(torch.from_numpy(x).double()).numpy()
    return state, x, y32, y64


@pytest.mark.parametrize("prec", ["fast", "fp32"])
def test_wide_variant(golden, wide_case, prec):
    state, x, y32, y64 = wide_case
    m = TVSpecNet(26, 128, 5, precision=prec).eval()
    m.load_state_dict(state)
    _check(m, golden["wide_x"], golden["wide_y"])
    out, _ = _run(m, x)
    if prec == "fast":
        assert band_rel_l2(out, y32).max() <= 1e-2
        return
    # The fp32 reference itself is 1.05e-5 from the exact (fp64) result on band 4
    # of this image (26 layers of fp32 rounding), so the 1e-5 gate is applied
    # against the fp64 reference; against the fp32 oracle the distance is the
    # oracle's own rounding error.
    assert band_rel_l2(y32, y64).max() > 1e-5  # documents the structural limit
    assert band_rel_l2(out, y64).max() <= 1e-5
    assert band_rel_l2(out, y32).max() <= 1.5e-5


@pytest.mark.parametrize("shape", [(2, 37, 300), (1, 130, 1), (3, 64, 128), (1, 1, 129)])
def test_wide_fp32_tcgen05_blocks(shape):
    """The wide variant's fp32-accurate mode on tcgen05 (every 128 -> 128 layer as
    2 x 2 blocks of the 64-channel split kernels, partial sums handed over in
    fp32) against the CUDA-core fp32 kernels (plan option wide_cuda=1: fp32 FFMA
    chunks combined in fp64) on ragged shapes, with a row window, the closure
    and both CTA layouts of the block kernel (modes 12 and 3, bitwise equal)."""
    state = build_seeded_state(26, 128, 5)
    x = torch.rand(*shape[:1], 1, *shape[1:], generator=torch.Generator().manual_seed(5)).cuda()
    outs = {}
    for name, opts in (("tc", {}), ("tc3", {"fp32_pairs": 0}), ("cuda", {"wide_cuda": 1})):
        m = TVSpecNet(26, 128, 5, precision="fp32", options=opts).eval()
        m.load_state_dict(state)
        bands, clos = m.forward_planes(x, closure=True)
        outs[name] = bands
        assert m.last_launch_count() == (26 if name == "cuda" else 1 + 2 + 24 * 4 + 2)
        np.testing.assert_allclose((bands.sum(1, keepdim=True) + clos).cpu().numpy(), x.cpu().numpy(), atol=1e-5)
        if shape[1] >= 30:
            b2, c2 = m.forward_planes(x, closure=True, rows=(9, 13))
            assert torch.equal(b2, bands[:, :, 9:22])
            assert torch.equal(c2, clos[:, :, 9:22])
    assert torch.equal(outs["tc"], outs["tc3"])
    err = band_rel_l2(outs["tc"].cpu().numpy(), outs["cuda"].cpu().numpy()).max()
    print(f"wide fp32 {shape}: tcgen05 blocks vs CUDA-core kernels {err:.3e}")
    # two fp32-class computations of the same 26 layers: each is within ~1e-5
    # of the exact result (tools/wide_fp32_probe.py), so of each other
    assert err <= 2e-5


@pytest.mark.parametrize("img", [1, 2, 3])
def test_wide_fp32_standing_exception_more_images(img):
    """The wide variant's fp32 mode vs the 1e-5 gate on more config-5 images
    (128x128 crops): the fp32 reference is itself >= ~1e-5 from the exact
    result on this 26-layer model, so the standing exception is checked as
    (a) <= 1e-5 against fp64 and (b) against the fp32 oracle no further than
    the oracle's own fp64 distance plus 1e-5."""
    state = build_seeded_state(26, 128, 5)
    x = make_image(CONFIGS["5w"], img)[None, None, 96:224, 160:288].copy()
    o32 = oracle_from_state(state, 26, 128, 5)
    o64 = oracle_from_state(state, 26, 128, 5).double()
    with torch.no_grad():
        y32 = o32(torch.from_numpy(x)).numpy()
        y64 = o64(torch.from_numpy(x).double()).numpy()
    m = TVSpecNet(26, 128, 5, precision="fp32").eval()
    m.load_state_dict(state)
    out, _ = _run(m, x)
    e64, e32, floor = band_rel_l2(out, y64).max(), band_rel_l2(out, y32).max(), band_rel_l2(y32, y64).max()
    print(f"wide fp32 img {img}: vs fp64 {e64:.3e}, vs fp32 oracle {e32:.3e}, oracle vs fp64 {floor:.3e}")
    assert e64 <= 1e-5
    assert e32 <= floor + 1e-5


@pytest.mark.parametrize("cfg,count", [(2, 4), (3, 1), (5, 2)])
def test_configs_vs_oracle(model, oracle, cfg, count):
    spec = CONFIGS[cfg]
    x = np.stack([make_image(spec, i) for i in range(count)])[:, None]
    with torch.no_grad():
        ref = oracle(torch.from_numpy(x)).numpy()
    _check(model, x, ref)


def test_config4_plane0_vs_oracle(model, oracle):
    x = make_image(CONFIGS[4], 0)[None, None]
    with torch.no_grad():
        ref = oracle(torch.from_numpy(x)).numpy()
    _check(model, x, ref)


@pytest.mark.parametrize("shape", [(1, 1, 5, 300), (2, 1, 129, 131), (1, 1, 300, 1), (1, 1, 1, 257), (3, 1, 33, 255)])
def test_ragged_shapes(model, oracle, shape):
    x = np.random.default_rng(sum(shape)).random(shape).astype(np.float32)
    with torch.no_grad():
        ref = oracle(torch.from_numpy(x)).numpy()
    _check(model, x, ref)


def test_translation_equivariance_interior(model):  # test_model.py:42-59
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal((48, 48)).astype(np.float32))
    shifted = torch.zeros_like(x)
    shifted[4:, :] = x[:-4, :]
    y = model(x[None, None].cuda())[0]
    y2 = model(shifted[None, None].cuda())[0]
    half = 35 // 2
    lo, hi = half + 4, 48 - half
    torch.testing.assert_close(y2[:, lo:hi, :], y[:, lo - 4 : hi - 4, :], atol=1e-5, rtol=1e-5)


def test_eval_is_deterministic(model):  # test_model.py:62-70
    x = torch.randn(2, 1, 64, 200, device="cuda")
    a, b = model(x), model(x)
    assert torch.equal(a, b)


def test_row_window_equals_full_rows(model):
    x = torch.rand(2, 1, 96, 140, device="cuda")
    full = model(x)
    bands, clos = model.forward_planes(x, closure=True, rows=(30, 17))
    assert torch.equal(bands, full[:, :, 30:47])
    torch.testing.assert_close(clos, x[:, :, 30:47] - full[:, :, 30:47].sum(1, keepdim=True))


def test_row_band_shards_equal_unsharded(model):
    """halo = depth rows makes every band bitwise equal to the full forward."""
    x = torch.from_numpy(make_image(CONFIGS[3], 0)[None, None]).cuda()
    full = model(x)
    for world in (2, 4, 8):
        parts = [forward_shard(model, x, r, world, "rows")[0] for r in range(world)]
        assert torch.equal(torch.cat(parts, dim=2), full), world


def test_batch_shards_equal_unsharded(model):
    x = torch.rand(5, 1, 64, 64, device="cuda")
    full = model(x)
    parts = [forward_shard(model, x, r, 4, "batch")[0] for r in range(4)]
    assert torch.equal(torch.cat(parts, dim=0), full)


def test_cpu_tensors_in_and_out(model, golden):
    x = torch.from_numpy(golden["nonsq_x"])
    y = model(x)
    assert y.device.type == "cpu" and y.shape == (1, 5, 32, 40)
    img = golden["small_x"][0, 0].astype(np.float64)
    out = predict_bands(model, img)  # inference.py:25-32 calling convention
    assert out.shape == (5, 16, 20) and np.isfinite(out).all()


@pytest.mark.parametrize("sched", [None, 3, (1, 4, 2, 1)])
def test_host_pipeline_schedules_match_device(model, sched):
    """CPU tensors in/out through the sub-batched H2D/forward/D2H pipeline give
    bitwise the device-path result, for the automatic and explicit schedules."""
    x = torch.rand(21, 1, 48, 160, generator=torch.Generator().manual_seed(7))
    ref_b, ref_c = model.forward_planes(x.cuda(), closure=True)
    old = model.host_chunks
    try:
        model.host_chunks = sched
        b, c = model.forward_planes(x, closure=True)
    finally:
        model.host_chunks = old
    assert b.device.type == "cpu" and b.is_pinned()
    assert torch.equal(b, ref_b.cpu()) and torch.equal(c, ref_c.cpu())


def test_predict_planes_stack(model):
    x = torch.rand(2, 1, 20, 30, device="cuda")
    planes = predict_planes(model, x)
    assert planes.shape == (2, 7, 20, 30)
    torch.testing.assert_close(planes[:, 1:].sum(1), planes[:, 0], atol=1e-5, rtol=0)


def test_host_buffer_abi_matches_device_path(model, golden):
    x = np.ascontiguousarray(golden["small_x"])
    plan = model._plan_for(torch.device("cuda", 0))
    bands = np.empty((2, 5, 16, 20), np.float32)
    clos = np.empty((2, 1, 16, 20), np.float32)
    plan.forward_host(x.ctypes.data, bands.ctypes.data, clos.ctypes.data, 2, 16, 20, 0)
    dev_b, dev_c = _run(model, x)
    np.testing.assert_array_equal(bands, dev_b)
    np.testing.assert_array_equal(clos, dev_c)


def test_weight_reload_invalidates_pack(seeded_state):
    m = TVSpecNet().eval()
    m.load_state_dict(seeded_state)
    x = torch.rand(1, 1, 32, 32, device="cuda")
    a = m(x)
    other = build_seeded_state(seed=1)
    m.load_state_dict(other)
    b = m(x)
    ref = oracle_from_state(other)(x.cpu()).detach().numpy()
    assert not torch.equal(a, b)
    assert band_rel_l2(b.cpu().numpy(), ref).max() < 1e-2


def test_nontrivial_batchnorm_stats(oracle):
    """Trained-looking BN stats (not the identity init) fold correctly."""
    torch.manual_seed(5)
    ref = oracle_from_state(build_seeded_state(seed=2))
    with torch.no_grad():
        for mod in ref.modules():
            if isinstance(mod, torch.nn.BatchNorm2d):
                mod.running_mean.uniform_(0.0, 0.3)
                mod.running_var.uniform_(0.5, 2.0)
                mod.weight.uniform_(0.7, 1.3)
                mod.bias.uniform_(-0.1, 0.1)
    x = np.random.default_rng(9).random((2, 1, 40, 70)).astype(np.float32)
    with torch.no_grad():
        y = ref(torch.from_numpy(x)).numpy()
    for prec in ("fast", "fp32"):
        m = TVSpecNet(precision=prec).eval()
        m.load_state_dict(ref.state_dict())
        _check(m, x, y)


def test_launch_accounting(model):
    x = torch.rand(1, 1, 64, 64, device="cuda")
    model(x)
    # input-scale + conv0 + (depth-2) hidden + head
    assert model.last_launch_count() == model.depth + 1


def test_conv0_tcgen05_matches_fp32_conv0(seeded_state):
    """The tcgen05 K1 (TF32 hi/lo split, conv0_tc.cu) against the CUDA-core fp32
    FFMA K1: both round the same fp32 pre-activation to fp16, so the first-layer
    activations may differ by one fp16 ulp where the sums differ in the last
    fp32 bits.  Signed inputs of larger magnitude exercise the hi/lo split."""
    outs = []
    for tc in (1, 0):
        m = TVSpecNet(depth=3, options={"conv0_tc": tc}).eval()  # conv0 -> 1 hidden -> head: conv0 dominates
        m.load_state_dict(build_seeded_state(3, 64, 5))
        outs.append(m)
    g = torch.Generator().manual_seed(3)
    for x in (torch.rand(2, 1, 40, 300, generator=g), torch.randn(2, 1, 40, 300, generator=g) * 30):
        x = x.cuda()
        a, b = outs[0](x), outs[1](x)
        rel = (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)).item()
        assert torch.isfinite(a).all() and rel < 1e-3, rel


def test_abi_errors_on_gpu(model):
    plan = model._plan_for(torch.device("cuda", 0))
    with pytest.raises(ValueError):
        plan.forward(0, 0, 0, 1, 8, 8, 0, -1, 0)
    x = torch.rand(1, 1, 8, 8, device="cuda")
    y = torch.empty(1, 5, 8, 8, device="cuda")
    with pytest.raises(ValueError):
        plan.forward(x.data_ptr(), y.data_ptr(), 0, 1, 8, 8, 6, 5, 0)  # window past H
    assert _native.load().tvs_abi_version() == 2
    with pytest.raises(ValueError):
        plan.set_option("no_such_option", 1)
    with pytest.raises(ValueError):
        plan.set_option("check", 7)


@pytest.mark.gpu
def test_fp32_cuda_core_kernels(golden):
    """The CUDA-core fp32 kernels (plan option fp32_cuda=1; the path of the wide
    variant's fp32 mode) on the 64-channel model: same 1e-5 gate as the default
    tcgen05 fp32 mode."""
    m = TVSpecNet(precision="fp32", options={"fp32_cuda": 1})
    m.load_state_dict(build_seeded_state())
    m = m.cuda().eval()
    for case in ("small", "nonsq", "cfg1"):
        with torch.no_grad():
            out = m(torch.from_numpy(golden[f"{case}_x"]).cuda()).cpu().numpy()
        assert band_rel_l2(out, golden[f"{case}_y"]).max() <= 1e-5, case


def _stack_model(seeded_state, stack, **opts):
    m = TVSpecNet(options={"stack": stack, **opts}).eval()
    m.load_state_dict(seeded_state)
    return m


@pytest.mark.parametrize("shape", [(2, 48, 160), (1, 37, 300), (3, 64, 128), (1, 5, 7), (2, 1, 130)])
def test_layer_stack_bitwise(seeded_state, shape):
    """The layer-stack kernel (conv_tc.cu mode 8: all hidden layers in one
    persistent launch, layers handed over through L2 under row flags) computes
    every output with the per-layer kernel's exact MMA sequence: bitwise equal,
    including ragged strips (W % 128 != 0), H < 3 and W < 128."""
    m0 = _stack_model(seeded_state, 0)
    m1 = _stack_model(seeded_state, 1)
    x = torch.rand(*shape[:1], 1, *shape[1:], generator=torch.Generator().manual_seed(sum(shape))).cuda()
    with torch.no_grad():
        y0, y1 = m0(x), m1(x)  # the default "check" option raises on a watchdog expiry
    torch.cuda.synchronize()
    assert not m0.last_used_stack() and m1.last_used_stack()
    assert m0.last_launch_count() == m0.depth + 1 and m1.last_launch_count() == 4
    assert torch.equal(y0, y1)


def test_layer_stack_auto_config2(seeded_state, oracle):
    """Config 2 (64 x 256^2) selects the layer stack by default (1920 items on
    148 SMs); parity against the oracle on two of its images."""
    m = TVSpecNet().eval()
    m.load_state_dict(seeded_state)
    x = np.stack([make_image(CONFIGS[2], i) for i in range(64)])[:, None]
    bands, clos = m.forward_planes(torch.from_numpy(x).cuda(), closure=True)
    torch.cuda.synchronize()
    assert m.last_used_stack() and m.last_launch_count() == 4
    with torch.no_grad():
        ref = oracle(torch.from_numpy(x[[0, 63]])).numpy()
    err = band_rel_l2(bands.cpu().numpy()[[0, 63]], ref)
    assert err.max() <= TOL["fast"], f"worst band rel-L2 {err.max():.3e}"
    np.testing.assert_allclose((bands.sum(1, keepdim=True) + clos).cpu().numpy(), x, atol=1e-5)


@pytest.mark.parametrize("pairs,tol", [(24, 1e-2), (12, 1e-2), (6, 1.5e-2), (0, 2e-2)])
def test_wide_pair_schedules(wide_case, pairs, tol):
    """Wide variant, fast mode: the first `pairs` hidden layers read fp16 hi/lo
    pair activations (conv_tc.cu mode 5), the rest single fp16 (mode 9, head
    mode 10).  24 (all) and 12 (the default) meet the 1e-2 gate; fewer pairs
    trade accuracy for MMA work (tools/emulate_wide.py: 6 -> ~1.06e-2, 0 ->
    1.1-1.3e-2, the plain-fp16 roofline probe)."""
    state, x, y32, _ = wide_case
    m = TVSpecNet(26, 128, 5, options={"wide_pair_layers": pairs}).eval()
    m.load_state_dict(state)
    out, clos = _run(m, x)
    err = band_rel_l2(out, y32).max()
    assert err <= tol, f"pairs={pairs}: worst band rel-L2 {err:.3e}"
    np.testing.assert_allclose(out.sum(1, keepdims=True) + clos, x[:, 0:1], atol=1e-5)


@pytest.mark.parametrize("prec", ["fast", "fp32"])
@pytest.mark.parametrize("bands", [1, 3, 8])
def test_band_counts(prec, bands):
    """Heads with 1..8 bands (the 8 hi + 8 lo weight columns per dy of the
    tcgen05 head, kMaxBands) against the oracle, on ragged shapes."""
    state = build_seeded_state(3, 64, bands)
    ref_m = oracle_from_state(state, 3, 64, bands)
    m = TVSpecNet(depth=3, out_bands=bands, precision=prec).eval()
    m.load_state_dict(state)
    x = np.random.default_rng(bands).random((2, 1, 37, 150)).astype(np.float32)
    with torch.no_grad():
        ref = ref_m(torch.from_numpy(x)).numpy()
    _check(m, x, ref)


@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (3, 1, 1, 300), (1, 1, 130, 1), (2, 1, 7, 129), (1, 1, 64, 257)])
def test_conv0_tcgen05_ragged(seeded_state, oracle, shape):
    """The tcgen05 K1 on ragged strips (partial 128-px strips, single rows and
    columns) stays within the fast-mode tolerance of the oracle."""
    m = TVSpecNet().eval()
    m.load_state_dict(seeded_state)
    x = np.random.default_rng(sum(shape)).random(shape).astype(np.float32)
    with torch.no_grad():
        ref = oracle(torch.from_numpy(x)).numpy()
    _check(m, x, ref)


@pytest.mark.parametrize("band_rows,skew", [(1, 0), (2, 1), (3, 2), (5, 0), (8, 2), (16, 3), (16, 0), (17, 2)])
@pytest.mark.parametrize("shape", [(1, 48, 160), (2, 37, 300), (1, 64, 256)])
def test_layer_stack_row_bands_bitwise(seeded_state, shape, band_rows, skew):
    """Row-band stack items (an item = R rows of one strip of one layer, band
    edges of layer j at rows = j*skew mod R; the batch-1 path): a band edge is
    a segment edge of the per-layer kernel too, so the outputs stay bitwise
    equal, for band heights down to one row, with and without skew."""
    m0 = _stack_model(seeded_state, 0)
    m1 = _stack_model(seeded_state, 1, stack_band_rows=band_rows, stack_skew=skew, watchdog_ms=500)
    x = torch.rand(*shape[:1], 1, *shape[1:], generator=torch.Generator().manual_seed(band_rows + sum(shape))).cuda()
    with torch.no_grad():
        y0, y1 = m0(x), m1(x)
    torch.cuda.synchronize()
    assert m1.last_used_stack()
    assert torch.equal(y0, y1)


def test_layer_stack_auto_batch1(seeded_state, oracle, golden):
    """Config 1 (one 256^2 image, 30 whole-column items) selects the row-band
    layer stack by default; parity against the reference-generated fixture."""
    m = TVSpecNet().eval()
    m.load_state_dict(seeded_state)
    with torch.no_grad():
        out = m(torch.from_numpy(golden["cfg1_x"]).cuda()).cpu().numpy()
    assert m.last_used_stack() and m.last_launch_count() == 4
    assert band_rel_l2(out, golden["cfg1_y"]).max() <= TOL["fast"]


def _recon_host(x, bands, clos):
    """The check's definition evaluated on the host from the returned planes:
    r = x - (sequential fp32 band sum + closure), sums of r^2 and x^2 in fp64."""
    s = bands[:, 0]
    for k in range(1, bands.shape[1]):
        s = s + bands[:, k]
    r = (x[:, 0] - (s + clos[:, 0])).double()
    return (r * r).sum((1, 2)), (x[:, 0].double() ** 2).sum((1, 2))


@pytest.mark.parametrize(
    "variant", ["fast", "fast_stack", "fast_bands", "fp32", "fp32_cuda", "wide", "wide_fp32", "unshuffle"])
def test_fused_reconstruction_check(seeded_state, variant):
    """tvs_forward_checked (north_star item 3): the head epilogue's residual
    sums equal the same check evaluated on the host from the stored planes,
    and the closure identity holds at the reference's 1e-5
    (pkg/trainer/tests/test_inference.py:31-38) for every head kernel."""
    from oracle.tvspecnet_oracle import build_seeded_state as bss

    opts, arch, state = {}, {}, seeded_state
    if variant == "fast_stack":
        opts = {"stack": 1}
    elif variant == "fast_bands":
        opts = {"stack": 1, "stack_band_rows": 8}
    elif variant == "fp32_cuda":
        opts = {"fp32_cuda": 1}
    elif variant in ("wide", "wide_fp32"):
        arch = dict(depth=26, channels=128)
        state = bss(**arch)
    elif variant == "unshuffle":
        arch = dict(unshuffle=2)
        state = bss(17, 64, 5, unshuffle=2)
    prec = "fp32" if "fp32" in variant else "fast"
    m = TVSpecNet(**arch, precision=prec, options=opts).eval()
    m.load_state_dict(state)
    x = torch.rand(3, 1, 40, 300, generator=torch.Generator().manual_seed(11)).cuda() * 3.0
    bands, clos, rel = m.forward_planes(x, check_reconstruction=True)
    torch.cuda.synchronize()
    if variant in ("fast_stack", "fast_bands"):
        assert m.last_used_stack()
    r2, x2 = _recon_host(x, bands, clos)
    got = torch.sqrt(r2 / x2)
    assert torch.allclose(rel, got.to(rel.device), rtol=1e-9, atol=1e-15), (rel, got)
    assert float(rel.max()) <= 1e-6
    np.testing.assert_allclose((bands.sum(1, keepdim=True) + clos).cpu().numpy(), x.cpu().numpy(), atol=1e-5)
    # a row window: the sums cover only the window's rows
    b2, c2, rel2 = m.forward_planes(x, rows=(8, 16), check_reconstruction=True)
    r2w, x2w = _recon_host(x[:, :, 8:24], b2, c2)
    assert torch.allclose(rel2, torch.sqrt(r2w / x2w).to(rel2.device), rtol=1e-9, atol=1e-15)


def test_predict_planes_reconstruction_gate(model):
    """predict_planes runs the fused check and returns [input, bands, closure]."""
    x = torch.rand(2, 1, 32, 48, generator=torch.Generator().manual_seed(3)).cuda()
    planes = predict_planes(model, x)
    assert planes.shape == (2, 7, 32, 48)
    np.testing.assert_allclose(planes[:, 1:].sum(1).cpu().numpy(), x[:, 0].cpu().numpy(), atol=1e-5)


@pytest.mark.parametrize("rows", [None, (5, 9)])
def test_head_gated_on_stack_flags_bitwise(seeded_state, rows):
    """The head launched after a layer stack acquires layer 14's rows through
    the stack's row flags (no grid-wide wait, it runs in the stack's tail);
    its output is bitwise the same as with the grid-wide dependency."""
    x = torch.rand(64, 1, 16, 256, generator=torch.Generator().manual_seed(8)).cuda()
    outs = []
    for gate in (0, 1):
        m = _stack_model(seeded_state, -1, head_gate=gate)
        b, c = m.forward_planes(x, closure=True, rows=rows)
        torch.cuda.synchronize()
        assert m.last_used_stack()
        outs.append((b, c))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("shape", [(64, 16, 256), (2, 37, 300), (1, 64, 256)])
def test_stack_flag_watcher_bitwise(seeded_state, shape):
    """The flag-watcher warp (plan option stack_watcher) only changes who polls
    the row flags: outputs are bitwise those of the producer-polled stack."""
    x = torch.rand(shape[0], 1, *shape[1:], generator=torch.Generator().manual_seed(sum(shape))).cuda()
    outs = []
    for w in (0, 1):
        m = _stack_model(seeded_state, 1, stack_watcher=w, watchdog_ms=500)
        with torch.no_grad():
            outs.append(m(x))
        assert m.last_used_stack()
    assert torch.equal(outs[0], outs[1])


def test_reconstruction_check_across_chunks(seeded_state):
    """The per-image check sums land at the right offsets when the batch is
    cut into activation chunks (plan option chunk_mb)."""
    m = TVSpecNet(options={"chunk_mb": 1}).eval()  # 40x300 fp16 activations: one image per chunk
    m.load_state_dict(seeded_state)
    x = torch.rand(3, 1, 40, 300, generator=torch.Generator().manual_seed(12)).cuda()
    x[1] *= 4.0
    bands, clos, rel = m.forward_planes(x, check_reconstruction=True)
    r2, x2 = _recon_host(x, bands, clos)
    assert torch.allclose(rel, torch.sqrt(r2 / x2).to(rel.device), rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("shape", [(2, 48, 300), (1, 1, 129), (3, 37, 256), (1, 130, 1)])
def test_fp32_cta_pairs_bitwise(seeded_state, shape):
    """The fp32-accurate hidden layer on CTA pairs (mode 12: both output-channel
    halves at once, input rows multicast to the pair) runs each output's MMA
    sequence of mode 3: bitwise equal."""
    x = torch.rand(shape[0], 1, *shape[1:], generator=torch.Generator().manual_seed(sum(shape))).cuda()
    outs = []
    for pr in (0, 1):
        m = TVSpecNet(precision="fp32", options={"fp32_pairs": pr}).eval()
        m.load_state_dict(seeded_state)
        with torch.no_grad():
            outs.append(m(x))
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("prec", ["fast", "fp32"])
def test_host_row_band_pipeline_bitwise(prec):
    """One large host image runs as row bands with `depth`-row halos through
    the H2D / compute / D2H streams (model._pipeline_rows): bitwise equal to
    the whole-image forward, closure plane included; automatic for config 3's
    shape, off for small results and batches."""
    m = TVSpecNet(precision=prec).eval()
    m.load_state_dict(build_seeded_state())
    x = torch.rand(1, 1, 300, 260, generator=torch.Generator().manual_seed(9))
    m.host_row_bands = 0
    b0, c0 = m.forward_planes(x, closure=True)
    for nb in (2, 3, 7):
        m.host_row_bands = nb
        b1, c1 = m.forward_planes(x, closure=True)
        assert torch.equal(b0, b1) and torch.equal(c0, c1), nb
    m.host_row_bands = None
    assert m._host_row_bands(1, 1024, 1024, 0, 1024, False) == 2
    assert m._host_row_bands(1, 2160, 3840, 0, 2160, False) == 4
    assert m._host_row_bands(1, 256, 256, 0, 256, False) == 1
    assert m._host_row_bands(2, 1024, 1024, 0, 1024, False) == 1
    assert m._host_row_bands(1, 1024, 1024, 0, 512, False) == 1


def test_model_pickles_and_deep_copies_after_host_forwards():
    """The per-process caches of the host paths (device staging buffers, streams,
    events) stay out of pickles and deep copies; the copy computes the same."""
    import copy
    import pickle

    m = TVSpecNet().eval()
    m.load_state_dict(build_seeded_state())
    x1 = torch.rand(1, 1, 40, 130, generator=torch.Generator().manual_seed(2))
    x8 = torch.rand(8, 1, 24, 40, generator=torch.Generator().manual_seed(3))
    y1, y8 = m(x1), m(x8)  # single-sub-batch path and sub-batch pipeline
    m.host_row_bands = 2
    yb = m(x1)
    assert torch.equal(yb, y1)
    for clone in (pickle.loads(pickle.dumps(m)), copy.deepcopy(m)):
        assert torch.equal(clone(x1), y1) and torch.equal(clone(x8), y8)


def test_empty_batch_returns_empty_planes_like_the_reference():
    m = TVSpecNet().eval()
    m.load_state_dict(build_seeded_state())
    ref = oracle_from_state(build_seeded_state())
    for x in (torch.zeros(0, 1, 8, 12), torch.zeros(0, 1, 8, 12).cuda()):
        with torch.no_grad():
            y = m(x)
        assert tuple(y.shape) == tuple(ref(torch.zeros(0, 1, 8, 12)).shape) == (0, 5, 8, 12) and y.device == x.device
        b, c = m.forward_planes(x, closure=True)
        assert tuple(b.shape) == (0, 5, 8, 12) and tuple(c.shape) == (0, 1, 8, 12)
