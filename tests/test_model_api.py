"""API contract of the drop-in (no GPU needed): the reference's
test_model.py structure/validation checks plus state_dict identity."""
import pytest
import torch

from oracle.tvspecnet_oracle import TVSpecNetOracle, build_seeded_state
from paper_2006_10004_b200 import ARCH_SPEC, TVSpecNet, receptive_field


def test_arch_spec_unchanged():
    assert ARCH_SPEC == {"depth": 17, "channels": 64, "kernel": 3, "out_bands": 5, "batch_norm": True,
                         "receptive_field": 35}


def test_layer_counts():  # test_model.py:16-23
    model = TVSpecNet()
    convs = [m for m in model.modules() if isinstance(m, torch.nn.Conv2d)]
    bns = [m for m in model.modules() if isinstance(m, torch.nn.BatchNorm2d)]
    assert len(convs) == ARCH_SPEC["depth"]
    assert len(bns) == ARCH_SPEC["depth"] - 2
    assert all(c.kernel_size == (3, 3) for c in convs)
    assert convs[-1].out_channels == ARCH_SPEC["out_bands"]


def test_receptive_field():  # test_model.py:26-28
    assert receptive_field(17, 3) == 35


def test_rejects_bad_input_shape():  # test_model.py:31-34 (raised before any device work)
    model = TVSpecNet().eval()
    with pytest.raises(ValueError):
        model(torch.zeros(2, 3, 16, 16))
    with pytest.raises(ValueError):
        model(torch.zeros(16, 16))


def test_rejects_shallow_depth():  # test_model.py:37-39
    with pytest.raises(ValueError):
        TVSpecNet(depth=2)


@pytest.mark.parametrize("arch", [(17, 64, 5), (26, 128, 5), (3, 64, 2)])
def test_state_dict_identical_to_reference_layout(arch):
    ours = TVSpecNet(*arch).state_dict()
    ref = TVSpecNetOracle(*arch).state_dict()
    assert list(ours) == list(ref)
    assert all(ours[k].shape == ref[k].shape and ours[k].dtype == ref[k].dtype for k in ref)


def test_load_state_dict_strict_and_cache_key():
    m = TVSpecNet().eval()
    k0 = m._weight_key(torch.device("cuda", 0))
    m.load_state_dict(build_seeded_state(), strict=True)
    assert m._weight_key(torch.device("cuda", 0)) != k0  # load bumps tensor versions -> repack


def test_layer_params_fold_matches_eval_bn():
    torch.manual_seed(1)
    m = TVSpecNet(depth=4).eval()
    with torch.no_grad():
        for mod in m.modules():
            if isinstance(mod, torch.nn.BatchNorm2d):
                mod.running_mean.uniform_(-0.5, 0.5)
                mod.running_var.uniform_(0.5, 2.0)
                mod.weight.uniform_(0.5, 1.5)
                mod.bias.uniform_(-0.2, 0.2)
    x = torch.randn(1, 64, 8, 8, dtype=torch.float64)
    conv, bn = m.body[2].double(), m.body[3].double()
    ref = bn(conv(x))
    w, s, b = m.layer_params()[1]
    y = torch.nn.functional.conv2d(x, w, padding=1) * s[None, :, None, None] + b[None, :, None, None]
    torch.testing.assert_close(y, ref, rtol=1e-12, atol=1e-12)


def test_no_cpu_fallback_and_dtype_rejected():
    m = TVSpecNet()
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):
            m(torch.zeros(1, 1, 8, 8))  # train mode needs the B200 training step: no CPU fallback
    m.eval()
    with pytest.raises(RuntimeError):
        m(torch.zeros(1, 1, 8, 8, dtype=torch.float64))


def test_precision_validation():
    with pytest.raises(ValueError):
        TVSpecNet(precision="bf16")
    m = TVSpecNet()
    m.precision = "fp32"
    assert m.precision == "fp32"


def test_unshuffle_variant_structure():
    """unshuffle=2 (the opt-in F-TVSpecNET-style variant): Conv2d(4, C)
    first layer, Conv2d(C, 4K) head, state_dict interchangeable with the torch
    composition oracle; fast mode only; the default stays the reference layout."""
    import torch

    from oracle.tvspecnet_oracle import UnshuffledOracle, build_seeded_state
    from paper_2006_10004_b200 import TVSpecNet

    m = TVSpecNet(unshuffle=2)
    sd = m.state_dict()
    assert sd["body.0.weight"].shape == (64, 4, 3, 3)
    assert sd["body.47.weight"].shape == (20, 64, 3, 3) and sd["body.47.bias"].shape == (20,)
    m.load_state_dict(build_seeded_state(unshuffle=2))
    assert UnshuffledOracle().state_dict().keys() == sd.keys()
    assert TVSpecNet().state_dict()["body.0.weight"].shape == (64, 1, 3, 3)
    with pytest.raises(ValueError):
        TVSpecNet(unshuffle=2, precision="fp32")
    with pytest.raises(ValueError):
        TVSpecNet(unshuffle=3)
    # the oracle composes exactly as torch's pixel_(un)shuffle: identity body check
    x = torch.randn(1, 1, 6, 8)
    assert torch.equal(torch.nn.functional.pixel_shuffle(torch.nn.functional.pixel_unshuffle(x, 2), 2), x)


@pytest.mark.parametrize("B", [1, 2, 3, 5, 16, 64, 129, 512])
def test_host_schedule_partitions_batch(B):
    """The host-tensor pipeline's automatic sub-batch schedule covers the batch
    exactly, and for config 2 (64 x 256^2) keeps a layer-stack-eligible big
    sub-batch and small tail sub-batches (the exposed last D2H)."""
    from paper_2006_10004_b200 import TVSpecNet

    for prec in ("fast", "fp32"):
        m = TVSpecNet(precision=prec)
        for H, W in ((256, 256), (48, 160), (1024, 1024)):
            sizes = m._host_schedule(B, H, W, H, False, 148)
            assert sum(sizes) == B and all(n > 0 for n in sizes)
    sizes = TVSpecNet()._host_schedule(64, 256, 256, 256, True, 148)
    big = max(sizes)
    items = big * 2 * 15
    assert items >= 6 * 148 and items >= 0.95 * 148 * -(-items // 148)
    assert sizes[-1] <= 8


def test_host_path_planning_is_pure_python():
    """Sub-batch schedules and the row-band rule of the host-tensor path
    (model._host_schedule / _host_row_bands) need no device."""
    m = TVSpecNet()
    for B in (1, 2, 3, 8, 17, 64, 65, 512):
        sizes = m._host_schedule(B, 256, 256, 256, False, 148)
        assert sum(sizes) == B and all(n > 0 for n in sizes), (B, sizes)
    assert m._host_schedule(64, 256, 256, 256, False, 148) == [4, 39, 17, 4]
    # one large image: 2 row bands, 4 from 6 MP; never for batches, windows or small results
    assert m._host_row_bands(1, 1024, 1024, 0, 1024, False) == 2
    assert m._host_row_bands(1, 2160, 3840, 0, 2160, True) == 4
    assert m._host_row_bands(1, 256, 256, 0, 256, True) == 1
    assert m._host_row_bands(4, 1024, 1024, 0, 1024, False) == 1
    assert m._host_row_bands(1, 1024, 1024, 8, 512, False) == 1
    m.host_row_bands = 3
    assert m._host_row_bands(1, 300, 260, 0, 300, False) == 3
    assert m._host_row_bands(2, 300, 260, 0, 300, False) == 1
