"""GPU parity of the opt-in unshuffle = 2 variant (north_star item 1; SURVEY
F2: not the reference architecture, so the reference is the torch composition
oracle.UnshuffledOracle: pixel_unshuffle -> conv stack -> pixel_shuffle).
Fast-mode gate: relative L2 <= 1e-2 per band, as for the reference layout."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-2


@pytest.fixture(scope="module")
def pair():
    from oracle.tvspecnet_oracle import UnshuffledOracle, build_seeded_state
    from paper_2006_10004_b200 import TVSpecNet

    state = build_seeded_state(unshuffle=2)
    m = TVSpecNet(unshuffle=2).eval()
    m.load_state_dict(state)
    o = UnshuffledOracle().eval()
    o.load_state_dict(state)
    return m.cuda(), o


def _ref(o, x):
    with torch.no_grad():
        return o(torch.from_numpy(x)).numpy()


@pytest.mark.parametrize("shape", [(1, 1, 16, 20), (2, 1, 32, 40), (1, 1, 64, 300), (1, 1, 2, 2)])
def test_unshuffle_vs_composition_oracle(pair, shape):
    from oracle.tvspecnet_oracle import band_rel_l2

    m, o = pair
    x = np.random.default_rng(sum(shape)).random(shape, dtype=np.float32)
    with torch.no_grad():
        out = m(torch.from_numpy(x).cuda()).cpu().numpy()
    assert out.shape == (shape[0], 5, shape[2], shape[3])
    assert band_rel_l2(out, _ref(o, x)).max() <= TOL


def test_unshuffle_config1_closure_and_rows(pair):
    """Config 1's image: bands vs the oracle, the fused closure plane
    (image - sum of bands, inference.py:34-42) and an even row window."""
    from oracle.tvspecnet_oracle import band_rel_l2
    from paper_2006_10004_b200.workloads import CONFIGS, make_image

    m, o = pair
    x = make_image(CONFIGS[1], 0)[None, None]
    xd = torch.from_numpy(x).cuda()
    with torch.no_grad():
        bands, clos = m.forward_planes(xd, closure=True)
        part, _ = m.forward_planes(xd, rows=(64, 96))
    bands, clos = bands.cpu(), clos.cpu()
    assert band_rel_l2(bands.numpy(), _ref(o, x)).max() <= TOL
    want = torch.from_numpy(x) - bands.sum(dim=1, keepdim=True)
    assert torch.allclose(clos, want, atol=1e-5)
    assert torch.equal(part.cpu(), bands[:, :, 64:160])


def test_unshuffle_host_tensors_and_errors(pair):
    m, o = pair
    x = np.random.default_rng(1).random((3, 1, 24, 28), dtype=np.float32)
    out = m(torch.from_numpy(x))  # CPU in, CPU out (pipelined host path)
    assert out.device.type == "cpu"
    with torch.no_grad():
        dev = m(torch.from_numpy(x).cuda()).cpu()
    assert torch.equal(out, dev)
    with pytest.raises(ValueError):
        m(torch.zeros(1, 1, 15, 16).cuda())
    with pytest.raises(ValueError):
        m.forward_planes(torch.zeros(1, 1, 16, 16).cuda(), rows=(1, 4))
