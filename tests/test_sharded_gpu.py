"""In-process multi-device forward (shard.ShardedForward) on one B200: two and
three plans on separate streams of device 0 stand in for devices.  Batch
shards and halo'd row bands must equal the unsharded forward bitwise
(the partition has no exchange and every kept pixel sees the same
arithmetic)."""
import pytest
import torch

from paper_2006_10004_b200 import TVSpecNet
from paper_2006_10004_b200.shard import ShardedForward

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def model(seeded_state):
    m = TVSpecNet().eval()
    m.load_state_dict(seeded_state)
    return m


@pytest.mark.parametrize("slots,mode,shape", [
    ([0, 0], "batch", (5, 1, 40, 150)),
    ([0, 0, 0], "batch", (2, 1, 33, 260)),   # one slot idle
    ([0, 0], "rows", (1, 1, 200, 140)),
    ([0, 0, 0], "rows", (2, 1, 97, 300)),
])
def test_sharded_equals_unsharded(model, slots, mode, shape):
    x = torch.rand(*shape, generator=torch.Generator().manual_seed(sum(shape))).cuda()
    want_b, want_c = model.forward_planes(x, closure=True)
    sf = ShardedForward(model, slots)
    got_b, got_c = sf.forward(x, closure=True, mode=mode)
    torch.cuda.synchronize()
    assert torch.equal(got_b, want_b)
    assert torch.equal(got_c, want_c)
    sf.close()


def test_sharded_host_input_and_weight_refresh(model, seeded_state):
    x = torch.rand(4, 1, 64, 128, generator=torch.Generator().manual_seed(9))
    sf = ShardedForward(model, [0, 0])
    got, _ = sf(x)
    assert torch.equal(got, model(x.cuda()))
    # a weight update repacks every slot's plan
    with torch.no_grad():
        model.body[0].bias.add_(0.01)
    try:
        got2, _ = sf(x)
        assert torch.equal(got2, model(x.cuda()))
        assert not torch.equal(got2, got)
    finally:
        model.load_state_dict(seeded_state)
    sf.close()
