"""Multi-rank partitioning, exercised on CPU: planning logic, halo exactness
on the oracle and a world_size-2 gloo run of the shard +
gather path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.tvspecnet_oracle import build_seeded_state, oracle_from_state
from paper_2006_10004_b200.shard import batch_shards, forward_shard, gather, row_bands


def test_batch_shards_cover_exactly():
    for b in (0, 1, 5, 64, 48, 512):
        for w in (1, 2, 4, 8):
            sh = batch_shards(b, w)
            assert len(sh) == w
            covered = [i for s, n in sh for i in range(s, s + n)]
            assert covered == list(range(b))


def test_row_bands_halo_and_cover():
    for h in (1, 7, 256, 1024, 2160):
        for w in (1, 2, 4, 8):
            bands = row_bands(h, w, 17)
            assert [r for bd in bands for r in range(bd.out0, bd.out1)] == list(range(h))
            for bd in bands:
                assert bd.src0 == max(0, bd.out0 - 17) and bd.src1 == min(h, bd.out1 + 17)
                assert 0 <= bd.valid_row0 and bd.valid_row0 + bd.rows <= bd.src1 - bd.src0


class _Shallow(torch.nn.Module):
    """depth-5 oracle wrapper so the halo test stays fast on CPU."""

    def __init__(self):
        super().__init__()
        self.m = oracle_from_state(build_seeded_state(5, 64, 5), 5, 64, 5)
        self.depth, self.out_bands = 5, 5

    def forward(self, x):
        return self.m(x)


@pytest.mark.parametrize("halo_ok", [True, False])
def test_row_band_halo_is_exact_on_oracle(halo_ok):
    net = _Shallow()
    x = torch.from_numpy(np.random.default_rng(0).random((1, 1, 40, 24)).astype(np.float32))
    with torch.no_grad():
        full = net(x)
    world = 4
    if not halo_ok:
        net.depth = 4  # one row short of the receptive-field radius
    parts = [forward_shard(net, x, r, world, "rows")[0] for r in range(world)]
    got = torch.cat(parts, dim=2)
    if halo_ok:
        assert torch.equal(got, full)
    else:
        assert not torch.equal(got, full)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, out_q, batch=3):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    net = _Shallow()
    x = torch.from_numpy(np.random.default_rng(1).random((batch, 1, 20, 18)).astype(np.float32))
    bands, clos = forward_shard(net, x, rank, world, mode, closure=True)
    dim = 0 if mode == "batch" else 2
    all_b = gather(bands, world, dim)
    all_c = gather(clos, world, dim)
    if rank != 0:
        assert all_b is None and all_c is None  # only the destination rank holds the result
    else:
        with torch.no_grad():
            full = net(x)
        out_q.put((torch.equal(all_b, full), float((all_b.sum(1, keepdim=True) + all_c - x).abs().max())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,batch", [("batch", 3), ("rows", 3), ("batch", 1)])
def test_gloo_world2_shard_and_gather(mode, batch):
    """batch=1 in batch mode leaves rank 1 with an empty shard (nothing sent)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q, batch)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    equal, clos_err = q.get(timeout=10)
    assert equal
    assert clos_err < 1e-5
