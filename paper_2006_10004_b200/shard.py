"""Multi-GPU partitioning of the TVSpecNET forward.

The forward shards with no data exchange:

* **batch shards** — contiguous slices of ceil(B/G) images per rank
  (configs 2, 4, 5);
* **row bands** — a single large image (config 3) is cut into G bands of
  output rows; each rank runs the forward on its band extended by
  ``halo = receptive_field(depth)//2 = depth`` rows per internal side
  (model.py:55-56), treats the extended slice as the whole image (zero
  padding only at true image edges, since the slice edge is >= halo rows
  away from every kept row) and stores only its own rows through the head
  kernel's row window.  The result is identical to the unsharded forward
  (every kept pixel sees the same inputs in the same arithmetic order).

No collective is on the data path.  Two ways to run it:

* **one process per GPU** (torchrun): ``forward_shard`` computes a rank's part
  and ``gather`` optionally collects the parts on rank 0 with point-to-point
  sends (NCCL between GPUs, gloo in the CPU tests); benchmarks measure the
  sharded forward without it;
* **one process, several devices**: ``ShardedForward`` owns one C-ABI plan and
  one stream per slot (a device, or a stream of a device), enqueues every
  shard's input copy, forward and result copy without host synchronisation,
  and gathers into the caller's output tensor with one peer copy per shard
  (cudaMemcpyPeerAsync under ``Tensor.copy_``).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = ["batch_shards", "RowBand", "row_bands", "forward_shard", "gather", "ShardedForward"]


def batch_shards(batch: int, world: int) -> list[tuple[int, int]]:
    """[(start, count)] per rank: contiguous, ceil-sized, possibly empty at the end."""
    per = -(-batch // world) if batch else 0
    out = []
    for r in range(world):
        s = min(batch, r * per)
        out.append((s, min(batch, s + per) - s))
    return out


@dataclass(frozen=True)
class RowBand:
    out0: int   # first output row this rank owns
    out1: int   # one past the last owned row
    src0: int   # first input row of the extended slice
    src1: int   # one past the last input row of the slice

    @property
    def valid_row0(self) -> int:  # owned rows inside the slice
        return self.out0 - self.src0

    @property
    def rows(self) -> int:
        return self.out1 - self.out0


def row_bands(height: int, world: int, halo: int) -> list[RowBand]:
    """Even split of ``height`` output rows; each slice extended by ``halo``."""
    bands = []
    for r in range(world):
        o0 = (height * r) // world
        o1 = (height * (r + 1)) // world
        bands.append(RowBand(o0, o1, max(0, o0 - halo), min(height, o1 + halo)))
    return bands


def forward_shard(model, x: torch.Tensor, rank: int, world: int, mode: str = "batch", closure: bool = False):
    """This rank's part of ``model(x)``.

    mode "batch": returns (bands, closure|None) for images [start, start+count).
    mode "rows" : returns (bands, closure|None) for output rows [out0, out1) of
                  every image, computed from the halo-extended slice.
    """
    if mode == "batch":
        s, n = batch_shards(x.shape[0], world)[rank]
        if n == 0:
            k = model.out_bands
            return x.new_empty((0, k) + tuple(x.shape[2:])), (x.new_empty((0, 1) + tuple(x.shape[2:])) if closure else None)
        return _planes(model, x[s : s + n], closure, None)
    if mode == "rows":
        halo = model.depth
        band = row_bands(x.shape[2], world, halo)[rank]
        xs = x[:, :, band.src0 : band.src1]
        return _planes(model, xs, closure, (band.valid_row0, band.rows))
    raise ValueError(f"unknown shard mode {mode!r}")


def _planes(model, x, closure, rows):
    if hasattr(model, "forward_planes"):
        return model.forward_planes(x, closure=closure, rows=rows)
    # oracle path (CPU tests): full slice forward then crop
    with torch.no_grad():
        y = model(x)
    if rows is not None:
        y = y[:, :, rows[0] : rows[0] + rows[1]]
    c = None
    if closure:
        xr = x if rows is None else x[:, :, rows[0] : rows[0] + rows[1]]
        c = xr - y.sum(1, keepdim=True)
    return y, c


def gather(local: torch.Tensor, world: int, dim: int, group=None, dst: int = 0) -> torch.Tensor | None:
    """Optional final collection of per-rank results along ``dim`` on rank
    ``dst`` (None on the other ranks).  Only the shard sizes are exchanged by
    a collective; the data moves by one send per rank, so no rank but ``dst``
    ever holds more than its own shard."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    size = torch.tensor([local.shape[dim]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(t.item()) for t in sizes]
    if rank != dst:
        if local.numel():
            dist.send(local.contiguous(), dst=dst, group=group)
        return None
    parts = []
    for r, n in enumerate(sizes):
        if r == dst:
            parts.append(local)
            continue
        shape = list(local.shape)
        shape[dim] = n
        buf = local.new_empty(shape)
        if buf.numel():
            dist.recv(buf, src=r, group=group)
        parts.append(buf)
    return torch.cat(parts, dim=dim)


class ShardedForward:
    """The forward of one ``TVSpecNet`` split over several slots of one process.

    ``slots`` lists device indices; a device may appear more than once (two
    plans on two streams of one GPU stand in for two devices in tests).  Each
    slot owns its plan (packed weights, scratch) and stream, so the shards
    run concurrently.  ``mode`` "batch" splits images (ceil(B/G) per slot),
    "rows" splits output rows into bands with ``depth``-row halos (one large
    image); "auto" picks rows for B < G.  Results are bitwise the
    unsharded forward's (the in-range input exponent is 0).
    """

    def __init__(self, model, slots=None):
        if slots is None:
            slots = list(range(torch.cuda.device_count()))
        if not slots:
            raise ValueError("ShardedForward needs at least one CUDA slot")
        self.model = model
        self.slots = []
        for d in slots:
            dev = torch.device("cuda", int(d))
            plan = model._new_plan(dev.index)
            plan.set_option("check", 2)  # statuses evaluated once at the end of forward()
            model._load_plan(plan, dev.index)
            self.slots.append((dev, torch.cuda.Stream(dev), plan))
        self._key = model._weight_key(self.slots[0][0])

    def _refresh(self):
        key = self.model._weight_key(self.slots[0][0])
        if key != self._key:
            for dev, _, plan in self.slots:
                self.model._load_plan(plan, dev.index)
            self._key = key

    def forward(self, x: torch.Tensor, closure: bool = False, mode: str = "auto"):
        """(bands, closure-or-None) on x's device (CUDA input) or on the first
        slot's device (CPU input)."""
        m = self.model
        m._check_input(x)
        self._refresh()
        G = len(self.slots)
        B, _, H, W = x.shape
        K = m.out_bands
        if mode == "auto":
            mode = "rows" if B < G else "batch"
        out_dev = x.device if x.is_cuda else self.slots[0][0]
        bands = torch.empty((B, K, H, W), device=out_dev)
        clos = torch.empty((B, 1, H, W), device=out_dev) if closure else None
        src_stream = torch.cuda.current_stream(out_dev)
        ready = torch.cuda.Event()
        ready.record(src_stream)
        done = []
        keep = []  # shard buffers stay referenced until the join
        for r, (dev, stream, plan) in enumerate(self.slots):
            if mode == "batch":
                s, n = batch_shards(B, G)[r]
                if n == 0:
                    continue
                xin, row0, nrows = x[s:s + n], 0, H
                dst_b = bands[s:s + n]
                dst_c = clos[s:s + n] if closure else None
            elif mode == "rows":
                band = row_bands(H, G, m.depth)[r]
                if band.rows == 0:
                    continue
                if m.unshuffle == 2 and (band.src0 % 2 or band.out0 % 2 or band.rows % 2):
                    raise ValueError("unshuffle=2 row bands need even band boundaries")
                xin, row0, nrows = x[:, :, band.src0:band.src1], band.valid_row0, band.rows
                dst_b = bands[:, :, band.out0:band.out1]
                dst_c = clos[:, :, band.out0:band.out1] if closure else None
            else:
                raise ValueError(f"unknown shard mode {mode!r}")
            with torch.cuda.device(dev), torch.cuda.stream(stream):
                stream.wait_event(ready)
                xs = xin.to(dev, non_blocking=True).contiguous()
                nb = xs.shape[0]
                ob = torch.empty((nb, K, nrows, W), device=dev)
                oc = torch.empty((nb, 1, nrows, W), device=dev) if closure else None
                plan.forward(xs.data_ptr(), ob.data_ptr(), oc.data_ptr() if closure else 0, nb, xs.shape[2], W,
                             row0, nrows, stream.cuda_stream)
                dst_b.copy_(ob, non_blocking=True)  # peer copy to the gather device
                if closure:
                    dst_c.copy_(oc, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            done.append(ev)
            keep.append((xs, ob, oc))
        for ev in done:
            src_stream.wait_event(ev)
        for dev, stream, plan in self.slots:  # raise any shard's failure (statuses were deferred)
            plan.sync(stream.cuda_stream)
        del keep
        return bands, clos

    __call__ = forward

    def close(self):
        for _, _, plan in self.slots:
            plan.close()
        self.slots = []
