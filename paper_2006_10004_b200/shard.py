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

No collective is on the data path.  ``gather`` is the optional final
collection to rank 0 (torch.distributed: NCCL between GPUs, gloo in the CPU
tests); benchmarks measure the sharded forward without it.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = ["batch_shards", "RowBand", "row_bands", "forward_shard", "gather"]


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


def gather(local: torch.Tensor, world: int, dim: int, group=None) -> torch.Tensor | None:
    """Optional final gather of per-rank results along ``dim`` (all ranks
    receive it; shards may differ in size along ``dim``)."""
    import torch.distributed as dist

    size = torch.tensor([local.shape[dim]], device=local.device)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad_shape = list(local.shape)
    pad_shape[dim] = mx
    padded = local.new_zeros(pad_shape)
    padded.narrow(dim, 0, local.shape[dim]).copy_(local)
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    return torch.cat([b.narrow(dim, 0, n) for b, n in zip(bufs, sizes)], dim=dim)
