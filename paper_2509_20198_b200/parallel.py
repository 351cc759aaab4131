"""Tile-grid sharding across GPUs + the one collective (tile gather).

SURVEY.md §8(e): heightmap tiles are independent given chunk points within
480 m, so the patch grid is cut into contiguous row bands, one per rank;
each rank also loads a one-tile halo row on each interior side (chunk
points of neighbouring tiles reach 480 m into a patch's padded square).
The only data exchange is gathering the finished tiles (heights + rgb,
B x 64 x 64 x 4 float32) to rank 0 -- NCCL over NVLink on the B200 box,
gloo in the CPU tests.  One process per GPU (torchrun), no other
collective on the data path.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Band:
    """Tile rows [row0, row1) owned by a rank, plus its halo rows."""
    rank: int
    row0: int
    row1: int
    halo0: int
    halo1: int

    @property
    def own_rows(self) -> int:
        return self.row1 - self.row0

    def owns(self, row: int) -> bool:
        return self.row0 <= row < self.row1


def band_for(rank: int, world: int, total_rows: int, halo: int = 1) -> Band:
    """Contiguous, balanced row band (rows differ by at most one)."""
    base, extra = divmod(total_rows, world)
    row0 = rank * base + min(rank, extra)
    row1 = row0 + base + (1 if rank < extra else 0)
    return Band(rank, row0, row1, max(0, row0 - halo),
                min(total_rows, row1 + halo))


def gather_tiles(out: torch.Tensor, dst: int = 0):
    """Gather every rank's finished tiles to `dst` (list on dst, else None).

    Ranks may own different tile counts: sizes are exchanged first so the
    payload gather is exact.
    """
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [out]
    world = dist.get_world_size()
    rank = dist.get_rank()
    if dist.get_backend() == "gloo" and out.is_cuda:  # gloo gathers host tensors
        res = gather_tiles(out.cpu(), dst)
        return None if res is None else [r.to(out.device) for r in res]
    n = torch.tensor([out.shape[0]], dtype=torch.int64, device=out.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    cap = int(max(s.item() for s in sizes))
    pad = out
    if out.shape[0] < cap:
        pad = torch.zeros((cap,) + tuple(out.shape[1:]), dtype=out.dtype,
                          device=out.device)
        pad[:out.shape[0]] = out
    if rank == dst:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.gather(pad, bufs, dst=dst)
        return [b[:int(s.item())] for b, s in zip(bufs, sizes)]
    dist.gather(pad, None, dst=dst)
    return None
