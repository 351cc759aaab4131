"""Multi-process (world_size 2, gloo, CPU) tests of the sharding + gather.

The B200 path runs the same functions over NCCL; here the collective is
exercised on CPU tensors so the host-side logic is covered without GPUs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_20198_b200.parallel import band_for, gather_tiles


def test_bands_partition_rows():
    for world in (1, 2, 3, 4, 8):
        for rows in (8, 31, 32, 1000):
            bands = [band_for(r, world, rows) for r in range(world)]
            owned = [row for b in bands for row in range(b.row0, b.row1)]
            assert owned == list(range(rows))
            for b in bands:
                assert b.halo0 == max(0, b.row0 - 1)
                assert b.halo1 == min(rows, b.row1 + 1)


def test_halo_covers_padded_squares():
    """Every patch's 960 m padded square lies inside its rank's halo band."""
    world, rows = 4, 32
    for r in range(world):
        b = band_for(r, world, rows)
        for row in range(b.row0, b.row1):
            cy = row * 640.0 + 320.0
            lo = int(np.floor((cy - 480.0) / 640.0))
            hi = int(np.floor((cy + 480.0) / 640.0))
            assert max(lo, 0) >= b.halo0 and min(hi, rows - 1) < b.halo1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        band = band_for(rank, world, 5)
        own = torch.full((band.own_rows * 3, 64, 64, 4), float(rank))
        own[:, 0, 0, 0] = torch.arange(len(own), dtype=torch.float32)
        got = gather_tiles(own, dst=0)
        if rank == 0:
            q.put([(g.shape[0], float(g[0, 1, 1, 1]), g[:, 0, 0, 0].tolist())
                   for g in got])
    finally:
        dist.destroy_process_group()


def test_gather_tiles_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # 5 rows over 2 ranks -> 3 + 2 rows, 3 tiles per row; ragged gather
    assert [r[0] for r in res] == [9, 6]
    assert [r[1] for r in res] == [0.0, 1.0]
    assert res[1][2] == [float(i) for i in range(6)]
