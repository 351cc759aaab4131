"""configs[3] driver, host side (no GPU): the streaming path's block staging
(pool images concatenated, record moves applied afterwards by
TilePool.move_records -- on the device in CountryRun, here on CPU tensors)
produces exactly the bytes of the reference-style host path images_for."""
import numpy as np
import torch

from paper_2509_20198_b200.country import TilePool


def test_staged_block_equals_host_images():
    pool = TilePool(side=2, chunks_per_tile=30, points_per_chunk=2000)
    rng = np.random.default_rng(5)
    cx = rng.integers(0, 1000, 40)
    cy = rng.integers(0, 1000, 40)
    want, wdesc = pool.images_for(cx, cy)
    buf, desc, meta = pool.stage(cx, cy, pin=False)
    pool.move_records(buf, meta)
    assert np.array_equal(buf.numpy(), want)
    assert np.array_equal(desc["file_offset"], wdesc["file_offset"])
    assert np.array_equal(desc["file_size"], wdesc["file_size"])
