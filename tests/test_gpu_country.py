"""configs[3] streaming driver (needs a B200): a grid streamed in blocks
with halo rings, split into row bands, equals one whole-grid pipeline run
bit for bit (heights, colours, c_z, status)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

COLS, ROWS = 10, 9


def test_streamed_blocks_and_bands_equal_whole_grid():
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.country import TILE, CountryRun, TilePool
    from paper_2509_20198_b200.pipeline import HeightmapPipeline
    from paper_2509_20198_b200.refiner import default_descriptor, random_weights
    pool = TilePool(side=3)
    pipe = HeightmapPipeline(random_weights(default_descriptor(), seed=3))
    cy, cx = np.meshgrid(np.arange(ROWS), np.arange(COLS), indexing="ij")
    buf, descs = pool.images_for(cx.ravel(), cy.ravel())
    tb = D.TileBatch.from_device(torch.from_numpy(buf).cuda(), descs)
    centers = np.stack([cx.ravel() * TILE + TILE / 2, cy.ravel() * TILE + TILE / 2], 1)
    cr = HeightmapPipeline.cell_range((0.0, 0.0), (COLS * TILE, ROWS * TILE))
    whole = pipe.run(tb, centers, cr)
    assert (whole["status"] == 0).all()
    for world, block in ((1, 4), (2, 3), (3, 5)):
        outs, czs = [], []
        for rank in range(world):
            run = CountryRun(pipe, pool, COLS, ROWS, block=block, rank=rank, world=world)
            assert run.run() == len(run.blocks)
            assert (run.status == 0).all()
            outs.append(run.out)
            czs.append(run.cz)
        torch.cuda.synchronize()
        assert torch.equal(torch.cat(outs), whole["out"]), (world, block)
        assert torch.equal(torch.cat(czs), whole["cz"]), (world, block)


def test_pool_tiles_move_records_exactly():
    """Virtual tile (cx, cy) = its pool tile with every first record moved
    by whole tiles: the extracted chunk points sit in the virtual footprint."""
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.country import TILE, TilePool
    pool = TilePool(side=2, chunks_per_tile=40)
    cx, cy = np.array([0, 7, 999, 123]), np.array([0, 3, 999, 456])
    buf, descs = pool.images_for(cx, cy)
    tb = D.TileBatch.from_device(torch.from_numpy(buf).cuda(), descs)
    tables = D.ChunkTables(tb)
    cp = D.ChunkPoints(tb, tables, records=False)
    xyz = cp.xyz.cpu().numpy().reshape(len(cx), 40, 3)
    k = pool.pick(cx, cy)
    for i in range(len(cx)):
        assert (xyz[i, :, 0] >= cx[i] * TILE).all() and (xyz[i, :, 0] < (cx[i] + 1) * TILE).all()
        assert (xyz[i, :, 1] >= cy[i] * TILE).all() and (xyz[i, :, 1] < (cy[i] + 1) * TILE).all()
        ref = pool.images[k[i]]
        # heights untouched
        rec = np.frombuffer(ref.tobytes(), np.uint8)
        z = np.array([np.frombuffer(rec[o + 8:o + 12].tobytes(), "<i4")[0]
                      for o in pool.rec_off[k[i]]]) * 0.01
        assert np.array_equal(xyz[i, :, 2], z)
