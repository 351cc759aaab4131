"""Row-band sharding reproduces the unsharded run bit for bit (needs a B200).

SURVEY §8(e): each rank processes a contiguous band of tile rows plus a
one-tile halo row on each interior side (a patch's padded square reaches
480 m < 640 m into its neighbours) and the finished tiles are gathered to
rank 0.  Here the ranks of a world of 2 and 4 run one after another on one
GPU; their owned tiles, concatenated in rank order (what
``parallel.gather_tiles`` returns on rank 0), must equal the 1-GPU run of
the whole grid exactly -- heights, colours, c_z and status.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

COLS, ROWS = 6, 8


def _run(tiles, own_rows, pipe):
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.lasio import parse_header
    from paper_2509_20198_b200.pipeline import HeightmapPipeline
    descs = np.concatenate([D.tile_desc(parse_header(t.data)) for t in tiles])
    tb = D.TileBatch([t.data for t in tiles], descs)
    own = [t for t in tiles if int(round(t.y0 / 640.0)) in own_rows]
    centers = np.array([[t.x0 + 320.0, t.y0 + 320.0] for t in own])
    x0s = [t.x0 for t in tiles]
    y0s = [t.y0 for t in tiles]
    cr = HeightmapPipeline.cell_range((min(x0s), min(y0s)),
                                      (max(x0s) + 640.0, max(y0s) + 640.0))
    res = pipe.run(tb, centers, cr)
    torch.cuda.synchronize()
    return res


@pytest.mark.parametrize("world", [2, 4])
def test_bands_equal_unsharded(world):
    from paper_2509_20198_b200 import synth
    from paper_2509_20198_b200.parallel import band_for
    from paper_2509_20198_b200.pipeline import HeightmapPipeline
    from paper_2509_20198_b200.refiner import default_descriptor, random_weights
    pipe = HeightmapPipeline(random_weights(default_descriptor(), seed=3))
    full = _run(synth.grid_tiles((0, COLS), (0, ROWS), chunks_per_tile=150),
                range(ROWS), pipe)
    outs, czs = [], []
    for rank in range(world):
        b = band_for(rank, world, ROWS)
        tiles = synth.grid_tiles((0, COLS), (b.halo0, b.halo1), chunks_per_tile=150)
        res = _run(tiles, range(b.row0, b.row1), pipe)
        assert (res["status"] == 0).all()
        outs.append(res["out"])
        czs.append(res["cz"])
    assert torch.equal(torch.cat(outs), full["out"])
    assert torch.equal(torch.cat(czs), full["cz"])
