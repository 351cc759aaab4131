"""WireHeightmap records written on the device (needs a B200).

``ts_wire_heightmaps`` against the reference's ``server.wire_heightmap``
bytes (tests/golden/wire.npz) and against the oracle on a refined pipeline
batch: bit-exact.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import wire as owire  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("name,colour", [("rgb", True), ("nocol", False)])
def test_wire_vs_reference_bytes(golden, name, colour):
    from paper_2509_20198_b200 import wire
    g = golden("wire.npz")
    out = np.concatenate([g[f"{name}_h"][..., None], g[f"{name}_rgb"]], axis=-1)
    buf = wire.wire_heightmaps(torch.from_numpy(np.ascontiguousarray(out)).cuda(),
                               g[f"{name}_cz"], g[f"{name}_ij"], g[f"{name}_stage"], colour)
    torch.cuda.synchronize()
    assert buf.cpu().numpy().tobytes() == g[f"{name}_wire"].tobytes()
    recs = wire.split_records(buf, colour)
    assert len(recs) == len(g[f"{name}_cz"])
    assert all(len(r) == (28686 if colour else 16398) for r in recs)


def test_wire_of_a_refined_batch():
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200 import synth, wire
    from paper_2509_20198_b200.lasio import parse_header
    from paper_2509_20198_b200.pipeline import HeightmapPipeline
    from paper_2509_20198_b200.refiner import default_descriptor, random_weights
    tiles = synth.chunked_terrain_tiles(3, 3, chunks_per_tile=150)
    descs = np.concatenate([D.tile_desc(parse_header(t.data)) for t in tiles])
    tb = D.TileBatch([t.data for t in tiles], descs)
    pipe = HeightmapPipeline(random_weights(default_descriptor(), seed=3), 4)
    centers = np.array([[t.x0 + 320.0, t.y0 + 320.0] for t in tiles])
    res = pipe.run(tb, centers)
    B = len(centers)
    ij = np.array([[k % 3, k // 3] for k in range(B)], np.int32)
    stage = np.full(B, 3, np.uint8)
    buf = wire.wire_heightmaps(res["out"], res["cz"], ij, stage, True)
    recs = wire.split_records(buf, True)
    out = res["out"].cpu().numpy()
    cz = res["cz"].cpu().numpy()
    for p in range(B):
        want = owire.wire_record(ij[p][0], ij[p][1], float(cz[p]), 3,
                                 out[p, :, :, 0], out[p, :, :, 1:4])
        assert recs[p] == want, p
