"""K1 on files (needs a B200): the drop-in reads files the way the
reference does (reader.py:146-160, 270-278) -- the chunk-table pointer and
table bytes, then one 4 KiB-aligned pread per chunk -- and uploads only
the table and a 64-byte window per chunk record, never the whole file.
Records equal the in-memory path and the reference's own bytes; cached
chunk_refs are honoured; errors keep the reference's classes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(data)
    return str(p)


def test_staged_batch_equals_in_memory_and_uploads_windows_only(tmp_path):
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200 import synth
    from paper_2509_20198_b200.lasio import parse_header, scan_tile
    from paper_2509_20198_b200.lasio.reader import StagedChunkPoints
    from paper_2509_20198_b200.lasio.writer import laz_image
    tiles = synth.grid_tiles((0, 3), (0, 2), chunks_per_tile=150)
    # realistic chunk bodies (~30 KB each: 4.5 MB files) so a whole-file
    # upload would be 70x the staged bytes
    rng = np.random.default_rng(3)
    paths, images = [], []
    for i, t in enumerate(tiles):
        img = laz_image(t.first_records, 2, 50_000, rng.integers(20_000, 40_000, 150))
        images.append(img)
        paths.append(_write(tmp_path, f"t{i}.laz", img))
    metas = [scan_tile(p, i) for i, p in enumerate(paths)]
    st = StagedChunkPoints(metas)
    cp = D.ChunkPoints(st.tb, st)
    descs = np.concatenate([D.tile_desc(parse_header(b)) for b in images])
    tb = D.TileBatch(images, descs)
    tables = D.ChunkTables(tb)
    ref = D.ChunkPoints(tb, tables)
    n = tables.total
    assert st.total == n
    assert torch.equal(cp.records[:n * 26], ref.records[:n * 26])
    assert torch.equal(cp.xyz[:n], ref.xyz[:n]) and torch.equal(cp.rgb[:n], ref.rgb[:n])
    assert torch.equal(cp.cells[:n], ref.cells[:n])
    assert st.staged_bytes <= 64 * n + 64
    assert sum(len(b) for b in images) > 50 * st.staged_bytes
    for m in metas:
        assert m.chunk_refs is not None and len(m.chunk_refs) == 150


def test_cached_chunk_refs_are_used(tmp_path):
    """An uncompressed LAS read with one stride, then read_chunk_points with
    another: the reference reads from the cached refs (reader.py:262-267)."""
    from paper_2509_20198_b200 import synth
    from paper_2509_20198_b200.lasio import ensure_chunk_refs, read_chunk_points, scan_tile
    from paper_2509_20198_b200.lasio.writer import las_image
    rec = synth.plane_records(0.1, 0.2, 5.0, 0.0, 0.0, 640.0, 1000, seed=2)
    path = _write(tmp_path, "a.las", las_image(rec, 2))
    tile = scan_tile(path, 0)
    ensure_chunk_refs(tile, las_stride=100)
    got = read_chunk_points(tile, las_stride=250)
    assert len(got) == 10
    assert got.tobytes() == rec[::100].tobytes()


def test_file_errors_keep_reference_classes(tmp_path):
    from paper_2509_20198_b200 import synth
    from paper_2509_20198_b200.errors import CorruptChunkTable, OutOfBoundsRead
    from paper_2509_20198_b200.lasio import parse_header, read_chunk_points, scan_tile
    from paper_2509_20198_b200.lasio.writer import las_image
    t = synth.grid_tiles((0, 1), (0, 1), chunks_per_tile=20)[0]
    pdo = parse_header(t.data).point_data_offset
    bad = bytearray(t.data)
    bad[pdo:pdo + 8] = (10 ** 12).to_bytes(8, "little")
    with pytest.raises(CorruptChunkTable):
        read_chunk_points(scan_tile(_write(tmp_path, "p.laz", bytes(bad)), 0))
    # -1 pointer: the table position lives in the last 8 bytes
    tpos = int.from_bytes(t.data[pdo:pdo + 8], "little")
    tail = bytearray(t.data)
    tail[pdo:pdo + 8] = (-1).to_bytes(8, "little", signed=True)
    tail += tpos.to_bytes(8, "little")
    got = read_chunk_points(scan_tile(_write(tmp_path, "m.laz", bytes(tail)), 0))
    assert got.tobytes() == t.first_records.tobytes()
    # LAS whose header claims more points than the file holds
    rec = synth.plane_records(0.0, 0.0, 1.0, 0.0, 0.0, 640.0, 300, seed=1)
    img = bytearray(las_image(rec, 2))
    img[107:111] = (900).to_bytes(4, "little")   # legacy point count
    with pytest.raises(OutOfBoundsRead):
        read_chunk_points(scan_tile(_write(tmp_path, "o.las", bytes(img)), 0), las_stride=100)
