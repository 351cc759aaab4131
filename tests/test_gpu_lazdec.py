"""Full LAZ chunk decode on the GPU (needs a B200): bit-exact with the
reference's load_tile_fullres / decode_chunk (reader.py:286-364, the
POINT10 / GPSTIME11 / RGB12 v2 item decoders of items.py) on
reference-compressed files (tests/golden/fullres.npz, formats 0-3, fixed
and variable chunking, branchy returns / classes / GPS sequences / colours),
in a batch of tiles (ts_lazdec) and through the drop-in functions."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_batched_decode_equals_reference(golden):
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.lasio import parse_header
    g = golden("fullres.npz")
    for fmt in range(4):
        ks = [k for k in range(int(g["n_files"])) if int(g[f"fmt{k}"]) == fmt]
        imgs = [g[f"file{k}"].tobytes() for k in ks] * 3   # repeated: many chunks
        descs = np.concatenate([D.tile_desc(parse_header(b)) for b in imgs])
        tb = D.TileBatch(imgs, descs)
        tables = D.ChunkTables(tb)
        assert not tables.status.any()
        fr = D.FullRecords(tb, tables)
        assert not fr.status.any(), fr.status.cpu().numpy()
        want = b"".join(g[f"rec{k}"].tobytes() for k in ks) * 3
        assert fr.records[:len(want)].cpu().numpy().tobytes() == want, fmt


def test_drop_in_load_tile_fullres_and_decode_chunk(golden, tmp_path):
    from paper_2509_20198_b200.lasio import (decode_chunk, ensure_chunk_refs,
                                             load_tile_fullres, scan_tile)
    g = golden("fullres.npz")
    for k in range(int(g["n_files"])):
        p = tmp_path / f"f{k}.laz"
        p.write_bytes(g[f"file{k}"].tobytes())
        tile = scan_tile(str(p), k)
        full = load_tile_fullres(tile)
        assert full.tobytes() == g[f"rec{k}"].tobytes(), k
        refs = ensure_chunk_refs(tile)
        dt = full.dtype
        one = decode_chunk(tile, refs[-1])
        start = sum(r.point_count for r in refs[:-1])
        assert one.tobytes() == full[start:].tobytes(), k


def test_corrupt_chunk_desyncs(golden):
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.lasio import parse_header
    g = golden("fullres.npz")
    img = bytearray(g["file2"].tobytes())
    h = parse_header(bytes(img))
    tb = D.TileBatch([bytes(img)], D.tile_desc(h))
    tables = D.ChunkTables(tb)
    off = tables.offsets[:tables.total].cpu().numpy()
    end = int(tables.end[0].item())
    # truncate the first chunk's stream: its decoder must run past the end
    # of its extent -> DecoderDesync, the other chunks still decode
    cut = D.TileBatch([bytes(img)], D.tile_desc(h))
    tab2 = D.ChunkTables(cut)
    tab2.offsets[1] = int(off[0]) + 40
    fr = D.FullRecords(cut, tab2)
    st = fr.status.cpu().numpy()
    assert st[0] == 10 and (st[2:] == 0).all(), st
    assert end > off[-1]


def test_realistic_tile_decode_sha(golden):
    """A reference-compressed 200,000-point tile (4 chunks of 50,000, the
    reference's chunk size) decodes to the reference's records (SHA-256)."""
    import hashlib

    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.lasio import parse_header
    g = golden("fullres_big.npz")
    img = g["laz"].tobytes()
    tb = D.TileBatch([img], D.tile_desc(parse_header(img)))
    fr = D.FullRecords(tb, D.ChunkTables(tb))
    assert not fr.status.any()
    rec = fr.records[:int(g["n"]) * 26].cpu().numpy().tobytes()
    assert hashlib.sha256(rec).digest() == g["sha256"].tobytes()


def test_model_heavy_chunk_takes_the_big_arena(golden):
    """Hundreds of lazily created byte models outgrow the first pass's
    arena: the chunk is queued and decoded again with the big arena, still
    bit-exact (and batched with ordinary chunks)."""
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.lasio import parse_header
    g = golden("fullres_models.npz")
    h = golden("fullres.npz")
    imgs = [g["laz"].tobytes(), h["file3"].tobytes(), g["laz"].tobytes()]
    descs = np.concatenate([D.tile_desc(parse_header(b)) for b in imgs])
    tb = D.TileBatch(imgs, descs)
    fr = D.FullRecords(tb, D.ChunkTables(tb))
    assert not fr.status.any(), fr.status.cpu().numpy()
    want = g["rec"].tobytes() + h["rec3"].tobytes() + g["rec"].tobytes()
    assert fr.records[:len(want)].cpu().numpy().tobytes() == want
