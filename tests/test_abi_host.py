"""CPU-only checks of the native library and the host-side logic.

No compute kernel is launched here (no GPU in the build container): the
library must load, export every symbol ``include/ts_b200.h`` declares,
and its host-callable predicate hooks must agree with exact rational
arithmetic.  Host helpers (descriptor/LSWB, key grid, stub writer) are
checked against the oracle and the reference's formats.
"""

import ctypes as C
import os
import re
from fractions import Fraction

import numpy as np
import pytest

from paper_2509_20198_b200._lib import LIB_PATH, SIGNATURES, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ts_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB_PATH), "run __graft_entry__.build() first"
    handle = C.CDLL(LIB_PATH)
    decl = declared_symbols()
    assert decl, "no declarations parsed"
    for name in decl:
        assert hasattr(handle, name), name
    assert decl == set(SIGNATURES), decl ^ set(SIGNATURES)
    lib()
    assert b"sm_100a" in lib().ts_version()
    assert [lib().ts_record_size(f) for f in range(5)] == [20, 28, 26, 34, -1]


def _frac_orient(a, b, c):
    a, b, c = [tuple(map(Fraction, p)) for p in (a, b, c)]
    d = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
    return (d > 0) - (d < 0)


def _frac_incircle(a, b, c, d):
    a, b, c, d = [tuple(map(Fraction, p)) for p in (a, b, c, d)]
    adx, ady = a[0] - d[0], a[1] - d[1]
    bdx, bdy = b[0] - d[0], b[1] - d[1]
    cdx, cdy = c[0] - d[0], c[1] - d[1]
    det = (adx * adx + ady * ady) * (bdx * cdy - cdx * bdy) + \
          (bdx * bdx + bdy * bdy) * (cdx * ady - adx * cdy) + \
          (cdx * cdx + cdy * cdy) * (adx * bdy - bdx * ady)
    return (det > 0) - (det < 0)


def _arr(p):
    return (C.c_double * 2)(*p)


def test_exact_predicates_match_rationals():
    rng = np.random.default_rng(7)
    cases = []
    # cocircular / collinear lattice points (fp64 filter cannot decide)
    for _ in range(300):
        pts = rng.integers(-4, 5, (4, 2)) / 4.0
        cases.append([tuple(p) for p in pts])
    # near-degenerate perturbations at the last ulp
    for _ in range(300):
        t = rng.uniform(0, 2 * np.pi, 4)
        pts = np.stack([np.cos(t), np.sin(t)], 1) * 0.7 + 0.1
        pts[3] = np.nextafter(pts[3], pts[3] + rng.choice([-1, 1], 2))
        cases.append([tuple(p) for p in pts])
    # patch-space-like values with exponent spread
    for _ in range(300):
        pts = rng.uniform(-1, 1, (4, 2)) * 10.0 ** rng.integers(-12, 0, (4, 1))
        cases.append([tuple(p) for p in pts])
    for a, b, c, d in cases:
        assert lib().ts_orient_sign(_arr(a), _arr(b), _arr(c)) == \
            _frac_orient(a, b, c)
        if _frac_orient(a, b, c) > 0:
            assert lib().ts_incircle_sign(_arr(a), _arr(b), _arr(c),
                                          _arr(d)) == \
                _frac_incircle(a, b, c, d), (a, b, c, d)


def test_descriptor_and_lswb_roundtrip(tmp_path):
    from oracle import refiner as oref
    from paper_2509_20198_b200 import refiner as R
    d = R.default_descriptor()
    assert d.parameter_count() == 2_432_868
    text = d.to_text()
    assert oref.layers_to_text(oref.text_to_layers(text)) == text
    b = R.random_weights(d, seed=3)
    p = tmp_path / "w.lswb"
    R.save_weights(str(p), b)
    b2 = R.load_weights(str(p))
    assert b2.descriptor.to_text() == text
    for k in b.tensors:
        assert np.array_equal(b.tensors[k], b2.tensors[k])
    from paper_2509_20198_b200.errors import BadMagic, UnsupportedVersion
    p.write_bytes(b"XXXX" + p.read_bytes()[4:])
    with pytest.raises(BadMagic):
        R.load_weights(str(p))
    with pytest.raises(UnsupportedVersion):
        R.ArchDescriptor.from_text("arch 2\n")


def test_stub_writer_roundtrip_through_oracle():
    from oracle import laz as olaz
    from paper_2509_20198_b200 import synth
    from paper_2509_20198_b200.lasio import parse_header
    tiles = synth.chunked_terrain_tiles(2, 1, chunks_per_tile=40)
    for t in tiles:
        rec = olaz.chunk_points(t.data)
        assert rec.tobytes() == t.first_records.tobytes()
        h = parse_header(t.data)
        assert h.point_count == 40 * 50_000
        assert h.laszip.chunk_size == 50_000


def test_key_grid_registers_every_window():
    from paper_2509_20198_b200.engine import key_grid
    rng = np.random.default_rng(3)
    centers = np.concatenate([
        np.stack(np.meshgrid(np.arange(4) * 640.0 + 320.0,
                             np.arange(3) * 640.0 + 320.0), -1).reshape(-1, 2),
        rng.uniform(-2000, 5000, (10, 2))])
    off, ids, gx0, gy0, gnx, gny, inner = key_grid(centers)
    pts = np.concatenate([rng.uniform(-3000, 6000, (20000, 2)),
                          np.round(rng.uniform(0, 2560, (4000, 2)) / 640.0) *
                          640.0 + rng.uniform(-0.05, 0.05, (4000, 2))])
    for x, y in pts:
        gx = int(np.floor((x - gx0) / 640.0))
        gy = int(np.floor((y - gy0) / 640.0))
        inside = np.nonzero(
            (np.floor((x - (centers[:, 0] - 320.0)) / 10.0) >= 0) &
            (np.floor((x - (centers[:, 0] - 320.0)) / 10.0) < 64) &
            (np.floor((y - (centers[:, 1] - 320.0)) / 10.0) >= 0) &
            (np.floor((y - (centers[:, 1] - 320.0)) / 10.0) < 64))[0]
        if len(inside) == 0:
            continue
        assert 0 <= gx < gnx and 0 <= gy < gny
        c = gy * gnx + gx
        listed = set(ids[off[c]:off[c + 1]].tolist())
        assert set(inside.tolist()) <= listed
        ox, oy = x - gx0 - 640.0 * gx, y - gy0 - 640.0 * gy
        if 0.02 <= ox <= 639.98 and 0.02 <= oy <= 639.98:
            assert set(inside.tolist()) <= set(ids[off[c]:off[c] + inner[c]])


def test_key_grid_interior_list_of_a_tiling_is_one_key():
    """A tiling of keys: every cell's interior list is just its own key."""
    from paper_2509_20198_b200.engine import key_grid
    centers = np.stack(np.meshgrid(np.arange(5) * 640.0 + 320.0 + 7e5,
                                   np.arange(4) * 640.0 + 320.0 + 4e6),
                       -1).reshape(-1, 2)
    off, ids, gx0, gy0, gnx, gny, inner = key_grid(centers)
    for k, (cx, cy) in enumerate(centers):
        c = int((cy - 320 - gy0) // 640) * gnx + int((cx - 320 - gx0) // 640)
        assert inner[c] == 1 and ids[off[c]] == k
        assert off[c + 1] - off[c] == 9 or k in (0, 4, 15, 19) or \
            off[c + 1] - off[c] == 6


def test_wire_record_sizes_and_split():
    """WireHeightmap record sizes (docs/wire.md: 14 + 16,384 [+ 12,288]) and
    the host-side split of a batch buffer (no GPU needed)."""
    from paper_2509_20198_b200 import wire
    assert wire.record_size(True) == 28686
    assert wire.record_size(False) == 16398
    buf = bytes(range(256)) * (2 * 28686 // 256) + bytes(2 * 28686 % 256)
    recs = wire.split_records(buf, True)
    assert len(recs) == 2 and b"".join(recs) == buf
    with pytest.raises(ValueError):
        wire.split_records(buf[:-1], True)
