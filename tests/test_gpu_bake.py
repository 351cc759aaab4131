"""K4 full-resolution texel update vs the oracle (needs a B200).

Tolerances: texel assignment exact (the covered
mask of a NaN prior is compared bit for bit), heights |dh| <= 1e-6 m, rgb
<= 1e-6.  The kernel accumulates in fixed point, so the result must also be
bit-identical under any permutation of the points.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import bake as obake  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _keys_and_bases(centers, cz=50.0, base_cz=40.0, colored=True, seed=0):
    from paper_2509_20198_b200.patches import PatchKey
    from paper_2509_20198_b200.refiner import RefinedPatch
    rng = np.random.default_rng(seed)
    keys, bases = [], []
    for p, c in enumerate(centers):
        keys.append(PatchKey(p, 0, tuple(c), cz))
        h = np.full((64, 64), np.nan, np.float32)
        rgb = rng.random((64, 64, 3), dtype=np.float32) if colored else None
        bases.append(RefinedPatch(PatchKey(p, 0, tuple(c), base_cz), h, rgb,
                                  "refined"))
    return keys, bases


def _grouped_points(side, per, seed, ox=0.0, oy=0.0):
    rng = np.random.default_rng(seed)
    xs, ys = [], []
    for j in range(side):
        for i in range(side):
            xs.append(np.round(ox + 640.0 * i + rng.random(per) * 640.0, 2))
            ys.append(np.round(oy + 640.0 * j + rng.random(per) * 640.0, 2))
    x, y = np.concatenate(xs), np.concatenate(ys)
    z = np.round(100.0 + 30.0 * np.sin(x / 300.0) + rng.normal(0, 2, len(x)), 2)
    rgb = rng.random((len(x), 3), dtype=np.float32)
    return np.stack([x, y, z], 1), rgb


def _check(out, xyz, rgb, keys, bases):
    for p, o in enumerate(out):
        h, c = obake.bake_one(xyz, rgb, bases[p].heights_rel, bases[p].key.c_z,
                              bases[p].rgb, keys[p].center, keys[p].c_z)
        assert np.array_equal(np.isnan(o.heights_rel), np.isnan(h)), p
        m = ~np.isnan(h)
        assert np.abs(o.heights_rel[m] - h[m]).max() <= 1e-6, p
        if c is not None:
            assert np.abs(o.rgb - c).max() <= 1e-6, p


def test_bake_grouped_and_permutation_invariant():
    from paper_2509_20198_b200.engine import bake_fullres
    side = 4
    centers = [(640.0 * i + 320.0, 640.0 * j + 320.0)
               for j in range(side) for i in range(side)]
    keys, bases = _keys_and_bases(centers)
    xyz, rgb = _grouped_points(side, 40000, 5)
    out = bake_fullres(xyz, rgb, bases, keys)
    _check(out, xyz, rgb, keys, bases)
    perm = np.random.default_rng(6).permutation(len(xyz))
    out2 = bake_fullres(xyz[perm], rgb[perm], bases, keys)
    for a, b in zip(out, out2):
        assert np.array_equal(a.heights_rel, b.heights_rel, equal_nan=True)
        assert np.array_equal(a.rgb, b.rgb)


def test_bake_overlapping_and_duplicate_keys():
    """Keys need not tile the plane: shifted and repeated keys each get
    every point their own predicate accepts."""
    from paper_2509_20198_b200.engine import bake_fullres
    centers = [(320.0, 320.0), (325.0, 317.5), (320.0, 320.0), (960.0, 320.0),
               (640.0, 640.0)]
    keys, bases = _keys_and_bases(centers, seed=2)
    xyz, rgb = _grouped_points(2, 30000, 8)
    out = bake_fullres(xyz, rgb, bases, keys)
    _check(out, xyz, rgb, keys, bases)
    assert np.array_equal(out[0].heights_rel, out[2].heights_rel,
                          equal_nan=True)


def test_bake_colour_sum_carry():
    """>256 unit-colour points in one texel wrap the 32-bit shared sums;
    the carry must land in the global sum (mean exactly 1.0)."""
    from paper_2509_20198_b200.engine import bake_fullres
    keys, bases = _keys_and_bases([(320.0, 320.0)], seed=3)
    n = 5000
    xyz = np.stack([np.full(n, 5.0), np.full(n, 5.0),
                    np.linspace(10.0, 20.0, n)], 1)
    rgb = np.ones((n, 3), np.float32)
    rgb[:, 1] = 0.999
    out = bake_fullres(xyz, rgb, bases, keys)
    _check(out, xyz, rgb, keys, bases)
    assert out[0].rgb[0, 0, 0] == 1.0


def test_bake_utm_seams_colourless():
    from paper_2509_20198_b200.engine import bake_fullres
    ox, oy = 712000.0, 4100000.0
    side = 3
    centers = [(ox + 640.0 * i + 320.0, oy + 640.0 * j + 320.0)
               for j in range(side) for i in range(side)]
    keys, bases = _keys_and_bases(centers, colored=False)
    xyz, _ = _grouped_points(side, 20000, 9, ox, oy)
    seam = np.random.default_rng(4)
    sx = ox + 640.0 * seam.integers(0, 4, 3000) + seam.choice([-1e-9, 0, 1e-9], 3000)
    sy = oy + seam.uniform(0, 1920, 3000)
    xyz = np.concatenate([xyz, np.stack([sx, sy, np.full(3000, 7.0)], 1)])
    out = bake_fullres(xyz, None, bases, keys)
    _check(out, xyz, None, keys, bases)
    assert all(o.rgb is None for o in out)


def test_bake_fast_path_edges_and_shifted_keys():
    """The splat's hot-patch fast path (points >= 2 cm inside a cell-aligned
    window skip the CSR walk) against the oracle: a 3 x 3 tiling with one key
    shifted by 3 mm (still within the 5 mm alignment tolerance) and one by
    7 mm (outside it: its cell has two interior keys), with points packed
    within +-3 cm of every window edge."""
    from paper_2509_20198_b200.engine import bake_fullres
    side = 3
    centers = [[640.0 * i + 320.0, 640.0 * j + 320.0]
               for j in range(side) for i in range(side)]
    centers[4][0] += 0.003
    centers[4][1] -= 0.002
    centers[2][0] += 0.007
    centers = [tuple(c) for c in centers]
    keys, bases = _keys_and_bases(centers, seed=4)
    xyz, rgb = _grouped_points(side, 20000, 11)
    rng = np.random.default_rng(12)
    n = 60000
    ex = 640.0 * rng.integers(0, side + 1, n) + rng.uniform(-0.03, 0.03, n)
    ey = rng.uniform(0.0, 640.0 * side, n)
    flip = rng.random(n) < 0.5
    ex, ey = np.where(flip, ey, ex), np.where(flip, ex, ey)
    edge = np.stack([ex, ey, rng.uniform(90.0, 110.0, n)], 1)
    xyz = np.concatenate([xyz, edge])
    rgb = np.concatenate([rgb, rng.random((n, 3), dtype=np.float32)])
    out = bake_fullres(xyz, rgb, bases, keys)
    _check(out, xyz, rgb, keys, bases)


def test_bin_points_groups_by_cell_and_keeps_the_bake():
    """ts_bake_bin: a permutation of the points, non-decreasing 640 m cell
    of the key grid (outside points last), and the bake of the binned
    points equals the bake of the shuffled ones bit for bit."""
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.engine import bake_device, bin_points, key_grid
    rng = np.random.default_rng(21)
    centers = np.stack(np.meshgrid(np.arange(5) * 640.0 + 320.0,
                                   np.arange(4) * 640.0 + 320.0), -1).reshape(-1, 2)
    m = 300_000
    xyz = np.stack([rng.uniform(-700, 3900, m), rng.uniform(-700, 3300, m),
                    rng.uniform(0, 100, m)], 1)
    rgb = rng.random((m, 3)).astype(np.float32)
    off, ids, gx0, gy0, gnx, gny, inner = key_grid(centers)
    dx, dc = D.upload(xyz), D.upload(rgb)
    bx, bc = bin_points(dx, dc, (gx0, gy0, gnx, gny))
    bxh, bch = bx.cpu().numpy(), bc.cpu().numpy()
    fx = np.floor((bxh[:, 0] - gx0) / 640.0)
    fy = np.floor((bxh[:, 1] - gy0) / 640.0)
    inside = (fx >= 0) & (fy >= 0) & (fx < gnx) & (fy < gny)
    cell = np.where(inside, fy * gnx + fx, gnx * gny)
    assert (np.diff(cell) >= 0).all()
    a = np.lexsort(np.hstack([xyz, rgb]).T)
    b = np.lexsort(np.hstack([bxh, bch]).T)
    assert np.array_equal(xyz[a], bxh[b]) and np.array_equal(rgb[a], bch[b])
    P = len(centers)
    prior = torch.zeros((P, 64, 64), device="cuda")
    prior_rgb = torch.zeros((P, 64, 64, 3), device="cuda")
    cz = torch.full((P,), 10.0, dtype=torch.float64, device="cuda")
    h1, c1 = bake_device(dx, dc, centers, prior, cz, cz, prior_rgb)
    h2, c2 = bake_device(bx, bc, centers, prior, cz, cz, prior_rgb)
    assert torch.equal(h1, h2) and torch.equal(c1, c2)
