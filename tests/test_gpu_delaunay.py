"""GPU Delaunay (ts_triangulate) under adversarial insertion orders and
patch sizes (needs a B200).

The kernel inserts points in index order (Bowyer-Watson, one warp per
patch).  Qhull (scipy.spatial.Delaunay, patches.py:316-326) is the oracle:
general-position inputs must give exactly Qhull's triangle set whatever the
order; degenerate inputs (cocircular, collinear) have several valid
triangulations, so there the result is checked for validity instead -- CCW
non-degenerate triangles tiling the padding square with every input point a
vertex and no point strictly inside any circumcircle (exact predicates).

Orders and sizes the shared-memory fast path does not see in the configs[1]
corpus: sorted x (flight-line sweeps), points on few parallel lines, a
circle, large patches (> 384 points: the global-memory mesh; > 32,767
points: vertex ids past 16 bits) and cavities past the shared-memory cavity
(176 triangles), which restart the patch in global memory.
"""
import ctypes as C

import numpy as np
import pytest
from scipy.spatial import Delaunay

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CORNERS = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0], [1.0, 1.0]])


def _gpu(xys):
    """Triangulate several patches in one launch; list of (tri, status)."""
    from paper_2509_20198_b200 import _device as D
    from paper_2509_20198_b200.patches import triangulate
    ns = [len(x) for x in xys]
    off = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
    xy = np.concatenate([np.asarray(x, np.float64).reshape(-1, 2) for x in xys])
    g = dict(n=len(xys), xy=D.upload(xy), h=D.upload(np.zeros(len(xy))),
             off=torch.from_numpy(off).cuda())
    t = triangulate(g)
    tri = t["tri"].cpu().numpy()
    ntri = t["ntri"].cpu().numpy()
    st = t["status"].cpu().numpy()
    out = []
    for p, n in enumerate(ns):
        base = 2 * off[p] + 8 * p
        out.append((tri[base:base + ntri[p]], int(st[p])))
    return out


def _tri_set(simp):
    return set(tuple(sorted(s)) for s in np.asarray(simp).tolist())


def _qhull(xy):
    return Delaunay(np.vstack([xy, CORNERS])).simplices


def _check_valid(xy, tri, check_empty_circle=True):
    from paper_2509_20198_b200._lib import lib
    allxy = np.vstack([xy, CORNERS])
    a, b, c = allxy[tri[:, 0]], allxy[tri[:, 1]], allxy[tri[:, 2]]
    det = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - \
        (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])
    assert (det > 0).all(), "CW or degenerate triangle"
    assert abs(det.sum() / 2 - 4.0) < 1e-9, "triangles do not tile the square"
    uniq = np.unique(allxy, axis=0, return_index=True)[1]
    assert set(np.unique(tri)) >= set(uniq.tolist()), "a point is no vertex"
    if not check_empty_circle:
        return
    c2 = lambda v: (C.c_double * 2)(*v)  # noqa: E731
    pts = [c2(p) for p in allxy]
    for t in tri:
        pa, pb, pc = pts[t[0]], pts[t[1]], pts[t[2]]
        for i in range(len(allxy)):
            if i in t:
                continue
            assert lib().ts_incircle_sign(pa, pb, pc, pts[i]) <= 0, (t, i)


@pytest.mark.parametrize("order", ["sorted_x", "sorted_y", "reverse_x", "spiral"])
def test_insertion_orders_match_qhull(order):
    rng = np.random.default_rng(5150)
    xy = rng.uniform(-0.95, 0.95, (330, 2))
    if order == "sorted_x":
        xy = xy[np.argsort(xy[:, 0])]
    elif order == "sorted_y":
        xy = xy[np.argsort(xy[:, 1])]
    elif order == "reverse_x":
        xy = xy[np.argsort(-xy[:, 0])]
    else:
        r = np.hypot(xy[:, 0], xy[:, 1])
        xy = xy[np.argsort(r)]
    (tri, st), = _gpu([xy])
    assert st == 0
    assert _tri_set(tri) == _tri_set(_qhull(xy))


def test_flight_lines_valid():
    """Points on a few parallel scan lines (collinear runs) in line order."""
    rng = np.random.default_rng(61)
    lines = []
    for y in np.linspace(-0.8, 0.8, 6):
        x = np.sort(rng.uniform(-0.9, 0.9, 50))
        lines.append(np.stack([x, np.full_like(x, y)], 1))
    xy = np.vstack(lines)
    (tri, st), = _gpu([xy])
    assert st == 0
    _check_valid(xy, tri)


def test_circle_valid():
    """Cocircular points (every incircle test of neighbours is exactly 0)."""
    t = np.linspace(0, 2 * np.pi, 64, endpoint=False)
    xy = np.stack([0.5 * np.cos(t), 0.5 * np.sin(t)], 1)
    xy = np.vstack([xy, [[0.0, 0.0]], xy[:8]])  # centre + exact duplicates
    (tri, st), = _gpu([xy])
    assert st == 0
    _check_valid(xy, tri)


def test_large_cavity_restarts_in_global_memory():
    """Points in sorted-x order along a parabola: each insertion's cavity
    holds every triangle of the lower hull so far (> 176 late in the run),
    so the shared-memory attempt overflows and the patch restarts on the
    global-memory mesh; the result must still equal Qhull's."""
    x = np.linspace(-0.9, 0.9, 370)
    xy = np.stack([x, 0.9 - 1.7 * x ** 2 + 1e-3 * np.sin(37 * x)], 1)
    (tri, st), = _gpu([xy])
    assert st == 0
    assert _tri_set(tri) == _tri_set(_qhull(xy))


@pytest.mark.parametrize("n", [385, 1500, 33000])
def test_large_patches_match_qhull(n):
    """Past the shared-memory mesh (385, 1500) and past 16-bit vertex ids
    (33,000 > 32,767), batched with a small patch."""
    rng = np.random.default_rng(n)
    big = rng.uniform(-0.99, 0.99, (n, 2))
    small = rng.uniform(-0.9, 0.9, (40, 2))
    (tb, sb), (ts, ss) = _gpu([big, small])
    assert sb == 0 and ss == 0
    assert _tri_set(tb) == _tri_set(_qhull(big))
    assert _tri_set(ts) == _tri_set(_qhull(small))
