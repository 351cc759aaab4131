"""Oracle: chunk-point index, gather/normalise and Algorithm 1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``pkg/src/terrascout/patches.py``:
  * ``ChunkPointIndex`` add/query order (``:99-160``),
  * ``gather_and_normalize`` (``:163-177``),
  * ``_nn_assign`` as exact d^2 argmin, ties -> lowest index (``:180-199``;
    rule pinned by ``pkg/tests/test_patches.py:15-18``),
  * ``grid_cell_centers`` (``:208-212``), ``_ccw`` (``:215-224``),
    ``_TriGeom`` (``:227-253``), flood fill passes (``:256-349``), padding
    removal + barycentric fill (``:351-380``), ``_finish`` (``:386-405``).

Two face-map routines are provided: ``face_map_flood`` is the reference's
order-dependent flood fill (used to time the CPU baseline and to pin the
rule), ``face_map_lowest_id`` is the "lowest triangle id wins" statement the
reference's acceptance oracle uses (``test_acceptance.py:165-191``).
"""

from __future__ import annotations

import numpy as np
from scipy.spatial import Delaunay, QhullError

PATCH = 640.0
TEXEL = 10.0
RES = 96
OUT = 64
RADIUS = 480.0
TOL = 1e-9
CORNERS = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0], [1.0, 1.0]])


class Index:
    """Append-only 640 m grid; iteration order matches patches.py:131-153."""

    def __init__(self):
        self.blocks = []      # (xyz, rgb)
        self.cells = {}       # (ci, cj) -> [(block, rows)]

    def add(self, xyz, rgb):
        xyz = np.asarray(xyz, np.float64)
        if len(xyz) == 0:
            return
        b = len(self.blocks)
        self.blocks.append((xyz, rgb))
        ci = np.floor(xyz[:, 0] / PATCH).astype(np.int64)
        cj = np.floor(xyz[:, 1] / PATCH).astype(np.int64)
        for key in sorted(set(zip(ci.tolist(), cj.tolist()))):
            rows = np.nonzero((ci == key[0]) & (cj == key[1]))[0]
            self.cells.setdefault(key, []).append((b, rows))

    def query(self, cx, cy, r=RADIUS):
        parts, cparts = [], []
        for ci in range(int(np.floor((cx - r) / PATCH)),
                        int(np.floor((cx + r) / PATCH)) + 1):
            for cj in range(int(np.floor((cy - r) / PATCH)),
                            int(np.floor((cy + r) / PATCH)) + 1):
                for b, rows in self.cells.get((ci, cj), ()):
                    xyz, rgb = self.blocks[b]
                    parts.append(xyz[rows])
                    if rgb is not None:
                        cparts.append(rgb[rows])
        has_rgb = bool(self.blocks) and self.blocks[0][1] is not None
        if not parts:
            return np.empty((0, 3)), (np.empty((0, 3), np.float32)
                                      if has_rgb else None)
        xyz = np.concatenate(parts)
        keep = (np.abs(xyz[:, 0] - cx) <= r) & (np.abs(xyz[:, 1] - cy) <= r)
        rgb = np.concatenate(cparts)[keep] if has_rgb else None
        return xyz[keep], rgb


def gather(center, index: Index):
    """(xy, h, rgb, c_z) in patch space, or None when empty."""
    xyz, rgb = index.query(center[0], center[1])
    if len(xyz) == 0:
        return None
    d2 = (xyz[:, 0] - center[0]) ** 2 + (xyz[:, 1] - center[1]) ** 2
    c_z = float(xyz[int(np.argmin(d2)), 2])
    xy = (xyz[:, :2] - np.asarray(center)) / RADIUS
    h = (xyz[:, 2] - c_z) / RADIUS
    return xy, h, rgb, c_z


def cell_centers(res=RES):
    c = -1.0 + (np.arange(res) + 0.5) * (2.0 / res)
    gx, gy = np.meshgrid(c, c)
    return np.stack([gx.ravel(), gy.ravel()], axis=1)


def nn_assign(xy, q, block=2048):
    """Exact argmin of (dx^2 + dy^2); np.argmin keeps the first minimum."""
    out = np.empty(len(q), np.int64)
    for s in range(0, len(q), block):
        qq = q[s:s + block]
        dx = qq[:, None, 0] - xy[None, :, 0]
        dy = qq[:, None, 1] - xy[None, :, 1]
        out[s:s + block] = np.argmin(dx * dx + dy * dy, axis=1)
    return out


def ccw(simp, pts):
    a, b, c = pts[simp[:, 0]], pts[simp[:, 1]], pts[simp[:, 2]]
    det = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - \
          (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])
    out = simp.copy()
    neg = det < 0
    out[neg, 1], out[neg, 2] = simp[neg, 2], simp[neg, 1]
    return out


class TriGeom:
    def __init__(self, pts, tri):
        self.a = pts[tri[:, 0]]
        self.ab = pts[tri[:, 1]] - self.a
        self.ac = pts[tri[:, 2]] - self.a
        det = self.ab[:, 0] * self.ac[:, 1] - self.ab[:, 1] * self.ac[:, 0]
        det[det == 0] = np.inf
        self.inv = 1.0 / det

    def bary(self, t, p):
        px = p[..., 0] - self.a[t, 0]
        py = p[..., 1] - self.a[t, 1]
        w1 = (px * self.ac[t, 1] - py * self.ac[t, 0]) * self.inv[t]
        w2 = (self.ab[t, 0] * py - self.ab[t, 1] * px) * self.inv[t]
        return 1.0 - w1 - w2, w1, w2

    def inside(self, t, p):
        w = self.bary(t, p)
        return np.logical_and.reduce([(x >= -TOL) & (x <= 1.0 + TOL)
                                      for x in w])


def face_map_flood(all_xy, tri, geom, res=RES):
    """The reference's two-pass flood fill (patches.py:330-349)."""
    centers = cell_centers(res)
    face = np.full(res * res, -2, np.int32)

    def fill(seed, t):
        stack = [seed]
        while stack:
            j = stack.pop()
            if face[j] != -2 or not geom.inside(t, centers[j]):
                continue
            face[j] = t
            y, x = divmod(j, res)
            for ny in (y - 1, y, y + 1):
                if 0 <= ny < res:
                    for nx in (x - 1, x, x + 1):
                        if 0 <= nx < res and (nx != x or ny != y) and \
                                face[ny * res + nx] == -2:
                            stack.append(ny * res + nx)

    def grid_span(lo, hi):
        a = int(np.ceil((lo + 1.0) * res / 2.0 - 0.5))
        b = int(np.floor((hi + 1.0) * res / 2.0 - 0.5))
        return max(a, 0), min(b, res - 1)

    for t in range(len(tri)):
        cx, cy = all_xy[tri[t]].mean(axis=0)
        gx = min(max(int(np.round((cx + 1.0) * res / 2.0 - 0.5)), 0), res - 1)
        gy = min(max(int(np.round((cy + 1.0) * res / 2.0 - 0.5)), 0), res - 1)
        if face[gy * res + gx] == -2:
            fill(gy * res + gx, t)
    for t in range(len(tri)):
        v = all_xy[tri[t]]
        x0, x1 = grid_span(max(v[:, 0].min(), -1.0), min(v[:, 0].max(), 1.0))
        y0, y1 = grid_span(max(v[:, 1].min(), -1.0), min(v[:, 1].max(), 1.0))
        for gy in range(y0, y1 + 1):
            for gx in range(x0, x1 + 1):
                j = gy * res + gx
                if face[j] == -2 and geom.inside(t, centers[j]):
                    fill(j, t)
    return face


def face_map_lowest_id(tri, geom, res=RES):
    """Vectorised 'lowest triangle id wins' over every cell centre."""
    centers = cell_centers(res)
    face = np.full(res * res, -2, np.int32)
    for t in range(len(tri)):
        open_ = face == -2
        ins = geom.inside(t, centers) & open_
        face[ins] = t
    return face


def interpolate(xy, h, rgb, c_z, key_center=None, res=RES, tri=None,
                flood=False):
    """Algorithm 1 (patches.py:290-405).  Returns a dict of rasters.

    ``tri``: optional precomputed simplices (else Qhull like the
    reference).  ``flood``: use the reference's flood fill instead of the
    equivalent lowest-id rule.
    """
    n = len(xy)
    centers = cell_centers(res)
    nn = nn_assign(xy, centers) if n > 1 else np.zeros(res * res, np.int64)
    hm_nn = h[nn].reshape(res, res)
    rgb_nn = rgb[nn].reshape(res, res, 3) if rgb is not None else None
    hm_lin = hm_nn.copy()
    rgb_lin = rgb_nn.copy() if rgb_nn is not None else None
    all_xy = np.vstack([xy, CORNERS])
    face = np.full(res * res, -1, np.int32)
    triangles = None
    try:
        simp = Delaunay(all_xy).simplices.astype(np.int64) if tri is None \
            else np.asarray(tri, np.int64)
    except QhullError:
        simp = None
    if simp is not None:
        triangles = ccw(simp, all_xy)
        geom = TriGeom(all_xy, triangles)
        face = face_map_flood(all_xy, triangles, geom, res) if flood else \
            face_map_lowest_id(triangles, geom, res)
        pad = (triangles >= n).any(axis=1)
        cov = face >= 0
        face[cov & pad[np.where(cov, face, 0)]] = -1
        face[face == -2] = -1
        inside = np.nonzero(face >= 0)[0]
        if len(inside):
            t = face[inside]
            p = centers[inside] - geom.a[t]
            w1 = (p[:, 0] * geom.ac[t, 1] - p[:, 1] * geom.ac[t, 0]) * \
                geom.inv[t]
            w2 = (geom.ab[t, 0] * p[:, 1] - geom.ab[t, 1] * p[:, 0]) * \
                geom.inv[t]
            w0 = 1.0 - w1 - w2
            v = triangles[t]
            hm_lin.ravel()[inside] = w0 * h[v[:, 0]] + w1 * h[v[:, 1]] + \
                w2 * h[v[:, 2]]
            if rgb_lin is not None:
                rgb_lin.reshape(-1, 3)[inside] = \
                    w0[:, None] * rgb[v[:, 0]] + w1[:, None] * rgb[v[:, 1]] \
                    + w2[:, None] * rgb[v[:, 2]]
    if key_center is not None:
        shift = float(hm_lin[res // 2, res // 2])
        hm_lin = hm_lin - shift
        hm_nn = hm_nn - shift
        c_z = c_z + shift * RADIUS
    return dict(hm_nn=hm_nn.astype(np.float32),
                hm_lin=hm_lin.astype(np.float32),
                rgb_nn=None if rgb_nn is None else rgb_nn.astype(np.float32),
                rgb_lin=None if rgb_lin is None else
                rgb_lin.astype(np.float32),
                face=face.reshape(res, res), c_z=c_z, nn=nn,
                triangles=triangles, n=n)


def reconstruct(center, index: Index, res=RES, flood=False):
    g = gather(center, index)
    if g is None:
        return None
    xy, h, rgb, c_z = g
    return interpolate(xy, h, rgb, c_z, key_center=center, res=res,
                       flood=flood)
