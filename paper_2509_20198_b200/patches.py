"""Patch-space heightmap reconstruction (Algorithm 1) on the GPU.

Drop-in for ``pkg/src/terrascout/patches.py``: same constants, value
types and functions.  Every computation runs in CUDA through the C ABI:
  * ``ChunkPointIndex``  device-resident points + stable cell sort
    (``ts_index_build``) replacing the dict-of-lists index (:99-160),
  * ``gather_and_normalize`` -> ``ts_gather_count``/``ts_gather_fill``
    (:163-177),
  * ``nearest_neighbor_query`` -> ``ts_nearest`` (:180-205),
  * ``interpolate_patch`` / ``reconstruct_patch`` -> ``ts_triangulate``
    (GPU Delaunay replacing Qhull) + ``ts_raster`` (:290-412).
``reconstruct_batch`` is the batched entry point the engine/bench use:
one launch per kernel for any number of patches, rasters stay on device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from .errors import EmptyPatch, EmptySet, raise_for_status

PATCH_SIZE = 640.0
TEXEL_SIZE = 10.0
RASTER_RES = 96
OUTPUT_RES = 64
PAD_RADIUS = RASTER_RES * TEXEL_SIZE / 2.0  # 480 m
BARY_TOL = 1e-9


@dataclass(frozen=True)
class PatchKey:
    i: int
    j: int
    center: tuple[float, float]
    c_z: float = 0.0

    def with_cz(self, c_z: float) -> "PatchKey":
        return PatchKey(self.i, self.j, self.center, c_z)


@dataclass
class PatchGrid:
    origin: tuple[float, float]
    ni: int
    nj: int

    def key(self, i: int, j: int, c_z: float = 0.0) -> PatchKey:
        return PatchKey(i, j, (self.origin[0] + (i + 0.5) * PATCH_SIZE,
                               self.origin[1] + (j + 0.5) * PATCH_SIZE), c_z)

    def keys(self) -> list[PatchKey]:
        return [self.key(i, j) for j in range(self.nj) for i in range(self.ni)]

    def contains(self, i: int, j: int) -> bool:
        return 0 <= i < self.ni and 0 <= j < self.nj


def patch_grid_for(bbox_min, bbox_max) -> PatchGrid:
    """640 m-aligned patch grid covering a bbox (patches.py:63-71)."""
    if bbox_min[0] >= bbox_max[0] or bbox_min[1] >= bbox_max[1]:
        raise ValueError("degenerate bbox")
    ox = np.floor(bbox_min[0] / PATCH_SIZE) * PATCH_SIZE
    oy = np.floor(bbox_min[1] / PATCH_SIZE) * PATCH_SIZE
    return PatchGrid((ox, oy), int(np.ceil((bbox_max[0] - ox) / PATCH_SIZE)),
                     int(np.ceil((bbox_max[1] - oy) / PATCH_SIZE)))


@dataclass
class PatchSpacePoints:
    xy: np.ndarray
    h: np.ndarray
    rgb: np.ndarray | None
    c_z: float = 0.0


@dataclass
class FaceMap:
    res: int
    cells: np.ndarray


@dataclass
class RawPatch:
    key: PatchKey
    hm_nn: np.ndarray
    hm_lin: np.ndarray
    rgb_nn: np.ndarray | None
    rgb_lin: np.ndarray | None
    face_map: FaceMap
    chunk_point_count: int


def grid_cell_centers(res: int = RASTER_RES) -> np.ndarray:
    """(res*res, 2) cell-centred sample positions (patches.py:208-212)."""
    c = -1.0 + (np.arange(res) + 0.5) * (2.0 / res)
    gx, gy = np.meshgrid(c, c)
    return np.stack([gx.ravel(), gy.ravel()], axis=1)


# ------------------------------------------------------------------ index

class ChunkPointIndex:
    """Device-resident chunk points with a stable 640 m cell order.

    Iteration order of a query equals the reference's: x-cell, y-cell,
    insertion block, row (patches.py:119-145) -- a stable sort of point ids
    by dense cell id reproduces it exactly.
    """

    def __init__(self):
        self._xyz: list[torch.Tensor] = []
        self._rgb: list[torch.Tensor | None] = []
        self._cells: list[torch.Tensor | None] = []
        self.count = 0
        self.has_rgb: bool | None = None
        self._built = None

    def add_points(self, xyz, rgb, cells=None):
        if len(xyz) == 0:
            return
        if self.has_rgb is None:
            self.has_rgb = rgb is not None
        xyz_t = xyz if isinstance(xyz, torch.Tensor) else \
            D.upload(np.asarray(xyz, dtype=np.float64))
        rgb_t = None
        if self.has_rgb:
            rgb_t = rgb if isinstance(rgb, torch.Tensor) else \
                D.upload(np.asarray(rgb, dtype=np.float32))
        self._xyz.append(xyz_t.reshape(-1, 3))
        self._rgb.append(rgb_t)
        self._cells.append(cells)
        self.count += len(xyz_t)
        self._built = None

    def device_points(self):
        if self._built is None:
            xyz = torch.cat(self._xyz) if len(self._xyz) > 1 else self._xyz[0]
            rgb = None
            if self.has_rgb:
                rgb = torch.cat(self._rgb) if len(self._rgb) > 1 \
                    else self._rgb[0]
            if all(c is not None for c in self._cells):
                cells = torch.cat(self._cells) if len(self._cells) > 1 \
                    else self._cells[0]
            else:
                # floor(x / 640) exactly like patches.py:119-120
                cells = D.empty((len(xyz), 2), torch.int64)
                D.call("ts_cell_keys", D.ptr(xyz.contiguous()), len(xyz),
                       D.ptr(cells), D.stream())
            self._built = DeviceIndex(xyz.contiguous(), rgb, cells.contiguous())
        return self._built

    def query_square(self, center, radius):
        if self.count == 0:
            return (np.empty((0, 3)),
                    np.empty((0, 3), np.float32) if self.has_rgb else None)
        g = self.device_points().gather(np.asarray([center], np.float64),
                                        radius=float(radius), want_xyz=True)
        n = int(g["off"][-1].item())
        xyz = D.host(g["xyz"][:n]) if n else np.empty((0, 3))
        rgb = None
        if self.has_rgb:
            rgb = D.host(g["prgb"][:n]) if n else np.empty((0, 3), np.float32)
        return xyz, rgb

    def all_points(self):
        if not self._xyz:
            return np.empty((0, 3)), None
        idx = self.device_points()
        return D.host(idx.xyz), (D.host(idx.rgb) if self.has_rgb else None)


class DeviceIndex:
    """xyz/rgb/cells on the device + the ts_index_build cell ranges."""

    def __init__(self, xyz: torch.Tensor, rgb, cells: torch.Tensor,
                 cell_range=None):
        """cell_range = (ci0, cj0, ci1, cj1) inclusive, e.g. from the LAS
        header bboxes; without it the range is reduced on the device (one
        host sync).  Points outside the range are not indexed."""
        self.xyz, self.rgb, self.cells = xyz, rgb, cells
        n = len(xyz)
        if cell_range is not None:
            lo_h, hi_h = list(cell_range[:2]), list(cell_range[2:])
        else:
            lo = cells.min(dim=0).values
            hi = cells.max(dim=0).values
            lo_h, hi_h = lo.tolist(), hi.tolist()   # sizes the grid
        self.ci0, self.cj0 = lo_h
        self.nci, self.ncj = hi_h[0] - lo_h[0] + 1, hi_h[1] - lo_h[1] + 1
        self.order = D.empty((max(n, 1),), torch.int32)
        self.start = D.empty((self.nci * self.ncj,), torch.int32)
        self.end = D.empty((self.nci * self.ncj,), torch.int32)
        D.call("ts_index_build", D.ptr(cells), n, self.ci0, self.cj0,
               self.nci, self.ncj, D.ptr(self.order), D.ptr(self.start),
               D.ptr(self.end), D.stream())

    def gather(self, centers, radius=PAD_RADIUS, want_xyz=False):
        """gather_and_normalize for many patches -> CSR device arrays."""
        keys = centers if isinstance(centers, torch.Tensor) else \
            D.upload(np.ascontiguousarray(centers, np.float64))
        P = len(keys)
        counts = D.empty((P,), torch.int32)
        D.call("ts_gather_count", D.ptr(self.xyz), D.ptr(self.order),
               D.ptr(self.start), D.ptr(self.end), self.ci0, self.cj0,
               self.nci, self.ncj, D.ptr(keys), P, radius, D.ptr(counts),
               D.stream())
        off = torch.zeros(P + 1, dtype=torch.int64, device=keys.device)
        torch.cumsum(counts, 0, out=off[1:])
        total = int(off[-1].item())             # one sync: sizes outputs
        nn = max(total, 1)
        out = dict(off=off, keys=keys, n=P,
                   xy=D.empty((nn, 2), torch.float64),
                   h=D.empty((nn,), torch.float64),
                   prgb=D.empty((nn, 3), torch.float32)
                   if self.rgb is not None else None,
                   cz=D.empty((P,), torch.float64),
                   xyz=D.empty((nn, 3), torch.float64) if want_xyz else None,
                   status=torch.zeros(P, dtype=torch.int32,
                                      device=keys.device))
        D.call("ts_gather_fill", D.ptr(self.xyz), D.ptr(self.rgb),
               D.ptr(self.order), D.ptr(self.start), D.ptr(self.end),
               self.ci0, self.cj0, self.nci, self.ncj, D.ptr(keys), P, radius,
               D.ptr(off), D.ptr(out["xy"]), D.ptr(out["h"]),
               D.ptr(out["prgb"]), D.ptr(out["cz"]), D.ptr(out["xyz"]),
               D.ptr(out["status"]), D.stream())
        return out


def triangulate(g) -> dict:
    """GPU Delaunay of every gathered patch (ts_triangulate)."""
    P = g["n"]
    total = len(g["h"])
    tri = D.empty((2 * total + 8 * P + 8, 3), torch.int32)
    ntri = D.empty((P,), torch.int32)
    st = torch.zeros(P, dtype=torch.int32, device=tri.device)
    from ._lib import lib
    scratch = D.empty((int(lib().ts_triangulate_scratch(total, P)),), torch.uint8)
    D.call("ts_triangulate", D.ptr(g["xy"]), D.ptr(g["off"]), P, D.ptr(tri),
           D.ptr(ntri), D.ptr(st), D.ptr(scratch), D.stream())
    tri_off = 3 * (2 * g["off"][:-1] + 8 * torch.arange(
        P, device=tri.device, dtype=torch.int64))
    return dict(tri=tri, ntri=ntri, tri_off=tri_off.contiguous(), status=st)


def raster(g, t, recenter: bool, cnn_in=None, api_outputs=False):
    """ts_raster over a gathered + triangulated batch."""
    P = g["n"]
    dev = g["xy"].device
    o = dict(cz=D.empty((P,), torch.float64),
             status=torch.zeros(P, dtype=torch.int32, device=dev))
    if api_outputs:
        o["hm_nn"] = D.empty((P, RASTER_RES, RASTER_RES), torch.float32)
        o["hm_lin"] = D.empty((P, RASTER_RES, RASTER_RES), torch.float32)
        o["face"] = D.empty((P, RASTER_RES, RASTER_RES), torch.int32)
        if g["prgb"] is not None:
            o["rgb_nn"] = D.empty((P, RASTER_RES, RASTER_RES, 3), torch.float32)
            o["rgb_lin"] = D.empty((P, RASTER_RES, RASTER_RES, 3),
                                   torch.float32)
    D.call("ts_raster", D.ptr(g["xy"]), D.ptr(g["h"]), D.ptr(g["prgb"]),
           D.ptr(g["off"]), D.ptr(t["tri"]), D.ptr(t["tri_off"]),
           D.ptr(t["ntri"]), D.ptr(g["cz"]), P, 1 if recenter else 0,
           D.ptr(cnn_in), D.ptr(o.get("hm_nn")), D.ptr(o.get("hm_lin")),
           D.ptr(o.get("rgb_nn")), D.ptr(o.get("rgb_lin")),
           D.ptr(o.get("face")), D.ptr(o["cz"]), D.ptr(o["status"]),
           D.stream())
    return o


def _raw_patches(g, o, keys: list | None, recenter: bool) -> list:
    P = g["n"]
    hm_nn, hm_lin = D.host(o["hm_nn"]), D.host(o["hm_lin"])
    face = D.host(o["face"])
    rgb_nn = D.host(o["rgb_nn"]) if "rgb_nn" in o else None
    rgb_lin = D.host(o["rgb_lin"]) if "rgb_lin" in o else None
    cz = D.host(o["cz"])
    counts = np.diff(D.host(g["off"]))
    out = []
    for p in range(P):
        if keys is not None and recenter:
            key = keys[p].with_cz(float(cz[p]))
        else:
            key = PatchKey(0, 0, (0.0, 0.0), float(cz[p]))
        out.append(RawPatch(
            key=key, hm_nn=hm_nn[p], hm_lin=hm_lin[p],
            rgb_nn=None if rgb_nn is None else rgb_nn[p],
            rgb_lin=None if rgb_lin is None else rgb_lin[p],
            face_map=FaceMap(RASTER_RES, face[p]),
            chunk_point_count=int(counts[p])))
    return out


# ------------------------------------------------------------------- API

def gather_and_normalize(key: PatchKey,
                         index: ChunkPointIndex) -> PatchSpacePoints:
    if index.count == 0:
        raise EmptyPatch(f"no chunk points near patch ({key.i},{key.j})")
    g = index.device_points().gather(np.asarray([key.center], np.float64))
    n = int(g["off"][-1].item())
    if n == 0:
        raise EmptyPatch(f"no chunk points near patch ({key.i},{key.j})")
    return PatchSpacePoints(
        xy=D.host(g["xy"][:n]), h=D.host(g["h"][:n]),
        rgb=D.host(g["prgb"][:n]) if g["prgb"] is not None else None,
        c_z=float(g["cz"][0].item()))


def nearest_neighbor_query(pts: PatchSpacePoints, q) -> int:
    xy = np.asarray(pts.xy, np.float64).reshape(-1, 2)
    if len(xy) == 0:
        raise EmptySet("no points for nearest-neighbor query")
    d_xy = D.upload(xy)
    d_q = D.upload(np.asarray(q, np.float64).reshape(1, 2))
    out = D.empty((1,), torch.int64)
    D.call("ts_nearest", D.ptr(d_xy), len(xy), D.ptr(d_q), 1, D.ptr(out),
           D.stream())
    return int(out.item())


def _check_res(res):
    if res != RASTER_RES:
        raise ValueError(f"the CUDA rasteriser is built for res={RASTER_RES}")


def interpolate_patch(pts: PatchSpacePoints, res: int = RASTER_RES,
                      key: PatchKey | None = None) -> RawPatch:
    """Algorithm 1 on the GPU for caller-supplied patch-space points."""
    _check_res(res)
    n = len(pts.xy)
    if n < 1:
        raise EmptyPatch("interpolate_patch requires at least one point")
    dev = D.device()
    g = dict(n=1, xy=D.upload(np.asarray(pts.xy, np.float64).reshape(-1, 2)),
             h=D.upload(np.asarray(pts.h, np.float64)),
             prgb=D.upload(np.asarray(pts.rgb, np.float32))
             if pts.rgb is not None else None,
             off=torch.tensor([0, n], dtype=torch.int64, device=dev),
             cz=torch.tensor([float(pts.c_z)], dtype=torch.float64,
                             device=dev))
    t = triangulate(g)
    D.raise_item_status(D.host(t["status"]), "triangulate")
    o = raster(g, t, recenter=key is not None, api_outputs=True)
    D.raise_item_status(D.host(o["status"]), "raster")
    return _raw_patches(g, o, [key] if key is not None else None,
                        key is not None)[0]


def reconstruct_batch(keys: list[PatchKey], index: ChunkPointIndex,
                      res: int = RASTER_RES) -> list:
    """reconstruct_patch for many keys in one pass; None for empty ones."""
    _check_res(res)
    if index.count == 0:
        return [None] * len(keys)
    g = index.device_points().gather(
        np.asarray([k.center for k in keys], np.float64))
    t = triangulate(g)
    o = raster(g, t, recenter=True, api_outputs=True)
    raws = _raw_patches(g, o, keys, True)
    st = D.host(o["status"])
    tst = D.host(t["status"])
    out = []
    for p, raw in enumerate(raws):
        if st[p] == 1:
            out.append(None)
            continue
        if tst[p] not in (0, 1):
            raise_for_status(int(tst[p]), f"triangulate patch {p}")
        out.append(raw)
    return out


def reconstruct_patch(key: PatchKey, index: ChunkPointIndex,
                      res: int = RASTER_RES) -> RawPatch:
    raw = reconstruct_batch([key], index, res)[0]
    if raw is None:
        raise EmptyPatch(f"no chunk points near patch ({key.i},{key.j})")
    return raw
