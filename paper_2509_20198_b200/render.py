"""Point and heightmap rendering on the GPU (drop-in for
``terrascout.render``, pkg/src/terrascout/render.py:25-268; SURVEY §8(f)
rank 3).

The framebuffer lives in device memory (``Framebuffer.keys``, a torch
uint64-as-int64 tensor); ``cells`` copies it to the host on demand.  Every
fragment is a 64-bit key (depth in the high 32 bits, 0xRRGGBBAA in the low
32) merged with atomicMin, so the resolved image is independent of
submission order and worker count, as in the reference.  The kernels
(``csrc/render.cu``) follow the reference's numpy expressions operation by
operation; the camera is reduced to its basis on the host.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _device as D
from ._lib import lib
from .patches import OUTPUT_RES, PATCH_SIZE, TEXEL_SIZE

EMPTY_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)
LARGE_TRIANGLE_PIXELS = 1024


class _Camera(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("right", C.c_double * 3),
                ("up", C.c_double * 3), ("fwd", C.c_double * 3),
                ("f", C.c_double), ("f_over_aspect", C.c_double),
                ("near", C.c_double), ("far", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class _Lut(C.Structure):
    _fields_ = [("v", C.c_uint8 * 256)]


def _camera(cam) -> _Camera:
    right, up, fwd = cam.basis()
    w, h = cam.viewport
    f = 1.0 / np.tan(cam.fov_y / 2)
    c = _Camera()
    c.pos[:] = [float(v) for v in cam.position]
    c.right[:] = [float(v) for v in right]
    c.up[:] = [float(v) for v in up]
    c.fwd[:] = [float(v) for v in fwd]
    c.f = float(f)
    c.f_over_aspect = float(f / (w / h))   # geometry.py:89 xe * (f / aspect)
    c.near, c.far = float(cam.near), float(cam.far)
    c.width, c.height = int(w), int(h)
    return c


class Framebuffer:
    """width x height min-key cells on the device (EMPTY_KEY initially)."""

    def __init__(self, width: int, height: int):
        self.width, self.height = width, height
        self.keys = torch.full((height, width), -1, dtype=torch.int64, device=D.device())

    @property
    def cells(self) -> np.ndarray:
        return self.keys.cpu().numpy().view(np.uint64)

    def merge_buffer(self, other: "Framebuffer"):
        # unsigned minimum of two key planes, elementwise on the device
        a = self.keys ^ (-(2 ** 63))
        b = other.keys ^ (-(2 ** 63))
        self.keys = torch.minimum(a, b) ^ (-(2 ** 63))


def pack_color(rgb: np.ndarray) -> np.ndarray:
    """Linear [0,1] -> packed 0xRRGGBBAA (render.py:44-49)."""
    q = np.clip(np.asarray(rgb) * 255.0 + 0.5, 0, 255).astype(np.uint64)
    return (q[..., 0] << np.uint64(24)) | (q[..., 1] << np.uint64(16)) | \
           (q[..., 2] << np.uint64(8)) | np.uint64(0xFF)


_GREY = int(pack_color(np.array([0.85, 0.85, 0.85])))


def rasterize_points(points_xyz, rgb, cam, fb: Framebuffer,
                     chunk_size: int = 50_000, workers: int = 1):
    """One fragment per in-frustum point, min-key merged (render.py:55-98;
    chunk_size / workers accepted for the signature: the result does not
    depend on them)."""
    xyz = points_xyz if isinstance(points_xyz, torch.Tensor) else \
        D.upload(np.asarray(points_xyz, np.float64).reshape(-1, 3))
    n = len(xyz)
    if n == 0:
        return
    d_rgb = None
    if rgb is not None:
        d_rgb = rgb if isinstance(rgb, torch.Tensor) else \
            D.upload(np.asarray(rgb, np.float32).reshape(-1, 3))
    c = _camera(cam)
    D.call("ts_render_points", D.ptr(xyz), D.ptr(d_rgb), n, C.byref(c), _GREY,
           D.ptr(fb.keys), D.stream())


def patch_mesh(patch):
    """Vertex grid at texel centres, triangles, packed colour per triangle
    (render.py:101-120; host utility -- the GPU raster builds the same mesh
    on the fly)."""
    res = OUTPUT_RES
    x0 = patch.key.center[0] - PATCH_SIZE / 2
    y0 = patch.key.center[1] - PATCH_SIZE / 2
    gx, gy = np.meshgrid(x0 + (np.arange(res) + 0.5) * TEXEL_SIZE,
                         y0 + (np.arange(res) + 0.5) * TEXEL_SIZE)
    hm = patch.heights_rel.astype(np.float64) + patch.key.c_z
    verts = np.stack([gx.ravel(), gy.ravel(), hm.ravel()], axis=1)
    idx = np.arange(res * res).reshape(res, res)
    a, b = idx[:-1, :-1].ravel(), idx[:-1, 1:].ravel()
    c, d = idx[1:, :-1].ravel(), idx[1:, 1:].ravel()
    tris = np.concatenate([np.stack([a, b, c], 1), np.stack([b, d, c], 1)])
    if patch.rgb is not None:
        packed = pack_color(patch.rgb[:-1, :-1].reshape(-1, 3))
    else:
        shade = np.clip(0.35 + 0.5 * (hm[:-1, :-1] - hm.min()) /
                        max(np.ptp(hm), 1e-9), 0, 1)
        packed = pack_color(np.stack([shade] * 3, axis=-1).reshape(-1, 3))
    return verts, tris, np.concatenate([packed, packed])


def rasterize_heightmaps(patches, cam, fb: Framebuffer):
    """Triangle-grid rasterisation of refined patches (render.py:193-239)."""
    if not patches:
        return
    for p in patches:
        if not np.isfinite(p.heights_rel).all():
            raise ValueError("non-finite heightmap cannot be rasterized")
    P = len(patches)
    heights = D.upload(np.stack([p.heights_rel for p in patches]).astype(np.float32))
    has = np.array([p.rgb is not None for p in patches], np.uint8)
    rgb = D.upload(np.stack([p.rgb if p.rgb is not None else
                             np.zeros((OUTPUT_RES, OUTPUT_RES, 3), np.float32)
                             for p in patches]).astype(np.float32))
    centers = D.upload(np.array([p.key.center for p in patches], np.float64))
    cz = D.upload(np.array([p.key.c_z for p in patches], np.float64))
    scratch = D.empty((int(lib().ts_render_heightmaps_scratch(P)),), torch.uint8)
    c = _camera(cam)
    D.call("ts_render_heightmaps", D.ptr(heights), D.ptr(rgb), D.ptr(D.upload(has)),
           D.ptr(centers), D.ptr(cz), P, C.byref(c), D.ptr(fb.keys),
           D.ptr(scratch), D.stream())


_SRGB = None


def _srgb_lut() -> np.ndarray:
    """The reference's linear -> sRGB byte table (render.py:245-251)."""
    global _SRGB
    if _SRGB is None:
        lin = np.arange(256) / 255.0
        srgb = np.where(lin <= 0.0031308, lin * 12.92,
                        1.055 * lin ** (1 / 2.4) - 0.055)
        _SRGB = np.clip(np.round(srgb * 255), 0, 255).astype(np.uint8)
    return _SRGB


def resolve(fb: Framebuffer, background=(0.12, 0.12, 0.15)) -> np.ndarray:
    """Colour bytes through the sRGB table, background where empty:
    (H, W, 4) uint8 (render.py:254-268), computed on the device."""
    lut = _Lut()
    lut.v[:] = [int(v) for v in _srgb_lut()]
    bg = np.clip(np.round(np.asarray(background) * 255), 0, 255).astype(np.uint8)
    out = D.empty((fb.height, fb.width, 4), torch.uint8)
    D.call("ts_render_resolve", D.ptr(fb.keys), fb.width * fb.height, C.byref(lut),
           (C.c_uint8 * 3)(*[int(v) for v in bg]), D.ptr(out), D.stream())
    return out.cpu().numpy()


def save_png(path: str, image: np.ndarray):
    from PIL import Image
    Image.fromarray(image, mode="RGBA").save(path)
