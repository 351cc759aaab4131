"""Oracle: point and heightmap rasterisation with 64-bit min keys.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``pkg/src/terrascout/render.py:25-268`` (Framebuffer min-key merge,
``pack_color``, ``rasterize_points``, ``patch_mesh``, ``_TriangleRaster``,
``rasterize_heightmaps``, ``resolve``) and the camera math it uses from
``geometry.py:13-102`` (``CameraState.basis``, ``eye_coords``, ``project``,
``depth_key``), with the same numpy expressions, so results are
bit-identical to the reference (pinned by ``tests/golden/render.npz``).
"""

from __future__ import annotations

import numpy as np

EMPTY_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)
LARGE = 1024
WORLD_UP = np.array([0.0, 0.0, 1.0])


class Camera:
    """CameraState fields from a flat vector (position, direction, fov_y,
    w, h, near, far), the layout the golden file stores."""

    def __init__(self, v):
        v = np.asarray(v, np.float64)
        self.position = v[0:3]
        d = v[3:6]
        self.direction = d / np.linalg.norm(d)
        self.fov_y = float(v[6])
        self.viewport = (int(v[7]), int(v[8]))
        self.near, self.far = float(v[9]), float(v[10])

    def basis(self):
        fwd = self.direction
        up_hint = WORLD_UP if abs(fwd @ WORLD_UP) < 0.999 else np.array([0.0, 1.0, 0.0])
        right = np.cross(fwd, up_hint)
        right /= np.linalg.norm(right)
        up = np.cross(right, fwd)
        return right, up, fwd


def project(cam, points):
    right, up, fwd = cam.basis()
    d = np.atleast_2d(points) - cam.position
    xe, ye, ze = d @ right, d @ up, d @ fwd
    w, h = cam.viewport
    f = 1.0 / np.tan(cam.fov_y / 2)
    aspect = w / h
    with np.errstate(divide="ignore", invalid="ignore"):
        ndc_x = xe * (f / aspect) / ze
        ndc_y = ye * f / ze
    return (ndc_x * 0.5 + 0.5) * w, (0.5 - ndc_y * 0.5) * h, ze


def depth_key(cam, depth):
    inv_n = 1.0 / cam.near
    inv_f = 1.0 / cam.far
    z = np.clip(depth, cam.near, cam.far)
    norm = (inv_n - 1.0 / z) / (inv_n - inv_f)
    return (norm * np.float64(0xFFFFFFFE)).astype(np.uint64)


def pack_color(rgb):
    q = np.clip(np.asarray(rgb) * 255.0 + 0.5, 0, 255).astype(np.uint64)
    return (q[..., 0] << np.uint64(24)) | (q[..., 1] << np.uint64(16)) | \
        (q[..., 2] << np.uint64(8)) | np.uint64(0xFF)


def new_fb(w, h):
    return np.full((h, w), EMPTY_KEY, np.uint64)


def rasterize_points(pts, rgb, cam, fb):
    n = len(pts)
    if n == 0:
        return
    packed = np.full(n, pack_color(np.array([0.85, 0.85, 0.85])), np.uint64) \
        if rgb is None else pack_color(rgb)
    px, py, ze = project(cam, pts)
    m = (ze > cam.near) & (ze <= cam.far)
    px, py, ze = px[m], py[m], ze[m]
    xi = np.floor(px).astype(np.int64)
    yi = np.floor(py).astype(np.int64)
    h, w = fb.shape
    inb = (xi >= 0) & (xi < w) & (yi >= 0) & (yi < h)
    keys = (depth_key(cam, ze[inb]) << np.uint64(32)) | packed[m][inb]
    np.minimum.at(fb, (yi[inb], xi[inb]), keys)


def patch_mesh(heights_rel, rgb, center, c_z):
    res = 64
    x0, y0 = center[0] - 320.0, center[1] - 320.0
    gx, gy = np.meshgrid(x0 + (np.arange(res) + 0.5) * 10.0,
                         y0 + (np.arange(res) + 0.5) * 10.0)
    hm = heights_rel.astype(np.float64) + c_z
    verts = np.stack([gx.ravel(), gy.ravel(), hm.ravel()], axis=1)
    idx = np.arange(res * res).reshape(res, res)
    a, b = idx[:-1, :-1].ravel(), idx[:-1, 1:].ravel()
    c, d = idx[1:, :-1].ravel(), idx[1:, 1:].ravel()
    tris = np.concatenate([np.stack([a, b, c], 1), np.stack([b, d, c], 1)])
    if rgb is not None:
        packed = pack_color(rgb[:-1, :-1].reshape(-1, 3))
    else:
        shade = np.clip(0.35 + 0.5 * (hm[:-1, :-1] - hm.min()) / max(np.ptp(hm), 1e-9), 0, 1)
        packed = pack_color(np.stack([shade] * 3, axis=-1).reshape(-1, 3))
    return verts, tris, np.concatenate([packed, packed])


def rasterize_heightmaps(patches, cam, fb):
    """patches: (heights_rel, rgb|None, center, c_z); the reference's
    small/large paths share the per-pixel arithmetic, so one path is
    restated (render.py:128-167)."""
    h_fb, w_fb = fb.shape
    for heights_rel, rgb, center, c_z in patches:
        verts, tris, colors = patch_mesh(heights_rel, rgb, center, c_z)
        px, py, ze = project(cam, verts)
        front = ze > cam.near
        inv_z = np.where(front, 1.0 / np.maximum(ze, 1e-12), -1.0)
        tri_front = front[tris].all(axis=1)
        txs, tys = px[tris], py[tris]
        x_lo = np.maximum(np.floor(txs.min(axis=1)), 0).astype(np.int64)
        x_hi = np.minimum(np.ceil(txs.max(axis=1)) - 1, w_fb - 1).astype(np.int64)
        y_lo = np.maximum(np.floor(tys.min(axis=1)), 0).astype(np.int64)
        y_hi = np.minimum(np.ceil(tys.max(axis=1)) - 1, h_fb - 1).astype(np.int64)
        valid = tri_front & (x_hi >= x_lo) & (y_hi >= y_lo)
        for t in np.nonzero(valid)[0]:
            vx, vy, vz = txs[t], tys[t], inv_z[tris[t]]
            d = (vy[1] - vy[2]) * (vx[0] - vx[2]) + (vx[2] - vx[1]) * (vy[0] - vy[2])
            if d == 0:
                continue
            xs = np.arange(x_lo[t], x_hi[t] + 1, dtype=np.float64) + 0.5
            for yi in range(y_lo[t], y_hi[t] + 1):
                pyc = yi + 0.5
                w0 = ((vy[1] - vy[2]) * (xs - vx[2]) + (vx[2] - vx[1]) * (pyc - vy[2])) / d
                w1 = ((vy[2] - vy[0]) * (xs - vx[2]) + (vx[0] - vx[2]) * (pyc - vy[2])) / d
                w2 = 1.0 - w0 - w1
                inside = (w0 >= 0) & (w1 >= 0) & (w2 >= 0)
                if not inside.any():
                    continue
                iz = w0 * vz[0] + w1 * vz[1] + w2 * vz[2]
                inside &= iz > 0
                (ix,) = np.nonzero(inside)
                if len(ix) == 0:
                    continue
                keys = (depth_key(cam, 1.0 / iz[ix]) << np.uint64(32)) | np.uint64(colors[t])
                np.minimum.at(fb, (np.full(len(ix), yi), ix + x_lo[t]), keys)


def srgb_lut():
    lin = np.arange(256) / 255.0
    srgb = np.where(lin <= 0.0031308, lin * 12.92, 1.055 * lin ** (1 / 2.4) - 0.055)
    return np.clip(np.round(srgb * 255), 0, 255).astype(np.uint8)


def resolve(fb, background=(0.12, 0.12, 0.15)):
    color = (fb & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    lut = srgb_lut()
    r = ((color >> 24) & 0xFF).astype(np.uint8)
    g = ((color >> 16) & 0xFF).astype(np.uint8)
    b = ((color >> 8) & 0xFF).astype(np.uint8)
    img = np.stack([lut[r], lut[g], lut[b], np.full_like(r, 255)], axis=-1)
    bg = np.clip(np.round(np.asarray(background) * 255), 0, 255).astype(np.uint8)
    img[fb == EMPTY_KEY] = np.array([lut[bg[0]], lut[bg[1]], lut[bg[2]], 255], np.uint8)
    return img
