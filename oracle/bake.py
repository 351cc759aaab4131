"""Oracle: full-resolution texel update.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``bake_fullres`` (``pkg/src/terrascout/engine.py:416-456``):
per key, texel index ``floor((x - (cx - 320)) / 10)`` in IEEE float64,
float64 ``bincount`` sums in point order, covered texels overwritten with
the mean, uncovered texels untouched, result re-expressed against
``key.c_z``.
"""

from __future__ import annotations

import numpy as np


def texel_ids(xyz, center, res=64):
    x0 = center[0] - 320.0
    y0 = center[1] - 320.0
    ix = np.floor((xyz[:, 0] - x0) / 10.0).astype(np.int64)
    iy = np.floor((xyz[:, 1] - y0) / 10.0).astype(np.int64)
    ok = (ix >= 0) & (ix < res) & (iy >= 0) & (iy < res)
    return ok, iy * res + ix


def bake_one(xyz, rgb, heights_rel, base_cz, prior_rgb, center, key_cz):
    """Returns (heights_rel float32 (64,64), rgb float32 (64,64,3)|None)."""
    res = 64
    ok, flat = texel_ids(xyz, center, res)
    heights = heights_rel.astype(np.float64) + base_cz
    out_rgb = None if prior_rgb is None else prior_rgb.copy()
    if ok.any():
        f = flat[ok]
        cnt = np.bincount(f, minlength=res * res)
        zs = np.bincount(f, weights=xyz[ok, 2], minlength=res * res)
        cov = cnt > 0
        heights.ravel()[cov] = zs[cov] / cnt[cov]
        if out_rgb is not None and rgb is not None:
            for ch in range(3):
                cs = np.bincount(f, weights=rgb[ok, ch], minlength=res * res)
                plane = out_rgb[:, :, ch].ravel()
                plane[cov] = (cs[cov] / cnt[cov]).astype(np.float32)
                out_rgb[:, :, ch] = plane.reshape(res, res)
    return (heights - key_cz).astype(np.float32), out_rgb
