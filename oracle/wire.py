"""Oracle: WireHeightmap records.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``wire_heightmap`` (``pkg/src/terrascout/server.py:126-142``) and
the "WireHeightmap" layout of ``pkg/docs/wire.md:25-45`` for one refined
patch given as arrays (the reference reads them from ``engine.refined`` and
``engine.patches``): a 14-byte little-endian head (i32 i, i32 j, f32 c_z,
u8 stage, u8 flags with bit 0 = colour plane), the float32 heights, then
the colour bytes clip(round(rgb * 255), 0, 255) -- numpy rounding (half to
even) of the float32 product -- when the patch has colour.
"""

from __future__ import annotations

import struct

import numpy as np


def wire_record(i: int, j: int, c_z: float, stage: int,
                heights_rel: np.ndarray, rgb: np.ndarray | None) -> bytes:
    flags = 0 if rgb is None else 1
    out = bytearray(struct.pack("<iifBB", int(i), int(j), float(c_z),
                                int(stage), flags))
    out += np.ascontiguousarray(heights_rel, dtype="<f4").tobytes()
    if rgb is not None:
        scaled = np.asarray(rgb, dtype=np.float32) * np.float32(255)
        out += np.clip(np.round(scaled), 0, 255).astype(np.uint8).tobytes()
    return bytes(out)
