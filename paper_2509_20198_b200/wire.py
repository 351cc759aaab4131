"""WireHeightmap records built on the device.

Mirrors ``wire_heightmap`` (``server.py:126-142``; layout
``docs/wire.md`` "WireHeightmap") for a whole batch of refined tiles: the
records are written by ``ts_wire_heightmaps`` straight from the refine /
bake output tensor, so serving a batch costs one device-to-host copy of the
finished bytes instead of a float download and a per-patch Python repack.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from ._lib import lib


def record_size(has_rgb: bool) -> int:
    """14 + 16,384 bytes, + 12,288 with the colour plane."""
    return int(lib().ts_wire_record_size(1 if has_rgb else 0))


def wire_heightmaps(out: torch.Tensor, cz, ij, stage, has_rgb: bool) -> torch.Tensor:
    """Device records of a batch, back to back (uint8, B * record_size).

    ``out``: B x 64 x 64 x 4 float32 CUDA tensor (heights_rel, r, g, b) as
    the refine / bake kernels leave it; ``cz`` (B,) float64 patch centre
    heights; ``ij`` (B, 2) int32 patch grid indices; ``stage`` (B,) uint8
    (0 empty .. 4 full-res-baked).  Host arrays are uploaded.
    """
    if out.dim() != 4 or tuple(out.shape[1:]) != (64, 64, 4) or out.dtype != torch.float32:
        raise ValueError("out must be B x 64 x 64 x 4 float32")
    out = out.contiguous()
    B = out.shape[0]
    dev = out.device

    def on_dev(a, dtype, shape):
        t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
        t = t.to(device=dev, dtype=dtype).contiguous()
        if tuple(t.shape) != shape:
            raise ValueError(f"expected shape {shape}, got {tuple(t.shape)}")
        return t

    cz_d = on_dev(cz, torch.float64, (B,))
    ij_d = on_dev(ij, torch.int32, (B, 2))
    st_d = on_dev(stage, torch.uint8, (B,))
    wire = torch.empty(B * record_size(has_rgb), dtype=torch.uint8, device=dev)
    D.call("ts_wire_heightmaps", D.ptr(out), D.ptr(cz_d), D.ptr(ij_d), D.ptr(st_d),
           1 if has_rgb else 0, B, D.ptr(wire), D.stream())
    return wire


def split_records(buf, has_rgb: bool) -> list[bytes]:
    """Per-patch ``bytes`` (what ``wire_heightmap`` returns) of a batch."""
    data = bytes(buf.cpu().numpy().tobytes() if isinstance(buf, torch.Tensor) else buf)
    n = record_size(has_rgb)
    if len(data) % n:
        raise ValueError("buffer is not a whole number of records")
    return [data[k:k + n] for k in range(0, len(data), n)]
