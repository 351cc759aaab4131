"""Device plumbing for the drop-in API: torch for memory/streams, the C ABI
(libts_b200.so) for every computation.

Nothing here computes a result on the host: host code only moves bytes,
sizes outputs and maps status codes onto the reference's exceptions.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import TABLE_POS_IN_IMAGE, TILE_DESC, lib
from .errors import raise_for_status


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2509_20198_b200 runs on a CUDA device only (no CPU "
            "fallback); no GPU is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p | None:
    return None if t is None else C.c_void_p(t.data_ptr())


def upload(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:  # e.g. np.frombuffer over bytes: copy, torch
        a = a.copy()           # cannot wrap a read-only buffer
    return torch.from_numpy(a).to(device())


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def call(name: str, *args) -> None:
    raise_for_status(getattr(lib(), name)(*args), name)


def host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def raise_item_status(status: np.ndarray, what: str) -> None:
    bad = np.nonzero(status)[0]
    if len(bad):
        raise_for_status(int(status[bad[0]]), f"{what} (item {bad[0]})")


# ------------------------------------------------------------ (1) records

def positions_host(records: np.ndarray, header) -> np.ndarray:
    """records.py:62-67 on the device."""
    n = len(records)
    if n == 0:
        return np.empty((0, 3), np.float64)
    raw = upload(np.frombuffer(records.tobytes(), np.uint8))
    out = empty((n, 3), torch.float64)
    scale = (C.c_double * 3)(*map(float, header.scale))
    offset = (C.c_double * 3)(*map(float, header.offset))
    call("ts_positions", ptr(raw), n, records.dtype.itemsize, scale, offset,
         ptr(out), stream())
    return host(out)


def colors_host(records: np.ndarray) -> np.ndarray:
    """records.py:70-86 on the device (per-batch 8/16-bit divisor)."""
    n = len(records)
    if n == 0:
        return np.empty((0, 3), np.float32)
    raw = upload(np.frombuffer(records.tobytes(), np.uint8))
    out = empty((n, 3), torch.float32)
    scratch = empty((1,), torch.int32)
    call("ts_colors", ptr(raw), n, records.dtype.itemsize,
         records.dtype.fields["red"][1], ptr(out), ptr(scratch), stream())
    return host(out)


class TileBatch:
    """File images of several tiles resident in one device byte buffer."""

    PAD = 64  # vector-window slack after the last image

    def __init__(self, images, descs: np.ndarray, file_sizes=None):
        """images: whole files, or (file_sizes given) sparse images whose
        descs carry image_base / table_pos (ts_tile_desc)."""
        sizes = np.array([len(b) for b in images], np.int64)
        offs = np.zeros(len(images), np.int64)
        # 16-byte aligned images keep the window loads aligned per tile
        aligned = (sizes + 15) // 16 * 16
        offs[1:] = np.cumsum(aligned)[:-1]
        total = int(aligned.sum()) + self.PAD
        host_buf = np.zeros(total, np.uint8)
        for o, b in zip(offs, images):
            host_buf[o:o + len(b)] = np.frombuffer(b, np.uint8)
        descs = descs.copy()
        descs["file_offset"] = offs
        descs["file_size"] = sizes if file_sizes is None else file_sizes
        self.descs = descs
        self.n = len(images)
        self.bytes = upload(host_buf)
        self.d_desc = upload(np.frombuffer(descs.tobytes(), np.uint8))

    @classmethod
    def from_device(cls, d_bytes: torch.Tensor, descs: np.ndarray):
        self = cls.__new__(cls)
        self.descs = descs
        self.n = len(descs)
        self.bytes = d_bytes
        self.d_desc = upload(np.frombuffer(descs.tobytes(), np.uint8))
        return self


def tile_desc(header, las_stride: int = 50_000) -> np.ndarray:
    """One ts_tile_desc row from a parsed LasHeader."""
    d = np.zeros(1, TILE_DESC)
    lz = header.laszip
    d["point_data_offset"] = header.point_data_offset
    d["point_count"] = header.point_count
    d["las_stride"] = las_stride
    d["chunk_size"] = lz.chunk_size if lz is not None else 0
    d["format"] = header.point_record_format
    d["record_length"] = header.point_record_length
    d["compressed"] = 1 if header.is_compressed else 0
    d["scale"] = header.scale
    d["offset"] = header.offset
    d["image_base"] = 0
    d["table_pos"] = TABLE_POS_IN_IMAGE
    return d


class ChunkTables:
    """Decoded chunk tables of a TileBatch (ts_chunk_counts + decode)."""

    def __init__(self, tb: TileBatch, sync_counts: bool = True):
        n = tb.n
        self.status = torch.zeros(n, dtype=torch.int32, device=device())
        counts = empty((n,), torch.int64)
        call("ts_chunk_counts", ptr(tb.bytes), ptr(tb.d_desc), n, ptr(counts),
             ptr(self.status), stream())
        base = torch.zeros(n + 1, dtype=torch.int64, device=device())
        torch.cumsum(counts, 0, out=base[1:])
        self.base = base
        self.total = int(base[-1].item())          # one sync: sizes outputs
        self.offsets = empty((max(self.total, 1),), torch.int64)
        self.points = empty((max(self.total, 1),), torch.int64)
        self.end = empty((n,), torch.int64)
        scratch = empty((int(lib().ts_chunk_decode_scratch(n)),), torch.uint8)
        call("ts_chunk_decode", ptr(tb.bytes), ptr(tb.d_desc), n, ptr(base),
             ptr(self.offsets), ptr(self.points), ptr(self.end),
             ptr(self.status), ptr(scratch), stream())


class FullRecords:
    """Every record of every chunk of a TileBatch of LAZ tiles, decoded on
    the GPU (ts_lazdec; load_tile_fullres).  ``records`` is the packed
    record_dtype(fmt) byte array, ``point_base`` the per-chunk record
    offsets (tile t's records: chunks tables.base[t] .. base[t + 1])."""

    def __init__(self, tb: TileBatch, tables: ChunkTables):
        fmts = set(int(f) for f in tb.descs["format"])
        if len(fmts) != 1:
            raise_for_status(8, "mixed point formats")
        self.format = fmts.pop()
        rs = int(lib().ts_record_size(self.format))
        if rs < 0:
            raise_for_status(8, f"point format {self.format}")
        n = tables.total
        pts = tables.points[:max(n, 1)]
        self.point_base = torch.zeros(n + 1, dtype=torch.int64, device=device())
        if n:
            torch.cumsum(pts[:n], 0, out=self.point_base[1:])
        self.n_points = int(self.point_base[-1].item())   # sizes the output
        self.records = empty((max(self.n_points, 1) * rs,), torch.uint8)
        self.status = torch.zeros(max(n, 1), dtype=torch.int32, device=device())
        scratch = empty((int(lib().ts_lazdec_scratch(n)),), torch.uint8)
        call("ts_lazdec", ptr(tb.bytes), ptr(tb.d_desc), tb.n, ptr(tables.base),
             ptr(tables.offsets), ptr(tables.points), ptr(tables.end),
             ptr(self.point_base), n, ptr(self.records), ptr(self.status),
             ptr(scratch), stream())
        self.tables = tables


class ChunkPoints:
    """Extracted chunk points of a TileBatch (ts_extract_chunk_points)."""

    def __init__(self, tb: TileBatch, tables: ChunkTables, records=True,
                 xyz=True, rgb=True, cells=True):
        fmts = set(int(f) for f in tb.descs["format"])
        n = tables.total
        self.n = n
        self.format = fmts.pop() if len(fmts) == 1 else None
        rs = int(lib().ts_record_size(self.format)) \
            if self.format is not None else -1
        if records and rs < 0:
            raise_for_status(8, "mixed or unsupported formats")
        nn = max(n, 1)
        self.records = empty((nn * max(rs, 1),), torch.uint8) \
            if records else None
        self.xyz = empty((nn, 3), torch.float64) if xyz else None
        has_rgb = any(int(f) in (2, 3) for f in tb.descs["format"])
        self.rgb = empty((nn, 3), torch.float32) if rgb and has_rgb else None
        self.cells = empty((nn, 2), torch.int64) if cells else None
        call("ts_extract_chunk_points", ptr(tb.bytes), ptr(tb.d_desc), tb.n,
             ptr(tables.base), ptr(tables.offsets), ptr(self.records),
             ptr(self.xyz), ptr(self.rgb), ptr(self.cells),
             ptr(tables.status), stream())
        self.status = tables.status
