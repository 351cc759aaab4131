"""LAS and stub-body LAZ file images for synthetic corpora (supporting).

The heightmap path never writes point clouds; these writers exist so the
benchmark and the parity tests can build inputs on the GPU box.  The
layout follows the LAS 1.2 public header and the LASzip chunked format the
reference writer emits (``pkg/src/terrascout/lasio/writer.py:26-194``):
header, LASzip VLR, 8-byte chunk-table pointer, chunks, chunk table.
Chunk bodies here are filler: only the raw first record of every chunk is
meaningful, which is all the chunk-point path reads.
"""

from __future__ import annotations

import struct

import numpy as np

from ..errors import UnsupportedFormat
from ._acenc import encode_chunk_table
from .header import (COMPRESSOR_POINTWISE_CHUNKED, ITEM_GPSTIME11,
                     ITEM_POINT10, ITEM_RGB12, LASZIP_RECORD_ID,
                     LASZIP_USER_ID, MIN_RECORD_LENGTH)
from .records import record_dtype

_HDR = struct.Struct("<4sHHIHH8sBB32s32sHHHIIBHI5I12d")


def _header(fmt_byte, rec_len, count, scale, offset, bmin, bmax, vlrs):
    pdo = 227 + sum(len(v) for v in vlrs)
    ident = b"paper_2509_20198_b200".ljust(32, b"\0")
    head = _HDR.pack(b"LASF", 0, 0, 0, 0, 0, bytes(8), 1, 2, ident, ident,
                     1, 2026, 227, pdo, len(vlrs), fmt_byte, rec_len,
                     count if count < 2 ** 32 else 0, 0, 0, 0, 0, 0,
                     *scale, *offset, bmax[0], bmin[0], bmax[1], bmin[1],
                     bmax[2], bmin[2])
    return head + b"".join(vlrs)


def _vlr(user_id: bytes, record_id: int, data: bytes) -> bytes:
    return struct.pack("<H16sHH32s", 0, user_id, record_id, len(data),
                       bytes(32)) + data


def _bbox(records, scale, offset):
    if len(records) == 0:
        return (0.0,) * 3, (0.0,) * 3
    lo = tuple(float(records[a].min()) * s + o
               for a, s, o in zip("xyz", scale, offset))
    hi = tuple(float(records[a].max()) * s + o
               for a, s, o in zip("xyz", scale, offset))
    return lo, hi


def las_image(records: np.ndarray, point_format: int,
              scale=(0.01, 0.01, 0.01), offset=(0.0, 0.0, 0.0)) -> bytes:
    """Uncompressed LAS 1.2 file image."""
    dt = record_dtype(point_format, records.dtype.itemsize)
    if records.dtype != dt:
        raise UnsupportedFormat("records dtype does not match point format")
    lo, hi = _bbox(records, scale, offset)
    return _header(point_format, dt.itemsize, len(records), scale, offset,
                   lo, hi, []) + records.tobytes()


def write_las(path, records, point_format, scale=(0.01, 0.01, 0.01),
              offset=(0.0, 0.0, 0.0)):
    with open(path, "wb") as fp:
        fp.write(las_image(records, point_format, scale, offset))


def laz_image(first_records: np.ndarray, point_format: int,
              points_per_chunk: int, body_sizes, scale=(0.01, 0.01, 0.01),
              offset=(0.0, 0.0, 0.0), bbox=None,
              chunk_counts=None) -> bytes:
    """Chunked-LAZ image with raw first records and filler chunk bodies.

    ``chunk_counts`` switches to variable chunking (counts in the table).
    """
    if point_format not in (0, 1, 2, 3):
        raise UnsupportedFormat(f"LAZ writer: format {point_format}")
    if first_records.dtype != record_dtype(point_format):
        raise UnsupportedFormat("records dtype does not match point format")
    n_chunks = len(first_records)
    items = [(ITEM_POINT10, 20, 2)]
    if point_format in (1, 3):
        items.append((ITEM_GPSTIME11, 8, 2))
    if point_format in (2, 3):
        items.append((ITEM_RGB12, 6, 2))
    variable = chunk_counts is not None
    if variable:
        counts = [int(c) for c in chunk_counts]
    else:
        counts = [points_per_chunk] * n_chunks
    total = int(sum(counts))
    lz = struct.pack("<HHBBHIIqqH", COMPRESSOR_POINTWISE_CHUNKED, 0, 2, 2, 0,
                     0, 0xFFFFFFFF if variable else points_per_chunk, -1, -1,
                     len(items))
    lz += b"".join(struct.pack("<HHH", *it) for it in items)
    if bbox is None:
        bbox = _bbox(first_records, scale, offset)
    head = _header(point_format | 0x80, MIN_RECORD_LENGTH[point_format],
                   total, scale, offset, bbox[0], bbox[1],
                   [_vlr(LASZIP_USER_ID, LASZIP_RECORD_ID, lz)])
    raw = first_records.tobytes()
    rl = first_records.dtype.itemsize
    parts = [head, b""]
    sizes = []
    filler = np.random.default_rng(len(raw)).integers(
        0, 256, int(np.max(body_sizes)) if n_chunks else 0,
        dtype=np.uint8).tobytes()
    for i in range(n_chunks):
        body = filler[:int(body_sizes[i])]
        parts.append(raw[i * rl:(i + 1) * rl] + body)
        sizes.append(rl + len(body))
    table_pos = len(head) + 8 + sum(sizes)
    parts[1] = struct.pack("<q", table_pos)
    table = struct.pack("<II", 0, n_chunks)
    if n_chunks:
        table += encode_chunk_table(sizes, counts if variable else None)
    parts.append(table)
    return b"".join(parts)
