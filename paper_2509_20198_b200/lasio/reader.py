"""Tile scanning (host metadata) and device chunk-point extraction.

Drop-in for ``pkg/src/terrascout/lasio/reader.py``:
  * ``scan_tile`` / ``scan_dataset`` read header bytes only (:89-129),
  * ``read_chunk_table`` decodes the LAZ chunk table on the GPU
    (``ts_chunk_decode``, replacing :132-209),
  * ``read_chunk_points`` runs the table decode and the vectorised
    first-record gather on the GPU (``ts_extract_chunk_points``, replacing
    :251-283) and returns the same structured record array, also filling
    ``tile.chunk_refs`` like the reference.
Full chunk decompression (``decode_chunk``/``load_tile_fullres``) is not
part of the heightmap hot path.
"""

from __future__ import annotations

import os
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from ..errors import UnsupportedFormat
from .header import COMPRESSOR_POINTWISE_CHUNKED, LasHeader, parse_header
from .records import record_dtype

DEFAULT_CHUNK_SIZE = 50_000
SECTOR = 4096
DECODABLE_FORMATS = frozenset({0, 1, 2, 3})


@dataclass
class ChunkRef:
    byte_offset: int
    point_count: int
    chunk_index: int
    byte_size: int = 0


@dataclass
class TileMeta:
    tile_id: int
    path: str
    header: LasHeader
    chunk_refs: list[ChunkRef] | None = None
    chunk_point_range: tuple[int, int] | None = None
    file_size: int = 0

    @property
    def is_compressed(self) -> bool:
        return self.header.is_compressed

    @property
    def chunk_size(self) -> int:
        lz = self.header.laszip
        if lz is not None and not lz.variable_chunks:
            return lz.chunk_size
        return DEFAULT_CHUNK_SIZE

    def num_chunks(self) -> int:
        if self.chunk_refs is not None:
            return len(self.chunk_refs)
        return -(-self.header.point_count // self.chunk_size)


@dataclass
class ScanResult:
    tiles: list[TileMeta]
    errors: list[tuple[str, Exception]] = field(default_factory=list)

    def dataset_bbox(self):
        if not self.tiles:
            return None
        lo = np.min([t.header.bbox_min for t in self.tiles], axis=0)
        hi = np.max([t.header.bbox_max for t in self.tiles], axis=0)
        return lo, hi


def _header_bytes(path: str) -> tuple[bytes, int]:
    with open(path, "rb") as fp:
        head = fp.read(375)
        size = os.fstat(fp.fileno()).st_size
        if len(head) >= 227:
            pdo, = struct.unpack_from("<I", head, 96)
            if pdo > len(head):
                head += fp.read(pdo - len(head))
    return head, size


def scan_tile(path: str, tile_id: int) -> TileMeta:
    raw, size = _header_bytes(path)
    return TileMeta(tile_id=tile_id, path=path, header=parse_header(raw),
                    file_size=size)


def scan_dataset(paths: list[str], max_workers: int = 8) -> ScanResult:
    """Header-only scan; per-file errors collected, input order kept."""
    slots: list = [None] * len(paths)
    errors: list = []

    def one(i):
        try:
            slots[i] = scan_tile(paths[i], i)
        except Exception as exc:  # noqa: BLE001 - per-file isolation
            errors.append((paths[i], exc))

    if paths:
        with ThreadPoolExecutor(max_workers=max_workers) as pool:
            list(pool.map(one, range(len(paths))))
    return ScanResult([t for t in slots if t is not None], errors)


def _check_laz(tile: TileMeta):
    lz = tile.header.laszip
    if lz is None:
        raise UnsupportedFormat("chunk tables exist only in LAZ files")
    if lz.compressor != COMPRESSOR_POINTWISE_CHUNKED:
        raise UnsupportedFormat(f"compressor {lz.compressor} not supported")


def _device_tables(tile: TileMeta, las_stride: int):
    from .. import _device as D
    with open(tile.path, "rb") as fp:
        image = fp.read()
    tb = D.TileBatch([image], D.tile_desc(tile.header, las_stride))
    tables = D.ChunkTables(tb)
    return D, tb, tables


def _refs_from(tables, tile: TileMeta) -> list[ChunkRef]:
    offs = tables.offsets[:tables.total].cpu().numpy()
    pts = tables.points[:tables.total].cpu().numpy()
    end = int(tables.end[0].item())
    refs = []
    for i in range(tables.total):
        nxt = int(offs[i + 1]) if i + 1 < tables.total else end
        size = int(pts[i]) * tile.header.point_record_length \
            if not tile.is_compressed else nxt - int(offs[i])
        refs.append(ChunkRef(int(offs[i]), int(pts[i]), i, size))
    return refs


def read_chunk_table(tile: TileMeta) -> list[ChunkRef]:
    """LAZ chunk table -> ChunkRefs, decoded on the GPU."""
    _check_laz(tile)
    D, _tb, tables = _device_tables(tile, DEFAULT_CHUNK_SIZE)
    D.raise_item_status(tables.status.cpu().numpy(), "read_chunk_table")
    tile.chunk_refs = _refs_from(tables, tile)
    return tile.chunk_refs


def ensure_chunk_refs(tile: TileMeta,
                      las_stride: int = DEFAULT_CHUNK_SIZE) -> list[ChunkRef]:
    if tile.chunk_refs is None:
        if tile.is_compressed:
            read_chunk_table(tile)
        else:
            D, _tb, tables = _device_tables(tile, las_stride)
            tile.chunk_refs = _refs_from(tables, tile)
    return tile.chunk_refs


def read_chunk_points(tile: TileMeta,
                      las_stride: int = DEFAULT_CHUNK_SIZE) -> np.ndarray:
    """Raw first record of every chunk (structured array), on the GPU."""
    fmt = tile.header.point_record_format
    if fmt not in DECODABLE_FORMATS:
        raise UnsupportedFormat(f"point format {fmt} not supported")
    if tile.is_compressed:
        _check_laz(tile)
    D, tb, tables = _device_tables(tile, las_stride)
    D.raise_item_status(tables.status.cpu().numpy(), "chunk table")
    cp = D.ChunkPoints(tb, tables, records=True, xyz=False, rgb=False,
                       cells=False)
    D.raise_item_status(cp.status.cpu().numpy(), "read_chunk_points")
    if tile.chunk_refs is None:
        tile.chunk_refs = _refs_from(tables, tile)
    dt = record_dtype(fmt)
    raw = cp.records[:tables.total * dt.itemsize].cpu().numpy()
    return raw.view(dt).copy()
