"""Tile scanning (host metadata) and device chunk-point extraction.

Drop-in for ``pkg/src/terrascout/lasio/reader.py``:
  * ``scan_tile`` / ``scan_dataset`` read header bytes only (:89-129),
  * ``read_chunk_table`` decodes the LAZ chunk table on the GPU
    (``ts_chunk_decode``, replacing :132-209) from the table bytes only
    (the reference's reads: pointer, table; sparse device images),
  * ``read_chunk_points`` reads each chunk's first record the way the
    reference does (one 4 KiB-aligned pread per chunk, :270-278), uploads
    a 64-byte window per record and gathers + decodes them on the GPU
    (``ts_extract_chunk_points``, replacing :251-283); it returns the same
    structured record array, fills ``tile.chunk_refs`` like the reference
    and reads from them when they are already set,
  * ``StagedChunkPoints`` is the batched form over many files,
  * ``decode_chunk`` / ``load_tile_fullres`` (:286-364) decode whole chunks
    on the GPU (``ts_lazdec``), reading the chunk
    bytes only.
"""

from __future__ import annotations

import os
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from ..errors import CorruptChunkTable, OutOfBoundsRead, UnsupportedFormat
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


def _table_image(tile: TileMeta, fd: int, size: int) -> tuple[bytes, int]:
    """The chunk table bytes [table_pos, EOF) by the reference's reads
    (reader.py:146-160): the 8-byte pointer at point_data_offset, the last
    8 bytes when it is -1, then the table.  Returns (image, table_pos)."""
    pdo = tile.header.point_data_offset
    raw = os.pread(fd, 8, pdo)
    if len(raw) < 8:
        raise CorruptChunkTable("missing chunk table pointer")
    table_pos = struct.unpack("<q", raw)[0]
    if table_pos == -1:
        table_pos = struct.unpack("<q", os.pread(fd, 8, size - 8))[0]
    if not pdo + 8 <= table_pos <= size - 8:
        raise CorruptChunkTable(f"chunk table pointer {table_pos} outside file")
    return os.pread(fd, size - table_pos, table_pos), table_pos


def _device_tables_files(tiles, las_stride: int, fds, sizes):
    """Chunk tables of several files decoded on the GPU from their table
    bytes only (sparse images: ts_tile_desc image_base / table_pos)."""
    from .. import _device as D
    images, descs = [], []
    for tile, fd, size in zip(tiles, fds, sizes):
        d = D.tile_desc(tile.header, las_stride)
        img = b""
        if tile.is_compressed:
            _check_laz(tile)
            img, pos = _table_image(tile, fd, size)
            d["image_base"] = pos
            d["table_pos"] = pos
        images.append(img)
        descs.append(d)
    tb = D.TileBatch(images, np.concatenate(descs),
                     file_sizes=np.asarray(sizes, np.int64))
    return D, D.ChunkTables(tb)


def _device_tables(tile: TileMeta, las_stride: int):
    fd = os.open(tile.path, os.O_RDONLY)
    try:
        return _device_tables_files([tile], las_stride, [fd],
                                    [os.fstat(fd).st_size])
    finally:
        os.close(fd)


def stage_first_records(tiles, offsets, fds, sizes, workers: int = 8):
    """Host staging of every chunk's first record, read as the reference
    reads it (one 4 KiB-aligned pread per chunk, reader.py:270-278).  Only
    the 64-byte window around each record (the device gather's vector
    window) is kept, so the upload is 64 B per chunk, not the file.

    offsets: per tile, the absolute chunk byte offsets.  Returns (staging
    bytes, per-chunk staged offsets).  Raises OutOfBoundsRead like the
    reference."""
    per = [len(o) for o in offsets]
    start = np.concatenate([[0], np.cumsum(per)]).astype(np.int64)
    staging = np.zeros(64 * int(start[-1]) + 64, np.uint8)
    staged = np.zeros(int(start[-1]), np.int64)

    def one(i):
        rl = tiles[i].header.point_record_length
        for j, off in enumerate(offsets[i]):
            off = int(off)
            if off + rl > sizes[i]:
                raise OutOfBoundsRead(f"chunk {j} offset beyond file end")
            aligned = (off // SECTOR) * SECTOR
            span = off - aligned + rl
            buf = os.pread(fds[i], ((span + SECTOR - 1) // SECTOR) * SECTOR, aligned)
            w0 = off & ~15                       # 16-byte aligned window
            piece = np.frombuffer(buf, np.uint8)[w0 - aligned:w0 - aligned + 64]
            k = int(start[i]) + j
            staging[64 * k:64 * k + len(piece)] = piece
            staged[k] = 64 * k + (off - w0)

    if len(tiles) > 1 and workers > 1:
        with ThreadPoolExecutor(max_workers=min(workers, len(tiles))) as pool:
            list(pool.map(one, range(len(tiles))))
    else:
        for i in range(len(tiles)):
            one(i)
    return staging, staged, start


class StagedChunkPoints:
    """Chunk tables + staged first records of files (two device phases):
    tables decoded from the table bytes, records gathered from 64-byte
    windows read by the reference's 4 KiB-aligned preads.  ``tb``/``base``/
    ``offsets`` feed ts_extract_chunk_points (D.ChunkPoints)."""

    def __init__(self, tiles, las_stride: int = DEFAULT_CHUNK_SIZE,
                 workers: int = 8):
        from .. import _device as D
        fds = [os.open(t.path, os.O_RDONLY) for t in tiles]
        try:
            sizes = [os.fstat(fd).st_size for fd in fds]
            cached = [t.chunk_refs for t in tiles]
            todo = [i for i, r in enumerate(cached) if r is None]
            offsets = [None] * len(tiles)
            if todo:
                _D, tables = _device_tables_files(
                    [tiles[i] for i in todo], las_stride,
                    [fds[i] for i in todo], [sizes[i] for i in todo])
                D.raise_item_status(tables.status.cpu().numpy(), "chunk table")
                offs = tables.offsets[:tables.total].cpu().numpy()
                base = tables.base.cpu().numpy()
                for k, i in enumerate(todo):
                    offsets[i] = offs[base[k]:base[k + 1]]
                    tiles[i].chunk_refs = _refs_from_host(
                        tables, k, offs[base[k]:base[k + 1]], tiles[i])
            for i, r in enumerate(cached):
                if r is not None:  # the reference reads from cached refs
                    offsets[i] = np.array([c.byte_offset for c in r], np.int64)
            staging, staged, start = stage_first_records(tiles, offsets, fds,
                                                         sizes, workers)
        finally:
            for fd in fds:
                os.close(fd)
        descs = np.concatenate([D.tile_desc(t.header, las_stride) for t in tiles])
        self.tb = D.TileBatch.from_device(D.upload(staging), _staged_descs(descs, len(staging)))
        self.base = D.upload(start)
        self.offsets = D.upload(staged) if len(staged) else D.empty((1,), torch_int64())
        self.total = int(start[-1])
        self.status = D.upload(np.zeros(len(tiles), np.int32))
        self.n_tiles = len(tiles)
        self.staged_bytes = len(staging)


def torch_int64():
    import torch
    return torch.int64


def _staged_descs(descs, n_bytes):
    d = descs.copy()
    d["file_offset"] = 0
    d["file_size"] = n_bytes
    d["image_base"] = 0
    return d


def _refs_from_host(tables, k, offs, tile) -> list[ChunkRef]:
    pts = tables.points[int(tables.base[k]):int(tables.base[k + 1])].cpu().numpy()
    end = int(tables.end[k].item())
    refs = []
    for i in range(len(offs)):
        nxt = int(offs[i + 1]) if i + 1 < len(offs) else end
        size = int(pts[i]) * tile.header.point_record_length \
            if not tile.is_compressed else nxt - int(offs[i])
        refs.append(ChunkRef(int(offs[i]), int(pts[i]), i, size))
    return refs


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
    D, tables = _device_tables(tile, DEFAULT_CHUNK_SIZE)
    D.raise_item_status(tables.status.cpu().numpy(), "read_chunk_table")
    tile.chunk_refs = _refs_from(tables, tile)
    return tile.chunk_refs


def ensure_chunk_refs(tile: TileMeta,
                      las_stride: int = DEFAULT_CHUNK_SIZE) -> list[ChunkRef]:
    if tile.chunk_refs is None:
        if tile.is_compressed:
            read_chunk_table(tile)
        else:
            D, tables = _device_tables(tile, las_stride)
            tile.chunk_refs = _refs_from(tables, tile)
    return tile.chunk_refs


def read_chunk_points(tile: TileMeta,
                      las_stride: int = DEFAULT_CHUNK_SIZE) -> np.ndarray:
    """Raw first record of every chunk (structured array): the chunk table
    is decoded on the GPU from the table bytes, each record is read by the
    reference's 4 KiB-aligned pread and gathered + decoded on the GPU
    (ts_extract_chunk_points).  Uses tile.chunk_refs when already set."""
    fmt = tile.header.point_record_format
    if fmt not in DECODABLE_FORMATS:
        raise UnsupportedFormat(f"point format {fmt} not supported")
    if tile.is_compressed:
        _check_laz(tile)
    from .. import _device as D
    st = StagedChunkPoints([tile], las_stride, workers=1)
    cp = D.ChunkPoints(st.tb, st, records=True, xyz=False, rgb=False, cells=False)
    D.raise_item_status(cp.status.cpu().numpy(), "read_chunk_points")
    dt = record_dtype(fmt)
    raw = cp.records[:st.total * dt.itemsize].cpu().numpy()
    return raw.view(dt).copy()


# ----------------------------------------------------------- full decode

_ITEMS = {0: [6], 1: [6, 7], 2: [6, 8], 3: [6, 7, 8]}  # POINT10, GPSTIME11, RGB12


def _check_items(tile: TileMeta):
    """decode_chunk's item-layout checks (reader.py:294-314)."""
    fmt = tile.header.point_record_format
    if fmt not in DECODABLE_FORMATS:
        raise UnsupportedFormat(f"compressed point format {fmt} not supported")
    lz = tile.header.laszip
    got = [t for t, _s, _v in lz.items]
    if got != _ITEMS[fmt]:
        raise UnsupportedFormat(f"unexpected LASzip item layout {lz.items}")
    for _t, _s, version in lz.items:
        if version != 2:
            raise UnsupportedFormat(
                f"LASzip item version {version}, only v2 is decodable")


class _Tables:
    """Chunk-table arrays of already known chunks (ChunkTables layout)."""

    def __init__(self, D, offsets, counts, ends_per_tile, base):
        import torch
        self.base = D.upload(np.asarray(base, np.int64))
        self.offsets = D.upload(np.asarray(offsets, np.int64))
        self.points = D.upload(np.asarray(counts, np.int64))
        self.end = D.upload(np.asarray(ends_per_tile, np.int64))
        self.total = len(offsets)
        self.status = torch.zeros(len(base) - 1, dtype=torch.int32, device=self.base.device)


def decode_chunk(tile: TileMeta, chunk: ChunkRef) -> np.ndarray:
    """One compressed chunk -> raw records (bit-exact), decoded on the GPU
    from the chunk's bytes only (reader.py:286-344)."""
    from .. import _device as D
    _check_items(tile)
    with open(tile.path, "rb") as fp:
        fp.seek(chunk.byte_offset)
        buf = fp.read(chunk.byte_size)
        size = os.fstat(fp.fileno()).st_size
    if len(buf) < chunk.byte_size:
        raise OutOfBoundsRead("chunk extends beyond file end")
    d = D.tile_desc(tile.header)
    d["image_base"] = chunk.byte_offset
    tb = D.TileBatch([buf], d, file_sizes=np.array([size], np.int64))
    tab = _Tables(D, [chunk.byte_offset], [chunk.point_count],
                  [chunk.byte_offset + chunk.byte_size], [0, 1])
    fr = D.FullRecords(tb, tab)
    D.raise_item_status(fr.status.cpu().numpy(), "decode_chunk")
    dt = record_dtype(tile.header.point_record_format)
    return fr.records[:fr.n_points * dt.itemsize].cpu().numpy().view(dt).copy()


def load_tile_fullres(tile: TileMeta, max_workers: int = 4) -> np.ndarray:
    """Every record of the tile (reader.py:347-364): LAS point block read
    directly, LAZ chunks decoded on the GPU in parallel (one thread per
    chunk); max_workers is accepted for the reference's signature."""
    header = tile.header
    if not tile.is_compressed:
        fmt = header.point_record_format
        dtype = record_dtype(fmt, header.point_record_length)
        with open(tile.path, "rb") as fp:
            fp.seek(header.point_data_offset)
            buf = fp.read(header.point_count * dtype.itemsize)
        if len(buf) < header.point_count * dtype.itemsize:
            raise OutOfBoundsRead("point data truncated")
        return np.frombuffer(buf, dtype=dtype)
    from .. import _device as D
    _check_laz(tile)
    _check_items(tile)
    refs = ensure_chunk_refs(tile)
    if not refs:
        return np.empty(0, dtype=record_dtype(header.point_record_format))
    lo = refs[0].byte_offset
    hi = max(r.byte_offset + r.byte_size for r in refs)
    with open(tile.path, "rb") as fp:
        size = os.fstat(fp.fileno()).st_size
        fp.seek(lo)
        buf = fp.read(hi - lo)   # the chunks only (header and table excluded)
    if len(buf) < hi - lo:
        raise OutOfBoundsRead("chunk extends beyond file end")
    d = D.tile_desc(header)
    d["image_base"] = lo
    tb = D.TileBatch([buf], d, file_sizes=np.array([size], np.int64))
    tab = _Tables(D, [r.byte_offset for r in refs], [r.point_count for r in refs],
                  [refs[-1].byte_offset + refs[-1].byte_size], [0, len(refs)])
    fr = D.FullRecords(tb, tab)
    D.raise_item_status(fr.status.cpu().numpy(), "load_tile_fullres")
    dt = record_dtype(header.point_record_format)
    return fr.records[:fr.n_points * dt.itemsize].cpu().numpy().view(dt).copy()
