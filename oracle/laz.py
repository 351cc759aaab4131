"""Oracle: LAZ chunk table + chunk-point extraction + model-space records.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  * ``ArithmeticDecoder`` / models / ``IntegerCompressor.decompress``
    (``pkg/src/terrascout/lasio/codec.py:43-281, 441-484``),
  * ``_read_chunk_table_fd`` (``lasio/reader.py:141-209``),
  * ``_las_chunk_refs`` (``reader.py:212-226``),
  * ``read_chunk_points`` + ``_raw_record`` (``reader.py:239-283``),
  * ``positions`` / ``colors`` (``lasio/records.py:62-86``),
operating on an in-memory file image (bytes) instead of a path.
"""

from __future__ import annotations

import struct

import numpy as np

_MIN = 0x01000000


class Desync(Exception):
    pass


class CorruptTable(Exception):
    pass


class BitModel:
    # codec.py:43-67
    def __init__(self):
        self.c0, self.n, self.p0, self.cyc, self.left = 1, 2, 4096, 4, 4

    def upd(self):
        self.n += self.cyc
        if self.n >= 8192:
            self.n = (self.n + 1) >> 1
            self.c0 = (self.c0 + 1) >> 1
            if self.c0 == self.n:
                self.n += 1
        self.p0 = (self.c0 * (0x80000000 // self.n)) >> 18
        self.cyc = min((5 * self.cyc) >> 2, 64)
        self.left = self.cyc


class SymModel:
    # codec.py:70-168 (decoder side, with the >16-symbol lookup table)
    def __init__(self, n):
        self.n = n
        self.cnt = [1] * n
        self.dist = [0] * n
        self.tot = 0
        self.tbits = 0
        if n > 16:
            tb = 3
            while n > (1 << (tb + 2)):
                tb += 1
            self.tbits = tb
            self.tshift = 15 - tb
            self.table = [0] * ((1 << tb) + 2)
        self.cyc = n
        self.upd()
        self.cyc = self.left = (n + 6) >> 1

    def upd(self):
        self.tot += self.cyc
        if self.tot > 32768:
            self.cnt = [(c + 1) >> 1 for c in self.cnt]
            self.tot = sum(self.cnt)
        scale = 0x80000000 // self.tot
        acc = 0
        for k in range(self.n):
            self.dist[k] = (scale * acc) >> 16
            acc += self.cnt[k]
        if self.tbits:
            size = 1 << self.tbits
            s = 0
            for k in range(self.n):
                w = self.dist[k] >> self.tshift
                while s < w:
                    s += 1
                    self.table[s] = k - 1
            self.table[0] = 0
            while s <= size:
                s += 1
                self.table[s] = self.n - 1
        self.cyc = min((5 * self.cyc) >> 2, (self.n + 6) << 3)
        self.left = self.cyc


class Decoder:
    # codec.py:173-281
    def __init__(self, buf, pos, end):
        self.b, self.p, self.end = buf, pos, end
        if pos + 4 > end:
            raise Desync("start")
        self.v = int.from_bytes(buf[pos:pos + 4], "big")
        self.p += 4
        self.len = 0xFFFFFFFF

    def _renorm(self):
        while self.len < _MIN:
            if self.p >= self.end:
                raise Desync("ran past end")
            self.v = ((self.v << 8) | self.b[self.p]) & 0xFFFFFFFF
            self.p += 1
            self.len <<= 8

    def bit(self, m: BitModel):
        x = m.p0 * (self.len >> 13)
        if self.v < x:
            s = 0
            self.len = x
            m.c0 += 1
        else:
            s = 1
            self.v -= x
            self.len -= x
        if self.len < _MIN:
            self._renorm()
        m.left -= 1
        if m.left == 0:
            m.upd()
        return s

    def sym(self, m: SymModel):
        hi = self.len
        self.len >>= 15
        unit = self.len
        if m.tbits:
            dv = self.v // unit
            t = dv >> m.tshift
            s = m.table[t]
            n = m.table[t + 1] + 1
            while n > s + 1:
                k = (s + n) >> 1
                if m.dist[k] > dv:
                    n = k
                else:
                    s = k
            lo = m.dist[s] * unit
            if s != m.n - 1:
                hi = m.dist[s + 1] * unit
        else:
            lo = s = 0
            n = m.n
            k = n >> 1
            while True:
                z = unit * m.dist[k]
                if z > self.v:
                    n = k
                    hi = z
                else:
                    s = k
                    lo = z
                k = (s + n) >> 1
                if k == s:
                    break
        self.v -= lo
        self.len = hi - lo
        if self.len < _MIN:
            self._renorm()
        m.cnt[s] += 1
        m.left -= 1
        if m.left == 0:
            m.upd()
        return s

    def bits(self, nb):
        if nb > 19:
            lo = self.bits(16)
            return (self.bits(nb - 16) << 16) | lo
        self.len >>= nb
        s = self.v // self.len
        self.v -= self.len * s
        if self.len < _MIN:
            self._renorm()
        return s


def decompress32(dec: Decoder, state: dict, pred: int, ctx: int) -> int:
    """IntegerCompressor(32 bits, bits_high 8).decompress (codec.py:441-484)."""
    km = state.get(("k", ctx))
    if km is None:
        km = state[("k", ctx)] = SymModel(33)
    k = dec.sym(km)
    if k == 0:
        bm = state.get(("c", 0))
        if bm is None:
            bm = state[("c", 0)] = BitModel()
        c = dec.bit(bm)
    elif k < 32:
        cm = state.get(("c", k))
        if cm is None:
            cm = state[("c", k)] = SymModel(1 << min(k, 8))
        if k <= 8:
            c = dec.sym(cm)
        else:
            lowb = k - 8
            c = (dec.sym(cm) << lowb) | dec.bits(lowb)
        if c >= (1 << (k - 1)):
            c += 1
        else:
            c -= (1 << k) - 1
    else:
        c = -0x80000000
    r = (pred + c) & 0xFFFFFFFF
    return r - (1 << 32) if r >= 0x80000000 else r


# --------------------------------------------------------------- headers

MIN_REC = {0: 20, 1: 28, 2: 26, 3: 34}


def header_fields(img: bytes) -> dict:
    """The handful of header fields the chunk-point path reads."""
    vmin = img[25]
    hsize, = struct.unpack_from("<H", img, 94)
    pdo, nvlr = struct.unpack_from("<II", img, 96)
    fmt = img[104] & 0x7F
    rec_len, = struct.unpack_from("<H", img, 105)
    count, = struct.unpack_from("<I", img, 107)
    so = struct.unpack_from("<6d", img, 131)
    if vmin >= 4:
        c14, = struct.unpack_from("<Q", img, 247)
        count = c14 or count
    chunk_size = None
    pos = hsize
    for _ in range(nvlr):
        uid = img[pos + 2:pos + 18].rstrip(b"\0")
        rid, ln = struct.unpack_from("<HH", img, pos + 18)
        if uid == b"laszip encoded" and rid == 22204:
            chunk_size, = struct.unpack_from("<I", img, pos + 54 + 12)
        pos += 54 + ln
    return dict(pdo=pdo, fmt=fmt, rec_len=rec_len, count=count,
                scale=so[:3], offset=so[3:], chunk_size=chunk_size,
                compressed=chunk_size is not None)


def chunk_table(img: bytes, h: dict):
    """(byte_offsets, point_counts) -- reader.py:141-209."""
    size = len(img)
    tpos, = struct.unpack_from("<q", img, h["pdo"])
    start = h["pdo"] + 8
    if tpos == -1:
        tpos, = struct.unpack_from("<q", img, size - 8)
    if not start <= tpos <= size - 8:
        raise CorruptTable("pointer outside file")
    version, n = struct.unpack_from("<II", img, tpos)
    if version != 0:
        raise CorruptTable("version")
    variable = h["chunk_size"] == 0xFFFFFFFF
    counts, sizes = [], []
    if n:
        dec = Decoder(img, tpos + 8, size)
        st: dict = {}
        pc = ps = 0
        try:
            for _ in range(n):
                if variable:
                    pc = decompress32(dec, st, pc, 0)
                    counts.append(pc)
                ps = decompress32(dec, st, ps, 1)
                sizes.append(ps)
        except Desync as e:
            raise CorruptTable(str(e)) from e
    if not variable:
        left = h["count"]
        for _ in range(n):
            c = min(h["chunk_size"], left)
            counts.append(c)
            left -= c
    if sum(counts) != h["count"]:
        raise CorruptTable("count mismatch")
    offs = []
    o = start
    for s in sizes:
        if s <= 0:
            raise CorruptTable("size")
        offs.append(o)
        o += s
    if o > tpos:
        raise CorruptTable("overlap")
    return np.array(offs, np.int64), np.array(counts, np.int64)


def record_dtype(fmt: int) -> np.dtype:
    f = [("x", "<i4"), ("y", "<i4"), ("z", "<i4"), ("intensity", "<u2"),
         ("bitfield", "u1"), ("classification", "u1"), ("scan_angle", "u1"),
         ("user_data", "u1"), ("point_source_id", "<u2")]
    if fmt in (1, 3):
        f.append(("gps_time", "<u8"))
    if fmt in (2, 3):
        f += [("red", "<u2"), ("green", "<u2"), ("blue", "<u2")]
    return np.dtype(f)


def chunk_points(img: bytes, las_stride: int = 50_000) -> np.ndarray:
    """First raw record of every chunk -- reader.py:251-283."""
    h = header_fields(img)
    fmt = h["fmt"]
    if fmt not in MIN_REC:
        raise ValueError("unsupported format")
    if h["compressed"]:
        offs, _ = chunk_table(img, h)
    else:
        n = -(-h["count"] // las_stride)
        offs = h["pdo"] + np.arange(n, dtype=np.int64) * las_stride * \
            h["rec_len"]
    dt = record_dtype(fmt)
    need = dt.itemsize
    if len(offs) and int(offs.max()) + h["rec_len"] > len(img):
        raise IndexError("offset beyond file end")
    buf = np.frombuffer(img, np.uint8)
    rows = np.stack([buf[o:o + need] for o in offs]) if len(offs) else \
        np.zeros((0, need), np.uint8)
    return rows.copy().view(dt).reshape(-1)


def positions(rec: np.ndarray, scale, offset) -> np.ndarray:
    """records.py:62-67: per axis x*s + o in float64 (two roundings)."""
    out = np.empty((len(rec), 3))
    for i, ax in enumerate("xyz"):
        out[:, i] = rec[ax].astype(np.float64) * scale[i] + offset[i]
    return out


def colors(rec: np.ndarray):
    """records.py:70-86 incl. the per-batch 8-bit heuristic."""
    if "red" not in (rec.dtype.names or ()):
        return None
    rgb = np.stack([rec["red"], rec["green"], rec["blue"]], axis=1)
    div = 255.0 if len(rgb) and rgb.max() <= 255 else 65535.0
    return (rgb / div).astype(np.float32)
