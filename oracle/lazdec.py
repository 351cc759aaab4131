"""Oracle: full LAZ chunk decode (POINT10 / GPSTIME11 / RGB12 v2 items).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``decode_chunk`` (``pkg/src/terrascout/lasio/reader.py:286-344``)
with the item decoders of ``lasio/items.py:108-606`` and the generic
``IntegerCompressor.decompress`` (``lasio/codec.py:441-484``) on top of the
arithmetic decoder and models already restated in ``oracle/laz.py``.
Pinned by ``tests/test_oracle_golden.py`` against ``tests/golden/
fullres.npz`` (reference-compressed files + the reference's decoded
records).  Pure Python: small inputs only.
"""

from __future__ import annotations

import struct

import numpy as np

from .laz import BitModel, Decoder, SymModel, chunk_table, header_fields, record_dtype

_NRM = (  # NUMBER_RETURN_MAP (items.py:26-35)
    (15, 14, 13, 12, 11, 10, 9, 8), (14, 0, 1, 3, 6, 10, 10, 9),
    (13, 1, 2, 4, 7, 11, 11, 10), (12, 3, 4, 5, 8, 12, 12, 11),
    (11, 6, 7, 8, 9, 13, 13, 12), (10, 10, 11, 12, 13, 14, 14, 13),
    (9, 10, 11, 12, 13, 14, 15, 14), (8, 9, 10, 11, 12, 13, 14, 15))
_NRL = tuple(tuple(abs(n - r) for r in range(8)) for n in range(8))  # items.py:37-46


def _i32(v):
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v >= 0x80000000 else v


class IC:
    """IntegerCompressor(bits, contexts, bits_high=8).decompress."""

    def __init__(self, bits=16, contexts=1, bits_high=8):
        self.bits_high = bits_high
        if 0 < bits < 32:
            self.corr_bits, self.corr_range = bits, 1 << bits
            self.corr_min = -(self.corr_range // 2)
        else:
            self.corr_bits, self.corr_range, self.corr_min = 32, 0, -0x80000000
        self.mk = {}
        self.mc = {}
        self.k = 0

    def decompress(self, dec: Decoder, pred: int, ctx: int = 0) -> int:
        m = self.mk.get(ctx)
        if m is None:
            m = self.mk[ctx] = SymModel(self.corr_bits + 1)
        k = dec.sym(m)
        self.k = k
        if k:
            if k < 32:
                cm = self.mc.get(k)
                if cm is None:
                    cm = self.mc[k] = SymModel(1 << min(k, self.bits_high))
                if k <= self.bits_high:
                    c = dec.sym(cm)
                else:
                    k1 = k - self.bits_high
                    c = (dec.sym(cm) << k1) | dec.bits(k1)
                if c >= (1 << (k - 1)):
                    c += 1
                else:
                    c -= (1 << k) - 1
            else:
                c = self.corr_min
        else:
            bm = self.mc.get(0)
            if bm is None:
                bm = self.mc[0] = BitModel()
            c = dec.bit(bm)
        real = pred + c
        if self.corr_range:
            if real < 0:
                real += self.corr_range
            elif real >= self.corr_range:
                real -= self.corr_range
            return real
        return _i32(real)


class Median5:
    # StreamingMedian5 (items.py:49-104)
    def __init__(self):
        self.v = [0, 0, 0, 0, 0]
        self.high = True

    def add(self, x):
        v = self.v
        if self.high:
            if x < v[2]:
                v[4], v[3] = v[3], v[2]
                if x < v[0]:
                    v[2], v[1], v[0] = v[1], v[0], x
                elif x < v[1]:
                    v[2], v[1] = v[1], x
                else:
                    v[2] = x
            else:
                if x < v[3]:
                    v[4], v[3] = v[3], x
                else:
                    v[4] = x
                self.high = False
        else:
            if x > v[2]:
                v[0], v[1] = v[1], v[2]
                if x > v[4]:
                    v[2], v[3], v[4] = v[3], v[4], x
                elif x > v[3]:
                    v[2], v[3] = v[3], x
                else:
                    v[2] = x
            else:
                if x > v[1]:
                    v[0], v[1] = v[1], x
                else:
                    v[0] = x
                self.high = True


class Point10:
    # Point10Codec.read (items.py:111-209)
    def __init__(self, first):
        self.mchg = SymModel(64)
        self.ic_int = IC(16, 4)
        self.msa = [SymModel(256), SymModel(256)]
        self.ic_psid = IC(16)
        self.mbit, self.mcls, self.mud = {}, {}, {}
        self.ic_dx, self.ic_dy, self.ic_z = IC(32, 2), IC(32, 22), IC(32, 20)
        self.mx = [Median5() for _ in range(16)]
        self.my = [Median5() for _ in range(16)]
        self.lint = [0] * 16
        self.lh = [0] * 8
        self.last = list(first)
        self.last[3] = 0

    @staticmethod
    def _m(tab, v):
        m = tab.get(v)
        if m is None:
            m = tab[v] = SymModel(256)
        return m

    def read(self, d):
        last = self.last
        cv = d.sym(self.mchg)
        if cv & 32:
            last[4] = d.sym(self._m(self.mbit, last[4]))
        bf = last[4]
        r, n = bf & 7, (bf >> 3) & 7
        mc, lvl = _NRM[n][r], _NRL[n][r]
        if cv & 16:
            last[3] = self.ic_int.decompress(d, self.lint[mc], mc if mc < 3 else 3)
            self.lint[mc] = last[3]
        else:
            last[3] = self.lint[mc]
        if cv & 8:
            last[5] = d.sym(self._m(self.mcls, last[5]))
        if cv & 4:
            last[6] = (d.sym(self.msa[(bf >> 6) & 1]) + last[6]) & 0xFF
        if cv & 2:
            last[7] = d.sym(self._m(self.mud, last[7]))
        if cv & 1:
            last[8] = self.ic_psid.decompress(d, last[8])
        n1 = 1 if n == 1 else 0
        diff = self.ic_dx.decompress(d, self.mx[mc].v[2], n1)
        last[0] = _i32(last[0] + diff)
        self.mx[mc].add(diff)
        kb = self.ic_dx.k
        diff = self.ic_dy.decompress(d, self.my[mc].v[2],
                                     n1 + ((kb & ~1) if kb < 20 else 20))
        last[1] = _i32(last[1] + diff)
        self.my[mc].add(diff)
        kb = (self.ic_dx.k + self.ic_dy.k) // 2
        last[2] = self.ic_z.decompress(d, self.lh[lvl], n1 + ((kb & ~1) if kb < 18 else 18))
        self.lh[lvl] = last[2]
        return tuple(last)


MULTI, MULTI_MINUS = 500, -10
MULTI_TOTAL = MULTI - MULTI_MINUS + 6
MULTI_UNCHANGED = MULTI - MULTI_MINUS + 1
MULTI_CODE_FULL = MULTI - MULTI_MINUS + 2


class Gps:
    # GpsTimeCodec.read (items.py:281-383)
    def __init__(self, first):
        self.mmulti = SymModel(MULTI_TOTAL)
        self.m0 = SymModel(6)
        self.ic = IC(32, 9)
        self.last = self.next = 0
        self.t = [first, 0, 0, 0]
        self.dt = [0, 0, 0, 0]
        self.cnt = [0, 0, 0, 0]

    def _full(self, d):
        self.next = (self.next + 1) & 3
        hi = self.ic.decompress(d, _i32(self.t[self.last] >> 32), 8)
        self.t[self.next] = ((hi & 0xFFFFFFFF) << 32) | d.bits(32)
        self.last = self.next
        self.dt[self.last] = 0
        self.cnt[self.last] = 0

    def read(self, d):
        while True:
            L = self.last
            if self.dt[L] == 0:
                m = d.sym(self.m0)
                if m == 1:
                    v = self.ic.decompress(d, 0, 0)
                    self.dt[L] = v
                    self.t[L] = (self.t[L] + v) & 0xFFFFFFFFFFFFFFFF
                    self.cnt[L] = 0
                elif m == 2:
                    self._full(d)
                elif m > 2:
                    self.last = (L + m - 2) & 3
                    continue
                return self.t[self.last]
            m = d.sym(self.mmulti)
            if m == 1:
                v = self.ic.decompress(d, self.dt[L], 1)
                self.t[L] = (self.t[L] + v) & 0xFFFFFFFFFFFFFFFF
                self.cnt[L] = 0
            elif m < MULTI_UNCHANGED:
                if m == 0:
                    g = self.ic.decompress(d, 0, 7)
                    self.cnt[L] += 1
                    if self.cnt[L] > 3:
                        self.dt[L] = g
                        self.cnt[L] = 0
                elif m < MULTI:
                    g = self.ic.decompress(d, _i32(m * self.dt[L]), 2 if m < 10 else 3)
                elif m == MULTI:
                    g = self.ic.decompress(d, _i32(MULTI * self.dt[L]), 4)
                    self.cnt[L] += 1
                    if self.cnt[L] > 3:
                        self.dt[L] = g
                        self.cnt[L] = 0
                else:
                    mm = MULTI - m
                    if mm > MULTI_MINUS:
                        g = self.ic.decompress(d, _i32(mm * self.dt[L]), 5)
                    else:
                        g = self.ic.decompress(d, _i32(MULTI_MINUS * self.dt[L]), 6)
                        self.cnt[L] += 1
                        if self.cnt[L] > 3:
                            self.dt[L] = g
                            self.cnt[L] = 0
                self.t[L] = (self.t[L] + g) & 0xFFFFFFFFFFFFFFFF
            elif m == MULTI_CODE_FULL:
                self._full(d)
            elif m > MULTI_CODE_FULL:
                self.last = (L + m - MULTI_CODE_FULL) & 3
                continue
            return self.t[self.last]


def _clamp(v):
    return 0 if v <= 0 else 255 if v >= 255 else v


def _cdiv2(v):
    return -((-v) >> 1) if v < 0 else v >> 1


class Rgb:
    # RgbCodec.read (items.py:514-561)
    def __init__(self, first):
        self.mused = SymModel(128)
        self.md = [SymModel(256) for _ in range(6)]
        self.last = tuple(first)

    def read(self, d):
        lr, lg, lb = self.last
        s = d.sym(self.mused)
        rl = (d.sym(self.md[0]) + (lr & 0xFF)) & 0xFF if s & 1 else lr & 0xFF
        rh = (d.sym(self.md[1]) + (lr >> 8)) & 0xFF if s & 2 else lr >> 8
        red = rl | (rh << 8)
        if s & 64:
            diff = rl - (lr & 0xFF)
            gl = (d.sym(self.md[2]) + _clamp(diff + (lg & 0xFF))) & 0xFF if s & 4 else lg & 0xFF
            if s & 16:
                diff = _cdiv2(diff + gl - (lg & 0xFF))
                bl = (d.sym(self.md[4]) + _clamp(diff + (lb & 0xFF))) & 0xFF
            else:
                bl = lb & 0xFF
            diff = rh - (lr >> 8)
            gh = (d.sym(self.md[3]) + _clamp(diff + (lg >> 8))) & 0xFF if s & 8 else lg >> 8
            if s & 32:
                diff = _cdiv2(diff + gh - (lg >> 8))
                bh = (d.sym(self.md[5]) + _clamp(diff + (lb >> 8))) & 0xFF
            else:
                bh = lb >> 8
            green, blue = gl | (gh << 8), bl | (bh << 8)
        else:
            green = blue = red
        self.last = (red, green, blue)
        return self.last


def decode_chunk(img: bytes, offset: int, size: int, count: int, fmt: int) -> np.ndarray:
    """decode_chunk (reader.py:286-344) of the chunk at [offset, offset+size)."""
    dt = record_dtype(fmt)
    buf = img[offset:offset + size]
    first = np.frombuffer(buf[:dt.itemsize], dt)[0]
    row0 = tuple(int(first[f]) for f in dt.names)
    rows = [row0]
    d = Decoder(buf, dt.itemsize, len(buf))
    p10 = Point10(row0[:9])
    cur = 9
    gps = rgb = None
    if fmt in (1, 3):
        gps = Gps(row0[cur])
        cur += 1
    if fmt in (2, 3):
        rgb = Rgb(row0[cur:cur + 3])
    for _ in range(count - 1):
        row = p10.read(d)
        if gps is not None:
            row += (gps.read(d),)
        if rgb is not None:
            row += rgb.read(d)
        rows.append(row)
    return np.array(rows, dtype=dt)


def load_fullres(img: bytes) -> np.ndarray:
    """load_tile_fullres (reader.py:347-364) of a LAZ image: every chunk."""
    h = header_fields(img)
    offs, counts = chunk_table(img, h)
    tpos = struct.unpack_from("<q", img, h["pdo"])[0]
    if tpos == -1:
        tpos = struct.unpack_from("<q", img, len(img) - 8)[0]
    ends = list(offs[1:]) + [tpos]
    parts = [decode_chunk(img, int(o), int(e - o), int(c), h["fmt"])
             for o, e, c in zip(offs, ends, counts)]
    return np.concatenate(parts) if parts else np.empty(0, record_dtype(h["fmt"]))


