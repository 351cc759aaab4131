"""LASzip-2 arithmetic *encoder* + integer compressor (corpus writer only).

Supporting code: synthetic corpora need an entropy-coded chunk table so
that the reference reader, the oracle and the CUDA decoder
(``csrc/laz_ac.cuh``) can all read the same files.  The model update rules
are the published LASzip ones the reference follows
(``pkg/src/terrascout/lasio/codec.py:43-168`` models, ``:284-383`` encoder,
``:486-508`` corrector coding); the decoder side lives in CUDA.
"""

from __future__ import annotations

MAX_LEN = 0xFFFFFFFF
MIN_LEN = 0x01000000
_BM_SHIFT = 13
_DM_SHIFT = 15
_M32 = 0xFFFFFFFF


class _BitModel:
    def __init__(self):
        self.zeros, self.total, self.p0 = 1, 2, 1 << (_BM_SHIFT - 1)
        self.cycle = self.left = 4

    def refresh(self):
        self.total += self.cycle
        if self.total >= (1 << _BM_SHIFT):
            self.total = (self.total + 1) >> 1
            self.zeros = (self.zeros + 1) >> 1
            if self.zeros == self.total:
                self.total += 1
        self.p0 = (self.zeros * (0x80000000 // self.total)) >> \
            (31 - _BM_SHIFT)
        self.cycle = min((5 * self.cycle) >> 2, 64)
        self.left = self.cycle


class _SymModel:
    """Adaptive frequency model (encoder side never needs the table)."""

    def __init__(self, n: int):
        self.n = n
        self.counts = [1] * n
        self.cdf = [0] * n
        self.total = 0
        self.cycle = n
        self.refresh()
        self.cycle = self.left = (n + 6) >> 1

    def refresh(self):
        self.total += self.cycle
        if self.total > (1 << _DM_SHIFT):
            self.counts = [(c + 1) >> 1 for c in self.counts]
            self.total = sum(self.counts)
        scale = 0x80000000 // self.total
        run = 0
        for k, c in enumerate(self.counts):
            self.cdf[k] = (scale * run) >> (31 - _DM_SHIFT)
            run += c
        self.cycle = min((5 * self.cycle) >> 2, (self.n + 6) << 3)
        self.left = self.cycle


class Encoder:
    def __init__(self):
        self.buf = bytearray()
        self.low = 0
        self.length = MAX_LEN

    def _carry(self):
        i = len(self.buf) - 1
        while self.buf[i] == 0xFF:
            self.buf[i] = 0
            i -= 1
        self.buf[i] += 1

    def _shift_out(self):
        while self.length < MIN_LEN:
            self.buf.append((self.low >> 24) & 0xFF)
            self.low = (self.low << 8) & _M32
            self.length = (self.length << 8) & _M32

    def _advance(self, add: int):
        old = self.low
        self.low = (self.low + add) & _M32
        if old > self.low:
            self._carry()

    def bit(self, m: _BitModel, b: int):
        x = m.p0 * (self.length >> _BM_SHIFT)
        if b:
            self._advance(x)
            self.length -= x
        else:
            self.length = x
            m.zeros += 1
        if self.length < MIN_LEN:
            self._shift_out()
        m.left -= 1
        if m.left == 0:
            m.refresh()

    def symbol(self, m: _SymModel, s: int):
        old = self.low
        if s == m.n - 1:
            x = m.cdf[s] * (self.length >> _DM_SHIFT)
            self.low = (self.low + x) & _M32
            self.length -= x
        else:
            unit = self.length >> _DM_SHIFT
            x = m.cdf[s] * unit
            self.low = (self.low + x) & _M32
            self.length = m.cdf[s + 1] * unit - x
        if old > self.low:
            self._carry()
        if self.length < MIN_LEN:
            self._shift_out()
        m.counts[s] += 1
        m.left -= 1
        if m.left == 0:
            m.refresh()

    def raw_bits(self, nbits: int, value: int):
        if nbits > 19:
            self.raw_bits(16, value & 0xFFFF)
            value >>= 16
            nbits -= 16
        self.length >>= nbits
        self._advance(value * self.length)
        if self.length < MIN_LEN:
            self._shift_out()

    def finish(self) -> bytes:
        old = self.low
        if self.length > 2 * MIN_LEN:
            self.low = (self.low + MIN_LEN) & _M32
            self.length = MIN_LEN >> 1
            extra = 1
        else:
            self.low = (self.low + (MIN_LEN >> 1)) & _M32
            self.length = MIN_LEN >> 9
            extra = 0
        if old > self.low:
            self._carry()
        self._shift_out()
        self.buf += bytes(2 + extra)
        return bytes(self.buf)


class IntCompressor32:
    """IntegerCompressor(bits=32, contexts, bits_high=8) encode side."""

    def __init__(self, enc: Encoder, contexts: int):
        self.enc = enc
        self.k_models = [None] * contexts
        self.c_models: dict[int, object] = {}

    def _corr_model(self, k: int):
        m = self.c_models.get(k)
        if m is None:
            m = _BitModel() if k == 0 else _SymModel(1 << min(k, 8))
            self.c_models[k] = m
        return m

    def compress(self, pred: int, real: int, ctx: int):
        c = (real - pred) & _M32
        if c >= 0x80000000:
            c -= 1 << 32
        if self.k_models[ctx] is None:
            self.k_models[ctx] = _SymModel(33)
        mag = -c if c <= 0 else c - 1
        k = mag.bit_length()
        self.enc.symbol(self.k_models[ctx], k)
        if k == 0:
            self.enc.bit(self._corr_model(0), c)
            return
        if k >= 32:
            return
        c = c - 1 if c >= 0 else c + (1 << k) - 1
        if k <= 8:
            self.enc.symbol(self._corr_model(k), c)
        else:
            low_bits = k - 8
            self.enc.symbol(self._corr_model(k), c >> low_bits)
            self.enc.raw_bits(low_bits, c & ((1 << low_bits) - 1))


def encode_chunk_table(sizes, counts=None) -> bytes:
    """Chunk-table payload (after the u32 version/count words)."""
    enc = Encoder()
    ic = IntCompressor32(enc, 2)
    prev_size = prev_count = 0
    for i, size in enumerate(sizes):
        if counts is not None:
            ic.compress(prev_count, int(counts[i]), 0)
            prev_count = int(counts[i])
        ic.compress(prev_size, int(size), 1)
        prev_size = int(size)
    return enc.finish()
