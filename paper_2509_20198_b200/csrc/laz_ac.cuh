// LASzip-2 arithmetic decoder + 32-bit IntegerCompressor for chunk tables.
//
// Device code (one thread decodes one tile's table).  Follows the
// published LASzip coder the reference restates in
// pkg/src/terrascout/lasio/codec.py:43-281 (models, decoder) and
// :441-484 (IntegerCompressor.decompress, bits=32, bits_high=8).
// Model state lives in a per-thread scratch pool (global memory) because a
// table may touch up to 31 corrector models of up to 256 symbols.
#pragma once

#include <stdint.h>

namespace ts {
namespace laz {

constexpr uint32_t kMinLen = 0x01000000u;
constexpr uint32_t kMaxLen = 0xFFFFFFFFu;

struct BitModel {
  uint32_t c0, n, p0, cyc, left;
  __host__ __device__ void init() { c0 = 1; n = 2; p0 = 1u << 12; cyc = left = 4; }
  __host__ __device__ void update() {
    n += cyc;
    if (n >= 8192u) {
      n = (n + 1) >> 1;
      c0 = (c0 + 1) >> 1;
      if (c0 == n) ++n;
    }
    p0 = (c0 * (0x80000000u / n)) >> 18;
    cyc = min((5u * cyc) >> 2, 64u);
    left = cyc;
  }
};

// Adaptive symbol model, decoder flavour (lookup table when n > 16).
struct SymModel {
  uint32_t n, tot, cyc, left, tbits, tshift;
  uint16_t* dist;   // n
  uint16_t* cnt;    // n
  uint16_t* table;  // (1 << tbits) + 2, only if tbits
  __host__ __device__ static uint32_t table_bits(uint32_t n) {
    if (n <= 16) return 0;
    uint32_t tb = 3;
    while (n > (1u << (tb + 2))) ++tb;
    return tb;
  }
  __host__ __device__ static uint32_t words16(uint32_t n) {
    uint32_t tb = table_bits(n);
    return 2 * n + (tb ? (1u << tb) + 2 : 0);
  }
  __host__ __device__ void init(uint32_t nsym, uint16_t* mem) {
    n = nsym;
    tbits = table_bits(n);
    tshift = tbits ? 15 - tbits : 0;
    dist = mem;
    cnt = mem + n;
    table = tbits ? mem + 2 * n : nullptr;
    for (uint32_t k = 0; k < n; ++k) cnt[k] = 1;
    tot = 0;
    cyc = n;
    update();
    cyc = left = (n + 6) >> 1;
  }
  __host__ __device__ void update() {
    tot += cyc;
    if (tot > 32768u) {
      tot = 0;
      for (uint32_t k = 0; k < n; ++k) {
        cnt[k] = (uint16_t)((cnt[k] + 1u) >> 1);
        tot += cnt[k];
      }
    }
    const uint32_t scale = 0x80000000u / tot;
    uint32_t acc = 0;
    if (!tbits) {
      for (uint32_t k = 0; k < n; ++k) {
        dist[k] = (uint16_t)((scale * acc) >> 16);
        acc += cnt[k];
      }
    } else {
      uint32_t s = 0;
      for (uint32_t k = 0; k < n; ++k) {
        const uint32_t d = (scale * acc) >> 16;
        dist[k] = (uint16_t)d;
        acc += cnt[k];
        const uint32_t w = d >> tshift;
        while (s < w) table[++s] = (uint16_t)(k - 1);
      }
      table[0] = 0;
      const uint32_t size = 1u << tbits;
      while (s <= size) table[++s] = (uint16_t)(n - 1);
    }
    cyc = min((5u * cyc) >> 2, (n + 6) << 3);
    left = cyc;
  }
};

struct Decoder {
  const uint8_t* buf;
  int64_t pos, end;
  uint32_t value, length;
  bool desync;

  __host__ __device__ bool start(const uint8_t* b, int64_t p, int64_t e) {
    buf = b; pos = p; end = e; desync = false;
    if (pos + 4 > end) { desync = true; return false; }
    value = ((uint32_t)buf[pos] << 24) | ((uint32_t)buf[pos + 1] << 16) |
            ((uint32_t)buf[pos + 2] << 8) | (uint32_t)buf[pos + 3];
    pos += 4;
    length = kMaxLen;
    return true;
  }
  __host__ __device__ void renorm() {
    while (length < kMinLen) {
      if (pos >= end) { desync = true; length = kMaxLen; return; }
      value = (value << 8) | buf[pos++];
      length <<= 8;
    }
  }
  __host__ __device__ uint32_t bit(BitModel& m) {
    const uint32_t x = m.p0 * (length >> 13);
    uint32_t s;
    if (value < x) { s = 0; length = x; ++m.c0; }
    else { s = 1; value -= x; length -= x; }
    if (length < kMinLen) renorm();
    if (--m.left == 0) m.update();
    return s;
  }
  __host__ __device__ uint32_t symbol(SymModel& m) {
    uint32_t hi = length;
    uint32_t lo, s;
    const uint32_t unit = length >> 15;
    length = unit;
    if (m.tbits) {
      const uint32_t dv = value / unit;
      const uint32_t t = dv >> m.tshift;
      s = m.table[t];
      uint32_t n = (uint32_t)m.table[t + 1] + 1;
      while (n > s + 1) {
        const uint32_t k = (s + n) >> 1;
        if (m.dist[k] > dv) n = k; else s = k;
      }
      lo = m.dist[s] * unit;
      if (s != m.n - 1) hi = m.dist[s + 1] * unit;
    } else {
      lo = 0; s = 0;
      uint32_t n = m.n, k = n >> 1;
      do {
        const uint32_t z = unit * m.dist[k];
        if (z > value) { n = k; hi = z; } else { s = k; lo = z; }
        k = (s + n) >> 1;
      } while (k != s);
    }
    value -= lo;
    length = hi - lo;
    if (length < kMinLen) renorm();
    ++m.cnt[s];
    if (--m.left == 0) m.update();
    return s;
  }
  __host__ __device__ uint32_t raw_bits_le19(uint32_t nb) {
    length >>= nb;
    const uint32_t s = value / length;
    value -= length * s;
    if (length < kMinLen) renorm();
    return s;
  }
  // read_bits (codec.py:258-267) without recursion: a static stack frame
  __host__ __device__ uint32_t raw_bits(uint32_t nb) {
    if (nb > 19) {
      const uint32_t lo = raw_bits_le19(16);
      return (raw_bits_le19(nb - 16) << 16) | lo;
    }
    return raw_bits_le19(nb);
  }
};

// Model pool of one decoding thread: k-models for 2 contexts, the k = 0
// bit model and corrector models k = 1..31, allocated on first use.
struct ChunkTableCoder {
  SymModel kmod[2];
  bool kmod_live[2];
  BitModel cbit;
  bool cbit_live;
  SymModel cmod[32];
  bool cmod_live[32];
  uint16_t* pool;      // fast pool (shared memory), `budget` words
  uint16_t* overflow;  // global-memory pool for models beyond the budget
  uint32_t used, budget, used_over;

  __host__ __device__ static uint32_t pool_words() {
    uint32_t w = 2 * SymModel::words16(33);
    for (uint32_t k = 1; k < 32; ++k) w += SymModel::words16(1u << (k < 8 ? k : 8));
    return w;
  }
  __host__ __device__ void init(uint16_t* mem) { init(mem, 0xFFFFFFFFu, nullptr); }
  __host__ __device__ void init(uint16_t* fast, uint32_t fast_words, uint16_t* over) {
    pool = fast; budget = fast_words; overflow = over; used = 0; used_over = 0;
    kmod_live[0] = kmod_live[1] = false;
    cbit_live = false;
    for (int k = 0; k < 32; ++k) cmod_live[k] = false;
  }
  __host__ __device__ SymModel& alloc(SymModel& m, bool& live, uint32_t n) {
    if (!live) {
      const uint32_t w = SymModel::words16(n);
      if (used + w <= budget) {
        m.init(n, pool + used);
        used += w;
      } else {
        m.init(n, overflow + used_over);
        used_over += w;
      }
      live = true;
    }
    return m;
  }
  // IntegerCompressor.decompress(pred, ctx) with 32-bit wraparound.
  __host__ __device__ int32_t decompress(Decoder& d, int32_t pred, int ctx) {
    const uint32_t k = d.symbol(alloc(kmod[ctx], kmod_live[ctx], 33));
    int64_t c;
    if (k == 0) {
      if (!cbit_live) { cbit.init(); cbit_live = true; }
      c = d.bit(cbit);
    } else if (k < 32) {
      SymModel& m = alloc(cmod[k], cmod_live[k], 1u << (k < 8 ? k : 8));
      if (k <= 8) {
        c = d.symbol(m);
      } else {
        const uint32_t lowb = k - 8;
        const uint32_t hi = d.symbol(m);
        const uint32_t lo = d.raw_bits(lowb);
        c = ((int64_t)hi << lowb) | lo;
      }
      if (c >= (int64_t(1) << (k - 1))) c += 1;
      else c -= (int64_t(1) << k) - 1;
    } else {
      c = -(int64_t)0x80000000LL;
    }
    return (int32_t)(uint32_t)((int64_t)pred + c);
  }
};


// ---------------------------------------------------------------------
// Warp-cooperative flavour (device only).  The 32 lanes of a warp hold
// identical decoder state in registers and take identical branches; the
// adaptive symbol models' tables (shared memory) are rebuilt by all lanes
// together (counts halving, the prefix sum behind dist[], the decode lookup
// table by binary search), and the decode path's count update is written
// by lane 0.  Produces exactly the serial coder's tables.
struct WSymModel {
  uint32_t n, tot, cyc, left, tbits, tshift;
  uint16_t* dist;
  uint16_t* cnt;
  uint16_t* table;
  __device__ void init(uint32_t nsym, uint16_t* mem, int lane) {
    n = nsym;
    tbits = SymModel::table_bits(n);
    tshift = tbits ? 15 - tbits : 0;
    dist = mem;
    cnt = mem + n;
    table = tbits ? mem + 2 * n : nullptr;
    for (uint32_t k = lane; k < n; k += 32) cnt[k] = 1;
    __syncwarp();
    tot = 0;
    cyc = n;
    update(lane);
    cyc = left = (n + 6) >> 1;
  }
  __device__ void update(int lane) {
    tot += cyc;
    if (tot > 32768u) {
      uint32_t part = 0;
      for (uint32_t k = lane; k < n; k += 32) {
        const uint32_t c = (cnt[k] + 1u) >> 1;
        cnt[k] = (uint16_t)c;
        part += c;
      }
      tot = __reduce_add_sync(0xFFFFFFFFu, part);
      __syncwarp();
    }
    const uint32_t scale = 0x80000000u / tot;
    uint32_t carry = 0;
    for (uint32_t b = 0; b < n; b += 32) {
      const uint32_t k = b + lane;
      const uint32_t c = k < n ? cnt[k] : 0u;
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
      }
      if (k < n) dist[k] = (uint16_t)((scale * (carry + incl - c)) >> 16);
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    __syncwarp();
    if (tbits) {
      // table[j] = (first k with dist[k] >> tshift >= j) - 1, or n - 1;
      // table[0] = 0 (the serial fill loop's result)
      const uint32_t size = 1u << tbits;
      for (uint32_t j = lane; j <= size + 1; j += 32) {
        uint32_t v;
        if (j == 0) {
          v = 0;
        } else {
          uint32_t lo = 0, hi = n;  // first k in [0, n] with w_k >= j
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (((uint32_t)dist[mid] >> tshift) >= j) hi = mid; else lo = mid + 1;
          }
          v = lo < n ? lo - 1 : n - 1;
        }
        table[j] = (uint16_t)v;
      }
      __syncwarp();
    }
    cyc = min((5u * cyc) >> 2, (n + 6) << 3);
    left = cyc;
  }
};

__device__ __forceinline__ uint32_t wsymbol(Decoder& d, WSymModel& m, int lane) {
  uint32_t hi = d.length;
  uint32_t lo, s;
  const uint32_t unit = d.length >> 15;
  d.length = unit;
  if (m.tbits) {
    const uint32_t dv = d.value / unit;
    const uint32_t t = dv >> m.tshift;
    s = m.table[t];
    uint32_t n = (uint32_t)m.table[t + 1] + 1;
    while (n > s + 1) {
      const uint32_t k = (s + n) >> 1;
      if (m.dist[k] > dv) n = k; else s = k;
    }
    lo = m.dist[s] * unit;
    if (s != m.n - 1) hi = m.dist[s + 1] * unit;
  } else {
    lo = 0; s = 0;
    uint32_t n = m.n, k = n >> 1;
    do {
      const uint32_t z = unit * m.dist[k];
      if (z > d.value) { n = k; hi = z; } else { s = k; lo = z; }
      k = (s + n) >> 1;
    } while (k != s);
  }
  d.value -= lo;
  d.length = hi - lo;
  if (d.length < kMinLen) d.renorm();
  __syncwarp();  // every lane has read the model before it changes
  if (lane == 0) ++m.cnt[s];
  __syncwarp();
  if (--m.left == 0) m.update(lane);
  return s;
}

struct WChunkTableCoder {
  WSymModel kmod[2];
  bool kmod_live[2];
  BitModel cbit;
  bool cbit_live;
  WSymModel cmod[32];
  bool cmod_live[32];
  uint16_t* pool;
  uint16_t* overflow;
  uint32_t used, budget, used_over;
  int lane;

  __device__ void init(uint16_t* fast, uint32_t fast_words, uint16_t* over, int ln) {
    pool = fast; budget = fast_words; overflow = over; used = 0; used_over = 0; lane = ln;
    kmod_live[0] = kmod_live[1] = false;
    cbit_live = false;
    for (int k = 0; k < 32; ++k) cmod_live[k] = false;
  }
  __device__ WSymModel& alloc(WSymModel& m, bool& live, uint32_t n) {
    if (!live) {
      const uint32_t w = SymModel::words16(n);
      if (used + w <= budget) {
        m.init(n, pool + used, lane);
        used += w;
      } else {
        m.init(n, overflow + used_over, lane);
        used_over += w;
      }
      live = true;
    }
    return m;
  }
  __device__ int32_t decompress(Decoder& d, int32_t pred, int ctx) {
    const uint32_t k = wsymbol(d, alloc(kmod[ctx], kmod_live[ctx], 33), lane);
    int64_t c;
    if (k == 0) {
      if (!cbit_live) { cbit.init(); cbit_live = true; }
      c = d.bit(cbit);
    } else if (k < 32) {
      WSymModel& m = alloc(cmod[k], cmod_live[k], 1u << (k < 8 ? k : 8));
      if (k <= 8) {
        c = wsymbol(d, m, lane);
      } else {
        const uint32_t lowb = k - 8;
        const uint32_t hi = wsymbol(d, m, lane);
        const uint32_t lo = d.raw_bits(lowb);
        c = ((int64_t)hi << lowb) | lo;
      }
      if (c >= (int64_t(1) << (k - 1))) c += 1;
      else c -= (int64_t(1) << k) - 1;
    } else {
      c = -(int64_t)0x80000000LL;
    }
    return (int32_t)(uint32_t)((int64_t)pred + c);
  }
};

}  // namespace laz
}  // namespace ts
