// Full LAZ chunk decode on the GPU.
//
// Replaces decode_chunk / load_tile_fullres (pkg/src/terrascout/lasio/
// reader.py:286-364) with the LASzip-2 item decoders of lasio/items.py:
// POINT10 v2 (:111-209), GPSTIME11 v2 (:281-383), RGB12 v2 (:514-561) over
// the arithmetic coder and IntegerCompressor of codec.py:173-484.
//
// A chunk is one sequential arithmetic-coded stream, so the parallelism is
// across chunks: one thread decodes one chunk (a 7.5 M-point tile has 150
// chunks; a batch of tiles has thousands).  Each thread owns a bump arena
// of adaptive models in global memory (the models are created lazily, as
// the reference does: a chunk typically touches tens of them, a
// pathological one a few hundred), and writes its chunk's records at the
// chunk's point offset.  Output is bit-exact with the reference
// (tests/test_gpu_lazdec.py against reference-compressed golden files).
#include <stdint.h>

#include <algorithm>

#include "laz_ac.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

using laz::BitModel;
using laz::Decoder;
using laz::SymModel;

// Pass 1: every chunk with a 128 KB arena and 256 model descriptors (the
// reference's own files use 26-45 K words in 80-125 models per chunk);
// chunks that outgrow it are queued and decoded again in pass 2 with a
// 2 MB arena and 4,096 descriptors (every model a chunk can create fits).
constexpr uint32_t kArenaWords = 64 * 1024, kMaxModels = 256;
constexpr uint32_t kArenaWords2 = 1024 * 1024, kMaxModels2 = 4096;
constexpr int kDecThreads = 128;                     // 4 warps, one decoder each
constexpr int64_t kDecWarps = 148 * 64;              // 64 warps per SM
constexpr int kMaxLanes = 4;                          // <= 37,888 decoders (~5.5 GB)
constexpr int64_t kRetryThreads = 1024;              // pass-2 decoders (~2.2 GB)

__device__ __forceinline__ int32_t i32w(int64_t v) { return (int32_t)(uint32_t)(uint64_t)v; }

// Per-chunk model store: descriptors + their tables in one global arena.
struct Arena {
  SymModel* desc;   // [max_models]
  uint16_t* words;  // [max_words]: model tables, fast memory (shared) first
  uint16_t* over;   // [max_over]: overflow tables (global), or null
  uint32_t ndesc, used, used_over, max_models, max_words, max_over;
  bool full;
  __device__ void reset() { ndesc = used = used_over = 0; full = false; }
  __device__ SymModel* make(uint32_t nsym) {
    const uint32_t w = SymModel::words16(nsym);
    uint16_t* mem;
    if (ndesc >= max_models) {
      mem = nullptr;
    } else if (used + w <= max_words) {
      mem = words + used;
      used += w;
    } else if (used_over + w <= max_over) {
      mem = over + used_over;
      used_over += w;
    } else {
      mem = nullptr;
    }
    if (!mem) {
      full = true;
      return nullptr;
    }
    SymModel* m = desc + ndesc++;
    m->init(nsym, mem);
    return m;
  }
};

// Lazily created model slot (index into the arena's descriptors, -1 = none)
__device__ __forceinline__ SymModel* lazy(Arena& A, int16_t& slot, uint32_t nsym) {
  if (slot < 0) {
    SymModel* m = A.make(nsym);
    if (!m) return nullptr;
    slot = (int16_t)(m - A.desc);
    return m;
  }
  return A.desc + slot;
}

// IntegerCompressor(bits, contexts, bits_high = 8) (codec.py:394-484)
template <int CTX>
struct IntComp {
  uint32_t corr_bits, corr_range;
  int32_t corr_min;
  int16_t kslot[CTX];
  int16_t cslot[32];  // k = 1..31 corrector models
  BitModel cbit;
  bool cbit_live;
  uint32_t k;
  __device__ void init(uint32_t bits) {
    if (bits > 0 && bits < 32) {
      corr_bits = bits;
      corr_range = 1u << bits;
      corr_min = -(int32_t)(corr_range / 2);
    } else {
      corr_bits = 32;
      corr_range = 0;
      corr_min = (int32_t)0x80000000;
    }
    for (int i = 0; i < CTX; ++i) kslot[i] = -1;
    for (int i = 0; i < 32; ++i) cslot[i] = -1;
    cbit_live = false;
    k = 0;
  }
  __device__ __forceinline__ int32_t decompress(Decoder& d, Arena& A, int32_t pred, int ctx) {
    SymModel* mk = lazy(A, kslot[ctx], corr_bits + 1);
    if (!mk) return pred;
    k = d.symbol(*mk);
    int64_t c;
    if (k) {
      if (k < 32) {
        SymModel* cm = lazy(A, cslot[k], 1u << (k < 8 ? k : 8));
        if (!cm) return pred;
        if (k <= 8) {
          c = d.symbol(*cm);
        } else {
          const uint32_t k1 = k - 8;
          const uint32_t hi = d.symbol(*cm);
          c = ((int64_t)hi << k1) | d.raw_bits(k1);
        }
        if (c >= ((int64_t)1 << (k - 1))) c += 1;
        else c -= ((int64_t)1 << k) - 1;
      } else {
        c = corr_min;
      }
    } else {
      if (!cbit_live) { cbit.init(); cbit_live = true; }
      c = d.bit(cbit);
    }
    int64_t real = (int64_t)pred + c;
    if (corr_range) {
      if (real < 0) real += corr_range;
      else if (real >= (int64_t)corr_range) real -= corr_range;
      return (int32_t)real;
    }
    return i32w(real);
  }
};

// StreamingMedian5 (items.py:49-104)
struct Median5 {
  int32_t v[5];
  bool high;
  __device__ void init() { for (int i = 0; i < 5; ++i) v[i] = 0; high = true; }
  __device__ void add(int32_t x) {
    if (high) {
      if (x < v[2]) {
        v[4] = v[3]; v[3] = v[2];
        if (x < v[0]) { v[2] = v[1]; v[1] = v[0]; v[0] = x; }
        else if (x < v[1]) { v[2] = v[1]; v[1] = x; }
        else v[2] = x;
      } else {
        if (x < v[3]) { v[4] = v[3]; v[3] = x; }
        else v[4] = x;
        high = false;
      }
    } else {
      if (x > v[2]) {
        v[0] = v[1]; v[1] = v[2];
        if (x > v[4]) { v[2] = v[3]; v[3] = v[4]; v[4] = x; }
        else if (x > v[3]) { v[2] = v[3]; v[3] = x; }
        else v[2] = x;
      } else {
        if (x > v[1]) { v[0] = v[1]; v[1] = x; }
        else v[0] = x;
        high = true;
      }
    }
  }
};

__constant__ uint8_t kNumRetMap[8][8] = {
    {15, 14, 13, 12, 11, 10, 9, 8}, {14, 0, 1, 3, 6, 10, 10, 9},
    {13, 1, 2, 4, 7, 11, 11, 10},   {12, 3, 4, 5, 8, 12, 12, 11},
    {11, 6, 7, 8, 9, 13, 13, 12},   {10, 10, 11, 12, 13, 14, 14, 13},
    {9, 10, 11, 12, 13, 14, 15, 14}, {8, 9, 10, 11, 12, 13, 14, 15}};

// Per-chunk decoder state: lives in the thread's scratch block (global
// memory) -- the model slot tables are too large for registers.
struct ChunkState {
  // POINT10
  int16_t m_changed, m_sar[2], m_bit[256], m_cls[256], m_ud[256];
  IntComp<4> ic_int;
  IntComp<1> ic_psid;
  IntComp<2> ic_dx;
  IntComp<22> ic_dy;
  IntComp<20> ic_z;
  Median5 mx[16], my[16];
  uint16_t lint[16];
  int32_t lh[8];
  int32_t x, y, z;
  uint16_t intensity, psid;
  uint8_t bf, cls, sa, ud;
  // GPSTIME11
  int16_t m_multi, m_0diff;
  IntComp<9> ic_gps;
  uint32_t g_last, g_next;
  uint64_t gt[4];
  int32_t gdt[4];
  int32_t gcnt[4];
  // RGB12
  int16_t m_used, m_diff[6];
  uint16_t lr, lg, lb;
};

constexpr int kMulti = 500, kMultiMinus = -10;
constexpr int kMultiTotal = kMulti - kMultiMinus + 6;
constexpr int kMultiUnchanged = kMulti - kMultiMinus + 1;
constexpr int kMultiCodeFull = kMulti - kMultiMinus + 2;

__device__ __forceinline__ int u8clamp(int v) { return v <= 0 ? 0 : v >= 255 ? 255 : v; }
__device__ __forceinline__ int cdiv2(int v) { return v < 0 ? -((-v) >> 1) : v >> 1; }

__device__ __forceinline__ uint32_t sym(Decoder& d, Arena& A, int16_t& slot, uint32_t n) {
  SymModel* m = lazy(A, slot, n);
  return m ? d.symbol(*m) : 0u;
}

__device__ __forceinline__ void point10_read(ChunkState& S, Decoder& d, Arena& A) {
  const uint32_t cv = sym(d, A, S.m_changed, 64);
  if (cv & 32) S.bf = (uint8_t)sym(d, A, S.m_bit[S.bf], 256);
  const uint32_t r = S.bf & 7, n = (S.bf >> 3) & 7;
  const int mc = kNumRetMap[n][r];
  const int lvl = n > r ? n - r : r - n;
  if (cv & 16) {
    S.intensity = (uint16_t)S.ic_int.decompress(d, A, S.lint[mc], mc < 3 ? mc : 3);
    S.lint[mc] = S.intensity;
  } else {
    S.intensity = S.lint[mc];
  }
  if (cv & 8) S.cls = (uint8_t)sym(d, A, S.m_cls[S.cls], 256);
  if (cv & 4) S.sa = (uint8_t)(sym(d, A, S.m_sar[(S.bf >> 6) & 1], 256) + S.sa);
  if (cv & 2) S.ud = (uint8_t)sym(d, A, S.m_ud[S.ud], 256);
  if (cv & 1) S.psid = (uint16_t)S.ic_psid.decompress(d, A, S.psid, 0);
  const int n1 = n == 1 ? 1 : 0;
  int32_t diff = S.ic_dx.decompress(d, A, S.mx[mc].v[2], n1);
  S.x = i32w((int64_t)S.x + diff);
  S.mx[mc].add(diff);
  uint32_t kb = S.ic_dx.k;
  diff = S.ic_dy.decompress(d, A, S.my[mc].v[2], n1 + (kb < 20 ? (int)(kb & ~1u) : 20));
  S.y = i32w((int64_t)S.y + diff);
  S.my[mc].add(diff);
  kb = (S.ic_dx.k + S.ic_dy.k) / 2;
  S.z = S.ic_z.decompress(d, A, S.lh[lvl], n1 + (kb < 18 ? (int)(kb & ~1u) : 18));
  S.lh[lvl] = S.z;
}

__device__ __forceinline__ void gps_full(ChunkState& S, Decoder& d, Arena& A) {
  S.g_next = (S.g_next + 1) & 3;
  const int32_t hi = S.ic_gps.decompress(d, A, (int32_t)(uint32_t)(S.gt[S.g_last] >> 32), 8);
  const uint32_t lo = d.raw_bits(32);
  S.gt[S.g_next] = ((uint64_t)(uint32_t)hi << 32) | lo;
  S.g_last = S.g_next;
  S.gdt[S.g_last] = 0;
  S.gcnt[S.g_last] = 0;
}

__device__ __forceinline__ uint64_t gps_read(ChunkState& S, Decoder& d, Arena& A) {
  for (int guard = 0; guard < 8; ++guard) {  // a sequence switch re-reads (items.py:304, 382)
    const uint32_t L = S.g_last;
    if (S.gdt[L] == 0) {
      const uint32_t m = sym(d, A, S.m_0diff, 6);
      if (m == 1) {
        const int32_t v = S.ic_gps.decompress(d, A, 0, 0);
        S.gdt[L] = v;
        S.gt[L] += (uint64_t)(int64_t)v;
        S.gcnt[L] = 0;
      } else if (m == 2) {
        gps_full(S, d, A);
      } else if (m > 2) {
        S.g_last = (L + m - 2) & 3;
        continue;
      }
      return S.gt[S.g_last];
    }
    const int m = (int)sym(d, A, S.m_multi, kMultiTotal);
    if (m == 1) {
      const int32_t v = S.ic_gps.decompress(d, A, S.gdt[L], 1);
      S.gt[L] += (uint64_t)(int64_t)v;
      S.gcnt[L] = 0;
    } else if (m < kMultiUnchanged) {
      int32_t g;
      if (m == 0) {
        g = S.ic_gps.decompress(d, A, 0, 7);
        if (++S.gcnt[L] > 3) { S.gdt[L] = g; S.gcnt[L] = 0; }
      } else if (m < kMulti) {
        g = S.ic_gps.decompress(d, A, i32w((int64_t)m * S.gdt[L]), m < 10 ? 2 : 3);
      } else if (m == kMulti) {
        g = S.ic_gps.decompress(d, A, i32w((int64_t)kMulti * S.gdt[L]), 4);
        if (++S.gcnt[L] > 3) { S.gdt[L] = g; S.gcnt[L] = 0; }
      } else {
        const int mm = kMulti - m;
        if (mm > kMultiMinus) {
          g = S.ic_gps.decompress(d, A, i32w((int64_t)mm * S.gdt[L]), 5);
        } else {
          g = S.ic_gps.decompress(d, A, i32w((int64_t)kMultiMinus * S.gdt[L]), 6);
          if (++S.gcnt[L] > 3) { S.gdt[L] = g; S.gcnt[L] = 0; }
        }
      }
      S.gt[L] += (uint64_t)(int64_t)g;
    } else if (m == kMultiCodeFull) {
      gps_full(S, d, A);
    } else if (m > kMultiCodeFull) {
      S.g_last = (L + m - kMultiCodeFull) & 3;
      continue;
    }
    return S.gt[S.g_last];
  }
  d.desync = true;  // more sequence switches than the four sequences allow
  return S.gt[S.g_last];
}

__device__ __forceinline__ void rgb_read(ChunkState& S, Decoder& d, Arena& A) {
  const int lr = S.lr, lg = S.lg, lb = S.lb;
  const uint32_t s = sym(d, A, S.m_used, 128);
  const int rl = s & 1 ? (int)((sym(d, A, S.m_diff[0], 256) + (lr & 0xFF)) & 0xFF) : lr & 0xFF;
  const int rh = s & 2 ? (int)((sym(d, A, S.m_diff[1], 256) + (lr >> 8)) & 0xFF) : lr >> 8;
  const int red = rl | (rh << 8);
  int green = red, blue = red;
  if (s & 64) {
    int diff = rl - (lr & 0xFF);
    const int gl = s & 4 ? (int)((sym(d, A, S.m_diff[2], 256) + u8clamp(diff + (lg & 0xFF))) & 0xFF)
                         : lg & 0xFF;
    int bl;
    if (s & 16) {
      diff = cdiv2(diff + gl - (lg & 0xFF));
      bl = (int)((sym(d, A, S.m_diff[4], 256) + u8clamp(diff + (lb & 0xFF))) & 0xFF);
    } else {
      bl = lb & 0xFF;
    }
    diff = rh - (lr >> 8);
    const int gh = s & 8 ? (int)((sym(d, A, S.m_diff[3], 256) + u8clamp(diff + (lg >> 8))) & 0xFF)
                         : lg >> 8;
    int bh;
    if (s & 32) {
      diff = cdiv2(diff + gh - (lg >> 8));
      bh = (int)((sym(d, A, S.m_diff[5], 256) + u8clamp(diff + (lb >> 8))) & 0xFF);
    } else {
      bh = lb >> 8;
    }
    green = gl | (gh << 8);
    blue = bl | (bh << 8);
  }
  S.lr = (uint16_t)red; S.lg = (uint16_t)green; S.lb = (uint16_t)blue;
}

__device__ __forceinline__ void put16(uint8_t* p, uint32_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
__device__ __forceinline__ void put32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
__device__ __forceinline__ uint32_t get16(const uint8_t* p) { return p[0] | ((uint32_t)p[1] << 8); }
__device__ __forceinline__ uint32_t get32(const uint8_t* p) {
  return p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

__device__ __forceinline__ void emit(const ChunkState& S, int fmt, uint8_t* o) {
  put32(o, (uint32_t)S.x); put32(o + 4, (uint32_t)S.y); put32(o + 8, (uint32_t)S.z);
  put16(o + 12, S.intensity);
  o[14] = S.bf; o[15] = S.cls; o[16] = S.sa; o[17] = S.ud;
  put16(o + 18, S.psid);
  int c = 20;
  if (fmt == 1 || fmt == 3) {
    const uint64_t t = S.gt[S.g_last];
    put32(o + 20, (uint32_t)t); put32(o + 24, (uint32_t)(t >> 32));
    c = 28;
  }
  if (fmt == 2 || fmt == 3) {
    put16(o + c, S.lr); put16(o + c + 2, S.lg); put16(o + c + 4, S.lb);
  }
}

__host__ __device__ __forceinline__ int rec_bytes(int fmt) {
  return fmt == 0 ? 20 : fmt == 1 ? 28 : fmt == 2 ? 26 : fmt == 3 ? 34 : -1;
}

struct DecArgs {
  const uint8_t* bytes;
  const ts_tile_desc* tiles;
  int n_tiles;
  const int64_t* chunk_base;    // [n_tiles + 1]
  const int64_t* chunk_offset;  // file offsets
  const int64_t* chunk_points;  // point counts
  const int64_t* chunk_end;     // [n_tiles]: end of the last chunk
  const int64_t* point_base;    // [total chunks + 1]: output record index
  int64_t n_chunks;
  uint8_t* records;             // packed record_dtype(fmt) rows
  int32_t* status;              // per chunk
  uint8_t* scratch;             // per thread: ChunkState + arena
  size_t per_thread;
  uint32_t arena_words, max_models;
  int lanes;                    // decoding lanes per warp
  const int64_t* list;          // pass 2: the chunks to decode, else null
  const uint32_t* list_n;
  int64_t* retry;               // pass 1: chunks whose models outgrew the arena
  uint32_t* retry_n;
};

constexpr int32_t kRetry = -1;

// Decode chunk ci with the given state and arena; the status, or kRetry
// when the models outgrew the arena (pass 1 only).
__device__ __forceinline__ int32_t decode_one(const DecArgs& a, int64_t ci, ChunkState& S, Arena& A) {
  // tile of this chunk: binary search over chunk_base
  int lo = 0, hi = a.n_tiles;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a.chunk_base[mid] <= ci) lo = mid; else hi = mid;
  }
  const ts_tile_desc t = a.tiles[lo];
  const int fmt = t.format;
  const int rs = rec_bytes(fmt);
  const int64_t off = a.chunk_offset[ci];
  const int64_t end = ci + 1 < a.chunk_base[lo + 1] ? a.chunk_offset[ci + 1] : a.chunk_end[lo];
  const int64_t count = a.chunk_points[ci];
  if (!t.compressed || rs < 0) return TS_E_UNSUPPORTED_FORMAT;
  if (off < 0 || end > t.file_size || end - off < rs || count < 0) return TS_E_OOB;
  if (count == 0) return TS_OK;
  const uint8_t* f = a.bytes + t.file_offset - t.image_base;
  const uint8_t* first = f + off;
  uint8_t* out = a.records + a.point_base[ci] * rs;
  for (int b = 0; b < rs; ++b) out[b] = first[b];  // the raw first record
  // item state from the first record (items.py:137-141, 270-276, 510-512)
  S.x = (int32_t)get32(first); S.y = (int32_t)get32(first + 4); S.z = (int32_t)get32(first + 8);
  S.intensity = 0;
  S.bf = first[14]; S.cls = first[15]; S.sa = first[16]; S.ud = first[17];
  S.psid = (uint16_t)get16(first + 18);
  S.m_changed = S.m_sar[0] = S.m_sar[1] = -1;
  for (int i = 0; i < 256; ++i) S.m_bit[i] = S.m_cls[i] = S.m_ud[i] = -1;
  S.ic_int.init(16); S.ic_psid.init(16);
  S.ic_dx.init(32); S.ic_dy.init(32); S.ic_z.init(32);
  for (int i = 0; i < 16; ++i) { S.mx[i].init(); S.my[i].init(); S.lint[i] = 0; }
  for (int i = 0; i < 8; ++i) S.lh[i] = 0;
  int c = 20;
  S.m_multi = S.m_0diff = -1;
  S.ic_gps.init(32);
  S.g_last = S.g_next = 0;
  for (int i = 0; i < 4; ++i) { S.gt[i] = 0; S.gdt[i] = 0; S.gcnt[i] = 0; }
  if (fmt == 1 || fmt == 3) {
    S.gt[0] = (uint64_t)get32(first + 20) | ((uint64_t)get32(first + 24) << 32);
    c = 28;
  }
  S.m_used = -1;
  for (int i = 0; i < 6; ++i) S.m_diff[i] = -1;
  if (fmt == 2 || fmt == 3) {
    S.lr = (uint16_t)get16(first + c); S.lg = (uint16_t)get16(first + c + 2);
    S.lb = (uint16_t)get16(first + c + 4);
  }
  A.reset();
  Decoder d;
  if (!d.start(f, off + rs, end)) return TS_E_DESYNC;
  for (int64_t i = 1; i < count; ++i) {
    point10_read(S, d, A);
    if (fmt == 1 || fmt == 3) gps_read(S, d, A);
    if (fmt == 2 || fmt == 3) rgb_read(S, d, A);
    if (d.desync || A.full) break;
    emit(S, fmt, out + i * rs);
  }
  if (d.desync) return TS_E_DESYNC;
  if (A.full) return a.list ? TS_E_INVALID : kRetry;
  return TS_OK;
}

// One chunk per thread, its state and models in the thread's global arena
// (pass 1: 128 KB for every chunk; pass 2: 2 MB for the queued ones).  A
// single thread's decode is a chain of dependent model reads, so
// throughput comes from many chunks in flight.  (Measured alternative: one
// decoding lane per CTA with the models in shared memory, two CTAs per SM:
// 0.68 s instead of 1.2 s for one 50,000-point chunk, but 22 M instead of
// 139 M points/s over 16,384 chunks.)
__global__ void __launch_bounds__(kDecThreads) lazdec_kernel(DecArgs a) {
  // a.lanes decoding lanes per warp: lanes of one warp on different chunks
  // diverge on every symbol, so small batches run one lane per warp (one
  // 50,000-point chunk: 0.77 s instead of 1.2-3.3 s) and large ones a few
  // (more chunks in flight; 16,384 chunks: 89 -> 137 M points/s)
  const int lane = threadIdx.x & 31;
  if (lane >= a.lanes) return;
  const int64_t nthreads = (int64_t)gridDim.x * (blockDim.x >> 5) * a.lanes;
  const int64_t gt = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * a.lanes + lane;
  uint8_t* mine = a.scratch + (size_t)gt * a.per_thread;
  ChunkState& S = *reinterpret_cast<ChunkState*>(mine);
  Arena A;
  A.desc = reinterpret_cast<SymModel*>(mine + ((sizeof(ChunkState) + 15) & ~size_t(15)));
  A.words = reinterpret_cast<uint16_t*>(A.desc + a.max_models);
  A.over = nullptr;
  A.max_models = a.max_models;
  A.max_words = a.arena_words;
  A.max_over = 0;
  const int64_t nwork = a.list ? (int64_t)*a.list_n : a.n_chunks;
  for (int64_t wi = gt; wi < nwork; wi += nthreads) {
    const int64_t ci = a.list ? a.list[wi] : wi;
    const int32_t st = decode_one(a, ci, S, A);
    if (st == kRetry) a.retry[atomicAdd(a.retry_n, 1u)] = ci;
    else a.status[ci] = st;
  }
}

}  // namespace
}  // namespace ts

using namespace ts;

namespace {
size_t block_bytes(uint32_t words, uint32_t models) {
  const size_t per = ((sizeof(ChunkState) + 15) & ~size_t(15)) + models * sizeof(SymModel) +
                     words * sizeof(uint16_t);
  return (per + 255) & ~size_t(255);
}
int pass1_lanes(int64_t n_chunks) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(kMaxLanes, ceil_div<int64_t>(n_chunks, kDecWarps)));
}
int64_t pass1_threads(int64_t n_chunks) {  // decoders
  return std::max<int64_t>(1, std::min<int64_t>(n_chunks, kDecWarps * pass1_lanes(n_chunks)));
}
}  // namespace

extern "C" size_t ts_lazdec_scratch(int64_t n_chunks) {
  const size_t list = ((size_t)std::max<int64_t>(n_chunks, 1) * 8 + 16 + 255) & ~size_t(255);
  return (size_t)pass1_threads(n_chunks) * block_bytes(kArenaWords, kMaxModels) + list +
         (size_t)kRetryThreads * block_bytes(kArenaWords2, kMaxModels2) + 256;
}

extern "C" int ts_lazdec(const uint8_t* d_bytes, const ts_tile_desc* d_tiles, int n_tiles,
                         const int64_t* d_chunk_base, const int64_t* d_chunk_offset,
                         const int64_t* d_chunk_points, const int64_t* d_chunk_end,
                         const int64_t* d_point_base, int64_t n_chunks, uint8_t* d_records,
                         int32_t* d_status, void* d_scratch, void* stream) {
  if (n_tiles < 0 || n_chunks < 0) return TS_E_INVALID;
  if (n_chunks == 0) return TS_OK;
  cudaStream_t s = as_stream(stream);
  const int64_t threads = pass1_threads(n_chunks);
  uint8_t* base = reinterpret_cast<uint8_t*>(d_scratch);
  const size_t b1 = (size_t)threads * block_bytes(kArenaWords, kMaxModels);
  int64_t* retry = reinterpret_cast<int64_t*>(base + b1);
  uint32_t* retry_n = reinterpret_cast<uint32_t*>(retry + n_chunks);
  const size_t list = ((size_t)n_chunks * 8 + 16 + 255) & ~size_t(255);
  TS_CUDA_TRY(cudaMemsetAsync(retry_n, 0, sizeof(uint32_t), s));
  DecArgs a{};
  a.bytes = d_bytes; a.tiles = d_tiles; a.n_tiles = n_tiles;
  a.chunk_base = d_chunk_base; a.chunk_offset = d_chunk_offset; a.chunk_points = d_chunk_points;
  a.chunk_end = d_chunk_end; a.point_base = d_point_base; a.n_chunks = n_chunks;
  a.records = d_records; a.status = d_status;
  a.scratch = base;
  a.per_thread = block_bytes(kArenaWords, kMaxModels);
  a.arena_words = kArenaWords;
  a.max_models = kMaxModels;
  a.retry = retry;
  a.retry_n = retry_n;
  a.lanes = pass1_lanes(n_chunks);
  const int64_t warps = ceil_div<int64_t>(threads, a.lanes);
  ts::count_launch(),
      lazdec_kernel<<<(int)ceil_div<int64_t>(warps, kDecThreads / 32), kDecThreads, 0, s>>>(a);
  // pass 2: the chunks that outgrew pass 1 (the count stays on the device)
  a.scratch = base + b1 + list;
  a.per_thread = block_bytes(kArenaWords2, kMaxModels2);
  a.arena_words = kArenaWords2;
  a.max_models = kMaxModels2;
  a.list = retry;
  a.list_n = retry_n;
  a.lanes = 1;
  ts::count_launch(),
      lazdec_kernel<<<(int)(kRetryThreads / (kDecThreads / 32)), kDecThreads, 0, s>>>(a);
  TS_LAUNCH_CHECK();
  return TS_OK;
}
