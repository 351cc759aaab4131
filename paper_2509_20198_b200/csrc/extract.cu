// Subsystem (1): chunk tables + chunk-first-point extraction.
//
//   ts_chunk_counts / ts_chunk_decode  <- reader.py:141-226 (table decode,
//                                         LAS stride refs)
//   ts_extract_chunk_points            <- reader.py:239-283 read_chunk_points
//                                         + records.py:62-86 positions/colors
//                                         + patches.py:119-120 cell keys
//
// Layout: the file images of all tiles are concatenated in one device byte
// buffer (padded by >= 64 bytes so the 16-byte vector window loads never
// leave the allocation).  One CTA per tile extracts its chunk points: each
// thread gathers one first record with four aligned 16-byte loads, funnel
// shifts it to byte 0 in registers and decodes the fields there.
#include "laz_ac.cuh"
#include <algorithm>

#include "ts_common.cuh"

namespace ts {
namespace {

__device__ __forceinline__ int64_t load_i64_unaligned(const uint8_t* p) {
  uint64_t v = 0;
#pragma unroll
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return (int64_t)v;
}
__device__ __forceinline__ uint32_t load_u32_unaligned(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
         ((uint32_t)p[3] << 24);
}

__host__ __device__ __forceinline__ int rec_size(int fmt) {
  return fmt == 0 ? 20 : fmt == 1 ? 28 : fmt == 2 ? 26 : fmt == 3 ? 34 : -1;
}

// Validated chunk-table position of a LAZ tile, or a negative status.
// f addresses file offsets (the image pointer minus image_base).
__device__ int64_t table_position(const uint8_t* f, const ts_tile_desc& t,
                                  int32_t* status) {
  if (t.point_data_offset + 8 > t.file_size) {
    *status = TS_E_CORRUPT_TABLE;
    return -1;
  }
  int64_t pos = t.table_pos;
  if (pos < -1) {  // the pointer is in the image (reader.py:146-157)
    pos = load_i64_unaligned(f + t.point_data_offset);
    if (pos == -1) pos = load_i64_unaligned(f + t.file_size - 8);
  }
  const int64_t start = t.point_data_offset + 8;
  if (!(start <= pos && pos <= t.file_size - 8)) {
    *status = TS_E_CORRUPT_TABLE;
    return -1;
  }
  return pos;
}

__global__ void chunk_count_kernel(const uint8_t* __restrict__ bytes,
                                   const ts_tile_desc* __restrict__ tiles,
                                   int n_tiles, int64_t* n_chunks,
                                   int32_t* status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_tiles) return;
  const ts_tile_desc t = tiles[i];
  int32_t st = TS_OK;
  int64_t n = 0;
  if (rec_size(t.format) < 0) {
    st = TS_E_UNSUPPORTED_FORMAT;
  } else if (!t.compressed) {
    n = t.las_stride > 0 ? (t.point_count + t.las_stride - 1) / t.las_stride : 0;
  } else {
    const uint8_t* f = bytes + t.file_offset - t.image_base;
    const int64_t pos = table_position(f, t, &st);
    if (pos >= 0) {
      const uint32_t version = load_u32_unaligned(f + pos);
      if (version != 0) st = TS_E_CORRUPT_TABLE;
      else n = load_u32_unaligned(f + pos + 4);
    }
  }
  n_chunks[i] = n;
  status[i] = st;
}

constexpr uint32_t kDecodeSmemWords = 12 * 1024;  // 24 KB of models per tile (warp)
constexpr int kDecodeWarps = 8;                     // 192 KB shared per CTA

// One warp per tile: the table is decoded by the 32 lanes in lockstep
// (laz::WChunkTableCoder), which rebuild each adaptive model's tables
// together; lane 0 writes the results.
__global__ void chunk_decode_kernel(const uint8_t* __restrict__ bytes,
                                    const ts_tile_desc* __restrict__ tiles,
                                    int n_tiles,
                                    const int64_t* __restrict__ base,
                                    int64_t* __restrict__ offsets,
                                    int64_t* __restrict__ counts,
                                    int64_t* __restrict__ chunk_end,
                                    int32_t* status, uint16_t* scratch,
                                    uint32_t scratch_words) {
  extern __shared__ __align__(16) uint16_t s_pool[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * kDecodeWarps + wib;
  const int nwarps = gridDim.x * kDecodeWarps;
  laz::WChunkTableCoder coder;
  for (int i = gwarp; i < n_tiles; i += nwarps) {
    if (status[i] != TS_OK) continue;
    const ts_tile_desc t = tiles[i];
    const int64_t b0 = base[i];
    const int64_t n = base[i + 1] - b0;
    int32_t st = TS_OK;
    if (!t.compressed) {
      for (int64_t k = lane; k < n; k += 32) {
        const int64_t left = t.point_count - k * (int64_t)t.las_stride;
        offsets[b0 + k] = t.point_data_offset + k * t.las_stride * t.record_length;
        counts[b0 + k] = left < t.las_stride ? left : t.las_stride;
      }
      if (chunk_end && lane == 0)
        chunk_end[i] = t.point_data_offset + t.point_count * t.record_length;
      continue;
    }
    const uint8_t* f = bytes + t.file_offset - t.image_base;
    const int64_t pos = table_position(f, t, &st);
    const bool variable = t.chunk_size == 0xFFFFFFFFu;
    int64_t off = t.point_data_offset + 8;
    if (st == TS_OK && n > 0) {
      laz::Decoder dec;
      coder.init(s_pool + (size_t)wib * kDecodeSmemWords, kDecodeSmemWords,
                 scratch + (size_t)gwarp * scratch_words, lane);
      if (!dec.start(f, pos + 8, t.file_size)) st = TS_E_CORRUPT_TABLE;
      int32_t pc = 0, ps = 0;
      int64_t total = 0;
      int64_t left = t.point_count;
      for (int64_t k = 0; k < n && st == TS_OK; ++k) {
        int64_t cnt;
        if (variable) {
          pc = coder.decompress(dec, pc, 0);
          cnt = pc;
        } else {
          cnt = left < (int64_t)t.chunk_size ? left : (int64_t)t.chunk_size;
          left -= cnt;
        }
        ps = coder.decompress(dec, ps, 1);
        if (dec.desync) { st = TS_E_CORRUPT_TABLE; break; }
        if (ps <= 0) { st = TS_E_CORRUPT_TABLE; break; }
        if (lane == 0) {
          offsets[b0 + k] = off;
          counts[b0 + k] = cnt;
        }
        off += ps;
        total += cnt;
      }
      if (st == TS_OK && (total != t.point_count || off > pos))
        st = TS_E_CORRUPT_TABLE;
      if (chunk_end && lane == 0) chunk_end[i] = off;
    } else if (st == TS_OK && t.point_count != 0) {
      st = TS_E_CORRUPT_TABLE;  // zero chunks but points declared
    }
    if (lane == 0) status[i] = st;
    __syncwarp();
  }
}

// Loads the (<= 34 byte) record at p into 9 little-endian words w[0..8]
// with four aligned 16-byte loads and a register funnel shift.
__device__ __forceinline__ void load_record(const uint8_t* p, uint32_t w[9]) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uint4* q = reinterpret_cast<const uint4*>(a);
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 v = __ldg(q + i);
    r[4 * i] = v.x; r[4 * i + 1] = v.y; r[4 * i + 2] = v.z; r[4 * i + 3] = v.w;
  }
  const uint32_t sh = reinterpret_cast<uintptr_t>(p) & 15;
  const uint32_t wsh = sh >> 2, bsh = (sh & 3) * 8;
  uint32_t t[10];
#define TS_PICK(W)                                                   \
  _Pragma("unroll") for (int i = 0; i < 10; ++i) t[i] = r[i + (W)];
  switch (wsh) {
    case 0: TS_PICK(0) break;
    case 1: TS_PICK(1) break;
    case 2: TS_PICK(2) break;
    default: TS_PICK(3) break;
  }
#undef TS_PICK
#pragma unroll
  for (int i = 0; i < 9; ++i) w[i] = __funnelshift_r(t[i], t[i + 1], bsh);
}

__device__ __forceinline__ void record_rgb(const uint32_t w[9], int fmt,
                                           uint32_t& r, uint32_t& g,
                                           uint32_t& b) {
  if (fmt == 2) { r = w[5] & 0xFFFF; g = w[5] >> 16; b = w[6] & 0xFFFF; }
  else { r = w[7] & 0xFFFF; g = w[7] >> 16; b = w[8] & 0xFFFF; }
}

__global__ void __launch_bounds__(128)
extract_kernel(const uint8_t* __restrict__ bytes,
               const ts_tile_desc* __restrict__ tiles,
               const int64_t* __restrict__ base,
               const int64_t* __restrict__ offsets,
               uint8_t* __restrict__ records, double* __restrict__ xyz,
               float* __restrict__ rgb, int64_t* __restrict__ cell,
               int32_t* status) {
  __shared__ uint32_t stage[128 * 9];
  const int ti = blockIdx.x;
  const ts_tile_desc t = tiles[ti];
  const int64_t b0 = base[ti], n = base[ti + 1] - b0;
  const int fmt = t.format;
  const int rs = rec_size(fmt);
  const bool has_rgb = fmt == 2 || fmt == 3;
  const uint8_t* f = bytes + t.file_offset - t.image_base;
  if (status[ti] != TS_OK) return;
  if (rs < 0) { if (threadIdx.x == 0) status[ti] = TS_E_UNSUPPORTED_FORMAT; return; }
  // pass 1: bounds + the per-batch colour heuristic (records.py:81-85)
  int big = 0, err = 0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
    const int64_t off = offsets[b0 + c];
    if (off < 0 || off + t.record_length > t.file_size) { err = 1; continue; }
    if (has_rgb) {
      uint32_t w[9], r, g, b;
      load_record(f + off, w);
      record_rgb(w, fmt, r, g, b);
      big |= (r > 255) | (g > 255) | (b > 255);
    }
  }
  if (__syncthreads_or(err)) {
    if (threadIdx.x == 0) status[ti] = TS_E_OOB;
    return;
  }
  const int div16 = __syncthreads_or(big);
  const double div = div16 ? 65535.0 : 255.0;
  const double sx = t.scale[0], sy = t.scale[1], sz = t.scale[2];
  const double ox = t.offset[0], oy = t.offset[1], oz = t.offset[2];
  for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
    const int64_t c = c0 + threadIdx.x;
    const bool live = c < n;
    uint32_t w[9];
    if (live) {
      load_record(f + offsets[b0 + c], w);
      const int64_t id = b0 + c;
      const double x = dadd(dmul((double)(int32_t)w[0], sx), ox);
      const double y = dadd(dmul((double)(int32_t)w[1], sy), oy);
      const double z = dadd(dmul((double)(int32_t)w[2], sz), oz);
      if (xyz) { xyz[3 * id] = x; xyz[3 * id + 1] = y; xyz[3 * id + 2] = z; }
      if (cell) {
        cell[2 * id] = floor_i64(ddiv(x, kPatch));
        cell[2 * id + 1] = floor_i64(ddiv(y, kPatch));
      }
      if (rgb && has_rgb) {
        uint32_t r, g, b;
        record_rgb(w, fmt, r, g, b);
        rgb[3 * id] = __double2float_rn(ddiv((double)r, div));
        rgb[3 * id + 1] = __double2float_rn(ddiv((double)g, div));
        rgb[3 * id + 2] = __double2float_rn(ddiv((double)b, div));
      }
#pragma unroll
      for (int i = 0; i < 9; ++i) stage[threadIdx.x * 9 + i] = w[i];
    }
    if (records) {
      __syncthreads();
      // coalesced byte copy of this round's packed rows
      const int64_t rows = (n - c0) < (int64_t)blockDim.x ? (n - c0) : (int64_t)blockDim.x;
      const uint8_t* s8 = reinterpret_cast<const uint8_t*>(stage);
      uint8_t* dst = records + (b0 + c0) * rs;
      for (int64_t k = threadIdx.x; k < rows * rs; k += blockDim.x) {
        const int64_t row = k / rs, col = k - row * rs;
        dst[k] = s8[row * 36 + col];
      }
      __syncthreads();
    }
  }
}

// positions() over device records (records.py:62-67).
__global__ void positions_kernel(const uint8_t* __restrict__ rec, int64_t n,
                                 int rs, double sx, double sy, double sz,
                                 double ox, double oy, double oz,
                                 double* __restrict__ xyz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* p = rec + i * rs;
    const int32_t x = (int32_t)load_u32_unaligned(p);
    const int32_t y = (int32_t)load_u32_unaligned(p + 4);
    const int32_t z = (int32_t)load_u32_unaligned(p + 8);
    xyz[3 * i] = dadd(dmul((double)x, sx), ox);
    xyz[3 * i + 1] = dadd(dmul((double)y, sy), oy);
    xyz[3 * i + 2] = dadd(dmul((double)z, sz), oz);
  }
}

__device__ __forceinline__ void rgb_of(const uint8_t* p, uint32_t& r, uint32_t& g,
                                       uint32_t& b) {
  r = p[0] | (p[1] << 8);
  g = p[2] | (p[3] << 8);
  b = p[4] | (p[5] << 8);
}

__global__ void rgb_max_kernel(const uint8_t* __restrict__ rec, int64_t n, int rs,
                               int ro, int32_t* big) {
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r, g, b;
    rgb_of(rec + i * rs + ro, r, g, b);
    local |= (r > 255) | (g > 255) | (b > 255);
  }
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(big, 1);
}

__global__ void colors_kernel(const uint8_t* __restrict__ rec, int64_t n, int rs,
                              int ro, const int32_t* big, float* __restrict__ rgb) {
  const double div = *big ? 65535.0 : 255.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r, g, b;
    rgb_of(rec + i * rs + ro, r, g, b);
    rgb[3 * i] = __double2float_rn(ddiv((double)r, div));
    rgb[3 * i + 1] = __double2float_rn(ddiv((double)g, div));
    rgb[3 * i + 2] = __double2float_rn(ddiv((double)b, div));
  }
}

constexpr int kDecodeThreads = 148 * kDecodeWarps;  // decoding warps

uint32_t decode_pool_words() {
  // mirror of ChunkTableCoder::pool_words() on the host
  auto words16 = [](uint32_t n) {
    uint32_t tb = 0;
    if (n > 16) { tb = 3; while (n > (1u << (tb + 2))) ++tb; }
    return 2 * n + (tb ? (1u << tb) + 2 : 0);
  };
  uint32_t w = 2 * words16(33);
  for (uint32_t k = 1; k < 32; ++k) w += words16(1u << (k < 8 ? k : 8));
  return (w + 7) & ~7u;  // 16-byte aligned per thread
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" int ts_record_size(int format) { return rec_size(format); }

extern "C" int ts_chunk_counts(const uint8_t* d_bytes, const ts_tile_desc* d_tiles,
                               int n_tiles, int64_t* d_n_chunks,
                               int32_t* d_status, void* stream) {
  if (n_tiles <= 0) return n_tiles == 0 ? TS_OK : TS_E_INVALID;
  ts::count_launch(), chunk_count_kernel<<<ceil_div(n_tiles, 128), 128, 0, as_stream(stream)>>>(
      d_bytes, d_tiles, n_tiles, d_n_chunks, d_status);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" size_t ts_chunk_decode_scratch(int n_tiles) {
  const int threads = n_tiles < kDecodeThreads ? n_tiles : kDecodeThreads;
  return (size_t)(threads > 0 ? threads : 1) * decode_pool_words() * sizeof(uint16_t);
}

extern "C" int ts_chunk_decode(const uint8_t* d_bytes, const ts_tile_desc* d_tiles,
                               int n_tiles, const int64_t* d_chunk_base,
                               int64_t* d_chunk_offset, int64_t* d_chunk_points,
                               int64_t* d_chunk_end, int32_t* d_status, void* d_scratch,
                               void* stream) {
  if (n_tiles <= 0) return n_tiles == 0 ? TS_OK : TS_E_INVALID;
  const int threads = n_tiles < kDecodeThreads ? n_tiles : kDecodeThreads;  // warps
  const int block = 32 * kDecodeWarps;
  const size_t smem = (size_t)kDecodeWarps * kDecodeSmemWords * sizeof(uint16_t);
  {  // per call: the attribute is per device (one process may drive several)
    TS_CUDA_TRY(cudaFuncSetAttribute(chunk_decode_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  ts::count_launch(), chunk_decode_kernel<<<ceil_div(threads, kDecodeWarps), block, smem, as_stream(stream)>>>(
      d_bytes, d_tiles, n_tiles, d_chunk_base, d_chunk_offset, d_chunk_points,
      d_chunk_end, d_status, reinterpret_cast<uint16_t*>(d_scratch), decode_pool_words());
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" int ts_extract_chunk_points(const uint8_t* d_bytes,
                                       const ts_tile_desc* d_tiles, int n_tiles,
                                       const int64_t* d_chunk_base,
                                       const int64_t* d_chunk_offset,
                                       uint8_t* d_records, double* d_xyz,
                                       float* d_rgb, int64_t* d_cell,
                                       int32_t* d_status, void* stream) {
  if (n_tiles <= 0) return n_tiles == 0 ? TS_OK : TS_E_INVALID;
  ts::count_launch(), extract_kernel<<<n_tiles, 128, 0, as_stream(stream)>>>(
      d_bytes, d_tiles, d_chunk_base, d_chunk_offset, d_records, d_xyz, d_rgb,
      d_cell, d_status);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" int ts_positions(const uint8_t* d_records, int64_t n, int record_stride,
                            const double scale[3], const double offset[3],
                            double* d_xyz, void* stream) {
  if (record_stride < 12) return TS_E_INVALID;
  if (n <= 0) return TS_OK;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 148 * 8);
  ts::count_launch(), positions_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      d_records, n, record_stride, scale[0], scale[1], scale[2], offset[0], offset[1],
      offset[2], d_xyz);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" int ts_colors(const uint8_t* d_records, int64_t n, int record_stride,
                         int rgb_offset, float* d_rgb, int32_t* d_scratch, void* stream) {
  if (rgb_offset < 0 || rgb_offset + 6 > record_stride) return TS_E_INVALID;
  cudaStream_t s = as_stream(stream);
  TS_CUDA_TRY(cudaMemsetAsync(d_scratch, 0, sizeof(int32_t), s));
  if (n <= 0) return TS_OK;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 148 * 8);
  ts::count_launch(), rgb_max_kernel<<<grid, 256, 0, s>>>(d_records, n, record_stride, rgb_offset, d_scratch);
  ts::count_launch(), colors_kernel<<<grid, 256, 0, s>>>(d_records, n, record_stride, rgb_offset, d_scratch,
                                     d_rgb);
  TS_LAUNCH_CHECK();
  return TS_OK;
}
