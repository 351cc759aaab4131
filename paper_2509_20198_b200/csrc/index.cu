// Subsystem (2a): chunk-point index + per-patch gather/normalise.
//
//   ts_index_build   <- ChunkPointIndex.add_points / query order
//                       (patches.py:99-153): stable sort of point ids by
//                       dense cell id (ci-major, like lexsort((cj, ci))),
//                       so a cell lists its points in insertion order.
//   ts_gather_count  <- gather_and_normalize pass 1 (patches.py:163-172)
//   ts_gather_fill   <- gather_and_normalize (patches.py:163-177): ordered
//                       warp compaction over the 3x3 cells, provisional
//                       c_z = z of the first d^2 argmin, IEEE fp64 patch-space
//                       transform.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "ts_common.cuh"

namespace ts {
namespace {

__global__ void cell_key_kernel(const int64_t* __restrict__ cell, int64_t n,
                                int64_t ci0, int64_t cj0, int64_t nci,
                                int64_t ncj, uint32_t* __restrict__ keys,
                                int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ci = cell[2 * i] - ci0, cj = cell[2 * i + 1] - cj0;
    const bool ok = ci >= 0 && ci < nci && cj >= 0 && cj < ncj;
    keys[i] = ok ? (uint32_t)(ci * ncj + cj) : 0xFFFFFFFFu;
    ids[i] = (int32_t)i;
  }
}

__global__ void cell_range_kernel(const uint32_t* __restrict__ keys, int64_t n,
                                  int32_t* __restrict__ start,
                                  int32_t* __restrict__ end) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    if (k == 0xFFFFFFFFu) continue;
    if (i == 0 || keys[i - 1] != k) start[k] = (int32_t)i;
    if (i == n - 1 || keys[i + 1] != k) end[k] = (int32_t)(i + 1);
  }
}

struct CellSpan {
  int64_t ci_lo, ci_hi, cj_lo, cj_hi;
};

// query_square's cell span (patches.py:133-137)
__device__ __forceinline__ CellSpan query_span(double cx, double cy, double r) {
  CellSpan s;
  s.ci_lo = floor_i64(ddiv(dsub(cx, r), kPatch));
  s.ci_hi = floor_i64(ddiv(dadd(cx, r), kPatch));
  s.cj_lo = floor_i64(ddiv(dsub(cy, r), kPatch));
  s.cj_hi = floor_i64(ddiv(dadd(cy, r), kPatch));
  return s;
}

__device__ __forceinline__ bool in_square(const double* p, double cx,
                                          double cy, double r) {
  return fabs(dsub(p[0], cx)) <= r && fabs(dsub(p[1], cy)) <= r;
}

// Visits every candidate (in reference order) of one patch with a full
// warp; fn(lane_has_point, point_id) is called warp-uniformly per batch.
template <typename Fn>
__device__ __forceinline__ void for_each_candidate(
    const CellSpan& s, const int32_t* __restrict__ order,
    const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
    int64_t ci0, int64_t cj0, int64_t nci, int64_t ncj, Fn fn) {
  const int lane = threadIdx.x & 31;
  for (int64_t ci = s.ci_lo; ci <= s.ci_hi; ++ci) {
    if (ci - ci0 < 0 || ci - ci0 >= nci) continue;
    for (int64_t cj = s.cj_lo; cj <= s.cj_hi; ++cj) {
      if (cj - cj0 < 0 || cj - cj0 >= ncj) continue;
      const int64_t c = (ci - ci0) * ncj + (cj - cj0);
      const int32_t b = cstart[c], e = cend[c];
      for (int32_t k = b; k < e; k += 32) {
        const bool has = k + lane < e;
        fn(has, has ? order[k + lane] : -1);
      }
    }
  }
}

__global__ void gather_count_kernel(const double* __restrict__ xyz,
                                    const int32_t* __restrict__ order,
                                    const int32_t* __restrict__ cstart,
                                    const int32_t* __restrict__ cend,
                                    int64_t ci0, int64_t cj0, int64_t nci,
                                    int64_t ncj,
                                    const ts_patch_key* __restrict__ keys,
                                    int n_patches, double radius,
                                    int32_t* counts) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= n_patches) return;
  const double cx = keys[warp].cx, cy = keys[warp].cy;
  const CellSpan s = query_span(cx, cy, radius);
  int total = 0;
  for_each_candidate(s, order, cstart, cend, ci0, cj0, nci, ncj,
                     [&](bool has, int32_t id) {
                       const bool keep = has && in_square(xyz + 3 * (int64_t)id, cx, cy, radius);
                       total += __popc(__ballot_sync(0xFFFFFFFFu, keep));
                     });
  if ((threadIdx.x & 31) == 0) counts[warp] = total;
}

__global__ void gather_fill_kernel(const double* __restrict__ xyz,
                                   const float* __restrict__ rgb,
                                   const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ cstart,
                                   const int32_t* __restrict__ cend,
                                   int64_t ci0, int64_t cj0, int64_t nci,
                                   int64_t ncj,
                                   const ts_patch_key* __restrict__ keys,
                                   int n_patches, double radius,
                                   const int64_t* __restrict__ pts_off,
                                   double* __restrict__ out_xy,
                                   double* __restrict__ out_h,
                                   float* __restrict__ out_rgb,
                                   double* __restrict__ out_cz,
                                   double* __restrict__ out_xyz,
                                   int32_t* status) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_patches) return;
  const double cx = keys[warp].cx, cy = keys[warp].cy;
  const CellSpan s = query_span(cx, cy, radius);
  const int64_t base = pts_off[warp];
  const int64_t n = pts_off[warp + 1] - base;
  if (n == 0) {
    if (lane == 0) { status[warp] = TS_E_EMPTY_PATCH; out_cz[warp] = 0.0; }
    return;
  }
  // pass A: ordered compaction of the point ids + first d^2 argmin
  double best = INFINITY;
  int64_t best_pos = INT64_MAX;
  int64_t w = 0;
  int32_t* ids = reinterpret_cast<int32_t*>(out_h + base);  // staging (N ints fit in N doubles)
  for_each_candidate(s, order, cstart, cend, ci0, cj0, nci, ncj,
                     [&](bool has, int32_t id) {
                       const double* p = xyz + 3 * (int64_t)(has ? id : 0);
                       const bool keep = has && in_square(p, cx, cy, radius);
                       const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
                       if (keep) {
                         const int64_t pos = w + __popc(m & ((1u << lane) - 1));
                         ids[pos] = id;
                         const double dx = dsub(p[0], cx), dy = dsub(p[1], cy);
                         const double d2 = dadd(dmul(dx, dx), dmul(dy, dy));
                         if (d2 < best) { best = d2; best_pos = pos; }
                       }
                       w += __popc(m);
                     });
  // warp argmin, ties -> earliest gathered position (np.argmin)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
    const int64_t op = __shfl_xor_sync(0xFFFFFFFFu, best_pos, o);
    if (ob < best || (ob == best && op < best_pos)) { best = ob; best_pos = op; }
  }
  __syncwarp();
  const int32_t cz_id = ids[best_pos];
  const double cz = xyz[3 * (int64_t)cz_id + 2];
  // pass B: patch-space transform.  Runs from the last block down: h[k]
  // overwrites staged ids 2k and 2k+1, which are >= k and so already read.
  for (int64_t k0 = ((n - 1) / 32) * 32; k0 >= 0; k0 -= 32) {
    const int64_t k = k0 + lane;
    int32_t id = 0;
    if (k < n) id = ids[k];
    __syncwarp();
    if (k < n) {
      const double* p = xyz + 3 * (int64_t)id;
      out_xy[2 * (base + k)] = ddiv(dsub(p[0], cx), kRadius);
      out_xy[2 * (base + k) + 1] = ddiv(dsub(p[1], cy), kRadius);
      out_h[base + k] = ddiv(dsub(p[2], cz), kRadius);
      if (out_xyz) {
        out_xyz[3 * (base + k)] = p[0];
        out_xyz[3 * (base + k) + 1] = p[1];
        out_xyz[3 * (base + k) + 2] = p[2];
      }
      if (out_rgb && rgb) {
        out_rgb[3 * (base + k)] = rgb[3 * (int64_t)id];
        out_rgb[3 * (base + k) + 1] = rgb[3 * (int64_t)id + 1];
        out_rgb[3 * (base + k) + 2] = rgb[3 * (int64_t)id + 2];
      }
    }
    __syncwarp();
  }
  if (lane == 0) { out_cz[warp] = cz; status[warp] = TS_OK; }
}

}  // namespace
}  // namespace ts

using namespace ts;

namespace ts {
// The stream-ordered pool returns freed memory to the driver at every
// synchronisation by default (release threshold 0); keep it instead so
// per-step scratch allocations stay cheap.
int keep_pool_memory() {
  static int done = 0;
  if (done) return TS_OK;
  int dev = 0;
  TS_CUDA_TRY(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  TS_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = ~0ull;
  TS_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done = 1;
  return TS_OK;
}
}  // namespace ts

extern "C" int ts_index_build(const int64_t* d_cell, int64_t n, int64_t ci0,
                              int64_t cj0, int64_t nci, int64_t ncj,
                              int32_t* d_order, int32_t* d_cell_start,
                              int32_t* d_cell_end, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (keep_pool_memory() != TS_OK) return TS_E_CUDA;
  if (nci <= 0 || ncj <= 0 || nci * ncj >= 0xFFFFFFFFLL) return TS_E_INVALID;
  TS_CUDA_TRY(cudaMemsetAsync(d_cell_start, 0, sizeof(int32_t) * nci * ncj, s));
  TS_CUDA_TRY(cudaMemsetAsync(d_cell_end, 0, sizeof(int32_t) * nci * ncj, s));
  if (n <= 0) return TS_OK;
  if (n >= (int64_t)INT32_MAX) return TS_E_INVALID;
  uint32_t *keys = nullptr, *keys_sorted = nullptr;
  int32_t* ids = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int bits = 1;
  while (bits < 32 && (1ull << bits) <= (unsigned long long)(nci * ncj)) ++bits;
  TS_CUDA_TRY(cudaMallocAsync(&keys, sizeof(uint32_t) * n * 2, s));
  keys_sorted = keys + n;
  TS_CUDA_TRY(cudaMallocAsync(&ids, sizeof(int32_t) * n, s));
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 148 * 8);
  ts::count_launch(), cell_key_kernel<<<grid, 256, 0, s>>>(d_cell, n, ci0, cj0, nci, ncj, keys, ids);
  TS_LAUNCH_CHECK();
  // out-of-range points (key 0xFFFFFFFF) need the full 32 bits
  bits = 32;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, ids,
                                  d_order, (int)n, 0, bits, s);
  TS_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  TS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted,
                                              ids, d_order, (int)n, 0, bits, s));
  ts::count_launch(), cell_range_kernel<<<grid, 256, 0, s>>>(keys_sorted, n, d_cell_start, d_cell_end);
  TS_LAUNCH_CHECK();
  TS_CUDA_TRY(cudaFreeAsync(tmp, s));
  TS_CUDA_TRY(cudaFreeAsync(ids, s));
  TS_CUDA_TRY(cudaFreeAsync(keys, s));
  return TS_OK;
}

extern "C" int ts_gather_count(const double* d_xyz, const int32_t* d_order,
                               const int32_t* d_cell_start,
                               const int32_t* d_cell_end, int64_t ci0,
                               int64_t cj0, int64_t nci, int64_t ncj,
                               const ts_patch_key* d_keys, int n_patches,
                               double radius, int32_t* d_counts, void* stream) {
  if (n_patches <= 0) return TS_OK;
  const int threads = 256;
  ts::count_launch(), gather_count_kernel<<<ceil_div(n_patches * 32, threads), threads, 0,
                        as_stream(stream)>>>(d_xyz, d_order, d_cell_start,
                                             d_cell_end, ci0, cj0, nci, ncj,
                                             d_keys, n_patches, radius, d_counts);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" int ts_gather_fill(const double* d_xyz, const float* d_rgb,
                              const int32_t* d_order, const int32_t* d_cell_start,
                              const int32_t* d_cell_end, int64_t ci0,
                              int64_t cj0, int64_t nci, int64_t ncj,
                              const ts_patch_key* d_keys, int n_patches,
                              double radius, const int64_t* d_pts_off, double* d_xy,
                              double* d_h, float* d_prgb, double* d_cz,
                              double* d_xyz_out, int32_t* d_status, void* stream) {
  if (n_patches <= 0) return TS_OK;
  const int threads = 256;
  ts::count_launch(), gather_fill_kernel<<<ceil_div(n_patches * 32, threads), threads, 0,
                       as_stream(stream)>>>(d_xyz, d_rgb, d_order, d_cell_start,
                                            d_cell_end, ci0, cj0, nci, ncj,
                                            d_keys, n_patches, radius, d_pts_off,
                                            d_xy, d_h, d_prgb, d_cz, d_xyz_out,
                                            d_status);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

namespace ts {
namespace {

__global__ void nearest_kernel(const double* __restrict__ xy, int64_t n,
                               const double* __restrict__ q, int64_t nq,
                               int64_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nq;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double qx = q[2 * j], qy = q[2 * j + 1];
    double best = INFINITY;
    int64_t bi = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double dx = dsub(qx, xy[2 * i]), dy = dsub(qy, xy[2 * i + 1]);
      const double d2 = dadd(dmul(dx, dx), dmul(dy, dy));
      if (d2 < best) { best = d2; bi = i; }
    }
    out[j] = bi;
  }
}

}  // namespace
}  // namespace ts

extern "C" int ts_nearest(const double* d_xy, int64_t n, const double* d_q, int64_t nq,
                          int64_t* d_idx, void* stream) {
  if (n <= 0) return TS_E_EMPTY_SET;
  if (nq <= 0) return TS_OK;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(nq, 128), 148 * 8);
  ts::count_launch(), nearest_kernel<<<grid, 128, 0, as_stream(stream)>>>(d_xy, n, d_q, nq, d_idx);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

namespace ts {
namespace {
__global__ void cell_of_kernel(const double* __restrict__ xyz, int64_t n,
                               int64_t* __restrict__ cell) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    cell[2 * i] = floor_i64(ddiv(xyz[3 * i], kPatch));
    cell[2 * i + 1] = floor_i64(ddiv(xyz[3 * i + 1], kPatch));
  }
}
}  // namespace
}  // namespace ts

extern "C" int ts_cell_keys(const double* d_xyz, int64_t n, int64_t* d_cell,
                            void* stream) {
  if (n <= 0) return TS_OK;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 148 * 8);
  ts::count_launch(), cell_of_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_xyz, n, d_cell);
  TS_LAUNCH_CHECK();
  return TS_OK;
}
