// K4: full-resolution texel update (bake_fullres, engine.py:416-456).
//
// Texel assignment.  Per point, candidate keys come from a host-built CSR
// grid (640 m cells; every key is registered in each cell its window
// [x0-1, x0+641] touches, so the cell may be computed approximately), and
// every candidate is tested with the reference predicate
//   ix = floor((x - (cx - 320)) / 10), 0 <= ix < 64   (IEEE fp64)
// so assignment is bit-exact for any key set, overlapping or not.  The
// divide is evaluated as x * 0.1 whenever that product lies more than 1e-9
// from an integer (both roundings are within 2e-14 of the true quotient,
// so their floors agree); otherwise by the IEEE divide.
//
// Accumulation.  Sums are fixed point, so the result is independent of the
// order in which points arrive (bit-identical run to run, any grid):
//   z:   int64, 2^-28 m per unit  (per-point rounding <= 1.9e-9 m;
//        |sum z| per texel must stay below 2^35 m)
//   rgb: 2^-24 per unit (per-point rounding <= 3e-8)
// against the reference's sequential fp64 bincount sums that is a mean
// difference <= 2e-9 m in height and <= 3e-8 in colour.
//
// One persistent CTA per SM walks a contiguous range of whole 1,984-point
// batches: 31 worker warps (two points per thread) and one staging warp.
// The staging warp bulk-copies positions into a double buffer
// (cp.async.bulk, mbarrier complete_tx) and, one batch ahead of the
// workers, decides whether a batch switches the CTA's "hot" patch (its
// first and last points belong to the same patch, not the current one);
// workers read the decision behind a per-buffer "ready" mbarrier and
// release buffers with per-warp arrivals, so there is no block-wide barrier
// per batch, only at the (rare) switches; the staging warp sleeps in its
// buffer waits (mbarrier suspend hint) instead of spinning on the issue
// slots the workers need.  Points >= 2 cm inside the hot key's window skip
// the CSR candidate walk when that window is its cell's only interior key
// (set_hot below; instructions per point 355 -> 210).  The hot patch's accumulators
// (count, z as lo/hi 32-bit words with the lo carry folded into hi, r/g/b
// u32 = 24 B x 4096 texels = 96 KB) live in shared memory and take native
// 32-bit shared atomics; other (point, key) pairs go straight to the global
// int64 accumulators.  A u32 colour sum that wraps adds its carry (2^32) to
// the global sum, so the shared sums are exact.  Input grouped by patch
// (engine._bake_one order, configs[2]) runs ~96% in shared memory;
// shuffled input never switches and degrades to global atomics.
#include <algorithm>

#include <cub/device/device_scan.cuh>

#include "tc_ptx.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int kTex = kOut * kOut;  // 4096 texels per patch
// one CTA per SM: 31 worker warps + 1 staging warp, two points per worker
// thread per batch, two staged batches.  Measured alternatives (r02):
// 24 warps x 3 buffers, 31 x 1 point x 4 buffers, colours staged with the
// positions (28 warps to fit) and decisions made a whole buffer ahead were
// all 5-10% slower: the kernel is latency bound and wants resident warps.
constexpr int kWorkers = 31 * 32;
constexpr int kBakeThreads = kWorkers + 32;
constexpr int kBakeU = 2;                   // points per worker thread per batch
constexpr int kBatch = kBakeU * kWorkers;   // 1,984 points
constexpr int kBufs = 2;                    // staged xyz batches (46.5 KB each)
static_assert(kBatch % 2 == 0, "16-byte aligned batches");
constexpr double kZScale = 268435456.0;          // 2^28
constexpr double kZInv = 1.0 / 268435456.0;
constexpr float kCScale = 16777216.0f;            // 2^24
constexpr double kCInv = 1.0 / 16777216.0;

struct BakeArgs {
  const double* xyz;
  const float* rgb;
  int64_t m;
  const ts_patch_key* keys;
  int n_patches;
  const int32_t* cell_off;
  const int32_t* cell_keys;
  const int32_t* cell_inner;  // nullable: leading interior keys per cell
  double gx0, gy0;
  int gnx, gny;
  int bulk;                      // arrays 16-byte aligned: stage by bulk copies
  uint32_t* cnt;                // [P][4096]
  unsigned long long* sum;      // [P][4][4096] fixed point (z, r, g, b)
};

// floor((d) / 10) exactly as numpy evaluates it (see header).
__device__ __forceinline__ int64_t texel_index(double d) {
  const double q = dmul(d, 0.1);
  const double f = floor(q);
  const double r = dsub(q, f);
  if (r > 1e-9 && r < 1.0 - 1e-9) return (int64_t)f;
  return floor_i64(ddiv(d, kTexel));
}

// Candidate key range of (x, y): the CSR slice of its (approximate) cell,
// cut to the cell's interior keys when the point is >= 2 cm inside it.
// Returns false when the point is outside the grid.
__device__ __forceinline__ bool candidates(const BakeArgs& A, double x, double y, int32_t& k0,
                                           int32_t& k1) {
  // approximate cell: the +-1 m registration margin absorbs the rounding
  const double fx = floor(dmul(dsub(x, A.gx0), 1.0 / kPatch));
  const double fy = floor(dmul(dsub(y, A.gy0), 1.0 / kPatch));
  if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)A.gnx && fy < (double)A.gny)) return false;
  const int64_t c = (int64_t)fy * A.gnx + (int64_t)fx;
  k0 = __ldg(A.cell_off + c);
  // points >= 2 cm inside their cell only test the cell's interior keys
  // (offsets are approximate to ~1e-10 m; the list uses a 1 cm square)
  const double ox = dsub(dsub(x, A.gx0), dmul(fx, kPatch));
  const double oy = dsub(dsub(y, A.gy0), dmul(fy, kPatch));
  if (A.cell_inner && ox >= 0.02 && ox <= kPatch - 0.02 && oy >= 0.02 && oy <= kPatch - 0.02)
    k1 = k0 + __ldg(A.cell_inner + c);
  else
    k1 = __ldg(A.cell_off + c + 1);
  return true;
}

// Texel of (x, y) under candidate k of the CSR list, or -1 (exact
// reference predicate).
__device__ __forceinline__ int texel_of(const BakeArgs& A, int32_t k, double x, double y,
                                        int& key) {
  key = __ldg(A.cell_keys + k);
  const double2 cc = __ldg(reinterpret_cast<const double2*>(A.keys) + key);
  const double dx = dsub(x, dsub(cc.x, 320.0));
  const double dy = dsub(y, dsub(cc.y, 320.0));
  // coarse reject: any hit has dx, dy in [-1e-13, 640 + 1e-13]
  if (!(dx > -0.5 && dx < 640.5 && dy > -0.5 && dy < 640.5)) return -1;
  const int64_t ix = texel_index(dx), iy = texel_index(dy);
  if (ix < 0 || ix >= kOut || iy < 0 || iy >= kOut) return -1;
  return (int)(iy * kOut + ix);
}

struct HotSmem {
  // hot-patch accumulators: count, z fixed point as lo/hi 32-bit words
  // (the lo word's carry goes into the hi word), colour sums
  uint32_t cnt[kTex], zlo[kTex], zhi[kTex], c[3][kTex];
  double xyz[kBufs][kBatch * 3];  // staged positions (bulk copies)
  uint64_t full[kBufs], ready[kBufs], empty[kBufs];
  int dec[kBufs];  // per staged batch: patch to switch the hot set to, or -1
};

// shared-window atomics on explicit shared addresses (no generic-address
// conversion per operation)
__device__ __forceinline__ void red_sh(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_sh(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void worker_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kWorkers) : "memory");
}

// first key whose window holds point i (-1: none)
__device__ __forceinline__ int first_key_of(const BakeArgs& A, double x, double y) {
  int32_t k0, k1;
  if (!candidates(A, x, y, k0, k1)) return -1;
  for (int32_t k = k0; k < k1; ++k) {
    int key;
    if (texel_of(A, k, x, y, key) >= 0) return key;
  }
  return -1;
}

__global__ void __launch_bounds__(kBakeThreads, 1) bake_splat_kernel(BakeArgs A) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  HotSmem& S = *reinterpret_cast<HotSmem*>(smem_raw);
  const int tid = threadIdx.x;
  for (int t = tid; t < kTex; t += kBakeThreads) {
    S.cnt[t] = 0; S.zlo[t] = 0; S.zhi[t] = 0; S.c[0][t] = 0; S.c[1][t] = 0; S.c[2][t] = 0;
  }
  // CTA ranges are whole batches, so every staged batch starts 16-byte
  // aligned (given 16-byte aligned arrays, checked by the host)
  const int64_t nbt = ceil_div<int64_t>(A.m, kBatch);
  const int64_t per = ceil_div<int64_t>(nbt, gridDim.x) * kBatch;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = min(A.m, lo + per);
  const int64_t nb = hi > lo ? ceil_div<int64_t>(hi - lo, kBatch) : 0;
  const bool has_rgb = A.rgb != nullptr;
  // full batches come in by cp.async.bulk; a ragged last batch (or
  // unaligned arrays) is read straight from global memory
  auto staged = [&](int64_t i) { return A.bulk && lo + (i + 1) * kBatch <= hi; };
  if (tid == 0) {
    for (int b = 0; b < kBufs; ++b) {
      tcx::mbar_init(&S.full[b], 1);
      tcx::mbar_init(&S.ready[b], 1);
      tcx::mbar_init(&S.empty[b], kWorkers / 32);
    }
    tcx::fence_barrier_init();
  }
  __syncthreads();

  if (tid >= kWorkers) {
    // ---------------- staging + hot-patch decisions (one warp) ----------------
    const int lane = tid & 31;
    auto issue = [&](int64_t i) {
      if (i < nb && staged(i) && lane == 0) {
        const int b = (int)(i % kBufs);
        const uint32_t bx = kBatch * 3 * sizeof(double);
        tcx::fence_proxy_async();
        tcx::mbar_arrive_tx(&S.full[b], bx);
        tcx::bulk_g2s(S.xyz[b], A.xyz + 3 * (lo + i * kBatch), bx, &S.full[b]);
      }
    };
    int hot = -1;
    auto decide = [&](int64_t i) {
      const int b = (int)(i % kBufs);
      const int64_t base = lo + i * kBatch, last = min(hi, base + kBatch) - 1;
      if (i >= kBufs && !staged(i) && lane == 0)
        tcx::mbar_wait_sleep(&S.empty[b], (uint32_t)(((i - kBufs) / kBufs) & 1), 20000);
      __syncwarp();
      int key = -1;
      if (lane < 2) {
        const int64_t q = lane ? last : base;
        double x, y;
        if (staged(i)) {
          tcx::mbar_wait(&S.full[b], (uint32_t)((i / kBufs) & 1));
          const int j = (int)(q - base);
          x = S.xyz[b][3 * j]; y = S.xyz[b][3 * j + 1];
        } else {
          x = A.xyz[3 * q]; y = A.xyz[3 * q + 1];
        }
        key = first_key_of(A, x, y);
      }
      const int ka = __shfl_sync(0xFFFFFFFFu, key, 0), kz = __shfl_sync(0xFFFFFFFFu, key, 1);
      const int sw = (ka >= 0 && ka == kz && ka != hot) ? ka : -1;
      if (sw >= 0) hot = sw;
      if (lane == 0) {
        S.dec[b] = sw;
        tcx::mbar_arrive(&S.ready[b]);
      }
      __syncwarp();
    };
    for (int q = 0; q < kBufs; ++q) issue(q);
    if (nb > 0) decide(0);
    for (int64_t i = 0; i < nb; ++i) {
      if (i + 1 < nb) decide(i + 1);
      if (i + kBufs < nb && staged(i + kBufs)) {
        if (lane == 0)
          tcx::mbar_wait_sleep(&S.empty[i % kBufs], (uint32_t)((i / kBufs) & 1), 20000);
        __syncwarp();
        issue(i + kBufs);
      }
    }
    return;
  }

  // ------------------------------ workers ------------------------------
  auto flush = [&](int hot) {
    for (int t = tid; t < kTex; t += kWorkers) {
      const uint32_t n = S.cnt[t];
      if (n) {
        atomicAdd(A.cnt + (int64_t)hot * kTex + t, n);
        unsigned long long* s = A.sum + (int64_t)hot * 4 * kTex + t;
        atomicAdd(s, ((unsigned long long)S.zhi[t] << 32) + S.zlo[t]);
        if (has_rgb) {
          atomicAdd(s + kTex, (unsigned long long)S.c[0][t]);
          atomicAdd(s + 2 * kTex, (unsigned long long)S.c[1][t]);
          atomicAdd(s + 3 * kTex, (unsigned long long)S.c[2][t]);
        }
      }
      S.cnt[t] = 0; S.zlo[t] = 0; S.zhi[t] = 0; S.c[0][t] = 0; S.c[1][t] = 0; S.c[2][t] = 0;
    }
  };
  int hot = -1;
  // Hot-patch fast path.  When the hot key's window lies within 5 mm of its
  // 640 m grid cell and is that cell's only interior key, a point >= 2 cm
  // inside the window (dx, dy as texel_of computes them) is >= 1.5 cm inside
  // the cell, where no other key's window (+-1e-6 m) reaches: its candidate
  // set is {hot}, so the CSR walk is skipped with the same result.
  double hx0 = 0.0, hy0 = 0.0;
  bool fast = false;
  auto set_hot = [&](int h) {
    const double2 cc = __ldg(reinterpret_cast<const double2*>(A.keys) + h);
    hx0 = dsub(cc.x, 320.0);
    hy0 = dsub(cc.y, 320.0);
    fast = false;
    if (!A.cell_inner) return;
    const double fx = floor(dmul(dsub(cc.x, A.gx0), 1.0 / kPatch));
    const double fy = floor(dmul(dsub(cc.y, A.gy0), 1.0 / kPatch));
    if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)A.gnx && fy < (double)A.gny)) return;
    const int64_t c = (int64_t)fy * A.gnx + (int64_t)fx;
    const double ox = dsub(hx0, dadd(A.gx0, dmul(fx, kPatch)));
    const double oy = dsub(hy0, dadd(A.gy0, dmul(fy, kPatch)));
    fast = fabs(ox) <= 0.005 && fabs(oy) <= 0.005 && __ldg(A.cell_inner + c) == 1 &&
           __ldg(A.cell_keys + __ldg(A.cell_off + c)) == h;
  };
  const uint32_t sh_cnt = tcx::su32(S.cnt), sh_zlo = tcx::su32(S.zlo), sh_zhi = tcx::su32(S.zhi),
                 sh_c = tcx::su32(S.c[0]);
  for (int64_t i = 0; i < nb; ++i) {
    const int b = (int)(i % kBufs);
    const int64_t base = lo + i * kBatch;
    // colours straight from global (coalesced 12-byte runs), issued before
    // the batch is waited for
    float cv[kBakeU][3];
    const bool stg = staged(i);
#pragma unroll
    for (int u = 0; u < kBakeU; ++u) {
      const int64_t q = base + u * kWorkers + tid;
      cv[u][0] = cv[u][1] = cv[u][2] = 0.f;
      if (has_rgb && q < hi) {
        cv[u][0] = __ldg(A.rgb + 3 * q); cv[u][1] = __ldg(A.rgb + 3 * q + 1);
        cv[u][2] = __ldg(A.rgb + 3 * q + 2);
      }
    }
    tcx::mbar_wait(&S.ready[b], (uint32_t)((i / kBufs) & 1));
    const int sw = S.dec[b];
    if (sw >= 0) {  // known to every worker: switch the hot patch
      worker_sync();  // all workers are done with the previous batch
      if (hot >= 0) flush(hot);
      worker_sync();
      hot = sw;
      set_hot(hot);
    }
#pragma unroll
    for (int u = 0; u < kBakeU; ++u) {
      const int j = u * kWorkers + tid;
      const int64_t q = base + j;
      if (q >= hi) continue;
      double x, y, z;
      if (stg) { x = S.xyz[b][3 * j]; y = S.xyz[b][3 * j + 1]; z = S.xyz[b][3 * j + 2]; }
      else { x = A.xyz[3 * q]; y = A.xyz[3 * q + 1]; z = A.xyz[3 * q + 2]; }
      const long long zf = __double2ll_rn(dmul(z, kZScale));
      int32_t k0 = 0, k1 = 0;
      int tfast = -1;
      if (fast) {
        const double dx = dsub(x, hx0), dy = dsub(y, hy0);
        if (dx >= 0.02 && dx <= 639.98 && dy >= 0.02 && dy <= 639.98)
          tfast = (int)(texel_index(dy) * kOut + texel_index(dx));
      }
      if (tfast < 0) {
        if (!candidates(A, x, y, k0, k1)) continue;
      } else {
        k1 = k0 + 1;  // one pass: the hot key, texel tfast
      }
      for (int32_t k = k0; k < k1; ++k) {
        int key = hot;
        const int t = tfast >= 0 ? tfast : texel_of(A, k, x, y, key);
        if (t < 0) continue;
        if (key == hot) {
          red_sh(sh_cnt + 4 * t, 1u);
          const uint32_t zl = (uint32_t)zf;
          const uint32_t old = atom_sh(sh_zlo + 4 * t, zl);
          red_sh(sh_zhi + 4 * t, (uint32_t)((unsigned long long)zf >> 32) + (old + zl < old ? 1u : 0u));
          if (has_rgb) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              const float v = cv[u][ch];
              if (v >= 0.f && v < 256.f) {
                const uint32_t qv = __float2uint_rn(v * kCScale);
                const uint32_t o = atom_sh(sh_c + 4 * (ch * kTex + t), qv);
                if (o + qv < o)  // carry out of the 32-bit shared sum
                  atomicAdd(A.sum + ((int64_t)key * 4 + ch + 1) * kTex + t, 1ull << 32);
              } else {
                atomicAdd(A.sum + ((int64_t)key * 4 + ch + 1) * kTex + t,
                          (unsigned long long)__double2ll_rn((double)v * (double)kCScale));
              }
            }
          }
        } else {
          unsigned long long* gs = A.sum + (int64_t)key * 4 * kTex + t;
          atomicAdd(A.cnt + (int64_t)key * kTex + t, 1u);
          atomicAdd(gs, (unsigned long long)zf);
          if (has_rgb)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
              atomicAdd(gs + (ch + 1) * kTex,
                        (unsigned long long)__double2ll_rn((double)cv[u][ch] * (double)kCScale));
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) tcx::mbar_arrive(&S.empty[b]);  // this warp is done with buffer b
  }
  worker_sync();
  if (hot >= 0) flush(hot);
}

__global__ void __launch_bounds__(256)
bake_finalize_kernel(const uint32_t* __restrict__ cnt, const unsigned long long* __restrict__ sum,
                     int n_patches, const float* __restrict__ prior_h,
                     const double* __restrict__ base_cz, const double* __restrict__ key_cz,
                     const float* __restrict__ prior_rgb, int has_pts_rgb,
                     float* __restrict__ out_h, float* __restrict__ out_rgb) {
  const int64_t total = (int64_t)n_patches * kTex;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / kTex, t = i - p * kTex;
    const uint32_t n = cnt[i];
    const unsigned long long* s = sum + p * 4 * kTex + t;
    double h;
    if (n > 0) h = ddiv(dmul((double)(long long)s[0], kZInv), (double)n);
    else h = dadd((double)prior_h[i], base_cz[p]);
    out_h[i] = __double2float_rn(dsub(h, key_cz[p]));
    if (prior_rgb && out_rgb) {
      if (n > 0 && has_pts_rgb) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
          out_rgb[3 * i + c] = __double2float_rn(
              ddiv(dmul((double)(long long)s[(c + 1) * kTex], kCInv), (double)n));
      } else {
        out_rgb[3 * i] = prior_rgb[3 * i];
        out_rgb[3 * i + 1] = prior_rgb[3 * i + 1];
        out_rgb[3 * i + 2] = prior_rgb[3 * i + 2];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Binning (ts_bake_bin): points in arbitrary order -> grouped by 640 m cell
// of the key grid, so the splat's shared-memory hot patch forms again.  Two
// counting-sort passes (most significant digit first): by cell row, then
// by cell.  Each pass: per-CTA bin histograms in shared memory, a column
// scan over CTAs, a scan over bins, then every CTA scatters its chunk
// through shared-memory cursors.  One pass over all cells would keep
// CTAs x cells partially written output lines in flight (4,357 cells x 592
// CTAs: 10x the L2) and write-amplify 6x; by rows first, every CTA of the
// second pass reads points of ~one row and writes ~gnx runs.  Points outside the grid go to the last bin (the
// splat skips them).  Order inside a cell is not defined -- the splat's
// fixed-point sums do not depend on it.
constexpr int kBinThreads = 512;
constexpr int kBinMaxCells = 16384;  // shared histogram: 64 KB

// bin of a point: its cell (rows: its cell row), outside the grid -> last
__device__ __forceinline__ int bin_cell(double x, double y, double gx0, double gy0, int gnx,
                                        int gny, bool rows) {
  const double fx = floor(dmul(dsub(x, gx0), 1.0 / kPatch));
  const double fy = floor(dmul(dsub(y, gy0), 1.0 / kPatch));
  if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)gnx && fy < (double)gny))
    return rows ? gny : gnx * gny;
  return rows ? (int)fy : (int)fy * gnx + (int)fx;
}

struct BinArgs {
  const double* xyz;
  const float* rgb;
  int64_t m, per;  // points, points per CTA
  double gx0, gy0;
  int gnx, gny, nb;  // nb bins: gnx * gny + 1 (cells) or gny + 1 (rows)
  int rows;          // pass 1: bin by cell row only
  uint32_t* hist;    // [grid][nb]: counts, then each CTA's offset within the bin
  uint32_t* total;   // [nb]
  uint32_t* start;   // [nb] exclusive scan of total
  double* xyz_out;
  float* rgb_out;
};

__global__ void __launch_bounds__(kBinThreads) bin_count_kernel(BinArgs A) {
  extern __shared__ uint32_t s_h[];
  for (int i = threadIdx.x; i < A.nb; i += kBinThreads) s_h[i] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * A.per, hi = min(A.m, lo + A.per);
  for (int64_t i0 = lo; i0 < hi; i0 += kBinThreads) {
    const int64_t i = i0 + threadIdx.x;
    const int bin = i < hi ? bin_cell(A.xyz[3 * i], A.xyz[3 * i + 1], A.gx0, A.gy0, A.gnx,
                                      A.gny, A.rows)
                           : -1;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
    if (bin >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(s_h + bin, (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < A.nb; i += kBinThreads)
    A.hist[(int64_t)blockIdx.x * A.nb + i] = s_h[i];
}

// per bin: exclusive prefix over CTAs (in place) and the bin total
__global__ void bin_column_kernel(BinArgs A, int grid) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= A.nb) return;
  uint32_t run = 0;
  for (int g = 0; g < grid; ++g) {
    uint32_t* h = A.hist + (int64_t)g * A.nb + c;
    const uint32_t v = *h;
    *h = run;
    run += v;
  }
  A.total[c] = run;
}

// Scatter through a shared-memory staging tile: kBinTile points are sorted
// by bin locally (counting sort), then written out run by run, so each
// bin's points of the tile leave as one coalesced run instead of one
// partial-line store per point.

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp) {
  // exclusive scan of one value per thread across the block (kBinThreads)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < kBinThreads / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kBinThreads / 32) s_warp[lane] = t;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t before = w ? s_warp[w - 1] : 0;
  __syncthreads();
  return before + x - v;
}

// kBinTile: 2,048 points for the row pass (two CTAs per SM), 4,096 for the
// cell pass (its per-tile bin bookkeeping covers every cell); measured
// 4.4 + 7.0 ms for 200 M points against 6.5 + 7.0 / 4.4 + 7.6
template <int kBinTile>
__global__ void __launch_bounds__(kBinThreads) bin_scatter_kernel(BinArgs A) {
  extern __shared__ __align__(16) uint8_t s_raw[];
  // [nb] global cursors, [nb] tile counts -> tile starts, [nb] tile fill
  // cursors, staged points (xyz, rgb, bin) of one tile
  uint32_t* s_cur = reinterpret_cast<uint32_t*>(s_raw);
  uint32_t* s_cnt = s_cur + A.nb;
  uint32_t* s_fill = s_cnt + A.nb;
  double* s_xyz = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(s_fill + A.nb) + 15) & ~uintptr_t(15));
  float* s_rgb = reinterpret_cast<float*>(s_xyz + 3 * kBinTile);
  int* s_bin = reinterpret_cast<int*>(s_rgb + 3 * kBinTile);
  __shared__ uint32_t s_warp[32];
  for (int i = threadIdx.x; i < A.nb; i += kBinThreads)
    s_cur[i] = A.start[i] + A.hist[(int64_t)blockIdx.x * A.nb + i];
  const int64_t lo = (int64_t)blockIdx.x * A.per, hi = min(A.m, lo + A.per);
  const int per_thread = (A.nb + kBinThreads - 1) / kBinThreads;
  for (int64_t t0 = lo; t0 < hi; t0 += kBinTile) {
    const int n = (int)(hi - t0 < kBinTile ? hi - t0 : kBinTile);
    for (int i = threadIdx.x; i < A.nb; i += kBinThreads) s_cnt[i] = 0;
    __syncthreads();
    // 1. bins of the tile's points + local histogram
    int bins[kBinTile / kBinThreads];
#pragma unroll
    for (int u = 0; u < kBinTile / kBinThreads; ++u) {
      const int j = u * kBinThreads + threadIdx.x;
      bins[u] = -1;
      if (j < n) {
        const int64_t i = t0 + j;
        bins[u] = bin_cell(A.xyz[3 * i], A.xyz[3 * i + 1], A.gx0, A.gy0, A.gnx, A.gny, A.rows);
        atomicAdd(s_cnt + bins[u], 1u);
      }
    }
    __syncthreads();
    // 2. tile starts per bin (block scan over nb bins, per_thread each)
    uint32_t mine = 0;
    for (int k = 0; k < per_thread; ++k) {
      const int b = threadIdx.x * per_thread + k;
      if (b < A.nb) mine += s_cnt[b];
    }
    uint32_t run = block_excl_scan(mine, s_warp);
    for (int k = 0; k < per_thread; ++k) {
      const int b = threadIdx.x * per_thread + k;
      if (b < A.nb) {
        const uint32_t c = s_cnt[b];
        s_cnt[b] = run;  // tile start of bin b
        s_fill[b] = run;
        run += c;
      }
    }
    __syncthreads();
    // 3. stage the points in bin order
#pragma unroll
    for (int u = 0; u < kBinTile / kBinThreads; ++u) {
      const int j = u * kBinThreads + threadIdx.x;
      if (j < n) {
        const int64_t i = t0 + j;
        const uint32_t q = atomicAdd(s_fill + bins[u], 1u);
        s_xyz[3 * q] = A.xyz[3 * i];
        s_xyz[3 * q + 1] = A.xyz[3 * i + 1];
        s_xyz[3 * q + 2] = A.xyz[3 * i + 2];
        if (A.rgb) {
          s_rgb[3 * q] = A.rgb[3 * i];
          s_rgb[3 * q + 1] = A.rgb[3 * i + 1];
          s_rgb[3 * q + 2] = A.rgb[3 * i + 2];
        }
        s_bin[q] = bins[u];
      }
    }
    __syncthreads();
    // 4. write runs: staged slot q of bin b -> global cursor[b] + (q - start[b])
    for (int e = threadIdx.x; e < 3 * n; e += kBinThreads) {
      const int q = e / 3, c = e - 3 * q, b = s_bin[q];
      const uint32_t g = s_cur[b] + (uint32_t)(q - (int)s_cnt[b]);
      A.xyz_out[3 * (int64_t)g + c] = s_xyz[e];
      if (A.rgb) A.rgb_out[3 * (int64_t)g + c] = s_rgb[e];
    }
    __syncthreads();
    for (int k = 0; k < per_thread; ++k) {  // advance the global cursors
      const int b = threadIdx.x * per_thread + k;
      if (b < A.nb) s_cur[b] += s_fill[b] - s_cnt[b];
    }
    __syncthreads();
  }
}

size_t bin_scatter_smem(int nb, int tile) {
  return (3 * (size_t)nb * 4 + 15) / 16 * 16 + (size_t)tile * (24 + 12 + 4);
}

int bin_grid(int64_t m) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 4, ceil_div<int64_t>(m, 4096)));
}

size_t bin_scan_bytes(int nb) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr, nb);
  return (tmp + 255) & ~size_t(255);
}

}  // namespace
}  // namespace ts

using namespace ts;

namespace {
size_t bin_words(int64_t m, int nb) { return (size_t)bin_grid(m) * nb + 2 * (size_t)nb; }
size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
}  // namespace

extern "C" size_t ts_bake_bin_scratch(int64_t m, int gnx, int gny) {
  if (m < 0 || gnx <= 0 || gny <= 0 || (int64_t)gnx * gny + 1 > kBinMaxCells) return 0;
  const int nb = gnx * gny + 1;
  // counters + scan temp (sized for the larger pass) + the pass-1 points
  return align256(bin_words(m, nb) * sizeof(uint32_t)) + bin_scan_bytes(nb) +
         align256((size_t)m * 3 * sizeof(double)) + align256((size_t)m * 3 * sizeof(float));
}

extern "C" int ts_bake_bin(const double* d_xyz, const float* d_rgb, int64_t m, double gx0,
                           double gy0, int gnx, int gny, double* d_xyz_out, float* d_rgb_out,
                           void* d_scratch, void* stream) {
  if (m < 0 || gnx <= 0 || gny <= 0 || (int64_t)gnx * gny + 1 > kBinMaxCells) return TS_E_INVALID;
  if (m >= ((int64_t)1 << 32)) return TS_E_INVALID;  // u32 positions
  if (m == 0) return TS_OK;
  if ((d_rgb == nullptr) != (d_rgb_out == nullptr)) return TS_E_INVALID;
  cudaStream_t s = as_stream(stream);
  const int ncell = gnx * gny + 1, grid = bin_grid(m);
  uint8_t* q = reinterpret_cast<uint8_t*>(d_scratch);
  uint32_t* w = reinterpret_cast<uint32_t*>(q);
  q += align256(bin_words(m, ncell) * sizeof(uint32_t));
  void* tmp = q;
  const size_t tmp_cap = bin_scan_bytes(ncell);
  q += tmp_cap;
  double* mid_xyz = reinterpret_cast<double*>(q);
  q += align256((size_t)m * 3 * sizeof(double));
  float* mid_rgb = d_rgb ? reinterpret_cast<float*>(q) : nullptr;
  for (int pass = 0; pass < 2; ++pass) {
    BinArgs a{};
    a.rows = pass == 0;
    a.nb = a.rows ? gny + 1 : ncell;
    a.xyz = pass == 0 ? d_xyz : mid_xyz;
    a.rgb = pass == 0 ? d_rgb : mid_rgb;
    a.xyz_out = pass == 0 ? mid_xyz : d_xyz_out;
    a.rgb_out = pass == 0 ? mid_rgb : d_rgb_out;
    a.m = m; a.per = ceil_div<int64_t>(m, grid);
    a.gx0 = gx0; a.gy0 = gy0; a.gnx = gnx; a.gny = gny;
    a.hist = w;
    a.total = w + (size_t)grid * a.nb;
    a.start = a.total + a.nb;
    size_t tmp_bytes = tmp_cap;
    const int smem = a.nb * (int)sizeof(uint32_t);
    const int smem2 = (int)bin_scatter_smem(a.nb, a.rows ? 2048 : 4096);
    TS_CUDA_TRY(cudaFuncSetAttribute(bin_count_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    TS_CUDA_TRY(cudaFuncSetAttribute(a.rows ? bin_scatter_kernel<2048> : bin_scatter_kernel<4096>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    ts::count_launch(), bin_count_kernel<<<grid, kBinThreads, smem, s>>>(a);
    ts::count_launch(), bin_column_kernel<<<ceil_div(a.nb, 256), 256, 0, s>>>(a, grid);
    TS_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, a.total, a.start, a.nb, s));
    if (a.rows) ts::count_launch(), bin_scatter_kernel<2048><<<grid, kBinThreads, smem2, s>>>(a);
    else ts::count_launch(), bin_scatter_kernel<4096><<<grid, kBinThreads, smem2, s>>>(a);
    TS_LAUNCH_CHECK();
  }
  return TS_OK;
}

extern "C" size_t ts_bake_workspace(int n_patches) {
  const size_t p = n_patches > 0 ? (size_t)n_patches : 1;
  return p * kTex * (sizeof(uint32_t) + 4 * sizeof(unsigned long long)) + 256;
}

extern "C" int ts_bake(const double* d_xyz, const float* d_rgb, int64_t m,
                       const ts_patch_key* d_keys, int n_patches,
                       const int32_t* d_cell_keys_off, const int32_t* d_cell_keys,
                       const int32_t* d_cell_inner, double gx0, double gy0, int gnx, int gny,
                       const float* d_prior_h, const double* d_base_cz,
                       const double* d_key_cz, const float* d_prior_rgb,
                       float* d_out_h, float* d_out_rgb, void* d_accum, void* stream) {
  if (n_patches <= 0) return TS_OK;
  if (gnx <= 0 || gny <= 0 || m < 0) return TS_E_INVALID;
  cudaStream_t s = as_stream(stream);
  unsigned long long* sum = reinterpret_cast<unsigned long long*>(d_accum);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sum + (size_t)n_patches * 4 * kTex);
  TS_CUDA_TRY(cudaMemsetAsync(d_accum, 0, ts_bake_workspace(n_patches) - 256, s));
  if (m > 0) {
    const int bulk = ((uintptr_t)d_xyz % 16 == 0) && ((uintptr_t)d_rgb % 16 == 0);
    BakeArgs a{d_xyz, d_rgb, m, d_keys, n_patches, d_cell_keys_off, d_cell_keys,
               d_cell_inner, gx0, gy0, gnx, gny, bulk, cnt, sum};
    int sms = 0;
    {  // per call: the SM count and the attribute are per device
      int dev = 0;
      TS_CUDA_TRY(cudaGetDevice(&dev));
      TS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      TS_CUDA_TRY(cudaFuncSetAttribute(bake_splat_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(HotSmem)));
    }
    // one CTA per SM, whole batches per CTA
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, ceil_div<int64_t>(m, kBatch)));
    ts::count_launch(), bake_splat_kernel<<<grid, kBakeThreads, sizeof(HotSmem), s>>>(a);
    TS_LAUNCH_CHECK();
  }
  const int64_t total = (int64_t)n_patches * kTex;
  const int grid2 = (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), 148 * 16);
  ts::count_launch(), bake_finalize_kernel<<<grid2, 256, 0, s>>>(cnt, sum, n_patches, d_prior_h, d_base_cz,
                                             d_key_cz, d_prior_rgb, d_rgb != nullptr,
                                             d_out_h, d_out_rgb);
  TS_LAUNCH_CHECK();
  return TS_OK;
}
