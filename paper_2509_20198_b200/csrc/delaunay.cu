// K2a: per-patch Delaunay triangulation on the GPU (one warp per patch).
//
// Replaces scipy.spatial.Delaunay (Qhull) + _ccw in interpolate_patch
// (patches.py:316-326).  Incremental Bowyer-Watson: start from the padding
// square split into two triangles, insert points 0..N-1 in index order.  For
// each point the warp tests every live triangle's circumcircle in parallel
// (exact incircle), compacts the cavity with ballots, finds its boundary
// edges and re-fans them to the new point, reusing the cavity's slots.
// Exact predicates keep the cavity star-shaped, so the mesh stays valid;
// an exact duplicate of an earlier point has an empty cavity and is
// skipped (the lowest index survives as the vertex).
//
// Compiled with --fmad=false: the predicate error bounds assume one
// rounding per operation.
#include <cstdlib>
#include <type_traits>

#include "predicates.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int kMaxCavity = 176;  // with the mesh: 31.5 KB, 7 patch-warps per SM
// Patches up to kSmemPoints keep their whole mesh (triangles + circumcircle
// cache, SoA) in shared memory: every insertion rewrites a few slots and the
// next one re-reads them, so a global-memory mesh turns each step into a
// chain of L1-miss latencies.  Larger patches spill to the caller's scratch.
// 384 points (~31 KB per warp) lets 7 patch-warps share an SM, so the
// 1,024 patches of a configs[1] batch (N ~ 310-340) run in ONE wave.
constexpr int kSmemPoints = 384;
constexpr int kSmemSlots = 2 * kSmemPoints + 8;
#ifndef TS_DL_ILP
#define TS_DL_ILP 6
#endif
constexpr int kScanIlp = TS_DL_ILP;  // circle tests per lane per cavity-scan pass (4: +2%, 8: +1% time)

constexpr size_t kDelaunaySmem = (size_t)kSmemSlots * (3 * sizeof(int) + 3 * sizeof(double)) +
                                 kMaxCavity * sizeof(int) + (kMaxCavity + 8) * sizeof(int2) +
                                 3 * kMaxCavity * sizeof(int);

struct PatchPts {
  const double* xy;
  int n;
  __device__ __forceinline__ void get(int v, double& x, double& y) const {
    if (v < n) { x = xy[2 * v]; y = xy[2 * v + 1]; }
    else {
      const int c = v - n;  // (-1,-1), (1,-1), (-1,1), (1,1)
      x = (c & 1) ? 1.0 : -1.0;
      y = (c & 2) ? 1.0 : -1.0;
    }
  }
};

// Circumcircle cache, structure of arrays.  An ill-conditioned triangle gets
// r2 = NaN, which makes both fast comparisons false -> exact predicate.
struct Mesh {
  int* tri;
  double *cx, *cy, *r2;
  __device__ __forceinline__ void set(const PatchPts& P, int slot, int a, int b, int c) {
    tri[3 * slot] = a;
    tri[3 * slot + 1] = b;
    tri[3 * slot + 2] = c;
    double ax, ay, bx, by, qx, qy;
    P.get(a, ax, ay);
    P.get(b, bx, by);
    P.get(c, qx, qy);
    const double ux = bx - ax, uy = by - ay, vx = qx - ax, vy = qy - ay;
    const double p1 = ux * vy, p2 = uy * vx;
    const double D = 2.0 * (p1 - p2);
    const bool ok = fabs(D) > 1e-6 * (fabs(p1) + fabs(p2)) && fabs(D) > 1e-200;
    const double l1 = ux * ux + uy * uy, l2 = vx * vx + vy * vy;
    // no IEEE divide: the cache only feeds the filter, whose 1e-6 relative
    // margin dwarfs the error of an approximate reciprocal refined by two
    // Newton steps (relative error ~1e-16; ill-conditioned D is flagged)
    double inv;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(D));
    inv = inv * (2.0 - D * inv);
    inv = inv * (2.0 - D * inv);
    const double ox = (vy * l1 - uy * l2) * inv, oy = (ux * l2 - vx * l1) * inv;
    cx[slot] = ax + ox;
    cy[slot] = ay + oy;
    r2[slot] = ok ? ox * ox + oy * oy : __longlong_as_double(0x7ff8000000000000LL);
  }
  // filter only (branch-free, so several tests overlap): 1 strictly inside,
  // -1 outside, 0 unsure (then in_circle_exact decides)
  __device__ __forceinline__ int in_circle_fast(int t, double px, double py) const {
    const double dx = px - cx[t], dy = py - cy[t], rr = r2[t];
    const double d2 = dx * dx + dy * dy;
    const double m = 1e-6 * (d2 + rr);
    return (d2 < rr - m) ? 1 : (d2 > rr + m) ? -1 : 0;
  }
  __device__ __forceinline__ int in_circle_exact(const PatchPts& P, int t, double px,
                                                 double py) const {
    double ax, ay, bx, by, qx, qy;
    P.get(tri[3 * t], ax, ay);
    P.get(tri[3 * t + 1], bx, by);
    P.get(tri[3 * t + 2], qx, qy);
    return pred::incircle(ax, ay, bx, by, qx, qy, px, py);
  }
};


constexpr int kOverflow = -1;  // shared-memory cavity full: retry in global memory

// Scratch layout (ts_triangulate_scratch): patch p owns triangle slots
// [base, base + cap), base = 2 off + 8 p, cap = 2 n + 8 (the most an n-point
// mesh can hold), and the byte block [60 base + 64 p, 60 (base + cap) +
// 64 (p + 1)) of the scratch:
//   circumcircle cache  3 x cap doubles (x, y, r^2 per slot)
//   cavity keys         3 x cap int64   (global-memory variant)
//   cavity edges        cap + 8 int2
//   cavity slots        cap int
// (60 base is a multiple of 8: base is even.)
constexpr int64_t kSlotBytes = 60, kPatchBytes = 64;

// SMEM: the mesh and the cavity live in shared memory (the instance's
// pointers all derive from the shared array, so its loads compile to LDS),
// the cavity holds kMaxCavity triangles and edge keys are u << 16 | w (ids <
// 2^16: n <= kSmemPoints).  Otherwise the mesh and a cavity of the mesh's
// full capacity live in the caller's scratch and keys are 64-bit, so no
// patch size or insertion order can overflow it.
template <bool SMEM>
__device__ __forceinline__ int triangulate_patch(unsigned char* smem,
                                                 const double* __restrict__ xy_all,
                                                 const int64_t* __restrict__ pts_off,
                                                 int32_t* tri_all, int32_t* ntri_out,
                                                 int32_t* status, uint8_t* scratch) {
  using Key = typename std::conditional<SMEM, int, long long>::type;
  constexpr int kShift = SMEM ? 16 : 32;
  const int lane = threadIdx.x;
  const int p = blockIdx.x;
  const int64_t off = pts_off[p];
  const int n = (int)(pts_off[p + 1] - off);
  const int64_t base = 2 * off + 8 * (int64_t)p;  // first triangle slot
  int* tri_out = tri_all + 3 * base;
  const PatchPts P{xy_all + 2 * off, n};
  const int cap = 2 * n + 8;
  constexpr bool in_smem = SMEM;
  const int max_cav = SMEM ? kMaxCavity : cap;
  Mesh M;
  int* bad;
  int2* edge;
  Key* ekey;
  if (SMEM) {
    double* s_cx = reinterpret_cast<double*>(smem);
    double* s_cy = s_cx + kSmemSlots;
    double* s_r2 = s_cy + kSmemSlots;
    int* s_tri = reinterpret_cast<int*>(s_r2 + kSmemSlots);
    M = Mesh{s_tri, s_cx, s_cy, s_r2};
    bad = s_tri + 3 * kSmemSlots;
    edge = reinterpret_cast<int2*>(bad + kMaxCavity);
    ekey = reinterpret_cast<Key*>(edge + kMaxCavity + 8);  // [3 * kMaxCavity]
  } else {
    uint8_t* blk = scratch + kSlotBytes * base + kPatchBytes * p;
    double* g = reinterpret_cast<double*>(blk);
    M = Mesh{tri_out, g, g + cap, g + 2 * cap};
    ekey = reinterpret_cast<Key*>(blk + 24 * (int64_t)cap);
    edge = reinterpret_cast<int2*>(blk + 48 * (int64_t)cap);
    bad = reinterpret_cast<int*>(blk + 56 * (int64_t)cap + 64);
  }
  if (lane == 0) M.set(P, 0, n, n + 1, n + 3);
  if (lane == 1) M.set(P, 1, n, n + 3, n + 2);
  int ntri = 2;
  int st = TS_OK;
  __syncwarp();
  for (int v = 0; v < n; ++v) {
    double px, py;
    P.get(v, px, py);
    // 1. cavity: triangles whose circumcircle strictly contains v
    //    (kScanIlp triangles per lane per pass: independent circle tests
    //    in flight; cavity order stays ascending)
    int nb = 0;
    const unsigned below = (1u << lane) - 1;
    for (int b0 = 0; b0 < ntri; b0 += 32 * kScanIlp) {
      bool in[kScanIlp];
      int f[kScanIlp];
#pragma unroll
      for (int j = 0; j < kScanIlp; ++j) {  // slots >= ntri hold stale data: masked
        const int t = min(b0 + lane + 32 * j, ntri - 1);
        f[j] = M.in_circle_fast(t, px, py);
      }
      bool unsure = false;
#pragma unroll
      for (int j = 0; j < kScanIlp; ++j) unsure |= f[j] == 0 && b0 + lane + 32 * j < ntri;
      if (__any_sync(0xFFFFFFFFu, unsure)) {  // rare: one warp-uniform branch
#pragma unroll
        for (int j = 0; j < kScanIlp; ++j) {
          const int t = b0 + lane + 32 * j;
          if (f[j] == 0 && t < ntri) f[j] = M.in_circle_exact(P, t, px, py);
        }
      }
      unsigned m[kScanIlp];
#pragma unroll
      for (int j = 0; j < kScanIlp; ++j) {
        in[j] = b0 + lane + 32 * j < ntri && f[j] > 0;
        m[j] = __ballot_sync(0xFFFFFFFFu, in[j]);
      }
#pragma unroll
      for (int j = 0; j < kScanIlp; ++j) {
        if (in[j]) {
          const int slot = nb + __popc(m[j] & below);
          if (slot < max_cav) bad[slot] = b0 + lane + 32 * j;
        }
        nb += __popc(m[j]);
      }
    }
    if (nb == 0) continue;  // exact duplicate of an inserted vertex
    if (nb > max_cav) { st = kOverflow; break; }  // (shared-memory cavity only)
    __syncwarp();
    // 2. boundary edges of the cavity (edges without a bad twin): every
    //    directed cavity edge is published as a key (u << kShift | w); an
    //    edge is interior iff its reverse key is present
    for (int e = lane; e < 3 * nb; e += 32) {
      const int i = e / 3, j = e - 3 * i;
      const int* t = M.tri + 3 * bad[i];
      ekey[e] = ((Key)t[j] << kShift) | (Key)t[j == 2 ? 0 : j + 1];
    }
    __syncwarp();
    int ne = 0;
    for (int e0 = 0; e0 < 3 * nb; e0 += 32) {
      const int e = e0 + lane;
      bool keep = false;
      int u = 0, w = 0;
      if (e < 3 * nb) {
        const Key key = ekey[e];
        u = (int)(key >> kShift);
        w = (int)(key & (((Key)1 << kShift) - 1));
        const Key twin = ((Key)w << kShift) | (Key)u;
        keep = true;
        // linear twin search over all keys (broadcast reads; measured
        // faster than __match_any_sync on the undirected keys)
        int hit = 0;
#pragma unroll 4
        for (int k = 0; k < 3 * nb; ++k) hit |= ekey[k] == twin;
        keep = !hit;
      }
      if (e < 3 * nb) {
        if (keep) {
          double ux, uy, wx, wy;
          P.get(u, ux, uy);
          P.get(w, wx, wy);
          // v on a hull edge: no zero-area triangle (patches.py:238 would
          // give it inv_det = 0)
          if (pred::orient(ux, uy, wx, wy, px, py) == 0) keep = false;
        }
      }
      const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
      if (keep) {
        const int slot = ne + __popc(m & ((1u << lane) - 1));
        if (slot < max_cav + 8) edge[slot] = make_int2(u, w);
      }
      ne += __popc(m);
    }
    if (ne > max_cav + 8) { st = kOverflow; break; }
    if (ne < nb || ntri + ne - nb > cap) {  // impossible with exact predicates
      st = TS_E_INVALID;
      break;
    }
    __syncwarp();
    // 3. fan the boundary to v: reuse cavity slots, then append
    for (int i = lane; i < ne; i += 32) {
      const int slot = i < nb ? bad[i] : ntri + (i - nb);
      const int2 ed = edge[i];
      M.set(P, slot, ed.x, ed.y, v);
    }
    ntri += ne - nb;
    __syncwarp();
  }
  if (st == kOverflow) return st;  // the caller retries in global memory
  if (in_smem && st == TS_OK)
    for (int i = lane; i < 3 * ntri; i += 32) tri_out[i] = M.tri[i];
  if (lane == 0) {
    ntri_out[p] = st == TS_OK ? ntri : 0;
    status[p] = st;
  }
  return st;
}

__global__ void __launch_bounds__(32)
delaunay_kernel(const double* __restrict__ xy_all,
                const int64_t* __restrict__ pts_off, int n_patches,
                int32_t* tri_all, int32_t* ntri_out, int32_t* status, uint8_t* scratch) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int p = blockIdx.x;
  const int n = (int)(pts_off[p + 1] - pts_off[p]);
  if (n == 0) {
    if (threadIdx.x == 0) { ntri_out[p] = 0; status[p] = TS_E_EMPTY_PATCH; }
    return;
  }
  // a cavity larger than the shared-memory one (rare insertion orders)
  // restarts the patch with the global-memory mesh
  if (n <= kSmemPoints &&
      triangulate_patch<true>(smem, xy_all, pts_off, tri_all, ntri_out, status, scratch) !=
          kOverflow)
    return;
  __syncwarp();
  triangulate_patch<false>(smem, xy_all, pts_off, tri_all, ntri_out, status, scratch);
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" size_t ts_triangulate_scratch(int64_t total_points, int n_patches) {
  const int64_t slots = 2 * total_points + 8 * (int64_t)n_patches + 8;
  return (size_t)(kSlotBytes * slots + kPatchBytes * (int64_t)(n_patches + 1));
}

extern "C" int ts_triangulate(const double* d_xy, const int64_t* d_pts_off,
                              int n_patches, int32_t* d_tri, int32_t* d_ntri,
                              int32_t* d_status, void* d_scratch, void* stream) {
  if (n_patches <= 0) return TS_OK;
  if (!d_scratch) return TS_E_INVALID;
  // per call: the attribute is per device (one process may drive several)
  TS_CUDA_TRY(cudaFuncSetAttribute(delaunay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kDelaunaySmem));
  TS_CUDA_TRY(cudaFuncSetAttribute(delaunay_kernel,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  ts::count_launch(),
      delaunay_kernel<<<n_patches, 32, kDelaunaySmem, as_stream(stream)>>>(
          d_xy, d_pts_off, n_patches, d_tri, d_ntri, d_status,
          reinterpret_cast<uint8_t*>(d_scratch));
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" int ts_incircle_sign(const double a[2], const double b[2],
                                const double c[2], const double d[2]) {
  return pred::incircle(a[0], a[1], b[0], b[1], c[0], c[1], d[0], d[1]);
}

extern "C" int ts_orient_sign(const double a[2], const double b[2],
                              const double c[2]) {
  return pred::orient(a[0], a[1], b[0], b[1], c[0], c[1]);
}

namespace ts {
namespace {
__global__ void predicate_kernel(const double* __restrict__ in, int64_t n, int mode,
                                 int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* p = in + 8 * i;
    out[i] = mode == 0 ? pred::orient(p[0], p[1], p[2], p[3], p[4], p[5])
                       : pred::incircle(p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7]);
  }
}
}  // namespace
}  // namespace ts

extern "C" int ts_predicates_device(const double* d_in, int64_t n, int mode,
                                    int32_t* d_out, void* stream) {
  if (n <= 0) return TS_OK;
  ts::count_launch(), predicate_kernel<<<(int)ceil_div<int64_t>(n, 128), 128, 0, as_stream(stream)>>>(
      d_in, n, mode, d_out);
  TS_LAUNCH_CHECK();
  return TS_OK;
}
