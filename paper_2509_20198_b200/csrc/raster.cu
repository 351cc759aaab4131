// K2b: Algorithm 1 rasterisation of one patch per CTA.
//
// Replaces interpolate_patch after the triangulation
// (patches.py:306-405):
//   * NN raster: exact d^2 = dx*dx + dy*dy argmin over the patch points,
//     strict '<' so the lowest index wins ties (_nn_assign, :180-199);
//   * face map: every triangle's clipped cell bbox (_cell_range, :283-287)
//     is tested with the _TriGeom barycentric formulas and 1e-9 tolerance
//     (:227-253); the lowest triangle id claims a cell (what the two flood
//     fill passes :330-349 compute; pinned by test_acceptance.py:165-191);
//   * padding-triangle blanking (:351-358), barycentric hm/rgb (:360-380),
//     re-centring on cell [48,48] and the float32 casts (_finish :386-405).
// Triangles are _ccw-normalised here (:215-224) so Qhull simplices can be
// fed in as well as ts_triangulate output.  Compiled with --fmad=false and
// explicit _rn intrinsics: every fp64 op rounds like numpy.
//
// Work split: the face map is rasterised over a flattened (triangle, cell)
// index space so one huge padding triangle does not serialise a thread; the
// NN search keeps the patch points in shared memory and scans them for
// four cells at a time.
#include <cfloat>
#include <climits>

#include "tc_ptx.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int kThreads = 256;
constexpr int kCells = kRes * kRes;
constexpr int kSmemPts = 384;          // points cached in shared memory (4 CTAs per SM)
constexpr int kSmemTri = 2 * kSmemPts + 8;
constexpr int kBins = 16;              // NN bin grid over [-1,1]^2

struct Tri {
  int v0, v1, v2;
};

struct Geo {
  double ax, ay, abx, aby, acx, acy, inv;
};

template <typename PT>
__device__ __forceinline__ void vtx(const PT* xy, int n, int v, double& x,
                                    double& y) {
  if (v < n) { x = xy[2 * v]; y = xy[2 * v + 1]; }
  else {
    const int c = v - n;
    x = (c & 1) ? 1.0 : -1.0;
    y = (c & 2) ? 1.0 : -1.0;
  }
}

// _ccw (patches.py:215-224) then _TriGeom (:230-239)
template <typename PT>
__device__ __forceinline__ Geo tri_geo(const PT* xy, int n, Tri& t) {
  double ax, ay, bx, by, cx, cy;
  vtx(xy, n, t.v0, ax, ay);
  vtx(xy, n, t.v1, bx, by);
  vtx(xy, n, t.v2, cx, cy);
  const double d = dsub(dmul(dsub(bx, ax), dsub(cy, ay)),
                        dmul(dsub(by, ay), dsub(cx, ax)));
  if (d < 0.0) {
    const int tmp = t.v1; t.v1 = t.v2; t.v2 = tmp;
    double tx = bx, ty = by;
    bx = cx; by = cy; cx = tx; cy = ty;
  }
  Geo g;
  g.ax = ax; g.ay = ay;
  g.abx = dsub(bx, ax); g.aby = dsub(by, ay);
  g.acx = dsub(cx, ax); g.acy = dsub(cy, ay);
  double det = dsub(dmul(g.abx, g.acy), dmul(g.aby, g.acx));
  if (det == 0.0) det = INFINITY;  // patches.py:238 -> inv_det = 0
  g.inv = ddiv(1.0, det);
  return g;
}

__device__ __forceinline__ void bary(const Geo& g, double qx, double qy,
                                     double& w0, double& w1, double& w2) {
  const double px = dsub(qx, g.ax), py = dsub(qy, g.ay);
  w1 = dmul(dsub(dmul(px, g.acy), dmul(py, g.acx)), g.inv);
  w2 = dmul(dsub(dmul(g.abx, py), dmul(g.aby, px)), g.inv);
  w0 = dsub(dsub(1.0, w1), w2);
}

__device__ __forceinline__ bool contains(const Geo& g, double qx, double qy) {
  double w0, w1, w2;
  bary(g, qx, qy, w0, w1, w2);
  const double lo = -kBaryTol, hi = 1.0 + kBaryTol;
  return w0 >= lo && w0 <= hi && w1 >= lo && w1 <= hi && w2 >= lo && w2 <= hi;
}

// _cell_range (patches.py:283-287) for res = 96
__device__ __forceinline__ void cell_range(double lo, double hi, int& a, int& b) {
  const double r = (double)kRes;
  a = (int)ceil(dsub(ddiv(dmul(dadd(lo, 1.0), r), 2.0), 0.5));
  b = (int)floor(dsub(ddiv(dmul(dadd(hi, 1.0), r), 2.0), 0.5));
  a = a < 0 ? 0 : a;
  b = b > kRes - 1 ? kRes - 1 : b;
}

struct RasterArgs {
  const double* xy;
  const double* h;
  const float* prgb;
  const int64_t* pts_off;
  const int32_t* tri;
  const int64_t* tri_off;
  const int32_t* ntri;
  const double* cz_in;
  int recenter;
  float* cnn_in;
  float* hm_nn;
  float* hm_lin;
  float* rgb_nn;
  float* rgb_lin;
  int32_t* face;
  double* cz_out;
  int32_t* status;
};

__global__ void __launch_bounds__(kThreads, 4)
raster_kernel(RasterArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  int* s_face = reinterpret_cast<int*>(smem);                       // 9216
  double* s_xy = reinterpret_cast<double*>(s_face + kCells);        // 2*512
  double* s_h = s_xy + 2 * kSmemPts;                                // 512
  int* s_pref = reinterpret_cast<int*>(s_h + kSmemPts);             // 1033
  uint32_t* s_rng = reinterpret_cast<uint32_t*>(s_pref + kSmemTri + 1);  // 1032
  int* s_bstart = reinterpret_cast<int*>(s_rng + kSmemTri);  // kBins^2 + 1
  short* s_bid = reinterpret_cast<short*>(s_bstart + kBins * kBins + 2);  // kSmemPts
  // bin-ordered copy of the cached points for the NN search; aliases
  // s_pref / s_rng, which are dead once the face map is done (>= 6,144 B,
  // 16-byte aligned)
  double2* s_bxy = reinterpret_cast<double2*>(s_pref);
  static_assert(sizeof(int) * (2 * kSmemTri + 1) >= sizeof(double2) * kSmemPts, "s_bxy alias");
  __shared__ double s_shift;
  __shared__ int s_total;
  __shared__ int s_wsum[kThreads / 32];
  __shared__ int s_cur[kThreads];

  const int p = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t off = A.pts_off[p];
  const int n = (int)(A.pts_off[p + 1] - off);
  if (n == 0) {
    if (tid == 0) {
      A.status[p] = TS_E_EMPTY_PATCH;
      if (A.cz_out) A.cz_out[p] = 0.0;
    }
    return;
  }
  const bool cached = n <= kSmemPts;
  const double* g_xy = A.xy + 2 * off;
  const double* g_h = A.h + off;
  const float* g_rgb = A.prgb ? A.prgb + 3 * off : nullptr;
  for (int i = tid; i < kCells; i += kThreads) s_face[i] = INT_MAX;
  if (cached) {
    for (int i = tid; i < n; i += kThreads) {
      s_xy[2 * i] = g_xy[2 * i];
      s_xy[2 * i + 1] = g_xy[2 * i + 1];
      s_h[i] = g_h[i];
    }
  }
  const double* xy = cached ? s_xy : g_xy;
  const double* hh = cached ? s_h : g_h;
  const int T = A.ntri ? A.ntri[p] : 0;
  const int32_t* tri = A.tri + A.tri_off[p];
  const bool tri_cached = T <= kSmemTri;
  __syncthreads();

  // ---- face map: lowest triangle id wins ----
  if (tri_cached) {
    // per-triangle clipped cell ranges + flattened work prefix
    int local = 0;
    const int per = ceil_div(T, kThreads);
    const int t0 = tid * per, t1 = min(T, t0 + per);
    for (int t = t0; t < t1; ++t) {
      Tri tr{tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
      double x[3], y[3];
      vtx(xy, n, tr.v0, x[0], y[0]);
      vtx(xy, n, tr.v1, x[1], y[1]);
      vtx(xy, n, tr.v2, x[2], y[2]);
      const double xl = fmax(fmin(fmin(x[0], x[1]), x[2]), -1.0);
      const double xh = fmin(fmax(fmax(x[0], x[1]), x[2]), 1.0);
      const double yl = fmax(fmin(fmin(y[0], y[1]), y[2]), -1.0);
      const double yh = fmin(fmax(fmax(y[0], y[1]), y[2]), 1.0);
      int gx0, gx1, gy0, gy1;
      cell_range(xl, xh, gx0, gx1);
      cell_range(yl, yh, gy0, gy1);
      int cnt = 0;
      if (gx1 >= gx0 && gy1 >= gy0) cnt = (gx1 - gx0 + 1) * (gy1 - gy0 + 1);
      else { gx0 = gy0 = 0; gx1 = gy1 = -1; }
      s_rng[t] = (uint32_t)gx0 | ((uint32_t)(gx1 - gx0 + 1) << 8) |
                 ((uint32_t)gy0 << 16);
      s_pref[t] = cnt;  // temporarily the count
      local += cnt;
    }
    // block exclusive scan of per-thread totals
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((tid & 31) >= o) incl += v;
    }
    if ((tid & 31) == 31) s_wsum[tid >> 5] = incl;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < (tid >> 5); ++w) wbase += s_wsum[w];
    if (tid == kThreads - 1) s_total = wbase + incl;
    int run = wbase + incl - local;
    for (int t = t0; t < t1; ++t) {
      const int c = s_pref[t];
      s_pref[t] = run;
      run += c;
    }
    __syncthreads();
    if (tid == 0) s_pref[T] = s_total;
    __syncthreads();
    // each thread takes one contiguous run of the flattened (triangle, cell)
    // items: one binary search, then a forward walk that rebuilds a
    // triangle's geometry only when the run crosses into the next triangle
    const int total = s_total;
    const int per_w = ceil_div(total, kThreads);
    const int w0 = tid * per_w, w1 = min(total, w0 + per_w);
    if (w0 < w1) {
      int lo = 0, hi = T;  // largest t with s_pref[t] <= w0
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pref[mid] <= w0) lo = mid; else hi = mid;
      }
      int t = lo;
      while (t + 1 < T && s_pref[t + 1] <= w0) ++t;  // skip empty triangles
      Tri tr{tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
      Geo g = tri_geo(xy, n, tr);
      for (int w = w0; w < w1; ++w) {
        if (w >= s_pref[t + 1]) {
          do { ++t; } while (w >= s_pref[t + 1]);
          tr = Tri{tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
          g = tri_geo(xy, n, tr);
        }
        const uint32_t rg = s_rng[t];
        const int width = (rg >> 8) & 0xFF;
        const int k = w - s_pref[t];
        const int gy = (int)(rg >> 16) + k / width;
        const int gx = (int)(rg & 0xFF) + k % width;
        if (contains(g, cell_center(gx, kRes), cell_center(gy, kRes)))
          atomicMin(&s_face[gy * kRes + gx], t);
      }
    }
  } else {
    for (int t = tid; t < T; t += kThreads) {
      Tri tr{tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
      double x[3], y[3];
      vtx(xy, n, tr.v0, x[0], y[0]);
      vtx(xy, n, tr.v1, x[1], y[1]);
      vtx(xy, n, tr.v2, x[2], y[2]);
      int gx0, gx1, gy0, gy1;
      cell_range(fmax(fmin(fmin(x[0], x[1]), x[2]), -1.0),
                 fmin(fmax(fmax(x[0], x[1]), x[2]), 1.0), gx0, gx1);
      cell_range(fmax(fmin(fmin(y[0], y[1]), y[2]), -1.0),
                 fmin(fmax(fmax(y[0], y[1]), y[2]), 1.0), gy0, gy1);
      const Geo g = tri_geo(xy, n, tr);
      for (int gy = gy0; gy <= gy1; ++gy)
        for (int gx = gx0; gx <= gx1; ++gx)
          if (contains(g, cell_center(gx, kRes), cell_center(gy, kRes)))
            atomicMin(&s_face[gy * kRes + gx], t);
    }
  }
  __syncthreads();

  // ---- per-cell values ----
  auto cell_value = [&](int j, int nn, double& hl, double* rl, int& f) {
    f = s_face[j];
    hl = hh[nn];
    if (g_rgb) {
      rl[0] = g_rgb[3 * nn]; rl[1] = g_rgb[3 * nn + 1]; rl[2] = g_rgb[3 * nn + 2];
    }
    if (f == INT_MAX) { f = -1; return; }
    Tri tr{tri[3 * f], tri[3 * f + 1], tri[3 * f + 2]};
    const Geo g = tri_geo(xy, n, tr);
    if (tr.v0 >= n || tr.v1 >= n || tr.v2 >= n) { f = -1; return; }
    double w0, w1, w2;
    bary(g, cell_center(j % kRes, kRes), cell_center(j / kRes, kRes), w0, w1, w2);
    hl = dadd(dadd(dmul(w0, hh[tr.v0]), dmul(w1, hh[tr.v1])), dmul(w2, hh[tr.v2]));
    if (g_rgb) {
      for (int c = 0; c < 3; ++c)
        rl[c] = dadd(dadd(dmul(w0, (double)g_rgb[3 * tr.v0 + c]),
                          dmul(w1, (double)g_rgb[3 * tr.v1 + c])),
                     dmul(w2, (double)g_rgb[3 * tr.v2 + c]));
    }
  };
  // Exact nearest neighbour (patches.py:180-199): the d^2 formula and the
  // lowest-index tie rule of a linear scan; with points cached in shared
  // memory they are binned on a 16x16 grid and searched ring by ring until
  // the next ring's lower bound exceeds the best d^2 (with a 1e-12 relative
  // safety margin, so ties on the bound are still visited).
  auto bin_of = [](double v) {
    int b = (int)floor((v + 1.0) * (kBins / 2));
    return b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
  };
  auto nn_of = [&](double qx, double qy) {
    double best = DBL_MAX;
    int bi = 0;
    if (!cached) {
      for (int i = 0; i < n; ++i) {
        const double dx = dsub(qx, xy[2 * i]), dy = dsub(qy, xy[2 * i + 1]);
        const double d2 = dadd(dmul(dx, dx), dmul(dy, dy));
        if (d2 < best) { best = d2; bi = i; }
      }
      return bi;
    }
    const int bx = bin_of(qx), by = bin_of(qy);
    const double hb = 2.0 / kBins;
    for (int r = 0; r < kBins; ++r) {
      const int x0 = max(bx - r, 0), x1 = min(bx + r, kBins - 1);
      const int y0 = max(by - r, 0), y1 = min(by + r, kBins - 1);
      for (int gy = y0; gy <= y1; ++gy) {
        const bool edge_row = (gy == by - r) || (gy == by + r);
        for (int gx = x0; gx <= x1; ++gx) {
          if (!edge_row && gx != bx - r && gx != bx + r) continue;  // ring only
          const int b = gy * kBins + gx;
          for (int k = s_bstart[b]; k < s_bstart[b + 1]; ++k) {
            const double2 q = s_bxy[k];  // no id -> coordinate indirection
            const int i = s_bid[k];
            const double dx = dsub(qx, q.x), dy = dsub(qy, q.y);
            const double d2 = dadd(dmul(dx, dx), dmul(dy, dy));
            if (d2 < best || (d2 == best && i < bi)) { best = d2; bi = i; }
          }
        }
      }
      double mind = DBL_MAX;
      if (bx - r > 0) mind = fmin(mind, qx - (-1.0 + (bx - r) * hb));
      if (bx + r < kBins - 1) mind = fmin(mind, (-1.0 + (bx + r + 1) * hb) - qx);
      if (by - r > 0) mind = fmin(mind, qy - (-1.0 + (by - r) * hb));
      if (by + r < kBins - 1) mind = fmin(mind, (-1.0 + (by + r + 1) * hb) - qy);
      if (mind == DBL_MAX) break;                      // every bin visited
      if (best < DBL_MAX && mind * mind > best * (1.0 + 1e-12)) break;
    }
    return bi;
  };
  if (cached) {
    // counting sort of point ids into bins, block-parallel: counts by
    // shared atomics, one 256-bin scan, placement by per-bin cursors (the
    // order inside a bin is free: nn_of breaks d^2 ties by lowest id)
    static_assert(kBins * kBins == kThreads, "one bin per thread in the scan");
    s_bstart[tid + 1] = 0;
    if (tid == 0) s_bstart[0] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kThreads)
      atomicAdd(&s_bstart[bin_of(xy[2 * i + 1]) * kBins + bin_of(xy[2 * i]) + 1], 1);
    __syncthreads();
    {  // inclusive scan of the 256 counts (warp shuffles + warp totals)
      int v = s_bstart[tid + 1];
      const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += y;
      }
      if (lane == 31) s_wsum[wid] = v;
      __syncthreads();
      int base = 0;
      for (int w = 0; w < wid; ++w) base += s_wsum[w];
      __syncthreads();
      const int prev = __shfl_up_sync(0xFFFFFFFFu, v, 1);  // all lanes take part
      s_bstart[tid + 1] = base + v;
      s_cur[tid] = base + (lane ? prev : 0);  // start of bin tid
    }
    __syncthreads();
    for (int i = tid; i < n; i += kThreads) {
      const int b = bin_of(xy[2 * i + 1]) * kBins + bin_of(xy[2 * i]);
      const int slot = atomicAdd(&s_cur[b], 1);
      s_bid[slot] = (short)i;
      s_bxy[slot] = make_double2(xy[2 * i], xy[2 * i + 1]);
    }
    __syncthreads();
  }

  if (tid == 0) {
    double shift = 0.0;
    if (A.recenter) {
      const int j = (kRes / 2) * kRes + kRes / 2;
      double hl, rl[3];
      int f;
      cell_value(j, nn_of(cell_center(kRes / 2, kRes), cell_center(kRes / 2, kRes)),
                 hl, rl, f);
      shift = hl;
    }
    s_shift = shift;
    if (A.cz_out)
      A.cz_out[p] = A.recenter ? dadd(A.cz_in[p], dmul(shift, kRadius)) : A.cz_in[p];
    A.status[p] = TS_OK;
  }
  __syncthreads();
  const double shift = s_shift;

  // Warp-cooperative NN for cached patches: a warp takes an 8 x 4 block of
  // cells, and all its lanes scan the SAME candidate points (the bins under
  // the block, then rings around them, until every lane's best d^2 is below
  // the next ring's bound): no divergence, broadcast shared loads.  Same
  // exact argmin with the lowest-index tie rule.
  const int lane = tid & 31, wid = tid >> 5;
  auto nn_block = [&](int cy0, int cx0) {
    const int cy = cy0 + (lane >> 3), cx = cx0 + (lane & 7);
    const double qx = cell_center(cx, kRes), qy = cell_center(cy, kRes);
    const int bx0 = bin_of(cell_center(cx0, kRes)), bx1 = bin_of(cell_center(cx0 + 7, kRes));
    const int by0 = bin_of(cell_center(cy0, kRes)), by1 = bin_of(cell_center(cy0 + 3, kRes));
    const double hb = 2.0 / kBins;
    double best = DBL_MAX;
    int bi = 0;
    for (int r = 0; r < kBins; ++r) {
      const int X0 = max(bx0 - r, 0), X1 = min(bx1 + r, kBins - 1);
      const int Y0 = max(by0 - r, 0), Y1 = min(by1 + r, kBins - 1);
      // points are in bin order, so a run of bins of one grid row is one
      // contiguous candidate range: a full row of the ring is one range,
      // an inner row its (up to) two edge bins
      auto scan = [&](int k0, int k1) {
#pragma unroll 2
        for (int k = k0; k < k1; ++k) {
          const double2 q = s_bxy[k];  // no id -> coordinate indirection
          const int i = s_bid[k];
          const double dx = dsub(qx, q.x), dy = dsub(qy, q.y);
          const double d2 = dadd(dmul(dx, dx), dmul(dy, dy));
          if (d2 < best || (d2 == best && i < bi)) { best = d2; bi = i; }
        }
      };
      for (int gy = Y0; gy <= Y1; ++gy) {
        const int row = gy * kBins;
        if (r == 0 || gy <= by0 - r || gy >= by1 + r) {
          scan(s_bstart[row + X0], s_bstart[row + X1 + 1]);
        } else {
          if (bx0 - r >= 0) scan(s_bstart[row + bx0 - r], s_bstart[row + bx0 - r + 1]);
          if (bx1 + r < kBins) scan(s_bstart[row + bx1 + r], s_bstart[row + bx1 + r + 1]);
        }
      }
      double mind = DBL_MAX;
      if (bx0 - r > 0) mind = fmin(mind, qx - (-1.0 + (bx0 - r) * hb));
      if (bx1 + r < kBins - 1) mind = fmin(mind, (-1.0 + (bx1 + r + 1) * hb) - qx);
      if (by0 - r > 0) mind = fmin(mind, qy - (-1.0 + (by0 - r) * hb));
      if (by1 + r < kBins - 1) mind = fmin(mind, (-1.0 + (by1 + r + 1) * hb) - qy);
      const bool done = mind == DBL_MAX || (best < DBL_MAX && mind * mind > best * (1.0 + 1e-12));
      if (__all_sync(0xFFFFFFFFu, done)) break;
    }
    return bi;
  };
  constexpr int kBlocksX = kRes / 8, kBlocks = kBlocksX * (kRes / 4);
  const int n_iter = cached ? ceil_div(kBlocks, kThreads / 32) : ceil_div(kCells, 4 * kThreads);
  for (int it = 0; it < n_iter; ++it) {
    int bi[4], jc[4];
    int nu = 4;
    if (cached) {  // one cell per lane of this warp's block
      const int blk = it * (kThreads / 32) + wid;
      nu = 1;
      jc[0] = -1;
      if (blk < kBlocks) {
        const int cy0 = (blk / kBlocksX) * 4, cx0 = (blk % kBlocksX) * 8;
        bi[0] = nn_block(cy0, cx0);
        jc[0] = (cy0 + (lane >> 3)) * kRes + cx0 + (lane & 7);
      }
    } else {
      const int j0 = it * 4 * kThreads + tid;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int jj = min(j0 + u * kThreads, kCells - 1);
        jc[u] = j0 + u * kThreads < kCells ? j0 + u * kThreads : -1;
        bi[u] = nn_of(cell_center(jj % kRes, kRes), cell_center(jj / kRes, kRes));
      }
    }
    for (int u = 0; u < nu; ++u) {
      const int j = jc[u];
      if (j < 0) continue;
      double hl, rl[3] = {0.0, 0.0, 0.0};
      int f;
      cell_value(j, bi[u], hl, rl, f);
      const float fnn = __double2float_rn(dsub(hh[bi[u]], shift));
      const float flin = __double2float_rn(dsub(hl, shift));
      float rn[3] = {0.f, 0.f, 0.f}, rli[3] = {0.f, 0.f, 0.f};
      if (g_rgb) {
        for (int c = 0; c < 3; ++c) {
          rn[c] = g_rgb[3 * bi[u] + c];
          rli[c] = __double2float_rn(rl[c]);
        }
      }
      const int64_t o = (int64_t)p * kCells + j;
      if (A.cnn_in) {
        const float cell[8] = {fnn, flin, rn[0], rn[1], rn[2], rli[0], rli[1], rli[2]};
        tcx::st_v8(A.cnn_in + 8 * o, cell);  // one 32-byte sector per cell
      }
      if (A.hm_nn) A.hm_nn[o] = fnn;
      if (A.hm_lin) A.hm_lin[o] = flin;
      if (A.face) A.face[o] = f;
      if (g_rgb && A.rgb_nn) {
        A.rgb_nn[3 * o] = rn[0]; A.rgb_nn[3 * o + 1] = rn[1]; A.rgb_nn[3 * o + 2] = rn[2];
      }
      if (g_rgb && A.rgb_lin) {
        A.rgb_lin[3 * o] = rli[0]; A.rgb_lin[3 * o + 1] = rli[1];
        A.rgb_lin[3 * o + 2] = rli[2];
      }
    }
  }
}

constexpr size_t kRasterSmem = sizeof(int) * kCells + sizeof(double) * 3 * kSmemPts +
                               sizeof(int) * (kSmemTri + 1) + sizeof(uint32_t) * kSmemTri +
                               sizeof(int) * (kBins * kBins + 2) + sizeof(short) * kSmemPts;

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" int ts_raster(const double* d_xy, const double* d_h, const float* d_prgb,
                         const int64_t* d_pts_off, const int32_t* d_tri,
                         const int64_t* d_tri_off, const int32_t* d_ntri,
                         const double* d_cz_in, int n_patches, int recenter,
                         float* d_cnn_in, float* d_hm_nn, float* d_hm_lin,
                         float* d_rgb_nn, float* d_rgb_lin, int32_t* d_face,
                         double* d_cz_out, int32_t* d_status, void* stream) {
  if (n_patches <= 0) return TS_OK;
  {  // per call: the attribute is per device (one process may drive several)
    TS_CUDA_TRY(cudaFuncSetAttribute(raster_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kRasterSmem));
    TS_CUDA_TRY(cudaFuncSetAttribute(raster_kernel,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
  RasterArgs a{d_xy, d_h, d_prgb, d_pts_off, d_tri, d_tri_off, d_ntri, d_cz_in,
               recenter, d_cnn_in, d_hm_nn, d_hm_lin, d_rgb_nn, d_rgb_lin, d_face,
               d_cz_out, d_status};
  ts::count_launch(), raster_kernel<<<n_patches, kThreads, kRasterSmem, as_stream(stream)>>>(a);
  TS_LAUNCH_CHECK();
  return TS_OK;
}
