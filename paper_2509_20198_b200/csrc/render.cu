// Rendering kernels: points and refined heightmaps
// into a 64-bit min-key framebuffer, and its resolve to RGBA8.
//
// Replaces render.py:55-98 (rasterize_points), :101-239 (patch_mesh,
// _TriangleRaster, rasterize_heightmaps: small / large triangle paths) and
// :254-268 (resolve), with the camera math of geometry.py:71-102.
//
// Every fragment is key = depth_key(eye depth) << 32 | 0xRRGGBBAA and a
// cell keeps the minimum key (atomicMin on u64), so the image does not
// depend on submission order or thread count -- the reference's
// determinism contract.  Arithmetic follows the reference's numpy
// expressions operation by operation (compiled without FMA contraction);
// the eye-space dot products are evaluated as (d0 r0 + d1 r1) + d2 r2.
//
// Heightmaps: one CTA per patch projects its 64 x 64 vertices into shared
// memory and walks its 7,938 triangles; triangles whose clipped bounding
// box covers fewer than 1,024 pixels are filled by one thread, larger ones
// are queued and filled by a whole CTA each afterwards (the reference's
// two paths, identical per-pixel arithmetic).
#include <stdint.h>

#include <algorithm>

#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int kPRes = 64;  // OUTPUT_RES vertices per side
constexpr int kTris = 2 * (kPRes - 1) * (kPRes - 1);
constexpr int kLargePixels = 1024;
constexpr int kPatchThreads = 256;

__device__ __forceinline__ double dot3(const double d[3], const double* v) {
  return dadd(dadd(dmul(d[0], v[0]), dmul(d[1], v[1])), dmul(d[2], v[2]));
}

// geometry.py:78-102: project + depth_key
struct Proj {
  double px, py, ze;
};
__device__ __forceinline__ Proj project(const ts_camera& c, double x, double y, double z) {
  const double d[3] = {dsub(x, c.pos[0]), dsub(y, c.pos[1]), dsub(z, c.pos[2])};
  const double xe = dot3(d, c.right), ye = dot3(d, c.up), ze = dot3(d, c.fwd);
  const double ndc_x = ddiv(dmul(xe, c.f_over_aspect), ze);
  const double ndc_y = ddiv(dmul(ye, c.f), ze);
  Proj p;
  p.px = dmul(dadd(dmul(ndc_x, 0.5), 0.5), (double)c.width);
  p.py = dmul(dsub(0.5, dmul(ndc_y, 0.5)), (double)c.height);
  p.ze = ze;
  return p;
}
__device__ __forceinline__ uint64_t depth_key(const ts_camera& c, double depth) {
  const double inv_n = ddiv(1.0, c.near), inv_f = ddiv(1.0, c.far);
  const double z = fmin(fmax(depth, c.near), c.far);
  const double norm = ddiv(dsub(inv_n, ddiv(1.0, z)), dsub(inv_n, inv_f));
  return (uint64_t)dmul(norm, 4294967294.0);  // numpy astype: truncation
}

// pack_color (render.py:44-49) of float32 rgb: float32 arithmetic
__device__ __forceinline__ uint32_t pack_f32(float r, float g, float b) {
  auto q = [](float v) -> uint32_t {
    const float t = __fadd_rn(__fmul_rn(v, 255.0f), 0.5f);
    const float cl = fminf(fmaxf(t, 0.0f), 255.0f);
    return (uint32_t)cl;
  };
  return (q(r) << 24) | (q(g) << 16) | (q(b) << 8) | 0xFFu;
}
// pack_color of float64 rgb (the shaded path)
__device__ __forceinline__ uint32_t pack_f64(double v3) {
  const double t = dadd(dmul(v3, 255.0), 0.5);
  const uint32_t q = (uint32_t)fmin(fmax(t, 0.0), 255.0);
  return (q << 24) | (q << 16) | (q << 8) | 0xFFu;
}

__global__ void render_points_kernel(const double* __restrict__ xyz,
                                     const float* __restrict__ rgb, int64_t n, ts_camera c,
                                     uint32_t grey, unsigned long long* fb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Proj p = project(c, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    if (!(p.ze > c.near && p.ze <= c.far)) continue;
    const double fx = floor(p.px), fy = floor(p.py);
    if (!(fx >= 0.0 && fx < (double)c.width && fy >= 0.0 && fy < (double)c.height)) continue;
    const uint32_t col = rgb ? pack_f32(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]) : grey;
    const unsigned long long key = (depth_key(c, p.ze) << 32) | col;
    atomicMin(fb + (int64_t)fy * c.width + (int64_t)fx, key);
  }
}

// One queued large triangle (screen-space setup of _TriangleRaster)
struct BigTri {
  double vx[3], vy[3], vz[3], d;
  int x0, x1, y0, y1;
  uint32_t color;
};

__device__ __forceinline__ void fragment(const ts_camera& c, const double* vx, const double* vy,
                                         const double* vz, double d, int ix, int iy,
                                         uint32_t color, unsigned long long* fb) {
  // _TriangleRaster._row (render.py:128-145) at pixel centre (ix+.5, iy+.5)
  const double px = dadd((double)ix, 0.5), py = dadd((double)iy, 0.5);
  const double w0 = ddiv(dadd(dmul(dsub(vy[1], vy[2]), dsub(px, vx[2])),
                              dmul(dsub(vx[2], vx[1]), dsub(py, vy[2]))), d);
  const double w1 = ddiv(dadd(dmul(dsub(vy[2], vy[0]), dsub(px, vx[2])),
                              dmul(dsub(vx[0], vx[2]), dsub(py, vy[2]))), d);
  const double w2 = dsub(dsub(1.0, w0), w1);
  if (!(w0 >= 0.0 && w1 >= 0.0 && w2 >= 0.0)) return;
  const double iz = dadd(dadd(dmul(w0, vz[0]), dmul(w1, vz[1])), dmul(w2, vz[2]));
  if (!(iz > 0.0)) return;
  const unsigned long long key = (depth_key(c, ddiv(1.0, iz)) << 32) | color;
  atomicMin(fb + (int64_t)iy * c.width + ix, key);
}

__global__ void __launch_bounds__(kPatchThreads)
render_patches_kernel(const float* __restrict__ heights, const float* __restrict__ rgb,
                      const uint8_t* __restrict__ has_rgb, const double* __restrict__ center,
                      const double* __restrict__ cz, ts_camera c, unsigned long long* fb,
                      BigTri* queue, uint32_t* queue_n, uint32_t queue_cap) {
  extern __shared__ __align__(16) double s_dyn[];
  double* s_px = s_dyn;                 // [4096] projected vertices
  double* s_py = s_px + kPRes * kPRes;
  double* s_iz = s_py + kPRes * kPRes;
  uint8_t* s_front = reinterpret_cast<uint8_t*>(s_iz + kPRes * kPRes);
  __shared__ double s_min[kPatchThreads / 32], s_max[kPatchThreads / 32];
  const int p = blockIdx.x;
  const float* hr = heights + (size_t)p * kPRes * kPRes;
  const double x0 = dsub(center[2 * p], 320.0), y0 = dsub(center[2 * p + 1], 320.0);
  const double c_z = cz[p];
  double lo = 1e300, hi = -1e300;
  for (int v = threadIdx.x; v < kPRes * kPRes; v += kPatchThreads) {
    // patch_mesh (render.py:101-120): texel-centre grid, hm = heights_rel + c_z
    const int iy = v / kPRes, ix = v - iy * kPRes;
    const double gx = dadd(x0, dmul(dadd((double)ix, 0.5), 10.0));
    const double gy = dadd(y0, dmul(dadd((double)iy, 0.5), 10.0));
    const double hm = dadd((double)hr[v], c_z);
    lo = fmin(lo, hm);
    hi = fmax(hi, hm);
    const Proj pr = project(c, gx, gy, hm);
    const bool front = pr.ze > c.near;
    s_px[v] = pr.px;
    s_py[v] = pr.py;
    s_front[v] = front;
    s_iz[v] = front ? ddiv(1.0, fmax(pr.ze, 1e-12)) : -1.0;
  }
  // hm.min() / np.ptp(hm) for the shaded colour path
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { s_min[threadIdx.x >> 5] = lo; s_max[threadIdx.x >> 5] = hi; }
  __syncthreads();
  lo = s_min[0];
  hi = s_max[0];
  for (int w = 1; w < kPatchThreads / 32; ++w) { lo = fmin(lo, s_min[w]); hi = fmax(hi, s_max[w]); }
  const double ptp = fmax(dsub(hi, lo), 1e-9);
  const bool colour = has_rgb && has_rgb[p];
  const float* cr = rgb + (size_t)p * kPRes * kPRes * 3;
  for (int t = threadIdx.x; t < kTris; t += kPatchThreads) {
    // tris = [a b c] for every quad, then [b d c] (render.py:112-118)
    const int q = t < kTris / 2 ? t : t - kTris / 2;
    const int qy = q / (kPRes - 1), qx = q - qy * (kPRes - 1);
    const int a = qy * kPRes + qx, b = a + 1, cc = a + kPRes, dd = cc + 1;
    int vi[3];
    if (t < kTris / 2) { vi[0] = a; vi[1] = b; vi[2] = cc; }
    else { vi[0] = b; vi[1] = dd; vi[2] = cc; }
    if (!(s_front[vi[0]] && s_front[vi[1]] && s_front[vi[2]])) continue;
    double vx[3], vy[3], vz[3];
    for (int k = 0; k < 3; ++k) { vx[k] = s_px[vi[k]]; vy[k] = s_py[vi[k]]; vz[k] = s_iz[vi[k]]; }
    const double mnx = fmin(fmin(vx[0], vx[1]), vx[2]), mxx = fmax(fmax(vx[0], vx[1]), vx[2]);
    const double mny = fmin(fmin(vy[0], vy[1]), vy[2]), mxy = fmax(fmax(vy[0], vy[1]), vy[2]);
    const double xl = fmax(floor(mnx), 0.0), yl = fmax(floor(mny), 0.0);
    const double xh = fmin(dsub(ceil(mxx), 1.0), (double)(c.width - 1));
    const double yh = fmin(dsub(ceil(mxy), 1.0), (double)(c.height - 1));
    if (!(xh >= xl && yh >= yl)) continue;
    const int x_lo = (int)xl, x_hi = (int)xh, y_lo = (int)yl, y_hi = (int)yh;
    const double d = dadd(dmul(dsub(vy[1], vy[2]), dsub(vx[0], vx[2])),
                          dmul(dsub(vx[2], vx[1]), dsub(vy[0], vy[2])));
    if (d == 0.0) continue;
    uint32_t color;
    const int qv = qy * kPRes + qx;  // quad colour: rgb[:-1, :-1]
    if (colour) {
      color = pack_f32(cr[3 * qv], cr[3 * qv + 1], cr[3 * qv + 2]);
    } else {
      const double hm = dadd((double)hr[qv], c_z);
      const double shade =
          fmin(fmax(dadd(0.35, ddiv(dmul(0.5, dsub(hm, lo)), ptp)), 0.0), 1.0);
      color = pack_f64(shade);
    }
    const int64_t pixels = (int64_t)(x_hi - x_lo + 1) * (y_hi - y_lo + 1);
    if (pixels < kLargePixels) {
      for (int iy = y_lo; iy <= y_hi; ++iy)
        for (int ix = x_lo; ix <= x_hi; ++ix) fragment(c, vx, vy, vz, d, ix, iy, color, fb);
    } else {
      const uint32_t slot = atomicAdd(queue_n, 1u);
      if (slot < queue_cap) {
        BigTri& bt = queue[slot];
        for (int k = 0; k < 3; ++k) { bt.vx[k] = vx[k]; bt.vy[k] = vy[k]; bt.vz[k] = vz[k]; }
        bt.d = d;
        bt.x0 = x_lo; bt.x1 = x_hi; bt.y0 = y_lo; bt.y1 = y_hi;
        bt.color = color;
      }
    }
  }
}

// the queued large triangles: one CTA per triangle, threads over its box
__global__ void render_big_kernel(ts_camera c, const BigTri* queue, const uint32_t* queue_n,
                                  unsigned long long* fb) {
  const uint32_t n = *queue_n;
  for (uint32_t t = blockIdx.x; t < n; t += gridDim.x) {
    const BigTri bt = queue[t];
    const int w = bt.x1 - bt.x0 + 1;
    const int64_t pixels = (int64_t)w * (bt.y1 - bt.y0 + 1);
    for (int64_t k = threadIdx.x; k < pixels; k += blockDim.x) {
      const int iy = bt.y0 + (int)(k / w), ix = bt.x0 + (int)(k % w);
      fragment(c, bt.vx, bt.vy, bt.vz, bt.d, ix, iy, bt.color, fb);
    }
  }
}

__global__ void resolve_kernel(const unsigned long long* __restrict__ fb, int64_t n,
                               ts_srgb_lut lut, uint32_t bg, uint32_t* __restrict__ img) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = fb[i];
    uint32_t o;
    if (k == 0xFFFFFFFFFFFFFFFFull) {
      o = bg;
    } else {
      const uint32_t col = (uint32_t)k;
      o = (uint32_t)lut.v[(col >> 24) & 0xFF] | ((uint32_t)lut.v[(col >> 16) & 0xFF] << 8) |
          ((uint32_t)lut.v[(col >> 8) & 0xFF] << 16) | 0xFF000000u;
    }
    img[i] = o;  // RGBA bytes in memory order
  }
}

// projected_bbox_area (geometry.py:128-164) for many boxes: 0 when all
// eight corners are behind one frustum plane, else the screen-space AABB
// of the corners (depth clamped to near) -> (area, diagonal)
__global__ void bbox_area_kernel(const double* __restrict__ boxes, int64_t n, ts_camera c,
                                 ts_frustum fr, double* __restrict__ area,
                                 double* __restrict__ diag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* b = boxes + 6 * i;
    double cx[8], cy[8], cz[8];
    for (int k = 0; k < 8; ++k) {  // meshgrid(..., indexing="ij") corner order
      cx[k] = b[(k >> 2) & 1 ? 3 : 0];
      cy[k] = b[(k >> 1) & 1 ? 4 : 1];
      cz[k] = b[k & 1 ? 5 : 2];
    }
    bool outside = false;
    for (int p = 0; p < 6 && !outside; ++p) {
      bool all_behind = true;
      for (int k = 0; k < 8; ++k) {
        const double v = dadd(dadd(dadd(dmul(cx[k], fr.plane[p][0]), dmul(cy[k], fr.plane[p][1])),
                                   dmul(cz[k], fr.plane[p][2])),
                              fr.plane[p][3]);
        all_behind = all_behind && v < 0.0;
      }
      outside = all_behind;
    }
    if (outside) {
      area[i] = 0.0;
      diag[i] = 0.0;
      continue;
    }
    double xlo = 1e308, xhi = -1e308, ylo = 1e308, yhi = -1e308;
    for (int k = 0; k < 8; ++k) {
      const double d[3] = {dsub(cx[k], c.pos[0]), dsub(cy[k], c.pos[1]), dsub(cz[k], c.pos[2])};
      const double xe = dot3(d, c.right), ye = dot3(d, c.up);
      const double ze = fmax(dot3(d, c.fwd), c.near);
      const double px = dmul(dadd(dmul(ddiv(dmul(xe, c.f_over_aspect), ze), 0.5), 0.5),
                             (double)c.width);
      const double py = dmul(dsub(0.5, dmul(ddiv(dmul(ye, c.f), ze), 0.5)), (double)c.height);
      xlo = fmin(xlo, px); xhi = fmax(xhi, px);
      ylo = fmin(ylo, py); yhi = fmax(yhi, py);
    }
    const double w = dsub(xhi, xlo), h = dsub(yhi, ylo);
    area[i] = dmul(w, h);
    diag[i] = hypot(w, h);
  }
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" int ts_bbox_areas(const double* d_boxes, int64_t n, const ts_camera* cam,
                             const ts_frustum* frustum, double* d_area, double* d_diag,
                             void* stream) {
  if (!cam || !frustum || n < 0) return TS_E_INVALID;
  if (n == 0) return TS_OK;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 148 * 16);
  ts::count_launch(), bbox_area_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      d_boxes, n, *cam, *frustum, d_area, d_diag);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" int ts_render_points(const double* d_xyz, const float* d_rgb, int64_t n,
                                const ts_camera* cam, uint32_t grey_color, uint64_t* d_fb,
                                void* stream) {
  if (!cam || n < 0 || cam->width <= 0 || cam->height <= 0) return TS_E_INVALID;
  if (n == 0) return TS_OK;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 148 * 16);
  ts::count_launch(), render_points_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      d_xyz, d_rgb, n, *cam, grey_color, reinterpret_cast<unsigned long long*>(d_fb));
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" size_t ts_render_heightmaps_scratch(int n_patches) {
  return 256 + (size_t)(n_patches > 0 ? n_patches : 1) * kTris * sizeof(BigTri);
}

extern "C" int ts_render_heightmaps(const float* d_heights, const float* d_rgb,
                                    const uint8_t* d_has_rgb, const double* d_center,
                                    const double* d_cz, int n_patches, const ts_camera* cam,
                                    uint64_t* d_fb, void* d_scratch, void* stream) {
  if (!cam || n_patches < 0 || cam->width <= 0 || cam->height <= 0) return TS_E_INVALID;
  if (n_patches == 0) return TS_OK;
  cudaStream_t s = as_stream(stream);
  uint32_t* queue_n = reinterpret_cast<uint32_t*>(d_scratch);
  BigTri* queue = reinterpret_cast<BigTri*>(reinterpret_cast<uint8_t*>(d_scratch) + 256);
  TS_CUDA_TRY(cudaMemsetAsync(queue_n, 0, sizeof(uint32_t), s));
  auto* fb = reinterpret_cast<unsigned long long*>(d_fb);
  const int smem = kPRes * kPRes * (3 * sizeof(double) + 1);
  TS_CUDA_TRY(cudaFuncSetAttribute(render_patches_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  ts::count_launch(), render_patches_kernel<<<n_patches, kPatchThreads, smem, s>>>(
      d_heights, d_rgb, d_has_rgb, d_center, d_cz, *cam, fb, queue, queue_n,
      (uint32_t)((size_t)n_patches * kTris));
  ts::count_launch(), render_big_kernel<<<148 * 4, 256, 0, s>>>(*cam, queue, queue_n, fb);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

extern "C" int ts_render_resolve(const uint64_t* d_fb, int64_t n_cells, const ts_srgb_lut* lut,
                                 const uint8_t background[3], uint8_t* d_rgba, void* stream) {
  if (!lut || n_cells < 0) return TS_E_INVALID;
  if (n_cells == 0) return TS_OK;
  const uint32_t bg = (uint32_t)lut->v[background[0]] | ((uint32_t)lut->v[background[1]] << 8) |
                      ((uint32_t)lut->v[background[2]] << 16) | 0xFF000000u;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n_cells, 256), 148 * 16);
  ts::count_launch(), resolve_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const unsigned long long*>(d_fb), n_cells, *lut, bg,
      reinterpret_cast<uint32_t*>(d_rgba));
  TS_LAUNCH_CHECK();
  return TS_OK;
}
