// K3 (CUDA-core path): fp32 implicit-GEMM convolution over NHWC views.
//
// Numerics follow refiner.py:330-396 (float32 cross-correlation + bias,
// leaky ReLU 0.01, nearest up2) with fp32 FMA accumulation.  GEMM view:
// M = output pixels of the window (x batch), N = C_out, K = k*k*C_in.
// CTA tile 64x64, K step 16, 4x4 register micro-tile per thread; the A
// tile is gathered im2col-style straight from the (optionally upsampled)
// input, zero outside the image (padding), the B tile from weights packed
// [K][C_out].  Used for layers the tensor-core path does not take and as
// the reference implementation of ts_conv2d.
#include "conv.cuh"
#include <algorithm>

#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256)
conv_simt_kernel(ConvOp op) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN];
  const int tid = threadIdx.x;
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int64_t M = (int64_t)op.batch * wy * wx;
  const int Cin = op.in.C, Cout = op.out.C;
  const int K = op.k * op.k * Cin;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int Hl = op.up2 ? 2 * op.in.H : op.in.H;
  const int Wl = op.up2 ? 2 * op.in.W : op.in.W;

  // this thread's A-load pixel (fixed across the K loop)
  const int am = tid & (BM - 1);
  const int ak = tid >> 6;  // 0..3, rows ak, ak+4, ak+8, ak+12
  const int64_t gm = m0 + am;
  const bool mvalid = gm < M;
  int b = 0, oy = 0, ox = 0;
  if (mvalid) {
    b = (int)(gm / ((int64_t)wy * wx));
    const int r = (int)(gm - (int64_t)b * wy * wx);
    oy = op.oy0 + r / wx;
    ox = op.ox0 + r % wx;
  }
  const int iy0 = oy * op.stride - op.pad, ix0 = ox * op.stride - op.pad;
  const float* inb = op.in.base + (int64_t)b * op.in.H * op.in.W * op.in.cstride + op.in.coff;

  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int kk = ak + 4 * r;
      const int k = k0 + kk;
      float v = 0.f;
      if (mvalid && k < K) {
        const int tap = k / Cin, ci = k - tap * Cin;
        const int ky = tap / op.k, kx = tap - ky * op.k;
        int iy = iy0 + ky, ix = ix0 + kx;
        if (iy >= 0 && iy < Hl && ix >= 0 && ix < Wl) {
          if (op.up2) { iy >>= 1; ix >>= 1; }
          v = inb[((int64_t)iy * op.in.W + ix) * op.in.cstride + ci];
        }
      }
      As[kk][am] = v;
    }
    for (int e = tid; e < BK * BN; e += 256) {
      const int kk = e / BN, nn = e - kk * BN;
      const int k = k0 + kk, n = n0 + nn;
      Bs[kk][nn] = (k < K && n < Cout) ? op.w[(int64_t)k * Cout + n] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
  // epilogue: bias (+ leaky ReLU), scatter to the output window
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gmo = m0 + ty * 4 + i;
    if (gmo >= M) continue;
    const int bo = (int)(gmo / ((int64_t)wy * wx));
    const int r = (int)(gmo - (int64_t)bo * wy * wx);
    const int y = op.oy0 + r / wx, x = op.ox0 + r % wx;
    float* o = op.out.base +
               (((int64_t)bo * op.out.H + y) * op.out.W + x) * op.out.cstride + op.out.coff;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= Cout) continue;
      float v = acc[i][j] + op.bias[n];
      if (op.lrelu) v = v >= 0.f ? v : 0.01f * v;
      o[n] = v;
    }
  }
}

}  // namespace

int launch_conv_simt(const ConvOp& op, void* stream) {
  if (op.in.planes || op.out.planes) return TS_E_INVALID;  // fp32 activations only
  if (op.out.s2d) return TS_E_INVALID;  // s2d outputs: direct / halo2 kernels only
  const int64_t M = (int64_t)op.batch * (op.oy1 - op.oy0) * (op.ox1 - op.ox0);
  if (M <= 0) return TS_OK;
  dim3 grid((unsigned)ceil_div<int64_t>(M, BM), (unsigned)ceil_div(op.out.C, BN));
  ts::count_launch(), conv_simt_kernel<<<grid, 256, 0, as_stream(stream)>>>(op);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

}  // namespace ts

// ---------------------------------------------------------------------------
// Direct convolution for thin layers (C_in <= 4 or C_out <= 16): one thread
// per output pixel keeps every output channel in registers, weights sit in
// shared memory (broadcast reads).  GEMM tiling would waste up to 16x of its
// N tile on these (enc*.0: 1/3 -> 48, fuse.2: 32 -> 4).
//
// A CTA owns an 8 x 16 output tile.  Its input halo ((8-1)s+k rows x
// (16-1)s+k columns x C_in) is staged into shared memory with coalesced
// loads first (zeros outside the image, nearest-up2 folded into the
// address): reading NHWC pixels straight from global memory would put each
// lane on its own cache line (channel-strided rows), which made the kernel
// L1-wavefront bound.  The halo's per-pixel channel pitch is padded so that
// neighbouring lanes hit different banks.
namespace ts {
namespace {

constexpr int kDTY = 8, kDTX = 16, kDThreads = kDTY * kDTX;

struct DirectGeom {
  int HY, HX, Cp;   // staged halo rows, columns, channel pitch (floats)
  int ntx, nty;     // tiles per window row / column
  int tiles;        // batch * nty * ntx
  int vec4;         // 16-byte input loads (C_in % 4 == 0, aligned)
  int halo_off, out_off;  // smem float offsets
};

// EXACT: C_out == CO and k == KS at compile time (the refiner's thin
// layers), so channel predicates fold away and weights load as float4.
template <int CO, bool EXACT, int KS>
__global__ void __launch_bounds__(kDThreads) conv_direct_kernel(ConvOp op, DirectGeom g) {
  extern __shared__ __align__(16) float sw[];
  const int Cin = op.in.C, Cout = EXACT ? CO : op.out.C, k = EXACT ? KS : op.k;
  const int st = op.stride;
  const int K = k * k * Cin;
  for (int i = threadIdx.x; i < K * Cout; i += kDThreads) sw[i] = op.w[i];
  float* sb = sw + K * Cout;
  for (int i = threadIdx.x; i < Cout; i += kDThreads) sb[i] = op.bias[i];
  float* halo = sw + g.halo_off;
  float* so = sw + g.out_off;            // [128][Cs] output staging
  const int Cs = Cout | 1;               // odd row pitch: conflict-free banks
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int Hl = op.up2 ? 2 * op.in.H : op.in.H;
  const int Wl = op.up2 ? 2 * op.in.W : op.in.W;
  const int ty = threadIdx.x / kDTX, tx = threadIdx.x % kDTX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
    const int b = tile / (g.nty * g.ntx);
    const int r = tile - b * g.nty * g.ntx;
    const int y0 = op.oy0 + (r / g.ntx) * kDTY, x0 = op.ox0 + (r % g.ntx) * kDTX;
    const int iy0 = y0 * st - op.pad, ix0 = x0 * st - op.pad;
    const float* inb =
        op.in.base + (int64_t)b * op.in.H * op.in.W * op.in.cstride + op.in.coff;
    __syncthreads();  // previous tile's halo and staging drained
    if (g.vec4) {
      const int n4 = Cin >> 2, n = g.HY * g.HX * n4;
      for (int e = threadIdx.x; e < n; e += kDThreads) {
        const int p = e / n4, q = e - p * n4;
        const int hy = p / g.HX, hx = p - hy * g.HX;
        int iy = iy0 + hy, ix = ix0 + hx;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (iy >= 0 && iy < Hl && ix >= 0 && ix < Wl) {
          if (op.up2) { iy >>= 1; ix >>= 1; }
          v = __ldg(reinterpret_cast<const float4*>(
              inb + ((int64_t)iy * op.in.W + ix) * op.in.cstride + 4 * q));
        }
        *reinterpret_cast<float4*>(halo + p * g.Cp + 4 * q) = v;
      }
    } else {
      const int n = g.HY * g.HX * Cin;
      for (int e = threadIdx.x; e < n; e += kDThreads) {
        const int p = e / Cin, ci = e - p * Cin;
        const int hy = p / g.HX, hx = p - hy * g.HX;
        int iy = iy0 + hy, ix = ix0 + hx;
        float v = 0.f;
        if (iy >= 0 && iy < Hl && ix >= 0 && ix < Wl) {
          if (op.up2) { iy >>= 1; ix >>= 1; }
          v = __ldg(inb + ((int64_t)iy * op.in.W + ix) * op.in.cstride + ci);
        }
        halo[p * g.Cp + ci] = v;
      }
    }
    __syncthreads();
    float acc[CO];
#pragma unroll
    for (int c = 0; c < CO; ++c) acc[c] = 0.f;
#pragma unroll 1
    for (int ky = 0; ky < k; ++ky) {
#pragma unroll 1
      for (int kx = 0; kx < k; ++kx) {
        const float* hp = halo + ((ty * st + ky) * g.HX + tx * st + kx) * g.Cp;
        const float* wt = sw + (ky * k + kx) * Cin * Cout;
        int ci = 0;
        if (EXACT && (CO & 3) == 0) {
          if (g.vec4) {  // wide-input thin layers (fuse3)
            for (; ci < Cin; ci += 4) {
              const float4 x4 = *reinterpret_cast<const float4*>(hp + ci);
              const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4* w4 = reinterpret_cast<const float4*>(wt + (ci + j) * CO);
#pragma unroll
                for (int c = 0; c < CO / 4; ++c) {
                  const float4 w = w4[c];
                  acc[4 * c] = fmaf(xs[j], w.x, acc[4 * c]);
                  acc[4 * c + 1] = fmaf(xs[j], w.y, acc[4 * c + 1]);
                  acc[4 * c + 2] = fmaf(xs[j], w.z, acc[4 * c + 2]);
                  acc[4 * c + 3] = fmaf(xs[j], w.w, acc[4 * c + 3]);
                }
              }
            }
          }
          for (; ci < Cin; ++ci) {
            const float x = hp[ci];
            const float4* w4 = reinterpret_cast<const float4*>(wt + ci * CO);
#pragma unroll
            for (int c = 0; c < CO / 4; ++c) {
              const float4 w = w4[c];
              acc[4 * c] = fmaf(x, w.x, acc[4 * c]);
              acc[4 * c + 1] = fmaf(x, w.y, acc[4 * c + 1]);
              acc[4 * c + 2] = fmaf(x, w.z, acc[4 * c + 2]);
              acc[4 * c + 3] = fmaf(x, w.w, acc[4 * c + 3]);
            }
          }
        }
        if (!EXACT && CO <= 16 && g.vec4) {
          for (; ci < Cin; ci += 4) {
            const float4 x4 = *reinterpret_cast<const float4*>(hp + ci);
            const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int c = 0; c < CO; ++c)
                if (c < Cout) acc[c] = fmaf(xs[j], wt[(ci + j) * Cout + c], acc[c]);
          }
        }
        for (; ci < Cin; ++ci) {
          const float x = hp[ci];
#pragma unroll
          for (int c = 0; c < CO; ++c)
            if (c < Cout) acc[c] = fmaf(x, wt[ci * Cout + c], acc[c]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CO; ++c) {
      if (c < Cout) {
        float v = acc[c] + sb[c];
        if (op.lrelu) v = v >= 0.f ? v : 0.01f * v;
        so[threadIdx.x * Cs + c] = v;
      }
    }
    __syncthreads();
    // coalesced write-back; a tile row's pixels are adjacent in memory
    const int64_t orow = (int64_t)op.out.W * op.out.cstride;
    float* ob = op.out.base + ((int64_t)b * op.out.H + y0) * orow +
                (int64_t)x0 * op.out.cstride + op.out.coff;
    if (op.out.s2d && Cout == CO && op.out.cstride == 4 * CO && op.out.coff == 0 &&
        ((y0 | x0) & 1) == 0) {
      // the 8 x 16 tile is 4 runs of 8 consecutive s2d pixels (4*CO floats
      // each): linear, coalesced stores
      const int64_t s2row = (int64_t)(op.out.W >> 1) * 4 * CO;
      float* sb0 = op.out.base + ((int64_t)b * (op.out.H >> 1) + (y0 >> 1)) * s2row +
                   (int64_t)(x0 >> 1) * 4 * CO;
      for (int e = threadIdx.x; e < kDThreads * CO; e += kDThreads) {
        const int r = e / (32 * CO), w = e - r * (32 * CO);
        const int j = w / (4 * CO), ph = (w / CO) & 3, c = w % CO;
        const int py = 2 * r + (ph >> 1), px = 2 * j + (ph & 1);
        if (y0 + py < op.oy1 && x0 + px < op.ox1)
          sb0[r * s2row + w] = so[(py * kDTX + px) * Cs + c];
      }
    } else if (op.out.s2d) {
      for (int t = warp; t < kDThreads; t += kDThreads / 32) {
        const int py = t / kDTX, px = t % kDTX;
        if (y0 + py >= op.oy1 || x0 + px >= op.ox1) continue;
        float* o = op.out.base + act_off(op.out, b, y0 + py, x0 + px);
        for (int c = lane; c < Cout; c += 32) o[c] = so[t * Cs + c];
      }
    } else if (Cout == CO && op.out.cstride == CO) {
      for (int e = threadIdx.x; e < kDThreads * CO; e += kDThreads) {
        const int t = e / CO, c = e - t * CO;
        const int py = t / kDTX, px = t % kDTX;
        if (y0 + py < op.oy1 && x0 + px < op.ox1) ob[py * orow + px * CO + c] = so[t * Cs + c];
      }
    } else {
      for (int t = warp; t < kDThreads; t += kDThreads / 32) {
        const int py = t / kDTX, px = t % kDTX;
        if (y0 + py >= op.oy1 || x0 + px >= op.ox1) continue;
        float* o = ob + py * orow + (int64_t)px * op.out.cstride;
        for (int c = lane; c < Cout; c += 32) o[c] = so[t * Cs + c];
      }
    }
  }
  (void)wy; (void)wx;
}

DirectGeom direct_geom(const ConvOp& op, size_t* smem) {
  DirectGeom g;
  const int Cin = op.in.C, s = op.stride;
  g.HY = (kDTY - 1) * s + op.k;
  g.HX = (kDTX - 1) * s + op.k;
  g.vec4 = (Cin & 3) == 0 && (op.in.cstride & 3) == 0 && (op.in.coff & 3) == 0 &&
           (reinterpret_cast<uintptr_t>(op.in.base) & 15) == 0;
  if (g.vec4) {
    g.Cp = Cin;
    if (((s * g.Cp / 4) & 1) == 0 && s == 1) g.Cp += 4;  // odd 16-byte lane stride
  } else {
    g.Cp = Cin;
    if (((s * g.Cp) & 1) == 0 && s == 1) g.Cp += 1;      // odd word lane stride
  }
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  g.ntx = (wx + kDTX - 1) / kDTX;
  g.nty = (wy + kDTY - 1) / kDTY;
  g.tiles = op.batch * g.nty * g.ntx;
  const int K = op.k * op.k * Cin;
  g.halo_off = (K * op.out.C + ((op.out.C + 3) & ~3) + 3) & ~3;
  g.out_off = g.halo_off + ((g.HY * g.HX * g.Cp + 3) & ~3);
  *smem = (size_t)(g.out_off + kDThreads * (op.out.C | 1)) * sizeof(float);
  return g;
}

}  // namespace

bool conv_direct_supported(const ConvOp& op) {
  if ((op.in.C > 4 && op.out.C > 16) || op.out.C > 64 || op.stride > 2 || op.k > 5)
    return false;
  if ((int64_t)op.batch * (op.oy1 - op.oy0) * (op.ox1 - op.ox0) >= (1LL << 30)) return false;
  size_t smem;
  direct_geom(op, &smem);
  return smem <= 200 * 1024;
}

int launch_conv_direct(const ConvOp& op, void* stream) {
  if (op.in.planes || op.out.planes) return TS_E_INVALID;  // fp32 activations only
  if (op.batch <= 0 || op.oy1 <= op.oy0 || op.ox1 <= op.ox0) return TS_OK;
  size_t smem;
  const DirectGeom g = direct_geom(op, &smem);
  const int per_sm = std::max(1, std::min(8, (int)((220 * 1024) / (smem + 1024))));
  const int grid = std::min(g.tiles, 148 * per_sm);
  cudaStream_t s = as_stream(stream);
#define TS_DIRECT(CO, EX, KS)                                                          \
  do {                                                                                 \
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_direct_kernel<CO, EX, KS>,                   \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                     (int)smem));                                      \
    ts::count_launch(),                                                                \
        conv_direct_kernel<CO, EX, KS><<<grid, kDThreads, smem, s>>>(op, g);           \
  } while (0)
  const int co = op.out.C;
  if (op.k == 3 && co == 4) TS_DIRECT(4, true, 3);
  else if (op.k == 3 && co == 16) TS_DIRECT(16, true, 3);
  else if (op.k == 3 && co == 32) TS_DIRECT(32, true, 3);
  else if (op.k == 3 && co == 48) TS_DIRECT(48, true, 3);
  else if (op.k == 3 && co == 64) TS_DIRECT(64, true, 3);
  else if (co <= 16) TS_DIRECT(16, false, 0);
  else TS_DIRECT(64, false, 0);
#undef TS_DIRECT
  TS_LAUNCH_CHECK();
  return TS_OK;
}

}  // namespace ts
