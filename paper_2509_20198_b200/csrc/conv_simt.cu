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
// 64-wide N tile on these (enc*.0: 1/3 -> 48, fuse.2: 32 -> 4).
namespace ts {
namespace {

template <int CO>
__global__ void __launch_bounds__(128) conv_direct_kernel(ConvOp op) {
  extern __shared__ float sw[];
  const int Cin = op.in.C, Cout = op.out.C;
  const int K = op.k * op.k * Cin;
  for (int i = threadIdx.x; i < K * Cout; i += blockDim.x) sw[i] = op.w[i];
  float* sb = sw + K * Cout;
  for (int i = threadIdx.x; i < Cout; i += blockDim.x) sb[i] = op.bias[i];
  float* so = sb + ((Cout + 3) & ~3);  // [128][Cs] output staging
  const int Cs = Cout | 1;              // odd row pitch: conflict-free banks
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int64_t M = (int64_t)op.batch * wy * wx;
  const int Hl = op.up2 ? 2 * op.in.H : op.in.H;
  const int Wl = op.up2 ? 2 * op.in.W : op.in.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t m0 = blockIdx.x * (int64_t)blockDim.x; m0 < M;
       m0 += (int64_t)gridDim.x * blockDim.x) {
    __syncthreads();  // weights loaded / previous staging drained
    const int64_t m = m0 + threadIdx.x;
    if (m < M) {
      const int b = (int)(m / ((int64_t)wy * wx));
      const int r = (int)(m - (int64_t)b * wy * wx);
      const int oy = op.oy0 + r / wx, ox = op.ox0 + r % wx;
      float acc[CO];
#pragma unroll
      for (int c = 0; c < CO; ++c) acc[c] = 0.f;
      const float* inb =
          op.in.base + (int64_t)b * op.in.H * op.in.W * op.in.cstride + op.in.coff;
      {
        for (int ky = 0; ky < op.k; ++ky) {
          int iy = oy * op.stride - op.pad + ky;
          if (iy < 0 || iy >= Hl) continue;
          if (op.up2) iy >>= 1;
          for (int kx = 0; kx < op.k; ++kx) {
            int ix = ox * op.stride - op.pad + kx;
            if (ix < 0 || ix >= Wl) continue;
            if (op.up2) ix >>= 1;
            const float* src = inb + ((int64_t)iy * op.in.W + ix) * op.in.cstride;
            const float* wt = sw + (ky * op.k + kx) * Cin * Cout;
            for (int ci = 0; ci < Cin; ++ci) {
              const float x = __ldg(src + ci);
#pragma unroll
              for (int c = 0; c < CO; ++c)
                if (c < Cout) acc[c] = fmaf(x, wt[ci * Cout + c], acc[c]);
            }
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
    }
    __syncthreads();
    // coalesced write-back: one warp per pixel, lanes over channels
    for (int t = warp; t < 128; t += 4) {
      const int64_t mm = m0 + t;
      if (mm >= M) break;
      const int b = (int)(mm / ((int64_t)wy * wx));
      const int r = (int)(mm - (int64_t)b * wy * wx);
      const int y = op.oy0 + r / wx, x = op.ox0 + r % wx;
      float* o = op.out.base + (((int64_t)b * op.out.H + y) * op.out.W + x) * op.out.cstride +
                 op.out.coff;
      for (int c = lane; c < Cout; c += 32) o[c] = so[t * Cs + c];
    }
  }
}

}  // namespace

bool conv_direct_supported(const ConvOp& op) {
  const int K = op.k * op.k * op.in.C;
  return (op.in.C <= 4 || op.out.C <= 16) && op.out.C <= 64 &&
         (size_t)(K + 1 + 128) * (op.out.C + 1) * sizeof(float) + 16 <= 160 * 1024;
}

int launch_conv_direct(const ConvOp& op, void* stream) {
  const int64_t M = (int64_t)op.batch * (op.oy1 - op.oy0) * (op.ox1 - op.ox0);
  if (M <= 0) return TS_OK;
  const size_t smem =
      ((size_t)(op.k * op.k * op.in.C) * op.out.C + ((op.out.C + 3) & ~3) +
       128 * (op.out.C | 1)) *
      sizeof(float);
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(M, 128), 148 * 16);
  cudaStream_t s = as_stream(stream);
#define TS_DIRECT(CO)                                                                  \
  do {                                                                                 \
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_direct_kernel<CO>,                           \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                     (int)smem));                                      \
    ts::count_launch(), conv_direct_kernel<CO><<<grid, 128, smem, s>>>(op);            \
  } while (0)
  if (op.out.C <= 4) TS_DIRECT(4);
  else if (op.out.C <= 16) TS_DIRECT(16);
  else if (op.out.C <= 32) TS_DIRECT(32);
  else TS_DIRECT(64);
#undef TS_DIRECT
  TS_LAUNCH_CHECK();
  return TS_OK;
}

}  // namespace ts
