// K3d: the refiner's last layer (fuse.2: 3x3 stride-1 pad-1, 32 -> 4
// channels, linear; refiner.py:430-441) on CUDA cores in fp32.
//
// Four output channels make a tensor-core tile almost all padding, and the
// layer is tiny (4.7 M MACs per tile), so the weights ride in the kernel
// parameters: every FMA takes its weight straight from the constant bank
// (uniform across the warp), and the only shared-memory traffic is the
// 18 x 18 x 32 input halo of a 16 x 16 output tile (pixel pitch 36 floats:
// conflict-free 16-byte reads).  fp32 FMAs, so this layer is as accurate
// as the reference's float32 GEMM.
#include <algorithm>

#include "conv.cuh"
#include "tc_ptx.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int kFT = 16;                 // output tile edge
constexpr int kFH = kFT + 2;            // halo edge
constexpr int kFCin = 32, kFCo = 4;
constexpr int kFPitch = kFCin + 4;      // floats per halo pixel

struct FinalArgs {
  float w[9 * kFCin * kFCo];  // [tap][ci][co]
  float b[kFCo];
  ActView in, out;
  int oy0, oy1, ox0, ox1, batch, lrelu;
};

__global__ void __launch_bounds__(kFT * kFT) conv_final_kernel(const __grid_constant__ FinalArgs A) {
  __shared__ __align__(16) float halo[kFH * kFH * kFPitch];
  const int wy = A.oy1 - A.oy0, wx = A.ox1 - A.ox0;
  const int nty = (wy + kFT - 1) / kFT, ntx = (wx + kFT - 1) / kFT;
  const int64_t b = blockIdx.x / (nty * ntx);
  const int r = blockIdx.x - (int)b * nty * ntx;
  const int y0 = A.oy0 + (r / ntx) * kFT, x0 = A.ox0 + (r % ntx) * kFT;
  // halo rows y0-1 .. y0+16, columns x0-1 .. x0+16, 32 channels (8 x 16 B)
  for (int e = threadIdx.x; e < kFH * kFH * (kFCin / 4); e += blockDim.x) {
    const int p = e >> 3, q = e & 7;
    const int hy = p / kFH, hx = p - hy * kFH;
    const int iy = y0 - 1 + hy, ix = x0 - 1 + hx;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (iy >= 0 && iy < A.in.H && ix >= 0 && ix < A.in.W)
      v = __ldg(reinterpret_cast<const float4*>(A.in.base + act_off(A.in, b, iy, ix)) + q);
    *reinterpret_cast<float4*>(halo + p * kFPitch + 4 * q) = v;
  }
  __syncthreads();
  const int ty = threadIdx.x / kFT, tx = threadIdx.x % kFT;
  const int y = y0 + ty, x = x0 + tx;
  if (y >= A.oy1 || x >= A.ox1) return;
  float acc[kFCo];
#pragma unroll
  for (int o = 0; o < kFCo; ++o) acc[o] = A.b[o];
#pragma unroll
  for (int ky = 0; ky < 3; ++ky)
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      const float* hp = halo + ((ty + ky) * kFH + tx + kx) * kFPitch;
#pragma unroll
      for (int g = 0; g < kFCin / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(hp + 4 * g);
        const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float* w = A.w + ((ky * 3 + kx) * kFCin + 4 * g + j) * kFCo;
          tcx::ffma2(acc[0], acc[1], xs[j], w[0], w[1]);  // packed fp32 FMAs
          tcx::ffma2(acc[2], acc[3], xs[j], w[2], w[3]);
        }
      }
    }
  if (A.lrelu)
#pragma unroll
    for (int o = 0; o < kFCo; ++o) acc[o] = acc[o] >= 0.f ? acc[o] : 0.01f * acc[o];
  *reinterpret_cast<float4*>(A.out.base + act_off(A.out, b, y, x)) =
      make_float4(acc[0], acc[1], acc[2], acc[3]);
}

}  // namespace

bool conv_final_supported(const ConvOp& op) {
  return op.k == 3 && op.stride == 1 && op.pad == 1 && !op.up2 && !op.ph &&
         op.in.C == kFCin && op.out.C == kFCo && !op.in.planes && !op.out.planes &&
         !op.in.s2d && !op.out.s2d && op.in.cstride % 4 == 0 && op.in.coff % 4 == 0 &&
         op.out.cstride % 4 == 0 && op.out.coff % 4 == 0;
}

int launch_conv_final(const ConvOp& op, const float* w_oikk_packed, const float* bias_host,
                      void* stream) {
  if (!conv_final_supported(op)) return TS_E_INVALID;
  if (op.batch <= 0 || op.oy1 <= op.oy0 || op.ox1 <= op.ox0) return TS_OK;
  FinalArgs a;
  memcpy(a.w, w_oikk_packed, sizeof(a.w));
  memcpy(a.b, bias_host, sizeof(a.b));
  a.in = op.in; a.out = op.out;
  a.oy0 = op.oy0; a.oy1 = op.oy1; a.ox0 = op.ox0; a.ox1 = op.ox1;
  a.batch = op.batch; a.lrelu = op.lrelu;
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int64_t tiles = (int64_t)op.batch * ((wy + kFT - 1) / kFT) * ((wx + kFT - 1) / kFT);
  ts::count_launch(),
      conv_final_kernel<<<(unsigned)tiles, kFT * kFT, 0, as_stream(stream)>>>(a);
  TS_LAUNCH_CHECK();
  return TS_OK;
}

}  // namespace ts
