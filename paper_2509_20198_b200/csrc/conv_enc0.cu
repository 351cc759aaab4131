// K3c: the four encoders' first layers in one launch (refiner.py:399-441,
// stages enc_hm_nn / enc_hm_lin / enc_rgb_nn / enc_rgb_lin, layer 0:
// 3x3 stride-2 pad-1 convolutions of 1, 1, 3, 3 raw input channels).
//
// The four layers read disjoint channels of the same B x 96 x 96 x 8 CNN
// input, so one CTA stages the input halo of a 4 x 16 output tile ONCE for
// all of them (the per-layer direct kernel read it four times) and its 16
// warps split as 4 encoders x C_out/16 output-channel groups (each thread: 2 pixels x 16 channels).  fp32 CUDA-core FMAs (thin K: 9
// or 27 MACs per output channel), outputs written straight into the
// space-to-depth layout the stride-2 tensor-core layers consume (a pixel's
// C_out channels are one contiguous run there: 32-byte stores).
// CTAs of 4 x C_out/16 warps, two per SM, so one CTA's halo load overlaps the
// other's FMAs.
//
// Shared memory: halo [8 ch][9 rows][2 column parities][20] (stride-2
// reads become stride-1 per parity plane: bank-conflict free), weights
// [K][C_out] per encoder.
#include <algorithm>
#include <cstdlib>

#include "conv.cuh"
#include "tc_ptx.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int kETY = 4, kETX = 16;          // output tile
constexpr int kEHY = 2 * kETY + 1;          // 9 halo rows
constexpr int kEPitch = 20;                 // floats per parity row (>= 17; 4*pitch = 16 mod 32)
constexpr int kEPlane = kEHY * 2 * kEPitch; // floats per channel
// threads per CTA: 4 encoders x C_out/16 channel groups of 16 (one warp each)
template <int CO>
__host__ __device__ constexpr int enc0_threads() { return 4 * (CO / 16) * 32; }

__device__ __forceinline__ float lrelu(float v) { return v >= 0.f ? v : 0.01f * v; }

// Two output pixels (rows ty and ty + 2 of the tile) x CH consecutive
// output channels per thread: every broadcast weight load feeds 8 FMAs.
template <int CIN, int CO, int CH>
__device__ __forceinline__ void enc0_accumulate(const float* __restrict__ halo, int ch0,
                                                const float* __restrict__ w, int ty, int tx,
                                                float (&acc)[2][CH]) {
#pragma unroll
  for (int ky = 0; ky < 3; ++ky)
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      // input column 2 tx + kx lives in parity plane kx & 1 at index tx + kx / 2
      const float* hp = halo + (2 * ty + ky) * 2 * kEPitch + (kx & 1) * kEPitch + tx + (kx >> 1);
#pragma unroll
      for (int ci = 0; ci < CIN; ++ci) {
        const float x0 = hp[(ch0 + ci) * kEPlane];
        const float x1 = hp[(ch0 + ci) * kEPlane + 4 * 2 * kEPitch];  // two output rows on
        const float4* w4 = reinterpret_cast<const float4*>(w + ((ky * 3 + kx) * CIN + ci) * CO);
#pragma unroll
        for (int o = 0; o < CH / 4; ++o) {  // packed fp32 FMAs (FFMA2)
          const float4 q = w4[o];
          tcx::ffma2(acc[0][4 * o], acc[0][4 * o + 1], x0, q.x, q.y);
          tcx::ffma2(acc[0][4 * o + 2], acc[0][4 * o + 3], x0, q.z, q.w);
          tcx::ffma2(acc[1][4 * o], acc[1][4 * o + 1], x1, q.x, q.y);
          tcx::ffma2(acc[1][4 * o + 2], acc[1][4 * o + 3], x1, q.z, q.w);
        }
      }
    }
}

template <int CO>
__global__ void __launch_bounds__(enc0_threads<CO>(), 2) conv_enc0_kernel(Enc0Op E) {
  constexpr int kEThreads = enc0_threads<CO>();
  extern __shared__ __align__(16) float sm[];
  float* halo = sm;                                   // 8 * kEPlane
  float* sw = halo + 8 * kEPlane;                     // weights, 4 encoders
  int woff[4];
  {
    int o = 0;
    for (int e = 0; e < 4; ++e) { woff[e] = o; o += 9 * E.cin[e] * CO; }
    for (int e = 0; e < 4; ++e)
      for (int i = threadIdx.x; i < 9 * E.cin[e] * CO; i += kEThreads) sw[woff[e] + i] = E.w[e][i];
    o = (o + 3) & ~3;
    for (int i = threadIdx.x; i < 4 * CO; i += kEThreads) sw[o + i] = E.bias[i / CO][i % CO];
  }
  const float* sbias = sw + ((woff[3] + 9 * E.cin[3] * CO + 3) & ~3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = warp & 3;                             // encoder of this warp
  constexpr int CH = 16;                              // channels per thread
  const int chalf = (warp >> 2) * CH;                 // which channel group
  const int ty = lane >> 4, tx = lane & 15;           // rows ty and ty + 2
  const int wy = E.oy1 - E.oy0, wx = E.ox1 - E.ox0;
  const int ntx = (wx + kETX - 1) / kETX, nty = (wy + kETY - 1) / kETY;
  const int64_t tiles = (int64_t)E.batch * nty * ntx;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    // tiles < 2^31 (checked by the host): 32-bit division
    const int64_t b = (int)tile / (nty * ntx);
    const int r = (int)tile - (int)b * nty * ntx;
    const int y0 = E.oy0 + (r / ntx) * kETY, x0 = E.ox0 + (r % ntx) * kETX;
    __syncthreads();  // previous tile's halo reads done
    // halo: input rows 2 y0 - 1 .. + 16, columns 2 x0 - 1 .. + 32, 8 channels
    const float* inb = E.in + b * (int64_t)E.H * E.W * 8;
    for (int i = threadIdx.x; i < kEHY * 33 * 2; i += kEThreads) {
      const int hy = i / 66, rem = i - hy * 66, hx = rem >> 1, half = rem & 1;
      const int iy = 2 * y0 - 1 + hy, ix = 2 * x0 - 1 + hx;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (iy >= 0 && iy < E.H && ix >= 0 && ix < E.W)
        v = __ldg(reinterpret_cast<const float4*>(inb + ((int64_t)iy * E.W + ix) * 8) + half);
      float* d = halo + hy * 2 * kEPitch + (hx & 1) * kEPitch + (hx >> 1) + 4 * half * kEPlane;
      d[0] = v.x; d[kEPlane] = v.y; d[2 * kEPlane] = v.z; d[3 * kEPlane] = v.w;
    }
    __syncthreads();
    float acc[2][CH];
#pragma unroll
    for (int o = 0; o < CH; ++o) acc[0][o] = acc[1][o] = sbias[e * CO + chalf + o];
    if (E.cin[e] == 1)
      enc0_accumulate<1, CO, CH>(halo, E.ch0[e], sw + woff[e] + chalf, ty, tx, acc);
    else
      enc0_accumulate<3, CO, CH>(halo, E.ch0[e], sw + woff[e] + chalf, ty, tx, acc);
    // space-to-depth store: the pixel's C_out channels are contiguous
    const ActView& ov = E.out[e];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int y = y0 + ty + 2 * r, x = x0 + tx;
      if (y >= E.oy1 || x >= E.ox1) continue;
      if (E.lrelu[e])
#pragma unroll
        for (int o = 0; o < CH; ++o) acc[r][o] = lrelu(acc[r][o]);
      if (ov.planes) {  // pre-split for the tensor-core consumer
        int64_t blk;
        int chan;
        act_block(ov, b, y, x, blk, chan);
#pragma unroll
        for (int o = 0; o < CH; o += 8)
          tcx::store8_planes(ov.base + blk, ov.cstride, chan + chalf + o, acc[r] + o,
                             ov.planes == 2);
      } else {
        float* op_ = ov.base + act_off(ov, b, y, x) + chalf;
#pragma unroll
        for (int o = 0; o < CH; o += 8) tcx::st_v8(op_ + o, acc[r] + o);
      }
    }
  }
}

// Store two pixels (rows y and y + 2) x CH channels starting at channel c0.
template <int CH>
__device__ __forceinline__ void enc0_store(const ActView& ov, int64_t b, int y, int x, int oy1,
                                           int ox1, int c0, bool lr, float (&acc)[2][CH]) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int yy = y + 2 * r;
    if (yy >= oy1 || x >= ox1) continue;
    if (lr)
#pragma unroll
      for (int o = 0; o < CH; ++o) acc[r][o] = lrelu(acc[r][o]);
    if (ov.planes) {
      int64_t blk;
      int chan;
      act_block(ov, b, yy, x, blk, chan);
#pragma unroll
      for (int o = 0; o < CH; o += 8)
        tcx::store8_planes(ov.base + blk, ov.cstride, chan + c0 + o, acc[r] + o,
                             ov.planes == 2);
    } else {
      float* op_ = ov.base + act_off(ov, b, yy, x) + c0;
#pragma unroll
      for (int o = 0; o < CH; o += 8) tcx::st_v8(op_ + o, acc[r] + o);
    }
  }
}

// Work-balanced variant for C_out = 48 and encoders of 1, 1, 3, 3 input
// channels (any order): a 1-channel encoder's 9 MACs per output take 2
// warps of CO/2 channels, a 3-channel encoder's 27 take 6 warps of CO/6,
// so all 16 warps do 216 MACs per pixel (the per-encoder mapping above
// leaves the 1-channel warps idle 2/3 of the time at every tile barrier).
// One CTA per SM; the next tile's halo is loaded into registers before this
// tile's FMAs (the loads' latency hides behind the compute).
constexpr int kBalWarps = 16, kBalThreads = kBalWarps * 32;

template <int CO>
__global__ void __launch_bounds__(kBalThreads, 1) conv_enc0_bal_kernel(Enc0Op E) {
  constexpr int CH1 = CO / 2, CH3 = CO / 6;
  extern __shared__ __align__(16) float sm[];
  float* halo = sm;                                   // 8 * kEPlane
  float* sw = halo + 8 * kEPlane;                     // weights, 4 encoders
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int e = 0, wi = warp, woff = 0, o = 0;
  for (int j = 0; j < 4; ++j) {
    for (int i = threadIdx.x; i < 9 * E.cin[j] * CO; i += kBalThreads) sw[o + i] = E.w[j][i];
    o += 9 * E.cin[j] * CO;
  }
  o = (o + 3) & ~3;
  float* sbias = sw + o;
  for (int i = threadIdx.x; i < 4 * CO; i += kBalThreads) sbias[i] = E.bias[i / CO][i % CO];
  for (; e < 3; ++e) {
    const int nw = E.cin[e] == 1 ? 2 : 6;
    if (wi < nw) break;
    wi -= nw;
    woff += 9 * E.cin[e] * CO;
  }
  const bool one = E.cin[e] == 1;
  const int c0 = wi * (one ? CH1 : CH3);
  const int ty = lane >> 4, tx = lane & 15;           // rows ty and ty + 2
  const int wy = E.oy1 - E.oy0, wx = E.ox1 - E.ox0;
  const int ntx = (wx + kETX - 1) / kETX, nty = (wy + kETY - 1) / kETY;
  const int64_t tiles = (int64_t)E.batch * nty * ntx;
  constexpr int kHaloPieces = kEHY * 33 * 2;
  constexpr int kPre = (kHaloPieces + kBalThreads - 1) / kBalThreads;
  float4 pre[kPre];
  auto load_halo = [&](int64_t t) {
    const int64_t b = (int)t / (nty * ntx);
    const int r = (int)t - (int)b * nty * ntx;
    const int y0 = E.oy0 + (r / ntx) * kETY, x0 = E.ox0 + (r % ntx) * kETX;
    const float* inb = E.in + b * (int64_t)E.H * E.W * 8;
#pragma unroll
    for (int j = 0; j < kPre; ++j) {
      const int i = threadIdx.x + j * kBalThreads;
      pre[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < tiles && i < kHaloPieces) {
        const int hy = i / 66, rem = i - hy * 66, hx = rem >> 1, half = rem & 1;
        const int iy = 2 * y0 - 1 + hy, ix = 2 * x0 - 1 + hx;
        if (iy >= 0 && iy < E.H && ix >= 0 && ix < E.W)
          pre[j] = __ldg(reinterpret_cast<const float4*>(inb + ((int64_t)iy * E.W + ix) * 8) + half);
      }
    }
  };
  load_halo(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    // tiles < 2^31 (checked by the host): 32-bit division
    const int64_t b = (int)tile / (nty * ntx);
    const int r = (int)tile - (int)b * nty * ntx;
    const int y0 = E.oy0 + (r / ntx) * kETY, x0 = E.ox0 + (r % ntx) * kETX;
    __syncthreads();  // previous tile's halo reads done
#pragma unroll
    for (int j = 0; j < kPre; ++j) {
      const int i = threadIdx.x + j * kBalThreads;
      if (i < kHaloPieces) {
        const int hy = i / 66, rem = i - hy * 66, hx = rem >> 1, half = rem & 1;
        float* d = halo + hy * 2 * kEPitch + (hx & 1) * kEPitch + (hx >> 1) + 4 * half * kEPlane;
        d[0] = pre[j].x; d[kEPlane] = pre[j].y; d[2 * kEPlane] = pre[j].z; d[3 * kEPlane] = pre[j].w;
      }
    }
    __syncthreads();
    load_halo(tile + gridDim.x);
    if (one) {
      float acc[2][CH1];
#pragma unroll
      for (int q = 0; q < CH1; ++q) acc[0][q] = acc[1][q] = sbias[e * CO + c0 + q];
      enc0_accumulate<1, CO, CH1>(halo, E.ch0[e], sw + woff + c0, ty, tx, acc);
      enc0_store<CH1>(E.out[e], b, y0 + ty, x0 + tx, E.oy1, E.ox1, c0, E.lrelu[e], acc);
    } else {
      float acc[2][CH3];
#pragma unroll
      for (int q = 0; q < CH3; ++q) acc[0][q] = acc[1][q] = sbias[e * CO + c0 + q];
      enc0_accumulate<3, CO, CH3>(halo, E.ch0[e], sw + woff + c0, ty, tx, acc);
      enc0_store<CH3>(E.out[e], b, y0 + ty, x0 + tx, E.oy1, E.ox1, c0, E.lrelu[e], acc);
    }
  }
}

bool enc0_balanced(const Enc0Op& E, int co) {
  int ones = 0;
  for (int e = 0; e < 4; ++e) ones += E.cin[e] == 1;
  return co == 48 && ones == 2;
}

size_t enc0_smem(const Enc0Op& E, int co) {
  int k = 0;
  for (int e = 0; e < 4; ++e) k += 9 * E.cin[e] * co;
  return sizeof(float) * ((size_t)8 * kEPlane + ((k + 3) & ~3) + 4 * co);
}

}  // namespace

bool conv_enc0_supported(const Enc0Op& E, int co) {
  if (co != 48 && co != 32 && co != 64) return false;
  for (int e = 0; e < 4; ++e) {
    if (E.cin[e] != 1 && E.cin[e] != 3) return false;
    if (E.ch0[e] < 0 || E.ch0[e] + E.cin[e] > 8) return false;
  }
  if ((E.oy0 | E.ox0) & 1) return false;  // space-to-depth pairs
  return enc0_smem(E, co) <= 220 * 1024;
}

int launch_conv_enc0(const Enc0Op& E, int co, void* stream) {
  if (!conv_enc0_supported(E, co)) return TS_E_INVALID;
  if (E.batch <= 0 || E.oy1 <= E.oy0 || E.ox1 <= E.ox0) return TS_OK;
  const size_t smem = enc0_smem(E, co);
  const int sms = sm_count();
  if (!sms) return TS_E_CUDA;
  const int64_t tiles = (int64_t)E.batch * ((E.oy1 - E.oy0 + kETY - 1) / kETY) *
                        ((E.ox1 - E.ox0 + kETX - 1) / kETX);
  if (tiles + 2 * (int64_t)sms >= (int64_t)INT32_MAX) return TS_E_INVALID;
  cudaStream_t s = as_stream(stream);
  if (enc0_balanced(E, co)) {
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_enc0_bal_kernel<48>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int g1 = (int)std::min<int64_t>(tiles, sms);
    ts::count_launch(), conv_enc0_bal_kernel<48><<<g1, kBalThreads, smem, s>>>(E);
    TS_LAUNCH_CHECK();
    return TS_OK;
  }
  const int grid = (int)std::min<int64_t>(tiles, 2 * sms);
#define TS_ENC0(CO)                                                                    \
  do {                                                                                 \
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_enc0_kernel<CO>,                             \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                     (int)smem));                                      \
    ts::count_launch(), conv_enc0_kernel<CO><<<grid, enc0_threads<CO>(), smem, s>>>(E); \
  } while (0)
  if (co == 48) TS_ENC0(48);
  else if (co == 32) TS_ENC0(32);
  else TS_ENC0(64);
#undef TS_ENC0
  TS_LAUNCH_CHECK();
  return TS_OK;
}

}  // namespace ts
