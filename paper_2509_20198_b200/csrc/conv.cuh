// Convolution layer descriptors shared by the refine planner and kernels.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include <cstring>
#include <vector>

namespace ts {

// One NHWC activation view: element (b, y, x, c) lives at
// base[((b * H + y) * W + x) * cstride + coff + c].
//
// s2d = 1: space-to-depth storage of an even-sized image (the input layout
// of a stride-2 3x3 layer run as a stride-1 2x2 convolution): element
// (b, y, x, c) of the logical H x W x C image lives at half-resolution pixel
// (y/2, x/2), channel ((y&1)*2 + (x&1))*C + c; cstride is then the physical
// pixel stride (>= 4C).
//
// planes = 1: pre-split storage for tensor-core consumers.  Same bytes per
// element as fp32: in the pixel block of cstride fp32 slots, bytes
// [2c, 2c+2) hold hi(c) = bf16_rn(v) and bytes [2 cstride + 2c, ...) hold
// lo(c) = bf16_rn(v - hi), the split the tensor-core producers would
// otherwise compute per halo row (so results are bit-identical).
struct ActView {
  float* base;
  int H, W, cstride, coff, C;
  int s2d;
  int planes;
};

__host__ __device__ inline int64_t act_off(const ActView& v, int64_t b, int y, int x) {
  if (!v.s2d) return ((b * v.H + y) * v.W + x) * v.cstride + v.coff;
  return ((b * (v.H >> 1) + (y >> 1)) * (v.W >> 1) + (x >> 1)) * v.cstride + v.coff +
         ((y & 1) * 2 + (x & 1)) * v.C;
}

// pixel block start (fp32 slots) and channel index of channel 0 within it
__host__ __device__ inline void act_block(const ActView& v, int64_t b, int y, int x,
                                          int64_t& block, int& chan) {
  if (!v.s2d) {
    block = ((b * v.H + y) * v.W + x) * v.cstride;
    chan = v.coff;
  } else {
    block = ((b * (v.H >> 1) + (y >> 1)) * (v.W >> 1) + (x >> 1)) * v.cstride;
    chan = v.coff + ((y & 1) * 2 + (x & 1)) * v.C;
  }
}

// A convolution launch (cross-correlation, refiner.py:330-380) with fused
// nearest x2 upsampling of the input (refiner.py:395), bias, optional
// leaky ReLU (refiner.py:391) and an output window (crop-aware execution).
struct ConvOp {
  ActView in;       // physical input
  ActView out;
  int up2;          // input is read through a nearest x2 upsample
  int k, stride, pad;
  int lrelu;
  int oy0, oy1, ox0, ox1;   // output window [oy0,oy1) x [ox0,ox1)
  const float* w;   // [K][C_out], K = (ky * k + kx) * C_in + ci
  const float* bias;
  int batch;
  const uint8_t* w_tc;  // tensor-core packed weights (conv_tc.cu), or null
  int w_layout;         // layout of w_tc: 0 regular, 1 halo (128 B rows), 2 halo2
  // phase form of "nearest x2 upsample -> 3x3 stride-1 pad-1 conv" (halo2
  // kernel only): ph = 1 runs output phase (ph_y, ph_x) as a 2x2 conv over
  // the low-resolution input, rows/cols offset by ph - 1 (pad 1 - ph), the
  // window [oy0,oy1) x [ox0,ox1) in low-resolution coordinates and output
  // pixel (2*oy + ph_y, 2*ox + ph_x) of op.out.
  int ph, ph_y, ph_x;
};

// Tap set of the phase form: low-resolution tap t (0 or 1) of output phase
// p collects the 3x3 taps k with (p + k - 1) >> 1 == p + t - 1, i.e.
// p=0: t0 <- {0}, t1 <- {1, 2};  p=1: t0 <- {0, 1}, t1 <- {2}.
inline bool phase_tap(int p, int t, int k) { return ((p + k + 1) >> 1) == p + t; }

inline uint16_t f2bf16_rn_host(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
inline float bf16_to_f_host(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

// FP16X3 weight planes (tc_ptx.cuh Mode<5>): w = h0 + 2^-11 h1
inline void split_f16_host(float v, uint16_t& h0, uint16_t& h1) {
  const __half a = __float2half_rn(v);
  const float r = (v - __half2float(a)) * 2048.f;
  const __half b = __float2half_rn(r);
  memcpy(&h0, &a, 2);
  memcpy(&h1, &b, 2);
}

// precision modes that run on the bf16/fp16 tensor-core kernels
inline bool tc16_mode(int precision) { return precision >= 2 && precision <= 5; }

// The four encoders' first layers (3x3 stride 2 pad 1 over 1/1/3/3 raw
// input channels) in one launch; outputs in space-to-depth layout.
struct Enc0Op {
  const float* in;          // B x H x W x 8 fp32 CNN input
  int H, W, batch;
  int ch0[4], cin[4], lrelu[4];
  const float* w[4];        // [9 * cin][C_out] packed like ConvOp::w
  const float* bias[4];
  ActView out[4];           // s2d views
  int oy0, oy1, ox0, ox1;   // common output window
};
bool conv_enc0_supported(const Enc0Op& e, int co);
int launch_conv_enc0(const Enc0Op& e, int co, void* stream);

// fuse.2-shaped layers (3x3 s1 p1, 32 -> 4): fp32 CUDA cores with the
// weights in the kernel parameters (conv_final.cu)
bool conv_final_supported(const ConvOp& op);
int launch_conv_final(const ConvOp& op, const float* w_packed, const float* bias_host,
                      void* stream);

int launch_conv_simt(const ConvOp& op, void* stream);
bool conv_direct_supported(const ConvOp& op);
int launch_conv_direct(const ConvOp& op, void* stream);
bool conv_tc_supported(const ConvOp& op, int precision);
int launch_conv_tc(const ConvOp& op, int precision, void* stream);
// Which tensor-core kernel (and so which packed weight layout) serves this
// layer shape: 0 regular implicit GEMM, 1 halo kernel (conv_tc.cu), 2 wide-M
// halo kernel (conv_tc2.cu).
int tc_weight_layout(const ConvOp& shape, int precision);
// Swizzled per-(n-tile, k-stage) shared-memory images of OIKK weights in the
// given layout (launch_conv_tc dispatches on op.w_layout).
std::vector<uint8_t> pack_tc_weights(const float* w_oikk, int co, int ci, int k,
                                     int precision, const ConvOp& shape_op, int layout);
bool conv_tc_halo_eligible(const ConvOp& op, int precision);
bool conv_tc_halo2_eligible(const ConvOp& op, int precision);
// TMEM accumulator buffers the wide-M halo kernel's plan gives op (0: not
// eligible)
int conv_tc_halo2_accbufs(const ConvOp& op, int precision);
std::vector<uint8_t> pack_tc_weights_halo2(const float* w_oikk, int co, int ci, int k,
                                           int precision, const ConvOp& op);
int launch_conv_tc_halo2(const ConvOp& op, int precision, void* stream);

}  // namespace ts
