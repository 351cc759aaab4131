// Convolution layer descriptors shared by the refine planner and kernels.
#pragma once

#include <stdint.h>

#include <vector>

namespace ts {

// One NHWC activation view: element (b, y, x, c) lives at
// base[((b * H + y) * W + x) * cstride + coff + c].
struct ActView {
  float* base;
  int H, W, cstride, coff, C;
};

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
};

int launch_conv_simt(const ConvOp& op, void* stream);
bool conv_direct_supported(const ConvOp& op);
int launch_conv_direct(const ConvOp& op, void* stream);
bool conv_tc_supported(const ConvOp& op, int precision);
int launch_conv_tc(const ConvOp& op, int precision, void* stream);
// Swizzled per-(n-tile, k-stage) shared-memory images of OIKK weights.
// chunk_major: K stages ordered (channel chunk, tap) for the halo kernel,
// else (tap, channel chunk).
std::vector<uint8_t> pack_tc_weights(const float* w_oikk, int co, int ci, int k,
                                     int precision, const ConvOp& shape_op,
                                     bool chunk_major);
bool conv_tc_halo_eligible(const ConvOp& op, int precision);

}  // namespace ts
