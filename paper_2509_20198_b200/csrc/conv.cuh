// Convolution layer descriptors shared by the refine planner and kernels.
#pragma once

#include <stdint.h>

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
};

int launch_conv_simt(const ConvOp& op, void* stream);

}  // namespace ts
