// Shared helpers for the ts_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ts_b200.h"

#define TS_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return TS_E_CUDA;                \
  } while (0)

#define TS_LAUNCH_CHECK() TS_CUDA_TRY(cudaGetLastError())

namespace ts {

// Number of kernels this library has launched (ts_launch_count).
void count_launch();

constexpr double kPatch = 640.0;
constexpr double kTexel = 10.0;
constexpr int kRes = 96;
constexpr int kOut = 64;
constexpr double kRadius = 480.0;
constexpr double kBaryTol = 1e-9;
constexpr int kCrop = 16;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// IEEE round-to-nearest fp64 ops that the compiler may never contract into
// an FMA: numpy evaluates every one of these with its own rounding.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// floor() of an fp64 into int64 the way numpy's floor + astype(int64) does.
__device__ __forceinline__ int64_t floor_i64(double v) { return (int64_t)floor(v); }

// cell centre coordinate -1 + (k + 0.5) * (2 / res)  (patches.py:210)
__device__ __forceinline__ double cell_center(int k, int res) {
  // 2 / 96 folded at compile time is the same correctly rounded double as
  // numpy's (and __ddiv_rn's) quotient; other resolutions divide
  const double step = res == kRes ? 2.0 / kRes : ddiv(2.0, (double)res);
  return dadd(-1.0, dmul((double)k + 0.5, step));
}

template <typename T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) { return (a + b - 1) / b; }

// SM count of the current device (cached per device; 0 on error)
inline int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  if (!cache[dev] &&
      cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  return cache[dev];
}

}  // namespace ts
