// WireHeightmap serialisation on the device (server.py:126-142
// wire_heightmap, docs/wire.md "WireHeightmap"): the refined tiles of a
// batch become their little-endian wire records in one launch, so a server
// copies finished bytes instead of pulling B x 64 x 64 x 4 floats to the host
// and repacking them per patch in Python.
//
// Record (packed, little-endian):
//   i32 i, i32 j, f32 c_z, u8 stage, u8 flags (bit 0: colour plane),
//   f32[64*64] heights_rel (row-major, row = y),
//   u8[64*64*3] rgb = clip(round_half_even(f32(rgb * 255)), 0, 255)  if flags & 1
// 14 + 16384 (+ 12288) bytes; records are written back to back.
//
// One CTA per record: the record is assembled in shared memory (its body
// starts at byte 14, so the floats are 2-byte aligned there) and streamed
// out with 16-bit stores (record sizes are even).
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int kWireHead = 14;
constexpr int kWireH = kOut * kOut * 4;
constexpr int kWireRgb = kOut * kOut * 3;
constexpr int kWireThreads = 256;

__global__ void __launch_bounds__(kWireThreads) wire_kernel(const float* __restrict__ out,
                                                            const double* __restrict__ cz,
                                                            const int32_t* __restrict__ ij,
                                                            const uint8_t* __restrict__ stage,
                                                            int has_rgb, uint8_t* wire) {
  __shared__ __align__(16) uint16_t rec[(kWireHead + kWireH + kWireRgb) / 2];
  uint8_t* rb = reinterpret_cast<uint8_t*>(rec);
  const int64_t p = blockIdx.x;
  const int size = kWireHead + kWireH + (has_rgb ? kWireRgb : 0);
  const float4* src = reinterpret_cast<const float4*>(out) + p * kOut * kOut;
  for (int t = threadIdx.x; t < kOut * kOut; t += kWireThreads) {
    const float4 v = __ldg(src + t);  // heights_rel, r, g, b
    const uint32_t hb = __float_as_uint(v.x);
    rec[(kWireHead + 4 * t) / 2] = (uint16_t)(hb & 0xFFFFu);
    rec[(kWireHead + 4 * t) / 2 + 1] = (uint16_t)(hb >> 16);
    if (has_rgb) {
      const float c[3] = {v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        // numpy: float32 * 255 (one rounding), np.round = half to even,
        // clip to [0, 255], astype(uint8)
        const float r = fminf(fmaxf(rintf(__fmul_rn(c[k], 255.0f)), 0.0f), 255.0f);
        rb[kWireHead + kWireH + 3 * t + k] = (uint8_t)r;
      }
    }
  }
  if (threadIdx.x == 0) {
    const int32_t hi = ij[2 * p], hj = ij[2 * p + 1];
    const float c = __double2float_rn(cz[p]);
    const uint32_t cb = __float_as_uint(c);
    rec[0] = (uint16_t)((uint32_t)hi & 0xFFFFu);
    rec[1] = (uint16_t)((uint32_t)hi >> 16);
    rec[2] = (uint16_t)((uint32_t)hj & 0xFFFFu);
    rec[3] = (uint16_t)((uint32_t)hj >> 16);
    rec[4] = (uint16_t)(cb & 0xFFFFu);
    rec[5] = (uint16_t)(cb >> 16);
    rec[6] = (uint16_t)(stage[p] | ((has_rgb ? 1u : 0u) << 8));  // stage, flags
  }
  __syncthreads();
  uint16_t* dst = reinterpret_cast<uint16_t*>(wire + p * (int64_t)size);
  for (int w = threadIdx.x; w < size / 2; w += kWireThreads) dst[w] = rec[w];
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" size_t ts_wire_record_size(int has_rgb) {
  return (size_t)(kWireHead + kWireH + (has_rgb ? kWireRgb : 0));
}

extern "C" int ts_wire_heightmaps(const float* d_out, const double* d_cz, const int32_t* d_ij,
                                  const uint8_t* d_stage, int has_rgb, int batch,
                                  uint8_t* d_wire, void* stream) {
  if (batch < 0) return TS_E_INVALID;
  if (batch == 0) return TS_OK;
  if (!d_out || !d_cz || !d_ij || !d_stage || !d_wire) return TS_E_INVALID;
  if ((reinterpret_cast<uintptr_t>(d_out) & 15) || (reinterpret_cast<uintptr_t>(d_wire) & 1))
    return TS_E_INVALID;
  ts::count_launch(), wire_kernel<<<batch, kWireThreads, 0, as_stream(stream)>>>(
                          d_out, d_cz, d_ij, d_stage, has_rgb ? 1 : 0, d_wire);
  TS_LAUNCH_CHECK();
  return TS_OK;
}
