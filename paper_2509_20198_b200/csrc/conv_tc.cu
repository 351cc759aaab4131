// K3 tensor-core path: tcgen05 implicit-GEMM convolution (sm_100a).
//
// Same operator as conv_simt.cu (refiner.py:330-396: cross-correlation +
// bias + leaky ReLU, nearest-up2 fused into the input read, crop-aware
// output window) mapped onto the 5th-gen tensor cores:
//
//   GEMM view   M = 128 output pixels per CTA tile, N = BN output channels,
//               K = (tap, channel) with channels innermost, BKC channels per
//               pipeline stage (one 128-byte K-major row per pixel).
//   producers   warps 0-3, one thread per tile row: im2col-gather the
//               pixel's 128 bytes of input (vector loads; zero outside the
//               image; up2 folded into the address), convert/split, store
//               into the SWIZZLE_128B K-major shared-memory image, publish
//               with fence.proxy.async + mbarrier arrive.  Thread 0 also
//               streams the stage's weight tile with one cp.async.bulk
//               (weights are pre-swizzled on the host into the exact smem
//               image) completing on the same mbarrier (expect_tx).
//   MMA         warp 4, one elected thread: tcgen05.mma (kind::tf32 or
//               kind::f16/bf16) from smem descriptors into a TMEM fp32
//               accumulator; tcgen05.commit releases the stage.
//   epilogue    warps 0-3 again: tcgen05.ld 32x32b (warp w owns TMEM lanes
//               32w..32w+31 = tile rows), + bias, leaky ReLU, fp32 NHWC store
//               at the concat channel offset.
//
// Precision modes:
//   TC_TF32X3  fp32-accurate "3xTF32": a = a_hi + a_lo (a_hi = rna-tf32(a)),
//              D += A_hi B_hi + A_hi B_lo + A_lo B_hi   (3 MMAs per k-step).
//   TC_BF16    operands rounded to bf16, fp32 accumulation (1 MMA/k-step).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "conv.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int BM = 128;
constexpr int kProducers = 128;          // 4 warps
constexpr int kThreads = kProducers + 32;  // + MMA warp
constexpr int kRowBytes = 128;           // one SW128 K-major row

// ------------------------------------------------------------------ PTX

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   su32(dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr),
               "r"(ncols));
}
template <int KIND>  // 0 = tf32, 1 = f16 (bf16 operands)
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
  if (KIND == 0)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// SWIZZLE_128B K-major smem descriptor (sm_100 UMMA layout: start>>4 at
// [0,14), LBO>>4 at [16,30), SBO>>4 at [32,46), version 1 at [46,48),
// layout type 2 = SWIZZLE_128B at [61,64)).  SBO = 8 rows x 128 B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor: D f32, A/B format (tf32 = 2, bf16 = 1), K-major
__host__ __device__ constexpr uint32_t make_idesc(uint32_t ab_fmt, int n) {
  return (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

struct TcArgs {
  ConvOp op;
  const uint8_t* wpk;     // packed weights [n_tile][kstage][split][BN][128B]
  int bn;                 // N tile (multiple of 16)
  int stages;             // pipeline depth
  int kiters;             // k-stages = taps * cchunks
  int cchunks;            // ceil(Cin / BKC)
};

template <int MODE>  // 0 = TF32X3, 1 = BF16
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(TcArgs T) {
  constexpr int NSPLIT = MODE == 0 ? 2 : 1;     // operand copies (hi, lo)
  constexpr int BKC = MODE == 0 ? 32 : 64;      // channels per stage
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ConvOp& op = T.op;
  const int BN = T.bn, S = T.stages;
  const int a_bytes = BM * kRowBytes * NSPLIT;
  const int b_bytes = BN * kRowBytes * NSPLIT;
  const int stage_bytes = a_bytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int64_t M = (int64_t)op.batch * wy * wx;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int Cin = op.in.C, Cout = op.out.C;
  uint32_t ncols = 32;
  while ((int)ncols < BN) ncols <<= 1;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, kProducers);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ---------------- producers: one thread = one tile row (pixel) ----
    const int64_t gm = m0 + tid;
    const bool valid = gm < M;
    int b = 0, oy = 0, ox = 0;
    if (valid) {
      b = (int)(gm / ((int64_t)wy * wx));
      const int r = (int)(gm - (int64_t)b * wy * wx);
      oy = op.oy0 + r / wx;
      ox = op.ox0 + r % wx;
    }
    const int Hl = op.up2 ? 2 * op.in.H : op.in.H;
    const int Wl = op.up2 ? 2 * op.in.W : op.in.W;
    const float* inb =
        op.in.base + (int64_t)b * op.in.H * op.in.W * op.in.cstride + op.in.coff;
    const uint8_t* wsrc = T.wpk + (size_t)blockIdx.y * T.kiters * b_bytes;
    const int r8 = tid & 7;
    const int row_off = (tid >> 3) * 1024 + r8 * kRowBytes;
    for (int it = 0; it < T.kiters; ++it) {
      const int s = it % S;
      const uint32_t ph = (it / S) & 1;
      mbar_wait(empty + s, ph ^ 1);
      uint8_t* sa = smem + s * stage_bytes;
      uint8_t* sb = sa + a_bytes;
      const int tap = it / T.cchunks;
      const int c0 = (it - tap * T.cchunks) * BKC;
      const int ky = tap / op.k, kx = tap - ky * op.k;
      int iy = oy * op.stride - op.pad + ky, ix = ox * op.stride - op.pad + kx;
      const bool inside = valid && iy >= 0 && iy < Hl && ix >= 0 && ix < Wl;
      if (op.up2) { iy >>= 1; ix >>= 1; }
      const float* src = inb + ((int64_t)iy * op.in.W + ix) * op.in.cstride + c0;
      const int nvalid = inside ? min(BKC, Cin - c0) : 0;  // multiple of 4
      if (MODE == 0) {
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          v[j] = (4 * j < nvalid) ? __ldg(reinterpret_cast<const float4*>(src) + j)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 hi = make_float4(to_tf32(v[j].x), to_tf32(v[j].y), to_tf32(v[j].z),
                                  to_tf32(v[j].w));
          float4 lo = make_float4(v[j].x - hi.x, v[j].y - hi.y, v[j].z - hi.z,
                                  v[j].w - hi.w);
          const int off = row_off + ((j ^ r8) << 4);
          *reinterpret_cast<float4*>(sa + off) = hi;
          *reinterpret_cast<float4*>(sa + BM * kRowBytes + off) = lo;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 p = make_float4(0.f, 0.f, 0.f, 0.f), q = p;
          if (8 * j < nvalid) p = __ldg(reinterpret_cast<const float4*>(src) + 2 * j);
          if (8 * j + 4 < nvalid) q = __ldg(reinterpret_cast<const float4*>(src) + 2 * j + 1);
          uint4 w;
          w.x = pack_bf16(p.x, p.y);
          w.y = pack_bf16(p.z, p.w);
          w.z = pack_bf16(q.x, q.y);
          w.w = pack_bf16(q.z, q.w);
          *reinterpret_cast<uint4*>(sa + row_off + ((j ^ r8) << 4)) = w;
        }
      }
      fence_proxy_async();
      if (tid == 0) {
        bulk_g2s(sb, wsrc + (size_t)it * b_bytes, b_bytes, full + s);
        mbar_arrive_tx(full + s, b_bytes);
      } else {
        mbar_arrive(full + s);
      }
    }
    // ---------------- epilogue: TMEM -> bias/lrelu -> NHWC fp32 -------
    mbar_wait(done, 0);
    tc_fence_after();
    float* o = op.out.base +
               (((int64_t)b * op.out.H + oy) * op.out.W + ox) * op.out.cstride + op.out.coff;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tmem_ld16(tmem + lane_base + c, v);  // warp-collective: every lane loads
      if (valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c + i;
          if (n < Cout) {
            float x = v[i] + op.bias[n];
            if (op.lrelu) x = x >= 0.f ? x : 0.01f * x;
            o[n] = x;
          }
        }
      }
    }
  } else {
    // ---------------- MMA issuer (warp 4, one thread) ----------------
    constexpr uint32_t fmt = MODE == 0 ? 2u : 1u;
    const uint32_t idesc = make_idesc(fmt, BN);
    if ((tid & 31) == 0) {
      for (int it = 0; it < T.kiters; ++it) {
        const int s = it % S;
        const uint32_t ph = (it / S) & 1;
        mbar_wait(full + s, ph);
        tc_fence_after();
        const uint32_t a0 = su32(smem + s * stage_bytes);
        const uint32_t b0 = a0 + a_bytes;
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 4 x 32-byte K steps per 128-B row
          const uint64_t ahi = sw128_desc(a0 + 32 * k);
          const uint64_t bhi = sw128_desc(b0 + 32 * k);
          const uint32_t acc = (it | k) ? 1u : 0u;
          if (MODE == 0) {
            const uint64_t alo = sw128_desc(a0 + BM * kRowBytes + 32 * k);
            const uint64_t blo = sw128_desc(b0 + BN * kRowBytes + 32 * k);
            umma<0>(tmem, ahi, bhi, idesc, acc);
            umma<0>(tmem, ahi, blo, idesc, 1u);
            umma<0>(tmem, alo, bhi, idesc, 1u);
          } else {
            umma<1>(tmem, ahi, bhi, idesc, acc);
          }
        }
        umma_commit(empty + s);
      }
      umma_commit(done);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, ncols);
  }
}

// ---------------------------------------------------------------- host

uint32_t f2tf32_rna(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return u;  // inf / nan
  u += 0x1000u;
  return u & 0xFFFFE000u;
}

uint16_t f2bf16_rn(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)(u >> 16 | ((u & 0xFFFF) ? 0x40 : 0));
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

struct TcPlan {
  int bn, stages, kiters, cchunks, ntiles, mode;
  size_t smem;
};

TcPlan plan_for(const ConvOp& op, int mode) {
  TcPlan p{};
  const int bkc = mode == 0 ? 32 : 64;
  const int nsplit = mode == 0 ? 2 : 1;
  const int n16 = (op.out.C + 15) / 16 * 16;
  const int cap = mode == 0 ? 128 : 256;
  p.ntiles = (n16 + cap - 1) / cap;
  p.bn = ((n16 + p.ntiles - 1) / p.ntiles + 15) / 16 * 16;
  p.cchunks = (op.in.C + bkc - 1) / bkc;
  p.kiters = op.k * op.k * p.cchunks;
  const size_t stage = (size_t)(BM + p.bn) * kRowBytes * nsplit;
  const size_t budget = 200 * 1024;
  p.stages = (int)std::min<size_t>(4, budget / stage);
  if (p.stages < 2) p.stages = 2;
  p.stages = std::min(p.stages, std::max(2, p.kiters));
  p.smem = p.stages * stage + 1024 + 8 * (2 * p.stages + 2) + 16;
  p.mode = mode;
  return p;
}

}  // namespace

bool conv_tc_supported(const ConvOp& op, int precision) {
  if (precision != 1 && precision != 2) return false;
  // vector loads need 16-byte aligned channel runs
  return op.in.C % 4 == 0 && op.in.cstride % 4 == 0 && op.in.coff % 4 == 0 &&
         op.out.C >= 8;
}

// Packs OIKK fp32 weights into the per-(n-tile, k-stage) swizzled smem image.
std::vector<uint8_t> pack_tc_weights(const float* w_oikk, int co, int ci, int k,
                                     int precision, const ConvOp& shape_op) {
  const int mode = precision == 1 ? 0 : 1;
  ConvOp op = shape_op;
  op.in.C = ci;
  op.out.C = co;
  op.k = k;
  const TcPlan p = plan_for(op, mode);
  const int bkc = mode == 0 ? 32 : 64;
  const int nsplit = mode == 0 ? 2 : 1;
  const size_t b_bytes = (size_t)p.bn * kRowBytes * nsplit;
  std::vector<uint8_t> out((size_t)p.ntiles * p.kiters * b_bytes, 0);
  for (int nt = 0; nt < p.ntiles; ++nt)
    for (int it = 0; it < p.kiters; ++it) {
      const int tap = it / p.cchunks, c0 = (it % p.cchunks) * bkc;
      const int ky = tap / k, kx = tap % k;
      uint8_t* base = out.data() + ((size_t)nt * p.kiters + it) * b_bytes;
      for (int r = 0; r < p.bn; ++r) {
        const int n = nt * p.bn + r;
        for (int e = 0; e < bkc; ++e) {
          const int c = c0 + e;
          float v = 0.f;
          if (n < co && c < ci) v = w_oikk[(((size_t)n * ci + c) * k + ky) * k + kx];
          const int esize = mode == 0 ? 4 : 2;
          const int byte = e * esize;
          const int chunk = byte >> 4, within = byte & 15;
          const size_t off = (size_t)(r >> 3) * 1024 + (r & 7) * kRowBytes +
                             ((chunk ^ (r & 7)) << 4) + within;
          if (mode == 0) {
            const uint32_t hi = f2tf32_rna(v);
            float hf;
            memcpy(&hf, &hi, 4);
            const float lo = v - hf;
            memcpy(base + off, &hi, 4);
            memcpy(base + (size_t)p.bn * kRowBytes + off, &lo, 4);
          } else {
            const uint16_t h = f2bf16_rn(v);
            memcpy(base + off, &h, 2);
          }
        }
      }
    }
  return out;
}

int launch_conv_tc(const ConvOp& op, int precision, void* stream) {
  const int mode = precision == 1 ? 0 : 1;
  const TcPlan p = plan_for(op, mode);
  const int64_t M = (int64_t)op.batch * (op.oy1 - op.oy0) * (op.ox1 - op.ox0);
  if (M <= 0) return TS_OK;
  TcArgs a{op, op.w_tc, p.bn, p.stages, p.kiters, p.cchunks};
  dim3 grid((unsigned)ceil_div<int64_t>(M, BM), (unsigned)p.ntiles);
  cudaStream_t s = as_stream(stream);
  if (mode == 0) {
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_tc_kernel<0>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)p.smem));
    ts::count_launch(), conv_tc_kernel<0><<<grid, kThreads, p.smem, s>>>(a);
  } else {
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_tc_kernel<1>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)p.smem));
    ts::count_launch(), conv_tc_kernel<1><<<grid, kThreads, p.smem, s>>>(a);
  }
  TS_LAUNCH_CHECK();
  return TS_OK;
}

}  // namespace ts
