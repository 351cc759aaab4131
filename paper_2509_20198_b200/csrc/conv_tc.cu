// K3 tensor-core path: persistent tcgen05 implicit-GEMM convolution.
//
// Same operator as conv_simt.cu (refiner.py:330-396: cross-correlation +
// bias + leaky ReLU, nearest-up2 folded into the input read, crop-aware
// output window) on the 5th-generation tensor cores.
//
//   GEMM view   M = 128 output pixels per tile, N = BN output channels,
//               K = (tap, channel), channels innermost; one pipeline stage =
//               one tap x KC channels = one 128-byte K-major row per pixel.
//   warps 0-7   producers, two threads per tile row: im2col-gather the
//               pixel's fp32 input (16-byte loads, zeros outside the image,
//               up2 folded into the address), split it into the operand
//               planes of the precision mode and store them into the
//               SWIZZLE_128B K-major smem image; publish with
//               fence.proxy.async + mbarrier arrive.  Thread 0 streams the
//               stage's pre-swizzled weight planes with one cp.async.bulk
//               completing on the same mbarrier (expect_tx).
//   warp 8      MMA issuer (one thread) + TMEM owner: tcgen05.mma from smem
//               descriptors into one of two TMEM fp32 accumulators;
//               tcgen05.commit frees smem stages and hands accumulators to
//               the epilogue, so the next tile's mainloop overlaps the
//               previous tile's epilogue.
//   warps 9-12  epilogue: tcgen05.ld 32x32b (warp w reads lane quadrant
//               w%4 = its 32 tile rows), + bias, leaky ReLU, fp32 NHWC store
//               at the concat channel offset, then release the accumulator.
//   grid        persistent: min(tiles, 148 x CTAs/SM), static tile stride.
//
// Precision modes (operand planes per tensor, MMAs per 32-byte K step):
//   1 TF32X3  a = hi + lo, hi = rna-tf32(a):  hi*hi + hi*lo + lo*hi   (2, 3)
//   2 BF16    a = bf16(a):                    a*b                    (1, 1)
//   3 BF16X3  a = a0 + a1 + a2 (exact 3-way bf16 split, 24 mantissa bits):
//             a0b0 + a0b1 + a1b0 + a1b1 + a0b2 + a2b0                 (3, 6)
// Modes 1 and 3 are fp32-accurate; 3 runs at the bf16 tensor rate.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "conv.cuh"
#include "tc_ptx.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

constexpr int BM = 128;
constexpr int kRowBytes = 128;
constexpr int kProdWarps = 8;
constexpr int kProd = kProdWarps * 32;      // 256 producer threads
constexpr int kMmaWarp = kProdWarps;        // warp 8
constexpr int kThreads = (kProdWarps + 1 + 4) * 32;

using namespace tcx;

struct TcArgs {
  ConvOp op;
  const uint8_t* wpk;   // [n_tile][kiter][plane][BN][128 B]
  int bn, stages, kiters, cchunks, n_tiles;
  int64_t m_tiles;
  int wide;  // MODE 4 with BN > 128: the three products accumulate into the
             // same BN columns (no plane stacking), N up to 256 per MMA
};

// Row table of one tile: input pixel origin of every output pixel.
struct RowInfo {
  int b, iy0, ix0;  // b < 0: row beyond M
};

// Stores one 16-byte fp32 source piece of a row into the operand planes.
template <int MODE>
__device__ __forceinline__ void store_piece(uint8_t* sa, int row, int piece, float4 a) {
  constexpr int plane_bytes = BM * kRowBytes;
  const int base = (row >> 3) * 1024 + (row & 7) * kRowBytes;
  if (MODE == 1) {  // 16 source bytes -> one 16-byte chunk per plane
    const int off = base + ((piece ^ (row & 7)) << 4);
    const float4 hi = make_float4(tf32_hi(a.x), tf32_hi(a.y), tf32_hi(a.z), tf32_hi(a.w));
    *reinterpret_cast<float4*>(sa + off) = hi;
    *reinterpret_cast<float4*>(sa + plane_bytes + off) =
        make_float4(a.x - hi.x, a.y - hi.y, a.z - hi.z, a.w - hi.w);
  } else {  // 4 floats -> 8 bytes (half a chunk) per plane
    const int off = base + (((piece >> 1) ^ (row & 7)) << 4) + ((piece & 1) << 3);
    if (MODE == 2) {
      *reinterpret_cast<uint2*>(sa + off) =
          make_uint2(hi_halves(rn_bf(a.x), rn_bf(a.y)), hi_halves(rn_bf(a.z), rn_bf(a.w)));
    } else if (Mode<MODE>::f16) {
      store_split_h(sa + off, plane_bytes, a);
    } else {
      store_split2(sa + off, plane_bytes, a);
    }
  }
}

__device__ __forceinline__ void prod_bar() {  // the 256 producer threads
  asm volatile("bar.sync 1, %0;" ::"n"(kProd) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(TcArgs T) {
  using Md = Mode<MODE>;
  constexpr int PA = Md::pa, PB = Md::pb;
  constexpr int KC = Md::kc;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array keeps the shared address
  // space (STS/LDS instead of generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const ConvOp& op = T.op;
  const int BN = T.bn, S = T.stages;
  const int a_bytes = PA * BM * kRowBytes;
  const int b_bytes = PB * BN * kRowBytes;
  const int stage_bytes = a_bytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;    // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // bias of every output column (zero past C_out), read by the epilogue
  // from shared memory instead of one global load per element
  float* s_bias = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(tmem_slot + 1) + 15) & ~uintptr_t(15));

  const int tid = threadIdx.x, warp = tid >> 5;
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int64_t M = (int64_t)op.batch * wy * wx;
  for (int i = tid; i < T.n_tiles * T.bn; i += blockDim.x)
    s_bias[i] = i < op.out.C ? __ldg(op.bias + i) : 0.f;
  const int Cin = op.in.C, Cout = op.out.C;
  const int64_t total_tiles = T.m_tiles * T.n_tiles;
  // MODE 4 stacks the two weight planes along N (one MMA per A plane,
  // N = 2 BN; the epilogue adds the halves): half the A-operand shared
  // memory reads of one MMA per plane pair
  // MODE 5 (FP16X3): [main | correction] column blocks, same stacking
  const int NST = ((MODE == 4 && !T.wide) || Md::f16) ? 2 : 1;
  // two accumulator buffers (epilogue overlaps the next tile) when they fit
  const int AB = 2 * NST * BN <= 512 ? 2 : 1;
  uint32_t ncols = 32;
  while ((int)ncols < AB * NST * BN) ncols <<= 1;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, kProdWarps);  // one arrival per producer warp
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, 4);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kProdWarps) {
    // ------------------------------ producers ------------------------------
    // Lanes of a warp cover consecutive 16-byte pieces of the same pixel
    // rows, so every global load instruction reads whole 128-byte lines.
    // Software-pipelined: stage k+1's loads are in flight while stage k is
    // split and stored.
    constexpr int PPR = KC / 4;               // fp32 pieces per row per stage
    constexpr int PIECES = BM * PPR / kProd;  // pieces per thread per stage
    const int Hl = op.up2 ? 2 * op.in.H : op.in.H;
    const int Wl = op.up2 ? 2 * op.in.W : op.in.W;
    const int sh = op.up2 ? 1 : 0;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int64_t mt = tile / T.n_tiles;
      const int nt = (int)(tile - mt * T.n_tiles);
      // per-piece pixel origin (registers): image base, iy0, ix0
      const float* pbase[PIECES];
      int py0[PIECES], px0[PIECES];
#pragma unroll
      for (int j = 0; j < PIECES; ++j) {
        const int p = j * kProd + tid;
        const int64_t gm = mt * BM + p / PPR;
        py0[j] = -(1 << 28);  // rows beyond M: always outside
        px0[j] = 0;
        pbase[j] = op.in.base;
        if (gm < M) {
          const int b = (int)(gm / ((int64_t)wy * wx));
          const int q = (int)(gm - (int64_t)b * wy * wx);
          py0[j] = (op.oy0 + q / wx) * op.stride - op.pad;
          px0[j] = (op.ox0 + q % wx) * op.stride - op.pad;
          pbase[j] = op.in.base + (int64_t)b * op.in.H * op.in.W * op.in.cstride +
                     op.in.coff + 4 * (p % PPR);
        }
      }
      const uint8_t* wsrc = T.wpk + (size_t)nt * T.kiters * b_bytes;
      auto load_stage = [&](int c0, int ky, int kx, float4* v) {
#pragma unroll
        for (int j = 0; j < PIECES; ++j) {
          const int iy = py0[j] + ky, ix = px0[j] + kx;
          const int c = c0 + 4 * ((j * kProd + tid) % PPR);
          v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (iy >= 0 && iy < Hl && ix >= 0 && ix < Wl && c < Cin)
            v[j] = __ldg(reinterpret_cast<const float4*>(
                pbase[j] + ((int64_t)(iy >> sh) * op.in.W + (ix >> sh)) * op.in.cstride + c0));
        }
      };
      int c0 = 0, ky = 0, kx = 0;  // (tap, channel chunk) walk, no division
      float4 cur[PIECES], nxt[PIECES];
      load_stage(0, 0, 0, cur);
      for (int kit = 0; kit < T.kiters; ++kit) {
        c0 += KC;
        if (c0 >= T.cchunks * KC) {
          c0 = 0;
          if (++kx == op.k) { kx = 0; ++ky; }
        }
        if (kit + 1 < T.kiters) load_stage(c0, ky, kx, nxt);
        mbar_wait(empty + s, ph ^ 1);
        uint8_t* sa = smem + s * stage_bytes;
#pragma unroll
        for (int j = 0; j < PIECES; ++j) {
          const int p = j * kProd + tid;
          store_piece<MODE>(sa, p / PPR, p % PPR, cur[j]);
        }
        fence_proxy_async();
        __syncwarp();
        if (tid == 0) {
          bulk_g2s(sa + a_bytes, wsrc + (size_t)kit * b_bytes, b_bytes, full + s);
          mbar_arrive_tx(full + s, b_bytes);
        } else if ((tid & 31) == 0) {
          mbar_arrive(full + s);
        }
        if (++s == S) { s = 0; ph ^= 1; }
#pragma unroll
        for (int j = 0; j < PIECES; ++j) cur[j] = nxt[j];
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------ MMA issuer -----------------------------
    // The whole warp walks the loop (uniform registers), one elected lane
    // issues; descriptors are integer offsets from precomputed bases.
    const int NMMA = Md::f16 ? 2 * BN : NST * BN;  // stacked B rows per MMA
    const uint32_t idesc = make_idesc(mode_fmt<MODE>(), NMMA > 256 ? 256 : NMMA);
    const uint32_t idesc_b0 = make_idesc(mode_fmt<MODE>(), BN);
    (void)idesc_b0;
    const uint64_t d_smem = sw128_desc(su32(smem));
    const uint32_t pa = (BM * kRowBytes) >> 4, pb = (BN * kRowBytes) >> 4;
    int s = 0, lt = 0;
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++lt) {
      const int acc = lt % AB;
      mbar_wait(acc_empty + acc, ((lt / AB) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * NST * BN;
      for (int kit = 0; kit < T.kiters; ++kit) {
        mbar_wait(full + s, ph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t a0 = d_smem + (uint64_t)((s * stage_bytes) >> 4);
          const uint64_t b0 = a0 + (uint64_t)(a_bytes >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 x 32-byte K steps per row
            const uint32_t first = (kit | k) ? 1u : 0u;
            const uint64_t ak = a0 + 2 * k, bk = b0 + 2 * k;
            if (MODE == 1) {
              umma<true>(d, ak, bk, idesc, first);
              umma<true>(d, ak, bk + pb, idesc, 1u);
              umma<true>(d, ak + pa, bk, idesc, 1u);
            } else if (MODE == 2) {
              umma<false>(d, ak, bk, idesc, first);
            } else if (Md::f16) {
              // a0 . [b0 | b1] -> [main | corr], a1 . b0 -> corr
              umma<false>(d, ak, bk, idesc, first);
              umma<false>(d + BN, ak + pa, bk, idesc_b0, 1u);
            } else if (MODE == 4) {
              // a0 . [b0 | b1] (N = 2 BN), then a1 . b0 (N = BN): the
              // a1 . b1 term (<= 2^-18 |ab|, the size of the split
              // residual) is dropped.  Wide tiles: the same three
              // products, each N = BN, into the same columns.
              if (T.wide) {
                umma<false>(d, ak, bk, idesc_b0, first);
                umma<false>(d, ak, bk + pb, idesc_b0, 1u);
              } else {
                umma<false>(d, ak, bk, idesc, first);
              }
              umma<false>(d, ak + pa, bk, idesc_b0, 1u);
            } else {
              umma<false>(d, ak + pa, bk + pb, idesc, first);  // small terms first
              umma<false>(d, ak, bk + 2 * pb, idesc, 1u);
              umma<false>(d, ak + pa, bk, idesc, 1u);
              umma<false>(d, ak, bk + pb, idesc, 1u);
              umma<false>(d, ak, bk, idesc, 1u);
            }
          }
          umma_commit(empty + s);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
      if (elect_one()) umma_commit(acc_full + acc);
      __syncwarp();
    }
  } else {
    // ------------------------------ epilogue -------------------------------
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const bool vec = (op.out.cstride % 4 == 0) && (op.out.coff % 4 == 0);
    const bool vec8 = (op.out.cstride % 8 == 0) && (op.out.coff % 8 == 0) &&
                      ((reinterpret_cast<uintptr_t>(op.out.base) & 31) == 0);
    int lt = 0;
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++lt) {
      const int acc = lt % AB;
      const int64_t mt = tile / T.n_tiles;
      const int nt = (int)(tile - mt * T.n_tiles);
      const int n0 = nt * BN;
      const int64_t gm = mt * BM + q * 32 + (tid & 31);
      const bool valid = gm < M;
      float* o = nullptr;
      float* oblk = nullptr;
      int ochan = 0;
      if (valid) {
        const int b = (int)(gm / ((int64_t)wy * wx));
        const int r = (int)(gm - (int64_t)b * wy * wx);
        const int y = op.oy0 + r / wx, x = op.ox0 + r % wx;
        o = op.out.base + (((int64_t)b * op.out.H + y) * op.out.W + x) * op.out.cstride +
            op.out.coff;
        int64_t blk;
        act_block(op.out, b, y, x, blk, ochan);
        oblk = op.out.base + blk;
      }
      mbar_wait(acc_full + acc, (lt / AB) & 1);
      tc_fence_after();
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(tmem + lane_base + acc * NST * BN + c, v);  // warp-collective
        if (NST >= 2) {
          float w[16];
          tmem_ld16(tmem + lane_base + acc * NST * BN + BN + c, w);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += Md::f16 ? w[i] * kF16LoInv : w[i];
        }
        if (valid) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = n0 + c + i;
            float x = v[i] + s_bias[n];
            if (op.lrelu) x = x >= 0.f ? x : 0.01f * x;
            v[i] = x;
          }
          if (op.out.planes) {
            if (n0 + c + 16 <= Cout) store16_planes(oblk, op.out.cstride, ochan + n0 + c, v, op.out.planes == 2);
          } else if (vec8 && n0 + c + 16 <= Cout) {
            st_v8(o + n0 + c, v);
            st_v8(o + n0 + c + 8, v + 8);
          } else if (vec && n0 + c + 16 <= Cout) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              *reinterpret_cast<float4*>(o + n0 + c + 4 * i) =
                  make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (n0 + c + i < Cout) o[n0 + c + i] = v[i];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(acc_empty + acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, ncols);
  }
}

// ===========================================================================
// Halo-reuse variant for stride-1 k x k convolutions (no up2).
//
// Output positions are linearised with a padded pitch Wp = wx + k - 1 and
// (wy + k - 1) rows per image, so the input of tap (ky, kx) for the 128
// consecutive positions of a tile is the contiguous run of "halo" rows
// starting at ky*Wp + kx.  Producers load each channel chunk's halo run
// (128 + (k-1)(Wp+1) rows) ONCE per tile into one SWIZZLE_128B image; the
// MMA issuer walks the k*k taps by sliding the A descriptor start address
// over that image (the swizzle is a function of absolute smem address
// bits), so every input element is gathered, split and stored once per
// tile instead of k*k times.  A dedicated warp streams the per-tap weight
// tiles through a small ring with cp.async.bulk.
// ===========================================================================

constexpr int kHThreads = (kProdWarps + 1 + 4 + 1) * 32;  // + B-loader warp 13

struct HaloArgs {
  ConvOp op;
  const uint8_t* wpk;   // [n_tile][chunk][tap][plane][BN][128 B]
  int bn, bstages, cchunks, taps, wp, lrows, n_tiles;
  int64_t m_tiles, positions;
};

template <int MODE>
__global__ void __launch_bounds__(kHThreads, 1) conv_tc_halo_kernel(HaloArgs T) {
  using Md = Mode<MODE>;
  constexpr int PA = Md::pa, PB = Md::pb;
  constexpr int KC = Md::kc;
  constexpr int PPR = KC / 4;  // fp32 pieces per halo row
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const ConvOp& op = T.op;
  const int BN = T.bn, SB = T.bstages, L = T.lrows;
  const int plane_a = L * kRowBytes;
  const int halo_bytes = PA * plane_a;  // one halo buffer (2 are resident)
  const int b_bytes = PB * BN * kRowBytes;
  uint8_t* halo = smem;
  uint8_t* bring = smem + 2 * halo_bytes;
  uint64_t* bfull = reinterpret_cast<uint64_t*>(bring + SB * b_bytes);
  uint64_t* bempty = bfull + SB;
  uint64_t* hfull = bempty + SB;       // [2]
  uint64_t* hempty = hfull + 2;        // [2]
  uint64_t* acc_full = hempty + 2;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int64_t* rowoff = reinterpret_cast<int64_t*>(tmem_slot + 4);  // [2][L]

  const int tid = threadIdx.x, warp = tid >> 5;
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int kk1 = op.k - 1;
  const int Wp = T.wp;
  const int64_t img_pos = (int64_t)(wy + kk1) * Wp;
  const int Cin = op.in.C, Cout = op.out.C;
  const int64_t total_tiles = T.m_tiles * T.n_tiles;
  uint32_t ncols = 32;
  while ((int)ncols < 2 * BN) ncols <<= 1;

  if (tid == 0) {
    for (int s = 0; s < SB; ++s) {
      mbar_init(bfull + s, 1);
      mbar_init(bempty + s, 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(hfull + h, kProdWarps);
      mbar_init(hempty + h, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, 4);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kProdWarps) {
    // ------------------------- halo producers -------------------------
    // Halo buffers alternate per (tile, chunk); each producer thread walks
    // the same sequence, so buffer hb and its phase are uniform.
    int hb = 0, lt = 0;
    uint32_t hmask = 0;  // bit hb = phase parity of halo buffer hb
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++lt) {
      const int64_t mt = tile / T.n_tiles;
      const int64_t j0 = mt * BM;
      int64_t* ro = rowoff + (lt & 1) * L;
      // ro[] of tile lt-2 was last read by loads published before this
      // thread passed prod_bar of tile lt-1
      for (int j = tid; j < L; j += kProd) {
        const int64_t pos = j0 + j;
        int64_t off = -1;
        const int64_t b = pos / img_pos;
        if (b < op.batch) {
          const int r = (int)(pos - b * img_pos);
          // halo position -> (up2-folded) source pixel; zero outside the image
          const int iy = op.oy0 - op.pad + r / Wp, ix = op.ox0 - op.pad + r % Wp;
          const int sh = op.up2 ? 1 : 0;
          if (iy >= 0 && iy < (op.in.H << sh) && ix >= 0 && ix < (op.in.W << sh))
            off = ((b * op.in.H + (iy >> sh)) * op.in.W + (ix >> sh)) * op.in.cstride +
                  op.in.coff;
        }
        ro[j] = off;
      }
      prod_bar();
      for (int c = 0; c < T.cchunks; ++c) {
        mbar_wait(hempty + hb, ((hmask >> hb) & 1u) ^ 1u);
        uint8_t* sa = halo + hb * halo_bytes;
        const int c0 = c * KC;
        for (int pc = tid; pc < L * PPR; pc += kProd * 8) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int q = pc + u * kProd;
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (q < L * PPR) {
              const int row = q / PPR, piece = q % PPR;
              const int64_t off = ro[row];
              const int ch = c0 + 4 * piece;
              if (off >= 0 && ch < Cin)
                v[u] = __ldg(reinterpret_cast<const float4*>(op.in.base + off + ch));
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int q = pc + u * kProd;
            if (q < L * PPR) {
              const int row = q / PPR, piece = q % PPR;
              const int base = (row >> 3) * 1024 + (row & 7) * kRowBytes;
              const float4 a = v[u];
              if (MODE == 1) {
                const int o = base + ((piece ^ (row & 7)) << 4);
                const float4 hi =
                    make_float4(tf32_hi(a.x), tf32_hi(a.y), tf32_hi(a.z), tf32_hi(a.w));
                *reinterpret_cast<float4*>(sa + o) = hi;
                *reinterpret_cast<float4*>(sa + plane_a + o) =
                    make_float4(a.x - hi.x, a.y - hi.y, a.z - hi.z, a.w - hi.w);
              } else {
                const int o = base + (((piece >> 1) ^ (row & 7)) << 4) + ((piece & 1) << 3);
                if (MODE == 2)
                  *reinterpret_cast<uint2*>(sa + o) = make_uint2(
                      hi_halves(rn_bf(a.x), rn_bf(a.y)), hi_halves(rn_bf(a.z), rn_bf(a.w)));
                else
                  store_split2(sa + o, plane_a, a);
              }
            }
          }
        }
        fence_proxy_async();
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(hfull + hb);
        hmask ^= 1u << hb;
        hb ^= 1;
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------- MMA issuer -------------------------
    const uint32_t idesc = make_idesc(Md::tf32 ? 2u : 1u, BN);
    const uint64_t d_halo = sw128_desc(su32(halo));
    const uint64_t d_ring = sw128_desc(su32(bring));
    const uint32_t pa = (uint32_t)plane_a >> 4, pb = (BN * kRowBytes) >> 4;
    int s = 0, lt = 0, hb = 0;
    uint32_t bph = 0;
    uint32_t hmask = 0;  // bit hb = phase parity of halo buffer hb
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      mbar_wait(acc_empty + acc, ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * BN;
      for (int c = 0; c < T.cchunks; ++c) {
        mbar_wait(hfull + hb, (hmask >> hb) & 1u);
        hmask ^= 1u << hb;
        tc_fence_after();
        const uint64_t d_hb = d_halo + (uint64_t)((hb * halo_bytes) >> 4);
        int ky = 0, kx = 0;
        for (int t = 0; t < T.taps; ++t) {
          mbar_wait(bfull + s, bph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t a0 = d_hb + (uint64_t)((ky * Wp + kx) * (kRowBytes >> 4));
            const uint64_t b0 = d_ring + (uint64_t)((s * b_bytes) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t first = (c | t | k) ? 1u : 0u;
              const uint64_t ak = a0 + 2 * k, bk = b0 + 2 * k;
              if (MODE == 1) {
                umma<true>(d, ak, bk, idesc, first);
                umma<true>(d, ak, bk + pb, idesc, 1u);
                umma<true>(d, ak + pa, bk, idesc, 1u);
              } else if (MODE == 2) {
                umma<false>(d, ak, bk, idesc, first);
              } else if (MODE == 4) {
                umma<false>(d, ak + pa, bk + pb, idesc, first);
                umma<false>(d, ak + pa, bk, idesc, 1u);
                umma<false>(d, ak, bk + pb, idesc, 1u);
                umma<false>(d, ak, bk, idesc, 1u);
              } else {
                umma<false>(d, ak + pa, bk + pb, idesc, first);
                umma<false>(d, ak, bk + 2 * pb, idesc, 1u);
                umma<false>(d, ak + pa, bk, idesc, 1u);
                umma<false>(d, ak, bk + pb, idesc, 1u);
                umma<false>(d, ak, bk, idesc, 1u);
              }
            }
            umma_commit(bempty + s);
          }
          __syncwarp();
          if (++s == SB) { s = 0; bph ^= 1; }
          if (++kx == op.k) { kx = 0; ++ky; }
        }
        if (elect_one()) umma_commit(hempty + hb);
        __syncwarp();
        hb ^= 1;
      }
      if (elect_one()) umma_commit(acc_full + acc);
      __syncwarp();
    }
  } else if (warp == kHThreads / 32 - 1) {
    // ------------------------- weight loader -------------------------
    if ((tid & 31) == 0) {
      int s = 0;
      uint32_t bph = 0;
      for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int nt = (int)(tile % T.n_tiles);
        const uint8_t* wsrc = T.wpk + (size_t)nt * T.cchunks * T.taps * b_bytes;
        for (int kt = 0; kt < T.cchunks * T.taps; ++kt) {
          mbar_wait(bempty + s, bph ^ 1);
          bulk_g2s(bring + s * b_bytes, wsrc + (size_t)kt * b_bytes, b_bytes, bfull + s);
          mbar_arrive_tx(bfull + s, b_bytes);
          if (++s == SB) { s = 0; bph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------- epilogue -------------------------
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const bool vec = (op.out.cstride % 4 == 0) && (op.out.coff % 4 == 0);
    int lt = 0;
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const int64_t mt = tile / T.n_tiles;
      const int nt = (int)(tile - mt * T.n_tiles);
      const int n0 = nt * BN;
      const int64_t pos = mt * BM + q * 32 + (tid & 31);
      float* o = nullptr;
      if (pos < T.positions) {
        const int64_t b = pos / img_pos;
        const int r = (int)(pos - b * img_pos);
        const int y = r / Wp, x = r % Wp;
        if (y < wy && x < wx)
          o = op.out.base +
              ((b * op.out.H + op.oy0 + y) * op.out.W + op.ox0 + x) * op.out.cstride +
              op.out.coff;
      }
      mbar_wait(acc_full + acc, (lt >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(tmem + lane_base + acc * BN + c, v);
        if (o) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = n0 + c + i;
            float x = v[i] + (n < Cout ? __ldg(op.bias + n) : 0.f);
            if (op.lrelu) x = x >= 0.f ? x : 0.01f * x;
            v[i] = x;
          }
          if (vec && n0 + c + 16 <= Cout) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              *reinterpret_cast<float4*>(o + n0 + c + 4 * i) =
                  make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (n0 + c + i < Cout) o[n0 + c + i] = v[i];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(acc_empty + acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, ncols);
  }
}

// ---------------------------------------------------------------- host

uint32_t f2tf32_rna(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return u;
  u += 0x1000u;
  return u & 0xFFFFE000u;
}

uint16_t f2bf16_rn(float x) { return f2bf16_rn_host(x); }
float bf16_to_f(uint16_t h) { return bf16_to_f_host(h); }

struct TcPlan {
  int bn, stages, kiters, cchunks, ntiles, pa, pb, kc, wide;
  size_t smem;
};

TcPlan plan_for(const ConvOp& op, int precision) {
  TcPlan p{};
  p.pa = precision == 2 ? 1 : 2;
  p.pb = precision == 2 ? 1 : precision == 3 ? 3 : 2;
  p.kc = precision == 1 ? 32 : 64;
  const int n16 = (op.out.C + 15) / 16 * 16;
  // BF16X4 1x1 layers (the merge GEMMs) take N tiles of up to 256 without
  // plane stacking: every N tile re-gathers and re-splits A, so fewer tiles
  // halve the producers' work
  const bool wide_ok = precision == 4 && op.k == 1;
  const int cap = wide_ok ? 256 : 128;
  p.ntiles = (n16 + cap - 1) / cap;
  p.bn = ((n16 + p.ntiles - 1) / p.ntiles + 15) / 16 * 16;
  p.wide = wide_ok && p.bn > 128;
  p.cchunks = (op.in.C + p.kc - 1) / p.kc;
  p.kiters = op.k * op.k * p.cchunks;
  const size_t stage = ((size_t)BM * p.pa + (size_t)p.bn * p.pb) * kRowBytes;
  const size_t budget = 218 * 1024;
  p.stages = (int)std::min<size_t>(6, budget / stage);
  p.stages = std::max(p.stages, 1);
  p.smem = p.stages * stage + 1024 + 8 * (2 * p.stages + 4) + 16 + 2 * BM * 12 + 16 +
           16 + 4 * (size_t)p.ntiles * p.bn;
  return p;
}

struct HaloPlan {
  TcPlan base;
  int wp, lrows, bstages;
  size_t smem;
  int64_t positions;
};

bool halo_plan(const ConvOp& op, int precision, HaloPlan* hp) {
  if (op.stride != 1 || op.k < 2 || op.pad * 2 + 1 != op.k) return false;
  if (precision >= 5) return false;  // FP16X3 runs on the wide-M halo kernel
  HaloPlan h{};
  h.base = plan_for(op, precision);
  const int wx = op.ox1 - op.ox0, wy = op.oy1 - op.oy0;
  h.wp = wx + op.k - 1;
  const int L = BM + (op.k - 1) * h.wp + (op.k - 1);
  h.lrows = (L + 7) / 8 * 8;
  const size_t halo = 2 * (size_t)h.base.pa * h.lrows * kRowBytes;  // double buffered
  const size_t bst = (size_t)h.base.pb * h.base.bn * kRowBytes;
  const size_t fixed = 1024 + 8 * 24 + 16 + 16 * (size_t)h.lrows + 64;
  const size_t cap = 225 * 1024;
  if (halo + 2 * bst + fixed > cap) return false;
  h.bstages = (int)std::min<size_t>(6, (cap - halo - fixed) / bst);
  h.smem = halo + h.bstages * bst + fixed;
  h.positions = (int64_t)op.batch * (wy + op.k - 1) * h.wp;
  *hp = h;
  return true;
}


}  // namespace

bool conv_tc_halo_eligible(const ConvOp& op, int precision) {
  HaloPlan h;
  return conv_tc_supported(op, precision) && halo_plan(op, precision, &h);
}

bool conv_tc_supported(const ConvOp& op, int precision) {
  if (precision < 1 || precision > 5) return false;
  return op.in.C % 4 == 0 && op.in.cstride % 4 == 0 && op.in.coff % 4 == 0;
}

std::vector<uint8_t> pack_tc_weights(const float* w_oikk, int co, int ci, int k,
                                     int precision, const ConvOp& shape_op, int layout) {
  if (layout == 2) return pack_tc_weights_halo2(w_oikk, co, ci, k, precision, shape_op);
  const bool chunk_major = layout == 1;
  ConvOp op = shape_op;
  op.in.C = ci;
  op.out.C = co;
  op.k = k;
  const TcPlan p = plan_for(op, precision);
  const size_t plane = (size_t)p.bn * kRowBytes;
  const size_t b_bytes = plane * p.pb;
  std::vector<uint8_t> out((size_t)p.ntiles * p.kiters * b_bytes, 0);
  for (int nt = 0; nt < p.ntiles; ++nt)
    for (int it = 0; it < p.kiters; ++it) {
      const int taps = k * k;
      const int tap = chunk_major ? it % taps : it / p.cchunks;
      const int c0 = (chunk_major ? it / taps : it % p.cchunks) * p.kc;
      const int ky = tap / k, kx = tap % k;
      uint8_t* base = out.data() + ((size_t)nt * p.kiters + it) * b_bytes;
      for (int r = 0; r < p.bn; ++r) {
        const int n = nt * p.bn + r;
        for (int e = 0; e < p.kc; ++e) {
          const int c = c0 + e;
          const float v =
              (n < co && c < ci) ? w_oikk[(((size_t)n * ci + c) * k + ky) * k + kx] : 0.f;
          const int esize = precision == 1 ? 4 : 2;
          const int byte = e * esize;
          const size_t off = (size_t)(r >> 3) * 1024 + (r & 7) * kRowBytes +
                             ((((byte >> 4) ^ (r & 7))) << 4) + (byte & 15);
          if (precision == 1) {
            const uint32_t hi = f2tf32_rna(v);
            float hf;
            memcpy(&hf, &hi, 4);
            const float lo = v - hf;
            memcpy(base + off, &hi, 4);
            memcpy(base + plane + off, &lo, 4);
          } else if (precision == 2) {
            const uint16_t h = f2bf16_rn(v);
            memcpy(base + off, &h, 2);
          } else if (precision >= 5) {
            uint16_t h0, h1;
            split_f16_host(v, h0, h1);
            memcpy(base + off, &h0, 2);
            memcpy(base + plane + off, &h1, 2);
          } else if (precision == 4) {  // RN split, like the device producers
            const uint16_t h0 = f2bf16_rn(v);
            const uint16_t h1 = f2bf16_rn(v - bf16_to_f(h0));
            memcpy(base + off, &h0, 2);
            memcpy(base + plane + off, &h1, 2);
          } else {
            // exact truncation split, like the device producers
            uint32_t u;
            memcpy(&u, &v, 4);
            const uint16_t h0 = (uint16_t)(u >> 16);
            const float r0 = v - bf16_to_f(h0);
            memcpy(&u, &r0, 4);
            const uint16_t h1 = (uint16_t)(u >> 16);
            const float r1 = r0 - bf16_to_f(h1);
            memcpy(&u, &r1, 4);
            const uint16_t h2 = (uint16_t)(u >> 16);
            memcpy(base + off, &h0, 2);
            memcpy(base + plane + off, &h1, 2);
            memcpy(base + 2 * plane + off, &h2, 2);
          }
        }
      }
    }
  return out;
}

int launch_conv_tc_halo(const ConvOp& op, int precision, void* stream) {
  HaloPlan h;
  if (!halo_plan(op, precision, &h)) return TS_E_INVALID;
  HaloArgs a{op, op.w_tc, h.base.bn, h.bstages, h.base.cchunks, op.k * op.k, h.wp,
             h.lrows, h.base.ntiles,
             ceil_div<int64_t>(h.positions, BM), h.positions};
  const int64_t tiles = a.m_tiles * h.base.ntiles;
  if (tiles <= 0) return TS_OK;
  const int sms = sm_count();
  if (!sms) return TS_E_CUDA;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
  cudaStream_t s = as_stream(stream);
#define TS_TCH_LAUNCH(MD)                                                             \
  do {                                                                                \
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_tc_halo_kernel<MD>,                         \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                     (int)h.smem));                                   \
    ts::count_launch(), conv_tc_halo_kernel<MD><<<grid, kHThreads, h.smem, s>>>(a);   \
  } while (0)
  if (precision == 1) TS_TCH_LAUNCH(1);
  else if (precision == 2) TS_TCH_LAUNCH(2);
  else if (precision == 4) TS_TCH_LAUNCH(4);
  else TS_TCH_LAUNCH(3);
#undef TS_TCH_LAUNCH
  TS_LAUNCH_CHECK();
  return TS_OK;
}

int tc_weight_layout(const ConvOp& shape, int precision) {
  if (conv_tc_halo2_eligible(shape, precision)) return 2;
  if (conv_tc_halo_eligible(shape, precision)) return 1;
  return 0;
}

int launch_conv_tc(const ConvOp& op, int precision, void* stream) {
  if (op.w_layout == 2) return launch_conv_tc_halo2(op, precision, stream);
  // the regular / halo kernels read fp32 activations only; planes outputs
  // only from the regular kernel (16-channel groups)
  if (op.in.planes || (op.out.planes && (op.w_layout != 0 || op.out.C % 16 ||
                                         op.out.cstride % 8 || op.out.coff % 8)))
    return TS_E_INVALID;
  if (op.out.s2d) return TS_E_INVALID;  // s2d outputs: direct / halo2 kernels only
  if (op.w_layout == 1) {
    if (!conv_tc_halo_eligible(op, precision)) return TS_E_INVALID;
    return launch_conv_tc_halo(op, precision, stream);
  }
  const TcPlan p = plan_for(op, precision);
  const int64_t M = (int64_t)op.batch * (op.oy1 - op.oy0) * (op.ox1 - op.ox0);
  if (M <= 0) return TS_OK;
  TcArgs a{op, op.w_tc, p.bn, p.stages, p.kiters, p.cchunks, p.ntiles,
           ceil_div<int64_t>(M, BM), p.wide};
  const int64_t tiles = a.m_tiles * p.ntiles;
  const int sms = sm_count();
  if (!sms) return TS_E_CUDA;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
  cudaStream_t s = as_stream(stream);
#define TS_TC_LAUNCH(MD)                                                              \
  do {                                                                                \
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_tc_kernel<MD>,                              \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                     (int)p.smem));                                   \
    ts::count_launch(), conv_tc_kernel<MD><<<grid, kThreads, p.smem, s>>>(a);         \
  } while (0)
  if (precision == 1) TS_TC_LAUNCH(1);
  else if (precision == 2) TS_TC_LAUNCH(2);
  else if (precision == 4) TS_TC_LAUNCH(4);
  else if (precision == 5) TS_TC_LAUNCH(5);
  else TS_TC_LAUNCH(3);
#undef TS_TC_LAUNCH
  TS_LAUNCH_CHECK();
  return TS_OK;
}

}  // namespace ts
