// K3b: halo-reuse tcgen05 convolution, wide-M variant (bf16 operand modes).
//
// Same operator as conv_tc.cu's halo kernel (refiner.py:330-396: stride-1
// k x k cross-correlation + bias + leaky ReLU, nearest-up2 folded into the
// input read, crop-aware output window), re-tiled for L2 bandwidth:
//
//   * one CTA tile = SUB x 128 consecutive output positions (SUB = 2 or 4
//     M=128 MMAs per K step), so every weight stage fetched from L2 feeds
//     SUB times more MMAs, and the halo overhead ((k-1)(Wp+1) extra rows
//     per tile) is amortised over 256-512 positions instead of 128;
//   * K chunks of 32 channels = 64-byte K-major rows in the SWIZZLE_64B
//     layout: channel padding is at most 28 (fuse.0's 72 channels run as
//     96, not 128) and 2-3 halo buffers fit next to the weight ring.
//
// Output positions are linearised with the padded pitch Wp = wx + k - 1
// and (wy + k - 1) rows per image, so tap (ky, kx) of a run of consecutive
// positions reads the contiguous run of halo rows starting at ky*Wp + kx:
// the MMA issuer slides the A descriptor over one staged halo image (the
// swizzle is a function of absolute smem address bits).
//
//   warps 0..P-1  producers (P = TS_H2_PRODW = 10): per (tile, chunk)
//               gather the halo rows' fp32 channels (32-byte loads, zeros
//               outside the image), split into the mode's bf16 planes,
//               store the SW64 image, arrive.
//   warp P      MMA issuer + TMEM owner (AB x SUB x BN fp32 columns).
//   warp P+1    weight loader: cp.async.bulk of pre-swizzled weight stages.
//   warps P+2.. epilogue (TS_H2_EPIW = 4): one warp per TMEM lane quadrant
//               (with 8 or 12, warps of a quadrant alternate 16-column
//               groups): tcgen05.ld of every B plane's columns, one wait,
//               + bias (shared), leaky ReLU, fp32 NHWC store.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "conv.cuh"
#include "tc_ptx.cuh"
#include "ts_common.cuh"

namespace ts {
namespace {

using namespace tcx;

constexpr int kRow = 64;   // bytes per K-major row (32 bf16 channels)
constexpr int kKC = 32;    // channels per K chunk
#ifndef TS_H2_PRODW
#define TS_H2_PRODW 10  // measured: 10 beats 8 and 12 on every layer (7.34 vs 7.40 / 7.48 ms per step)
#endif
constexpr int kProdW = TS_H2_PRODW;
#ifndef TS_H2_PF
#define TS_H2_PF 1  // L2 prefetch of the next chunk / next tile's first chunk
#endif
#ifndef TS_H2_IN8
#define TS_H2_IN8 4
#endif
constexpr int kProdT = kProdW * 32;
constexpr int kInflight = 8;  // 16-byte loads in flight per producer thread
constexpr int kMmaW = kProdW;
constexpr int kLoadW = kProdW + 1;
#ifndef TS_H2_EPIW
#define TS_H2_EPIW 4  // measured: 4 beats 8 and 12 (7.15 vs 7.38 / 7.45 ms of halo2 launches per step)
#endif
constexpr int kEpiW0 = kProdW + 2, kEpiWarps = TS_H2_EPIW;  // multiple of 4
static_assert(kEpiWarps % 4 == 0, "epilogue warps cover the 4 TMEM lane quadrants");
static_assert(kProdW % 2 == 0, "row stride must keep the swizzle phase");
constexpr int kThreads = (kEpiW0 + kEpiWarps) * 32;
constexpr int kHdr = 1024;         // packed-weight header: u32 count, u32 0, u16 list
constexpr int kMaxStages = (kHdr - 8) / 2 - 1;  // + sentinel

// Build-time wait profile (make PROFILE=1 -> -DTS_H2_PROF): cycles each
// role spends in its mbarrier waits, summed per CTA, printed per launch by
// ts_h2_prof_dump().  Compiled out of the product library.
#ifdef TS_H2_PROF
enum { kPrProdWait, kPrMmaAcc, kPrMmaHalo, kPrMmaW, kPrEpiWait, kPrLoadWait, kPrTotal, kPrN };
__device__ unsigned long long g_h2_prof[kPrN];
#define TS_PROF_WAIT(slot, call)                                          \
  do {                                                                    \
    const long long t0_ = clock64();                                      \
    call;                                                                 \
    if ((threadIdx.x & 31) == 0)                                          \
      atomicAdd(&g_h2_prof[slot], (unsigned long long)(clock64() - t0_)); \
  } while (0)
#else
#define TS_PROF_WAIT(slot, call) call
#endif

struct Halo2Args {
  ConvOp op;
  const uint8_t* wpk;  // packed weights: kHdr-byte stage list, then
                       // [n_tile][stage][plane][BN][64 B] SW64 images
  int bn, sub, hbufs, bstages, cchunks, taps, wp, lrows, n_tiles, accbufs;
  int stack;  // 1: B planes stacked along N (PB*BN columns per sub-tile);
              // 0: every product accumulates into the same BN columns
  int cgrp;   // MODE 5: channel chunks per accumulator group (promotion unit)
  int64_t m_tiles, positions;
};

__device__ __forceinline__ void prod_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kProdT) : "memory");
}

template <int MODE, int SUB, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_halo2_kernel(Halo2Args T) {
  using Md = Mode<MODE>;
  constexpr int PA = Md::pa, PB = Md::pb;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
#ifdef TS_H2_PROF
  const long long t_start = clock64();
#endif
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const ConvOp& op = T.op;
  const int BN = T.bn, HB = T.hbufs, SB = T.bstages, L = T.lrows;
  const int plane_a = L * kRow;          // multiple of 512 (L % 8 == 0)
  const int halo_bytes = PA * plane_a;
  // weight ring slot: one stage's B planes, or (PAIR) this CTA's halves
  const int b_bytes = PAIR ? 3 * BN * kRow / 2 : PB * BN * kRow;
  uint8_t* halo = smem;
  uint8_t* bring = smem + HB * halo_bytes;
  uint64_t* bfull = reinterpret_cast<uint64_t*>(bring + SB * b_bytes);
  uint64_t* bempty = bfull + SB;
  uint64_t* hfull = bempty + SB;
  uint64_t* hempty = hfull + HB;
  uint64_t* acc_full = hempty + HB;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bpeer = acc_empty + 2;  // PAIR: the peer's weight stage landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bpeer + SB);
  int64_t* rowoff = reinterpret_cast<int64_t*>(tmem_slot + 4);  // [2][L]
  // stage table: (chunk, tap) pairs with nonzero weights, chunk-major,
  // decoded once into the chunk id and the A-descriptor row offset of the tap
  uint32_t* s_aoff = reinterpret_cast<uint32_t*>(rowoff + 2 * L);  // [nst]
  uint16_t* s_chunk = reinterpret_cast<uint16_t*>(s_aoff + kMaxStages);
  const int nst = (int)reinterpret_cast<const uint32_t*>(T.wpk)[0];
  constexpr int G = 1;  // output phases per launch (stage-list encoding keeps the field)
  {
    // entry = (chunk * G + phase) * taps + tap, bit 15 = the phase's first
    // stage (its MMAs overwrite the accumulator); decoded into the A
    // descriptor offset (bits 0-27), the phase (28-29) and that flag (30)
    const uint16_t* gl = reinterpret_cast<const uint16_t*>(T.wpk + 8);
    for (int i = threadIdx.x; i < nst; i += blockDim.x) {
      const int e = gl[i] & 0x7FFF, c = e / (G * T.taps);
      const int g = (e - c * G * T.taps) / T.taps, t = e % T.taps;
      const int ky = t / op.k, kx = t - ky * op.k;
      s_chunk[i] = (uint16_t)c;
      s_aoff[i] = (uint32_t)((ky * T.wp + kx) * (kRow >> 4)) | ((uint32_t)g << 28) |
                  ((uint32_t)(gl[i] >> 15) << 30);
    }
    s_chunk[nst] = 0xFFFF;  // sentinel
  }
  float* s_bias = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(s_chunk + kMaxStages + 1) + 15) & ~uintptr_t(15));
  for (int i = threadIdx.x; i < T.n_tiles * T.bn; i += blockDim.x)
    s_bias[i] = i < T.op.out.C ? __ldg(T.op.bias + i) : 0.f;
  const uint8_t* wdata = T.wpk + kHdr;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int wy = op.oy1 - op.oy0, wx = op.ox1 - op.ox0;
  const int Wp = T.wp;
  const int64_t img_pos = (int64_t)(wy + op.k - 1) * Wp;
  const int Cin = op.in.C, Cout = op.out.C;
  const int MT = SUB * 128;
  const int64_t total_tiles = T.m_tiles * T.n_tiles;
  // This CTA's tiles: units u = unit0, unit0 + n_units_step, ... < units.
  // PAIR: a unit is (m-tile pair, n-tile); rank r of the CTA pair computes
  // m-tile 2 mp + r (an odd last m-tile leaves the peer's half empty:
  // its positions lie past the end, gathered as zeros and not stored).
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int64_t unit_step = PAIR ? gridDim.x / 2 : gridDim.x;
  const int64_t unit0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t units = PAIR ? (T.m_tiles + 1) / 2 * T.n_tiles : total_tiles;
  auto tile_of = [&](int64_t u) -> int64_t {
    if (!PAIR) return u;
    const int64_t mp = u / T.n_tiles;
    return (2 * mp + rank) * T.n_tiles + (u - mp * T.n_tiles);
  };
  // arrivals on a barrier the leader waits on (the peer's go across the pair)
  auto arrive_leader = [&](uint64_t* bar) {
    if (PAIR && !leader) mbar_arrive_remote(mapa_shared(bar, 0));
    else mbar_arrive(bar);
  };
  const int AB = T.accbufs;
  // accumulator column blocks per sub-tile (MODE 5: main + correction)
  const int PBS = Md::f16 ? 2 : T.stack ? PB : 1;
  const int acc_cols = SUB * G * PBS * BN;  // per accumulator buffer
  uint32_t ncols = 32;
  while ((int)ncols < AB * acc_cols) ncols <<= 1;

  // FP16X3 over 32-byte aligned fp32 input with short halos (1x1 and
  // SUB-1 2x2 layers, L <= 160 rows): grouped producers (below).  Measured:
  // merge.0 1127 -> 906 us, merge.1 579 -> 463 us; longer halos (SUB 2-4)
  // got slower (dec*.2 134 -> 153 us): their chunks already outlast a round
  // trip, and a group has half the loads in flight per chunk
  const bool grouped = MODE == 5 && L <= 160 && !op.in.planes && Cin % 8 == 0 &&
                       op.in.cstride % 8 == 0 && op.in.coff % 8 == 0 &&
                       (reinterpret_cast<uintptr_t>(op.in.base) & 31) == 0;
  if (tid == 0) {
    for (int s = 0; s < SB; ++s) {
      mbar_init(bfull + s, 1);
      mbar_init(bempty + s, 1);
    }
    for (int h = 0; h < HB; ++h) {
      // one arrival per producer warp (per warp of the filling group)
      mbar_init(hfull + h, (grouped ? kProdW / 2 : kProdW) * (PAIR ? 2 : 1));
      mbar_init(hempty + h, 1);
    }
    for (int a = 0; a < AB; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, kEpiWarps * (PAIR ? 2 : 1));
    }
    for (int st = 0; st < SB; ++st) mbar_init(bpeer + st, 1);
    fence_barrier_init();
  }
  if (warp == kMmaW) {
    if (PAIR) tmem_alloc2(tmem_slot, ncols);
    else tmem_alloc(tmem_slot, ncols);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // both CTAs' barriers and TMEM ready
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // FP16X3: the epilogue warp group (warps 12-15) holds each group's
  // promoted sums in registers; the other three groups give theirs up
  static_assert(MODE != 5 || (kEpiW0 == 12 && kEpiWarps == 4), "epilogue = warp group 3");

  if (warp < kProdW) {
    if constexpr (MODE == 5) reg_dealloc<96>();
    // ------------------------- halo producers -------------------------
    // buffers are used round-robin per (tile, chunk); hph bit h = phase of
    // buffer h
    int hb = 0, lt = 0;
    uint32_t hph = 0;
    // pre-split input: chunks whose cp.async copies are still in flight
    // (publication lag kLag <= HB - 1, so the producer never waits on a
    // buffer the MMA cannot yet have been handed)
    const int lag = HB >= 3 ? 2 : 1;
    int pend[3] = {0, 0, 0}, npend = 0;
    constexpr int PPR = kKC / 4;  // float4 pieces per row
    const int pad_y = op.ph ? 1 - op.ph_y : op.pad, pad_x = op.ph ? 1 - op.ph_x : op.pad;
    // 32-byte aligned 8-channel pieces available
    const bool v8in = Cin % 8 == 0 && op.in.cstride % 8 == 0 && op.in.coff % 8 == 0 &&
                      (reinterpret_cast<uintptr_t>(op.in.base) & 31) == 0;
    // row table of this CTA's tile lt_ (parity lt_ & 1); with pf, the first
    // chunk's row lines are prefetched into L2 as they are computed
    auto build_rows = [&](int lt_, bool pf) {
      const int64_t tile_ = tile_of(unit0 + (int64_t)lt_ * unit_step);
      const int64_t j0 = (tile_ / T.n_tiles) * MT;
      int64_t* ro_ = rowoff + (lt_ & 1) * L;
      for (int j = tid; j < L; j += kProdT) {
        const int64_t pos = j0 + j;
        int64_t off = -1;
        // positions < 2^31 (checked by the host): 32-bit divisions
        const int64_t b = (int64_t)((uint32_t)pos / (uint32_t)img_pos);
        if (b < op.batch) {
          const int r = (int)(pos - b * img_pos);
          const int iy = op.oy0 - pad_y + r / Wp, ix = op.ox0 - pad_x + r % Wp;
          const int sh = op.up2 ? 1 : 0;
          if (iy >= 0 && iy < (op.in.H << sh) && ix >= 0 && ix < (op.in.W << sh))
            off = ((b * op.in.H + (iy >> sh)) * op.in.W + (ix >> sh)) * op.in.cstride +
                  op.in.coff;
        }
        ro_[j] = off;
        if (TS_H2_PF && pf && off >= 0 && !op.in.planes)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(op.in.base + off));
      }
    };
    if (grouped) {
      // FP16X3 fp32 input: two producer groups of kProdW / 2 warps fill
      // alternate (tile, chunk) units, so two chunks' loads are in flight
      // per round trip (the 1x1 and 2x2 layers' MMAs per chunk are shorter
      // than one L2 round trip); unit n uses halo buffer n % HB, phase
      // (n / HB) & 1
      constexpr int kGW = kProdW / 2, kGT = kGW * 32, kStep = kGT / 4;
      static_assert(kStep % 8 == 0, "rows per pass keep the swizzle phase");
      const int pg = warp / kGW, gt = tid - pg * kGT;
      const int piece = gt & 3, row0 = gt >> 2;
      const int obase = row0 * kRow + ((piece ^ ((row0 >> 1) & 3)) << 4);
      constexpr int kIn = TS_H2_IN8;
      int64_t n = 0;
      for (int64_t u = unit0; u < units; u += unit_step, ++lt) {
        const int64_t* ro = rowoff + (lt & 1) * L;
        if (lt == 0) build_rows(0, false);
        prod_sync();
        for (int c = 0; c < T.cchunks; ++c, ++n) {
          if (c == T.cchunks - 1 && u + unit_step < units) build_rows(lt + 1, true);
          if ((int)(n & 1) != pg) continue;
          const int h = (int)(n % HB);
          TS_PROF_WAIT(kPrProdWait, mbar_wait(hempty + h, (uint32_t)((n / HB) & 1) ^ 1u));
          uint8_t* sa = halo + h * halo_bytes + obase;
          const int ch = c * kKC + 8 * piece;
          const bool ch_ok = ch < Cin;
          const bool pf_ok = c + 1 < T.cchunks && ch + kKC < Cin;
          const float* src = op.in.base + ch;
          for (int r0 = row0; r0 < L; r0 += kStep * kIn) {
            float v[kIn][8];
#pragma unroll
            for (int u = 0; u < kIn; ++u) {
              const int row = r0 + u * kStep;
#pragma unroll
              for (int i = 0; i < 8; ++i) v[u][i] = 0.f;
              if (row < L) {
                const int64_t off = ro[row];
                if (off >= 0 && ch_ok) ld_v8(src + off, v[u]);
                if (TS_H2_PF && off >= 0 && pf_ok)
                  asm volatile("prefetch.global.L2 [%0];" ::"l"(src + off + kKC));
              }
            }
#pragma unroll
            for (int u = 0; u < kIn; ++u) {
              if (r0 + u * kStep < L) {
                uint8_t* d = sa + (r0 - row0 + u * kStep) * kRow;
                uint32_t hw[4], lw[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) split_h2(v[u][2 * i], v[u][2 * i + 1], hw[i], lw[i]);
                *reinterpret_cast<uint4*>(d) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4*>(d + plane_a) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
              }
            }
          }
          fence_proxy_async();
          __syncwarp();
          if ((tid & 31) == 0) arrive_leader(hfull + h);
        }
      }
    } else
    for (int64_t u = unit0; u < units; u += unit_step, ++lt) {
      int64_t* ro = rowoff + (lt & 1) * L;
      if (lt == 0) build_rows(0, false);
      prod_sync();
      for (int c = 0; c < T.cchunks; ++c) {
        // during the last chunk, the next tile's row table (other parity)
        // and an L2 prefetch of its first chunk
        if (c == T.cchunks - 1 && u + unit_step < units) build_rows(lt + 1, true);
        TS_PROF_WAIT(kPrProdWait, mbar_wait(hempty + hb, ((hph >> hb) & 1u) ^ 1u));
        uint8_t* sa = halo + hb * halo_bytes;
        if (op.in.planes) {
          // pre-split input: 16-byte piece p of a row is 8 channels of plane
          // p >> 2, copied as is by cp.async (zero-fill outside the image);
          // the chunk is published kLag chunks later (below), so several
          // chunks' copies are in flight per producer
          const int piece = tid & 7, pl = piece >> 2, sub = piece & 3;
          const int ch = c * kKC + 8 * sub;
          const bool ok = ch < Cin && pl < PA;
          const uint8_t* src = reinterpret_cast<const uint8_t*>(op.in.base) +
                               2 * (ch - op.in.coff) + 2 * (int64_t)pl * op.in.cstride;
          const int row0 = tid >> 3;
          const uint32_t dst0 = su32(sa + pl * plane_a + row0 * kRow) +
                                ((sub ^ ((row0 >> 1) & 3)) << 4);
          constexpr int kRowStep = kProdT / PPR;  // rows per pass (multiple of 8)
          if (pl < PA) {
            for (int r = row0; r < L; r += kRowStep) {
              const int64_t off = ro[r];
              const bool in = off >= 0 && ok;
              cp_async16(dst0 + (r - row0) * kRow, in ? src + 4 * off : src, in ? 16u : 0u);
            }
          }
        } else if (v8in) {
          // 32-byte pieces (8 channels): LDG.256, one STS.128 per plane.
          // Each thread owns one piece column (kProdT % 4 == 0); rows advance
          // by kProdT / 4 (a multiple of 8: the swizzle phase repeats).
          const int piece = tid & 3;
          const int ch = c * kKC + 8 * piece;
          const bool ch_ok = ch < Cin;
          const bool pf_ok = c + 1 < T.cchunks && ch + kKC < Cin;
          const float* src = op.in.base + ch;
          const int row0 = tid >> 2;
          const int obase = row0 * kRow + ((piece ^ ((row0 >> 1) & 3)) << 4);
          constexpr int kStep8 = kProdT / 4;
          constexpr int kIn8 = TS_H2_IN8;  // 32-byte loads in flight per thread
          for (int r0 = row0; r0 < L; r0 += kStep8 * kIn8) {
            float v[kIn8][8];
#pragma unroll
            for (int u = 0; u < kIn8; ++u) {
              const int row = r0 + u * kStep8;
#pragma unroll
              for (int i = 0; i < 8; ++i) v[u][i] = 0.f;
              if (row < L) {
                const int64_t off = ro[row];
                if (off >= 0 && ch_ok) ld_v8(src + off, v[u]);
                if (TS_H2_PF && off >= 0 && pf_ok)
                  asm volatile("prefetch.global.L2 [%0];" ::"l"(src + off + kKC));
              }
            }
            uint8_t* so = sa + obase + (r0 - row0) * kRow;
#pragma unroll
            for (int u = 0; u < kIn8; ++u) {
              if (r0 + u * kStep8 < L) {
                uint8_t* d = so + u * kStep8 * kRow;
                uint32_t h[4];
                if (Md::f16) {
                  uint32_t l[4];
#pragma unroll
                  for (int i = 0; i < 4; ++i) split_h2(v[u][2 * i], v[u][2 * i + 1], h[i], l[i]);
                  *reinterpret_cast<uint4*>(d) = make_uint4(h[0], h[1], h[2], h[3]);
                  *reinterpret_cast<uint4*>(d + plane_a) = make_uint4(l[0], l[1], l[2], l[3]);
                } else {
#pragma unroll
                  for (int i = 0; i < 4; ++i) h[i] = pack_bf2(v[u][2 * i], v[u][2 * i + 1]);
                  *reinterpret_cast<uint4*>(d) = make_uint4(h[0], h[1], h[2], h[3]);
                  if (MODE != 2) {
                    uint32_t l[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                      l[i] = pack_bf2(v[u][2 * i] - __uint_as_float(h[i] << 16),
                                      v[u][2 * i + 1] - __uint_as_float(h[i] & 0xFFFF0000u));
                    *reinterpret_cast<uint4*>(d + plane_a) = make_uint4(l[0], l[1], l[2], l[3]);
                  }
                }
              }
            }
          }
        } else {
        // each thread owns one 16-byte piece column (kProdT % 8 == 0): its
        // channel, validity and swizzled byte offset within a row are fixed,
        // and rows advance by kProdT / 8 = 32 (the swizzle phase repeats)
        const int piece = tid & 7;
        const int ch = c * kKC + 4 * piece;
        const bool ch_ok = ch < Cin;
        const bool pf_ok = c + 1 < T.cchunks && ch + kKC < Cin;
        const float* src = op.in.base + ch;
        const int row0 = tid >> 3;
        const int obase = row0 * kRow + (((piece >> 1) ^ ((row0 >> 1) & 3)) << 4) +
                          ((piece & 1) << 3);
        constexpr int kRowStep = kProdT / PPR;  // rows per pass (multiple of 8)
        for (int r0 = row0; r0 < L; r0 += kRowStep * kInflight) {
          float4 v[kInflight];
#pragma unroll
          for (int u = 0; u < kInflight; ++u) {
            const int row = r0 + u * kRowStep;
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < L) {
              const int64_t off = ro[row];
              if (off >= 0 && ch_ok) v[u] = __ldg(reinterpret_cast<const float4*>(src + off));
              // the next chunk's piece of this row into L2 while this one
              // is converted (the fill is otherwise one DRAM latency per
              // chunk)
              if (off >= 0 && pf_ok)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(src + off + kKC));
            }
          }
          uint8_t* so = sa + obase + (r0 - row0) * kRow;
#pragma unroll
          for (int u = 0; u < kInflight; ++u) {
            if (r0 + u * kRowStep < L) {
              const float4 a = v[u];
              uint8_t* d = so + u * kRowStep * kRow;
              if (MODE == 2)
                *reinterpret_cast<uint2*>(d) =
                    make_uint2(pack_bf2(a.x, a.y), pack_bf2(a.z, a.w));
              else if (Md::f16)
                store_split_h(d, plane_a, a);
              else
                store_split2(d, plane_a, a);
            }
          }
        }
        }
        if (op.in.planes) {
          // publish the chunk issued kLag chunks ago once its copies landed
          cp_async_commit();
          pend[npend++] = hb;
          if (npend > lag) {
            if (lag == 2) cp_async_wait<2>();
            else cp_async_wait<1>();
            fence_proxy_async();
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(hfull + pend[0]);
            pend[0] = pend[1];
            pend[1] = pend[2];
            --npend;
          }
        } else {
          fence_proxy_async();
          __syncwarp();
          if ((tid & 31) == 0) arrive_leader(hfull + hb);
        }
        hph ^= 1u << hb;
        if (++hb == HB) hb = 0;
      }
    }
    if (op.in.planes && npend) {
      cp_async_wait<0>();
      fence_proxy_async();
      __syncwarp();
      if ((tid & 31) == 0)
        for (int i = 0; i < npend; ++i) mbar_arrive(hfull + pend[i]);
    }
  } else if (warp == kMmaW && MODE == 5 && PAIR && !leader) {
    // ---------- the peer's weight-stage forwarder (CTA pair) ----------
    // its loader's bulk copies complete on this CTA's bfull; the leader's
    // MMA issuer learns of them through bpeer
    reg_dealloc<96>();
    if ((tid & 31) == 0) {
      int s = 0;
      uint32_t bph = 0;
      for (int64_t u = unit0; u < units; u += unit_step)
        for (int kt = 0; kt < nst; ++kt) {
          mbar_wait(bfull + s, bph);
          mbar_arrive_remote(mapa_shared(bpeer + s, 0));
          if (++s == SB) { s = 0; bph ^= 1; }
        }
    }
    __syncwarp();
  } else if (warp == kMmaW && MODE == 5) {
    // ------------------- MMA issuer (FP16X3, promoted) -------------------
    // PAIR: the leader issues M = 256 MMAs for both CTAs (cta_group::2):
    // each CTA supplies its own 128 A rows and half of every B operand
    // ([b0 | b1]: b0 here, b1 in the peer; b0 for a1 . b0: its first half
    // here, its second in the peer), commits arrive in both CTAs
    reg_dealloc<96>();
    // Per sub-tile u and K step: a0 . [b0 | b1] -> [main | corr] (one
    // stacked MMA, N = 2 BN) and a1 . b0 -> corr (N = BN).  The accumulator
    // pair rotates per GROUP of T.cgrp channel chunks (<= 18 K steps): the
    // group's first K step overwrites it, the epilogue promotes it.
    const uint32_t idesc = make_idesc(mode_fmt<MODE>(), 2 * BN, PAIR ? 256 : 128);
    const uint32_t idesc_b0 = make_idesc(mode_fmt<MODE>(), BN, PAIR ? 256 : 128);
    const uint64_t d_halo = sw64_desc(su32(halo));
    const uint64_t d_ring = sw64_desc(su32(bring));
    const uint32_t pa = (uint32_t)plane_a >> 4;
    const uint32_t b_step = (uint32_t)b_bytes >> 4, h_step = (uint32_t)halo_bytes >> 4;
    // B of the a1 . b0 MMA: the same b0 rows (single CTA) or this CTA's
    // half of b0 stored after its BN rows of [b0 | b1] (pair)
    const uint32_t b2_off = PAIR ? (uint32_t)(BN * kRow) >> 4 : 0u;
    int s = 0, hb = 0;
    uint32_t bph = 0, hph = 0, gc = 0;
    for (int64_t u_ = unit0; u_ < units; u_ += unit_step) {
      int si = 0;
      uint32_t d = 0, acc_f = 0;
      for (int c = 0; c < T.cchunks; ++c) {
        const bool g_first = c % T.cgrp == 0;
        const bool g_last = c % T.cgrp == T.cgrp - 1 || c == T.cchunks - 1;
        if (g_first) {
          TS_PROF_WAIT(kPrMmaAcc, mbar_wait(acc_empty + (gc & 1u), ((gc >> 1) & 1u) ^ 1u));
          tc_fence_after();
          d = tmem + (gc & 1u) * acc_cols;
          acc_f = 0;
        }
        TS_PROF_WAIT(kPrMmaHalo, mbar_wait(hfull + hb, (hph >> hb) & 1u));
        hph ^= 1u << hb;
        tc_fence_after();
        const uint64_t d_hb = d_halo + (uint64_t)(hb * h_step);
        const int nk = (c == T.cchunks - 1 && Cin - c * kKC <= 16) ? 1 : 2;
        for (; s_chunk[si] == c; ++si) {
          TS_PROF_WAIT(kPrMmaW, mbar_wait(bfull + s, bph));
          if (PAIR) TS_PROF_WAIT(kPrMmaW, mbar_wait(bpeer + s, bph));
          tc_fence_after();
          if (elect_one()) {
            const uint64_t a0 = d_hb + (uint64_t)(s_aoff[si] & 0x0FFFFFFFu);
            const uint64_t b0 = d_ring + (uint64_t)(s * b_step);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              if (k >= nk) break;
#pragma unroll
              for (int u = 0; u < SUB; ++u) {
                const uint64_t ak = a0 + (uint64_t)(u * (128 * kRow >> 4) + 2 * k);
                const uint32_t du = d + u * 2 * BN;
                if (PAIR) {
                  umma2(du, ak, b0 + 2 * k, idesc, (acc_f | k) ? 1u : 0u);
                  umma2(du + BN, ak + pa, b0 + b2_off + 2 * k, idesc_b0, 1u);
                } else {
                  umma<false>(du, ak, b0 + 2 * k, idesc, (acc_f | k) ? 1u : 0u);
                  umma<false>(du + BN, ak + pa, b0 + 2 * k, idesc_b0, 1u);
                }
              }
            }
            if (PAIR) umma_commit2(bempty + s);
            else umma_commit(bempty + s);
          }
          __syncwarp();
          acc_f = 1;
          if (++s == SB) { s = 0; bph ^= 1; }
        }
        if (elect_one()) {
          if (PAIR) {
            umma_commit2(hempty + hb);
            if (g_last) umma_commit2(acc_full + (gc & 1u));
          } else {
            umma_commit(hempty + hb);
            if (g_last) umma_commit(acc_full + (gc & 1u));
          }
        }
        __syncwarp();
        if (g_last) ++gc;
        if (++hb == HB) hb = 0;
      }
    }
  } else if (warp == kMmaW) {
    // ------------------------- MMA issuer -------------------------
    // one MMA per A plane against all PB weight planes stacked along N:
    // D[:, p*BN + n] accumulates A . b_p, summed by the epilogue.  Same
    // MACs as one MMA per (A plane, B plane) pair at N = BN, but every
    // 4 KB A read from shared memory now feeds PB*BN columns.
    // stacked B planes: all PB (bf16 modes) or [b0 | b1] (fp16 modes)
    const uint32_t idesc = make_idesc(mode_fmt<MODE>(), (Md::f16 ? 2 : PB) * BN);
    const uint32_t idesc_b0 = make_idesc(mode_fmt<MODE>(), BN);
    const uint64_t d_halo = sw64_desc(su32(halo));
    const uint64_t d_ring = sw64_desc(su32(bring));
    const uint32_t pa = (uint32_t)plane_a >> 4;
    int s = 0, lt = 0, hb = 0;
    uint32_t bph = 0, hph = 0;
    const uint32_t b_step = (uint32_t)b_bytes >> 4, h_step = (uint32_t)halo_bytes >> 4;
    const uint32_t b_plane16 = (uint32_t)(BN * kRow) >> 4;  // one B plane
    for (int64_t u_ = unit0; u_ < units; u_ += unit_step, ++lt) {
      const int acc = lt % AB;
      mbar_wait(acc_empty + acc, ((lt / AB) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * acc_cols;
      int si = 0;
      for (int c = 0; c < T.cchunks; ++c) {
        mbar_wait(hfull + hb, (hph >> hb) & 1u);
        hph ^= 1u << hb;
        tc_fence_after();
        const uint64_t d_hb = d_halo + (uint64_t)(hb * h_step);
        // the last chunk may hold <= 16 real channels (fuse.0: 72 = 2 x 32
        // + 8): its second K step would multiply zeros
        const int nk = (c == T.cchunks - 1 && Cin - c * kKC <= 16) ? 1 : 2;
        for (; s_chunk[si] == c; ++si) {
          mbar_wait(bfull + s, bph);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t ent = s_aoff[si];
            const uint64_t a0 = d_hb + (uint64_t)(ent & 0x0FFFFFFFu);
            const uint64_t b0 = d_ring + (uint64_t)(s * b_step);
            const uint32_t first = (ent >> 30) ? 0u : 1u;  // accumulate flag of K step 0
            const uint32_t dg = d + ((ent >> 28) & 3u) * PBS * BN;
#pragma unroll
            for (int k = 0; k < 2; ++k) {  // 2 x 32-byte K steps per row
              if (k >= nk) break;
#pragma unroll
              for (int u = 0; u < SUB; ++u) {
                const uint64_t ak = a0 + (uint64_t)(u * (128 * kRow >> 4) + 2 * k);
                const uint32_t du = dg + u * G * PBS * BN;
                if (T.stack) {
                  umma<false>(du, ak, b0 + 2 * k, idesc, k ? 1u : first);
                } else {  // a0 . b_p for every plane into the same columns
                  umma<false>(du, ak, b0 + 2 * k, idesc_b0, k ? 1u : first);
#pragma unroll
                  for (int q = 1; q < PB; ++q)
                    umma<false>(du, ak, b0 + (uint64_t)(q * b_plane16) + 2 * k, idesc_b0, 1u);
                }
                // second A plane against b0 only (N = BN): a1 . b_{p>0}
                // terms are below the split residual and are dropped
                if (PA == 2) umma<false>(du, ak + pa, b0 + 2 * k, idesc_b0, 1u);
              }
            }
            umma_commit(bempty + s);
          }
          __syncwarp();
          if (++s == SB) { s = 0; bph ^= 1; }
        }
        if (elect_one()) umma_commit(hempty + hb);
        __syncwarp();
        if (++hb == HB) hb = 0;
      }
      if (elect_one()) umma_commit(acc_full + acc);
      __syncwarp();
    }
  } else if (warp == kLoadW) {
    // ------------------------- weight loader -------------------------
    if constexpr (MODE == 5) reg_dealloc<96>();
    if ((tid & 31) == 0) {
      int s = 0;
      uint32_t bph = 0;
      // PAIR: this CTA's image of each stage (its halves, 1.5 BN rows)
      const int img = b_bytes;
      for (int64_t u = unit0; u < units; u += unit_step) {
        const int nt = (int)(tile_of(u) % T.n_tiles);
        const uint8_t* wsrc = wdata + (size_t)nt * nst * (PAIR ? 2 * img : img);
        for (int kt = 0; kt < nst; ++kt) {
          TS_PROF_WAIT(kPrLoadWait, mbar_wait(bempty + s, bph ^ 1));
          const uint8_t* src = PAIR ? wsrc + ((size_t)kt * 2 + rank) * img
                                    : wsrc + (size_t)kt * b_bytes;
          bulk_g2s(bring + s * b_bytes, src, img, bfull + s);
          mbar_arrive_tx(bfull + s, img);
          if (++s == SB) { s = 0; bph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (MODE == 5 && warp >= kEpiW0) {
    // -------------------- epilogue (FP16X3, promoted) --------------------
    // Per group: main + 2^-11 corr of every column into fp32 registers (RN
    // adds), the TMEM pair released; after the tile's last group: bias,
    // leaky ReLU, fp32 NHWC stores.
    reg_alloc<224>();
    constexpr int NB = 128 / SUB / 16;  // 16-column blocks held per sub-tile
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const bool vec = (op.out.cstride % 4 == 0) && (op.out.coff % 4 == 0);
    const bool vec8 = (op.out.cstride % 8 == 0) && (op.out.coff % 8 == 0) &&
                      (op.out.C % 8 == 0) && ((reinterpret_cast<uintptr_t>(op.out.base) & 31) == 0);
    const int groups = (T.cchunks + T.cgrp - 1) / T.cgrp;
    uint32_t gc = 0;
    for (int64_t u_ = unit0; u_ < units; u_ += unit_step) {
      const int64_t tile = tile_of(u_);
      const int64_t mt = tile / T.n_tiles;
      const int n0 = (int)(tile - mt * T.n_tiles) * BN;
      float R[SUB][NB][16];
#pragma unroll
      for (int u = 0; u < SUB; ++u)
#pragma unroll
        for (int j = 0; j < NB; ++j)
#pragma unroll
          for (int i = 0; i < 16; ++i) R[u][j][i] = 0.f;
      for (int g = 0; g < groups; ++g, ++gc) {
        TS_PROF_WAIT(kPrEpiWait, mbar_wait(acc_full + (gc & 1u), (gc >> 1) & 1u));
        tc_fence_after();
        const uint32_t tb = tmem + lane_base + (gc & 1u) * acc_cols;
#pragma unroll
        for (int u = 0; u < SUB; ++u)
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            if (16 * j >= BN) break;
            uint32_t m[16], r[16];
            tmem_ld16_nw(tb + u * 2 * BN + 16 * j, m);
            tmem_ld16_nw(tb + u * 2 * BN + BN + 16 * j, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i)
              R[u][j][i] += __fmaf_rn(__uint_as_float(r[i]), kF16LoInv, __uint_as_float(m[i]));
          }
        tc_fence_before();
        __syncwarp();
        if ((tid & 31) == 0) arrive_leader(acc_empty + (gc & 1u));
      }
#pragma unroll
      for (int u = 0; u < SUB; ++u) {
        const int64_t pos = mt * MT + u * 128 + q * 32 + (tid & 31);
        float* o = nullptr;
        float* oblk = nullptr;
        int ochan = 0;
        if (pos < T.positions) {
          const int64_t b = (int64_t)((uint32_t)pos / (uint32_t)img_pos);
          const int r = (int)(pos - b * img_pos);
          const int y = r / Wp, x = r % Wp;
          if (y < wy && x < wx) {
            int oy = op.oy0 + y, ox = op.ox0 + x;
            if (op.ph == 1) {
              oy = 2 * oy + op.ph_y;
              ox = 2 * ox + op.ph_x;
            }
            o = op.out.base + act_off(op.out, b, oy, ox);
            int64_t blk;
            act_block(op.out, b, oy, ox, blk, ochan);
            oblk = op.out.base + blk;
          }
        }
        if (!o) continue;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const int c = 16 * j;
          if (c >= BN) break;
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x = R[u][j][i] + s_bias[n0 + c + i];
            if (op.lrelu) x = x >= 0.f ? x : 0.01f * x;
            v[i] = x;
          }
          if (op.out.planes) {
            if (n0 + c + 16 <= Cout)
              store16_planes(oblk, op.out.cstride, ochan + n0 + c, v, op.out.planes == 2);
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
    }
  } else if (MODE != 5) {
    // ------------------------- epilogue -------------------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = (warp - kEpiW0) >> 2;  // which 16-column groups
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const bool vec = (op.out.cstride % 4 == 0) && (op.out.coff % 4 == 0);
    const bool vec8 = (op.out.cstride % 8 == 0) && (op.out.coff % 8 == 0) &&
                      (op.out.C % 8 == 0) && ((reinterpret_cast<uintptr_t>(op.out.base) & 31) == 0);
    int lt = 0;
    for (int64_t u_ = unit0; u_ < units; u_ += unit_step, ++lt) {
      const int64_t tile = tile_of(u_);
      const int acc = lt % AB;
      const int64_t mt = tile / T.n_tiles;
      const int nt = (int)(tile - mt * T.n_tiles);
      const int n0 = nt * BN;
      mbar_wait(acc_full + acc, (lt / AB) & 1);
      tc_fence_after();
      for (int u = 0; u < SUB; ++u) {
        const int64_t pos = mt * MT + u * 128 + q * 32 + (tid & 31);
        float* o = nullptr;
        float* oblk = nullptr;
        int ochan = 0;
        if (pos < T.positions) {
          const int64_t b = (int64_t)((uint32_t)pos / (uint32_t)img_pos);
          const int r = (int)(pos - b * img_pos);
          const int y = r / Wp, x = r % Wp;
          if (y < wy && x < wx) {
            int oy = op.oy0 + y, ox = op.ox0 + x;
            if (op.ph == 1) {
              oy = 2 * oy + op.ph_y;
              ox = 2 * ox + op.ph_x;
            }
            o = op.out.base + act_off(op.out, b, oy, ox);
            int64_t blk;
            act_block(op.out, b, oy, ox, blk, ochan);
            oblk = op.out.base + blk;
          }
        }
        for (int c = 16 * half; c < BN; c += 16 * (kEpiWarps / 4)) {
          uint32_t r[3][16];
          const uint32_t ta = tmem + lane_base + acc * acc_cols + u * PBS * BN + c;
#pragma unroll
          for (int p = 0; p < 3; ++p)
            if (p < PBS) tmem_ld16_nw(ta + p * BN, r[p]);
          tmem_wait_ld();
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x = __uint_as_float(r[0][i]);
#pragma unroll
            for (int p = 1; p < PB; ++p)
              if (p < PBS) x += __uint_as_float(r[p][i]);
            x += s_bias[n0 + c + i];
            if (op.lrelu) x = x >= 0.f ? x : 0.01f * x;
            v[i] = x;
          }
          if (o && op.out.planes) {
            if (n0 + c + 16 <= Cout) store16_planes(oblk, op.out.cstride, ochan + n0 + c, v, op.out.planes == 2);
          } else if (o) {
            if (vec8 && n0 + c + 16 <= Cout) {
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
      }
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(acc_empty + acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the leader's last MMAs wrote the peer's TMEM
  if (warp == kMmaW) {
    tc_fence_after();
    if (PAIR) tmem_dealloc2(tmem, ncols);
    else tmem_dealloc(tmem, ncols);
  }
#ifdef TS_H2_PROF
  if (tid == 0) atomicAdd(&g_h2_prof[kPrTotal], (unsigned long long)(clock64() - t_start));
#endif
}

// weight-ring depth of the CTA-pair kernel (its slots are 1.5 BN rows)
#ifndef TS_H2_PAIR_STAGES
#define TS_H2_PAIR_STAGES 8
#endif
constexpr int kPairStages = TS_H2_PAIR_STAGES;

// CTA pairs (cta_group::2) for the FP16X3 halo kernel: opt-in with
// TS_H2_PAIR=1 (read once per process).  Bit-identical to the single-CTA
// kernel, 23% fewer shared-memory operand reads, but measured slower (CNN
// 11.7 vs 9.7 ms per 1,024 tiles, fuse.0 2.38 vs 1.53 ms: tensor pipe 27%
// active, the leader's MMA issuer waiting on the weight ring 40% of the
// time; profiles/r02_notes.md)
bool pair_enabled() {
  static const bool on = [] {
    const char* e = getenv("TS_H2_PAIR");
    return e && e[0] == '1';
  }();
  return on;
}

struct Halo2Plan {
  int bn, ntiles, pa, pb, sub, hbufs, bstages, cchunks, wp, lrows, accbufs, stack, cgrp;
  int pair;  // FP16X3 on CTA pairs: M = 256 MMAs, B halves per CTA
  size_t smem;
  int64_t positions;
};

bool plan2(const ConvOp& op, int precision, Halo2Plan* out) {
  if (precision < 2 || precision > 5) return false;
  // stride-1 k >= 2 (incl. the 2x2 space-to-depth form of stride-2 layers);
  // 1x1 layers stay on the regular kernel (no halo to reuse, and their
  // multi-N-tile shapes re-read A per N tile here)
  if (op.stride != 1 || op.k < 1 || op.pad < 0 || op.pad >= op.k) return false;
  constexpr int G = 1;
  // 1x1 layers: the bf16-class modes measured slower here than on the
  // regular kernel (A re-read per N tile); FP16X3 runs them here for the
  // promoted accumulation
  if (op.k == 1 && precision != 5) return false;
  if (op.in.C % 4 || op.in.cstride % 4 || op.in.coff % 4) return false;
  if (op.in.planes && (op.in.C % 8 || op.in.cstride % 8 || op.in.coff % 8)) return false;
  if (op.out.planes && (op.out.C % 16 || op.out.cstride % 8 || op.out.coff % 8)) return false;
  Halo2Plan p{};
  p.pa = precision == 2 ? 1 : 2;
  p.pb = precision == 2 ? 1 : precision == 3 ? 3 : 2;
  const int n16 = (op.out.C + 15) / 16 * 16;
  {  // widest N tile: up to 256 (one MMA) so a layer's A halo is gathered
     // and read once for all its columns (enc*.2, N = 192: 235 -> 192 us
     // against two 96-column tiles); FP16X3 stacks its two weight planes
     // into one MMA (N = 2 BN <= 256)
    const int bmax = precision == 5 ? 128 : 256;
    p.ntiles = (n16 + bmax - 1) / bmax;
  }
  p.bn = ((n16 + p.ntiles - 1) / p.ntiles + 15) / 16 * 16;
  p.cchunks = (op.in.C + kKC - 1) / kKC;
  const int wx = op.ox1 - op.ox0, wy = op.oy1 - op.oy0;
  p.wp = wx + op.k - 1;
  p.positions = (int64_t)op.batch * (wy + op.k - 1) * p.wp;
  const size_t cap = 225 * 1024;
  const size_t bst = (size_t)p.pb * p.bn * kRow;
  // (sub-tiles, accumulator buffers): the epilogue must overlap the next
  // tile's MMAs (two accumulator buffers), then prefer M >= 256
  // B planes stacked along N feed one MMA per A plane (fewer, wider MMAs);
  // measured better only for thin N (BN <= 32).  Wider layers accumulate
  // every product into the same BN columns, which doubles the sub-tiles
  // per TMEM buffer and amortises the MMA issuer's per-stage overhead.
  p.stack = p.pb * p.bn <= 64 && 4 * G * p.pb * p.bn <= 512;
  if (precision == 5) p.stack = 1;          // [b0 | b1] rows (BN <= 128)
  else if (p.pb * p.bn > 256) p.stack = 0;  // MMA N limit
  const int cols = G * (precision == 5 ? 2 * p.bn : p.stack ? p.pb * p.bn : p.bn);
  // FP16X3: promotion group = the channel chunks of <= 18 K steps (2 per
  // 32-channel chunk and tap): 1 for 3x3, 2 for 2x2, 8 for 1x1
  p.cgrp = precision == 5 ? std::max(1, 16 / (2 * op.k * op.k)) : 1;
  const int cand[6][2] = {{4, 2}, {2, 2}, {1, 2}, {4, 1}, {2, 1}, {1, 1}};
  for (const auto& cb : cand) {
    const int sub = cb[0], ab = cb[1];
    if (ab * sub * cols > 512) continue;
    // FP16X3: two group buffers, and the epilogue holds SUB x BN sums
    if (precision == 5 && (ab != 2 || sub * p.bn > 128)) continue;
    const int L = (128 * sub + (op.k - 1) * (p.wp + 1) + 7) / 8 * 8;
    const size_t hbuf = (size_t)p.pa * L * kRow;
    const size_t fixed = 1024 + 8 * 40 + 16 + 16 * (size_t)L + 6 * kMaxStages + 64 +
                         4 * (size_t)p.ntiles * p.bn + 16;
    // halo buffers: 3, else 2 (measured: 4-8 no faster); weight ring: up to
    // 4 stages (measured: 3-4 about 1% faster than 8).  Layers the kernel
    // fills with two producer groups (FP16X3, L <= 160, 8-channel aligned
    // input: conv_tc_halo2_kernel `grouped`) take an even count, so each
    // buffer is always filled by the same group's threads
    const bool grouped = precision == 5 && L <= 160 && !op.in.planes && op.in.C % 8 == 0 &&
                         op.in.cstride % 8 == 0 && op.in.coff % 8 == 0;
    const int hbs[2] = {grouped ? 4 : 3, 2};  // (4 vs 3: same time, within noise)
    for (int hb : hbs) {
      const size_t used = hb * hbuf + fixed;
      if (used + 3 * bst > cap) continue;
      p.sub = sub;
      p.accbufs = ab;
      p.hbufs = hb;
      p.lrows = L;
      p.bstages = (int)std::min<size_t>(4, (cap - used) / bst);
      // pairs need B halves of >= 8 rows (BN a multiple of 16: always) and
      // the plain fp32 producers (the pre-split cp.async path publishes
      // chunks with a lag the pair's arrival counts do not model).  A
      // pair's ring slot holds one CTA's halves (1.5 BN rows), and the ring
      // is deeper: a slot's reuse also waits for the peer's copy to be
      // forwarded
      p.pair = precision == 5 && pair_enabled() && !op.in.planes && p.bn % 16 == 0;
      if (p.pair) {
        const size_t slot = (size_t)3 * p.bn * kRow / 2;
        p.bstages = (int)std::min<size_t>(kPairStages, (cap - used) / slot);
        p.smem = used + p.bstages * slot;
      } else {
        p.smem = used + p.bstages * bst;
      }
      *out = p;
      return true;
    }
  }
  return false;
}

}  // namespace

bool conv_tc_halo2_eligible(const ConvOp& op, int precision) {
  Halo2Plan p;
  return plan2(op, precision, &p);
}

int conv_tc_halo2_accbufs(const ConvOp& op, int precision) {
  Halo2Plan p;
  return plan2(op, precision, &p) ? p.accbufs : 0;
}

std::vector<uint8_t> pack_tc_weights_halo2(const float* w_oikk, int co, int ci, int k,
                                           int precision, const ConvOp& op) {
  Halo2Plan p;
  if (!plan2(op, precision, &p)) return {};
  const size_t plane = (size_t)p.bn * kRow;
  const size_t b_bytes = plane * p.pb;
  const int taps = k * k;
  constexpr int G = 1;
  const size_t wg = (size_t)co * ci * taps;  // floats per phase tensor
  // (chunk, phase, tap) stages whose weights are all zero in every n-tile
  // are skipped (the space-to-depth form of a stride-2 3x3 layer has 7 such
  // taps of 16 per 4 channel groups; a phase of a group uses 4 of 9 taps)
  std::vector<uint16_t> list;
  std::vector<char> seen(G, 0);
  for (int c = 0; c < p.cchunks; ++c)
    for (int g = 0; g < G; ++g) {
      bool any = false;  // FP16X3: every chunk keeps a stage (its group's
                         // first MMA must write the accumulators)
      for (int t = 0; t < taps; ++t) {
        const int ky = t / k, kx = t % k;
        bool nz = false;
        for (int n = 0; n < co && !nz; ++n)
          for (int e = 0; e < kKC && !nz; ++e) {
            const int ch = c * kKC + e;
            if (ch < ci && w_oikk[g * wg + (((size_t)n * ci + ch) * k + ky) * k + kx] != 0.f)
              nz = true;
          }
        // an all-zero phase keeps one (zero) stage so its columns are written
        const bool keep = precision == 5 ? (t == taps - 1 && !any)
                                         : (c == p.cchunks - 1 && t == taps - 1 && !seen[g]);
        if (!nz && !keep) continue;
        list.push_back((uint16_t)(((c * G + g) * taps + t) | (seen[g] ? 0 : 0x8000)));
        seen[g] = 1;
        any = true;
      }
    }
  if ((int)list.size() > kMaxStages) return {};
  const int nst = (int)list.size();
  // CTA pair: per stage two images of 1.5 BN rows, [b0 | b0 rows 0..BN/2)
  // for rank 0 and [b1 | b0 rows BN/2..BN) for rank 1 (each CTA's half of
  // the [b0 | b1] and b0 B operands; conv_tc_halo2_kernel PAIR)
  const size_t img = p.pair ? (size_t)3 * p.bn * kRow / 2 : b_bytes;
  const size_t stage_bytes = p.pair ? 2 * img : b_bytes;
  std::vector<uint8_t> out(kHdr + (size_t)p.ntiles * nst * stage_bytes, 0);
  auto put = [&](uint8_t* image, int r, int e, uint16_t v) {  // SW64 row r, channel e
    const int byte = 2 * e;
    const size_t off = (size_t)r * kRow + (size_t)(((byte >> 4) ^ ((r >> 1) & 3)) << 4) +
                       (byte & 15);
    memcpy(image + off, &v, 2);
  };
  const uint32_t hdr[2] = {(uint32_t)nst, 0u};
  memcpy(out.data(), hdr, 8);
  memcpy(out.data() + 8, list.data(), 2 * list.size());
  for (int nt = 0; nt < p.ntiles; ++nt)
    for (int i = 0; i < nst; ++i) {
      const int e = list[i] & 0x7FFF, c = e / (G * taps);
      const int g = (e - c * G * taps) / taps, t = e % taps;
      const int ky = t / k, kx = t % k;
      uint8_t* base = out.data() + kHdr + ((size_t)nt * nst + i) * stage_bytes;
      for (int r = 0; r < p.bn; ++r) {
        const int n = nt * p.bn + r;
        for (int e = 0; e < kKC; ++e) {
          const int ch = c * kKC + e;
          const float v =
              (n < co && ch < ci) ? w_oikk[g * wg + (((size_t)n * ci + ch) * k + ky) * k + kx]
                                  : 0.f;
          uint16_t h[3] = {0, 0, 0};
          if (precision == 2) {
            h[0] = f2bf16_rn_host(v);
          } else if (precision == 5) {
            split_f16_host(v, h[0], h[1]);

          } else if (precision == 4) {  // RN split, like the device producers
            h[0] = f2bf16_rn_host(v);
            h[1] = f2bf16_rn_host(v - bf16_to_f_host(h[0]));
          } else {  // exact truncation split
            uint32_t u;
            float rr = v;
            for (int pl = 0; pl < 3; ++pl) {
              memcpy(&u, &rr, 4);
              h[pl] = (uint16_t)(u >> 16);
              rr -= bf16_to_f_host(h[pl]);
            }
          }
          if (p.pair) {
            put(base, r, e, h[0]);                 // rank 0: b0 row r
            put(base + img, r, e, h[1]);           // rank 1: b1 row r
            if (r < p.bn / 2) put(base, p.bn + r, e, h[0]);
            else put(base + img, p.bn + r - p.bn / 2, e, h[0]);
          } else {
            for (int pl = 0; pl < p.pb; ++pl) put(base + pl * plane, r, e, h[pl]);
          }
        }
      }
    }
  return out;
}

int launch_conv_tc_halo2(const ConvOp& op, int precision, void* stream) {
  Halo2Plan p;
  if (!plan2(op, precision, &p)) return TS_E_INVALID;
  if (p.positions + 128 * p.sub + p.lrows >= (int64_t)INT32_MAX) return TS_E_INVALID;
  Halo2Args a{op, op.w_tc, p.bn, p.sub, p.hbufs, p.bstages, p.cchunks, op.k * op.k, p.wp,
              p.lrows, p.ntiles, p.accbufs, p.stack, p.cgrp,
              ceil_div<int64_t>(p.positions, 128 * p.sub), p.positions};
  const int64_t tiles = a.m_tiles * p.ntiles;
  if (tiles <= 0) return TS_OK;
  const int sms = sm_count();
  if (!sms) return TS_E_CUDA;
  unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
  cudaStream_t s = as_stream(stream);
  if (p.pair && precision == 5) {
    // one CTA pair (2-CTA cluster, same TPC) per two SMs
    const int64_t units = (a.m_tiles + 1) / 2 * p.ntiles;
    grid = 2 * (unsigned)std::min<int64_t>(units, sms / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define TS_TCH2_PAIR(SB_)                                                                 \
  do {                                                                                    \
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_tc_halo2_kernel<5, SB_, true>,                  \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                                     (int)p.smem));                                       \
    ts::count_launch();                                                                   \
    TS_CUDA_TRY(cudaLaunchKernelEx(&cfg, conv_tc_halo2_kernel<5, SB_, true>, a));         \
  } while (0)
    if (p.sub == 1) TS_TCH2_PAIR(1);
    else if (p.sub == 2) TS_TCH2_PAIR(2);
    else TS_TCH2_PAIR(4);
#undef TS_TCH2_PAIR
  } else {
#define TS_TCH2_LAUNCH(MD, SB_)                                                       \
  do {                                                                                \
    TS_CUDA_TRY(cudaFuncSetAttribute(conv_tc_halo2_kernel<MD, SB_>,                   \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                     (int)p.smem));                                   \
    ts::count_launch(), conv_tc_halo2_kernel<MD, SB_><<<grid, kThreads, p.smem, s>>>(a); \
  } while (0)
#define TS_TCH2_SUB(MD)                                 \
  do {                                                  \
    if (p.sub == 1) TS_TCH2_LAUNCH(MD, 1);              \
    else if (p.sub == 2) TS_TCH2_LAUNCH(MD, 2);         \
    else TS_TCH2_LAUNCH(MD, 4);                         \
  } while (0)
  if (precision == 2) TS_TCH2_SUB(2);
  else if (precision == 4) TS_TCH2_SUB(4);
  else if (precision == 5) TS_TCH2_SUB(5);
  else TS_TCH2_SUB(3);
#undef TS_TCH2_SUB
#undef TS_TCH2_LAUNCH
  }
  TS_LAUNCH_CHECK();
#ifdef TS_H2_PROF
  {  // per-launch wait profile (profiling build only): cycles per CTA
    unsigned long long h[kPrN];
    TS_CUDA_TRY(cudaStreamSynchronize(s));
    TS_CUDA_TRY(cudaMemcpyFromSymbol(h, g_h2_prof, sizeof(h)));
    const unsigned long long z[kPrN] = {};
    TS_CUDA_TRY(cudaMemcpyToSymbol(g_h2_prof, z, sizeof(z)));
    const double n = (double)grid, tot = (double)h[kPrTotal] / n;
    fprintf(stderr,
            "h2prof k=%d ci=%d co=%d sub=%d bn=%d nt=%d hb=%d sb=%d L=%d cgrp=%d tiles=%lld | "
            "total %.0f kcyc | prod-wait-buf %.2f (x%d warps) | mma: acc %.2f halo %.2f wts "
            "%.2f | epi-wait %.2f (x4) | load-wait %.2f\n",
            op.k, op.in.C, op.out.C, p.sub, p.bn, p.ntiles, p.hbufs, p.bstages, p.lrows, p.cgrp,
            (long long)tiles, tot / 1e3, h[kPrProdWait] / n / kProdW / tot, kProdW,
            h[kPrMmaAcc] / n / tot, h[kPrMmaHalo] / n / tot, h[kPrMmaW] / n / tot,
            h[kPrEpiWait] / n / 4 / tot, h[kPrLoadWait] / n / tot);
  }
#endif
  return TS_OK;
}

}  // namespace ts
