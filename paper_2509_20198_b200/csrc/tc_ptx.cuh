// tcgen05 / TMEM / mbarrier / bulk-copy PTX wrappers and the operand-split
// helpers shared by the implicit-GEMM convolution kernels (conv_tc.cu,
// conv_tc2.cu).  sm_100a only.
#pragma once

#include <stdint.h>

namespace ts {
namespace tcx {

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
// Same wait with a suspend-time hint: the waiting warp sleeps (woken by the
// phase flip or after ~ns) instead of re-polling, for waiters whose
// latency does not matter (a staging warp that is a buffer ahead).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, uint32_t ns) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity), "r"(ns)
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
// 16-byte asynchronous global -> shared copy (LDGSTS); bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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
template <bool TF32>
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
  if (TF32)
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
// Packed fp32 FMA (sm_100 FFMA2): {a0, a1} = fma({x, x}, {w0, w1}, {a0, a1}),
// each lane an IEEE fp32 fma (the same results as two fmaf calls, in half
// the instructions)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x, float w0, float w1) {
  uint64_t a = ((uint64_t)__float_as_uint(a1) << 32) | __float_as_uint(a0);
  const uint64_t xx = ((uint64_t)__float_as_uint(x) << 32) | __float_as_uint(x);
  const uint64_t ww = ((uint64_t)__float_as_uint(w1) << 32) | __float_as_uint(w0);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(xx), "l"(ww));
  a0 = __uint_as_float((uint32_t)a);
  a1 = __uint_as_float((uint32_t)(a >> 32));
}

// ---- CTA pairs (cta_group::2): two CTAs of a 2-CTA cluster share one
// M = 256 MMA stream.  The leader (rank 0) issues every MMA; A rows come from
// each CTA's own shared memory, the B (N) columns are split between them,
// and each CTA's TMEM holds its own 128 rows of D.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of the same shared-memory object in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(p)), "r"(rank));
  return a;
}
// arrive on an mbarrier of another CTA of the cluster (release, cluster scope)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// wait whose phase was completed by arrivals from other CTAs (acquire at
// cluster scope)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   su32(dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr),
               "r"(ncols));
}
__device__ __forceinline__ void umma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                      uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// commit of the pair's MMAs, arriving on the barrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(su32(bar)),
      "h"((uint16_t)3)
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

// tcgen05.ld without the wait: several loads can be in flight before one
// tmem_wait_ld()
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Warp-group register reallocation (setmaxnreg): every warp of a warp group
// must execute the same instruction.  The launch-bounds budget is the
// starting point; ptxas allocates each region within its new limit.
template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

// SWIZZLE_128B K-major UMMA smem descriptor: start>>4 [0,14), LBO>>4
// [16,30) (unused for swizzled K-major), SBO>>4 [32,46) = 1024 B per 8-row
// group, version 1 [46,48), layout SWIZZLE_128B = 2 at [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor: D = f32, A/B format (bf16 = 1, tf32 = 2), both
// K-major, N >> 3 at [17,23), M >> 4 at [24,29)
__host__ __device__ constexpr uint32_t make_idesc(uint32_t ab_fmt, int n, int m = 128) {
  return (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// SWIZZLE_64B K-major descriptor: 64-byte rows, SBO = 512 B per 8-row group,
// layout SWIZZLE_64B = 4 at [61,64).  The swizzle XORs address bits [4,6)
// with bits [7,9), i.e. 16-byte chunk c of row r sits at chunk c ^ ((r>>1)&3)
// for a 512-byte aligned image.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// Operand splitting with integer ALU ops only (no F2F/XU conversions).
// tf32 hi: round-to-nearest-away on the 13 dropped bits; bf16 planes: exact
// truncation split a = a0 + a1 + a2 (each 8 significant bits), bf16 RN for
// the single-plane mode.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ uint32_t hi_halves(float a, float b) {  // {a.hi16, b.hi16}
  return __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x7632);
}
// bf16 round-to-nearest-even; the result's high 16 bits are the bf16 value
// (low bits are garbage until bf_keep clears them)
__device__ __forceinline__ float rn_bf(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float(u + 0x7FFFu + ((u >> 16) & 1u));
}
__device__ __forceinline__ float bf_keep(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFF0000u);
}

// 32-byte global store (STG.256, sm_100): one full sector per lane
__device__ __forceinline__ void st_v8(float* p, const float* v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

// 32-byte read-only global load (LDG.256)
__device__ __forceinline__ void ld_v8(const float* p, float* v) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                 "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

// {bf16_rn(lo), bf16_rn(hi)} packed (lo in the low half): one F2FP
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// a = a0 + a1 + e, a0 = bf16_rn(a), a1 = bf16_rn(a - a0), |e| <= 2^-18 |a|
// (hardware RN conversions: 2 F2FP + 4 unpack/subtract per pair)
__device__ __forceinline__ void store_split2(uint8_t* dst, int plane_bytes, float4 a) {
  const uint32_t h01 = pack_bf2(a.x, a.y), h23 = pack_bf2(a.z, a.w);
  const uint32_t l01 = pack_bf2(a.x - __uint_as_float(h01 << 16),
                                a.y - __uint_as_float(h01 & 0xFFFF0000u));
  const uint32_t l23 = pack_bf2(a.z - __uint_as_float(h23 << 16),
                                a.w - __uint_as_float(h23 & 0xFFFF0000u));
  *reinterpret_cast<uint2*>(dst) = make_uint2(h01, h23);
  *reinterpret_cast<uint2*>(dst + plane_bytes) = make_uint2(l01, l23);
}

// a pair -> the two plane words of an ActView planes format (1: bf16 RN
// hi/lo, 2: FP16X3 hi / 2^11-scaled lo, the split the halo producers would
// compute from the fp32 value)
__device__ __forceinline__ void split_pair(float x, float y, bool f16, uint32_t& h,
                                           uint32_t& l);
// 16 consecutive channels (chan % 8 == 0) into a planes pixel block
// (conv.cuh ActView): 32 bytes of hi, 32 bytes of lo, 16-byte stores
__device__ __forceinline__ void store16_planes(float* block, int cstride, int chan,
                                               const float* v, bool f16) {
  uint32_t h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) split_pair(v[2 * i], v[2 * i + 1], f16, h[i], l[i]);
  uint4* hp = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(block) + 2 * chan);
  uint4* lp = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(block) + 2 * (cstride + chan));
  hp[0] = make_uint4(h[0], h[1], h[2], h[3]);
  hp[1] = make_uint4(h[4], h[5], h[6], h[7]);
  lp[0] = make_uint4(l[0], l[1], l[2], l[3]);
  lp[1] = make_uint4(l[4], l[5], l[6], l[7]);
}
// 8 channels (chan % 8 == 0): 16 bytes of hi, 16 of lo
__device__ __forceinline__ void store8_planes(float* block, int cstride, int chan,
                                              const float* v, bool f16) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_pair(v[2 * i], v[2 * i + 1], f16, h[i], l[i]);
  *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(block) + 2 * chan) =
      make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(block) + 2 * (cstride + chan)) =
      make_uint4(l[0], l[1], l[2], l[3]);
}

// integer-ALU form of store_split2 (same values)
__device__ __forceinline__ void store_split2_alu(uint8_t* dst, int plane_bytes, float4 a) {
  const float x0 = bf_keep(rn_bf(a.x)), y0 = bf_keep(rn_bf(a.y)), z0 = bf_keep(rn_bf(a.z)),
              w0 = bf_keep(rn_bf(a.w));
  const float x1 = rn_bf(a.x - x0), y1 = rn_bf(a.y - y0), z1 = rn_bf(a.z - z0),
              w1 = rn_bf(a.w - w0);
  *reinterpret_cast<uint2*>(dst) = make_uint2(hi_halves(x0, y0), hi_halves(z0, w0));
  *reinterpret_cast<uint2*>(dst + plane_bytes) =
      make_uint2(hi_halves(x1, y1), hi_halves(z1, w1));
}

template <int MODE>
struct Mode;
template <>
struct Mode<1> {  // TF32X3: A hi/lo, B hi/lo
  static constexpr int pa = 2, pb = 2, kc = 32;
  static constexpr bool tf32 = true, f16 = false;
};
template <>
struct Mode<2> {  // BF16
  static constexpr int pa = 1, pb = 1, kc = 64;
  static constexpr bool tf32 = false, f16 = false;
};
template <>
struct Mode<3> {  // BF16X3: A = a0 + a1 (RN, residual <= 2^-18 |a|), B = b0+b1+b2
  static constexpr int pa = 2, pb = 3, kc = 64;
  static constexpr bool tf32 = false, f16 = false;
};
template <>
struct Mode<4> {  // BF16X4: A = a0 + a1, B = b0 + b1 (both RN, residual <= 2^-18)
  static constexpr int pa = 2, pb = 2, kc = 64;
  static constexpr bool tf32 = false, f16 = false;
};
// FP16X3 (the fp32-class mode): fp16 planes with a scaled correction plane,
// a = a0 + 2^-11 a1, a0 = fp16_rn(a), a1 = fp16_rn((a - a0) 2^11), so both
// planes are in fp16's normal range and |a - a0 - 2^-11 a1| <= 2^-24 |a|
// (fp32's own rounding); same for the weights.  Products: a0 b0 into a MAIN
// column block, a0 b1 + a1 b0 into a CORRECTION block (scaled by 2^11).
// Each tcgen05 MMA truncates its fp32 accumulation (scripts/mma_numerics.cu
// measures the bias), so a long K chain in one accumulator drifts: the
// kernels restart both blocks every <= 18 K steps (a "group" of channel
// chunks) and the epilogue warps promote each group's main + 2^-11 corr into
// fp32 registers with round-to-nearest adds.
template <>
struct Mode<5> {
  static constexpr int pa = 2, pb = 2, kc = 64;
  static constexpr bool tf32 = false, f16 = true;
};
constexpr float kF16Lo = 2048.f;         // correction-plane scale 2^11
constexpr float kF16LoInv = 1.f / 2048.f;

// instruction-descriptor operand format of a mode: tf32 2, bf16 1, fp16 0
template <int MODE>
__host__ __device__ constexpr uint32_t mode_fmt() {
  return Mode<MODE>::tf32 ? 2u : Mode<MODE>::f16 ? 0u : 1u;
}

// {fp16_rn(lo), fp16_rn(hi)} packed (lo in the low half): one F2FP
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// a pair -> main plane word h and scaled correction word l
__device__ __forceinline__ void split_h2(float x, float y, uint32_t& h, uint32_t& l) {
  h = pack_h2(x, y);
  float hx, hy;
  asm("{\n.reg .f16 a, b;\nmov.b32 {a, b}, %2;\ncvt.f32.f16 %0, a;\ncvt.f32.f16 %1, b;\n}\n"
      : "=f"(hx), "=f"(hy)
      : "r"(h));
  // x - hx is exact (hx = x rounded to 11 bits); the 2^11 scale is exact
  l = pack_h2((x - hx) * kF16Lo, (y - hy) * kF16Lo);
}
__device__ __forceinline__ void split_pair(float x, float y, bool f16, uint32_t& h,
                                           uint32_t& l) {
  if (f16) {
    split_h2(x, y, h, l);
  } else {
    h = pack_bf2(x, y);
    l = pack_bf2(x - __uint_as_float(h << 16), y - __uint_as_float(h & 0xFFFF0000u));
  }
}
// 4 floats -> 8 bytes of each plane
__device__ __forceinline__ void store_split_h(uint8_t* dst, int plane_bytes, float4 a) {
  uint32_t h01, l01, h23, l23;
  split_h2(a.x, a.y, h01, l01);
  split_h2(a.z, a.w, h23, l23);
  *reinterpret_cast<uint2*>(dst) = make_uint2(h01, h23);
  *reinterpret_cast<uint2*>(dst + plane_bytes) = make_uint2(l01, l23);
}


}  // namespace tcx
}  // namespace ts
