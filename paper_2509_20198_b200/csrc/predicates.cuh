// Exact orientation / incircle predicates for the GPU Delaunay (K2a).
//
// Fast path: fp64 evaluation with Shewchuk-style static error bounds.
// Slow path (|det| under the bound): the doubles are scaled by a common
// power of two into integers (< 2^111) and the determinant is evaluated in
// exact 512-bit two's-complement arithmetic.  Inputs whose exponent spread
// exceeds 110 bits (never produced by patch-space transforms of real data)
// keep the fp64 sign; that fallback is counted in the status.
//
// The reference delegates triangulation to Qhull (patches.py:319), which
// is not exact; with exact predicates the triangulation equals the unique
// Delaunay triangulation whenever no four points are cocircular.
#pragma once

#include <stdint.h>
#include <string.h>

namespace ts {
namespace pred {

#ifdef __CUDACC__
#define TS_HD __host__ __device__ __forceinline__
#else
#define TS_HD inline
#endif

typedef unsigned __int128 u128;
typedef __int128 i128;

struct I512 {
  uint64_t w[8];  // little-endian limbs, two's complement
};

TS_HD I512 from_i128(i128 v) {
  I512 r;
  r.w[0] = (uint64_t)v;
  r.w[1] = (uint64_t)(v >> 64);
  const uint64_t ext = v < 0 ? ~0ull : 0ull;
  for (int i = 2; i < 8; ++i) r.w[i] = ext;
  return r;
}
TS_HD bool neg(const I512& a) { return (a.w[7] >> 63) != 0; }
TS_HD I512 add(const I512& a, const I512& b) {
  I512 r;
  uint64_t carry = 0;
  for (int i = 0; i < 8; ++i) {
    const u128 s = (u128)a.w[i] + b.w[i] + carry;
    r.w[i] = (uint64_t)s;
    carry = (uint64_t)(s >> 64);
  }
  return r;
}
TS_HD I512 negate(const I512& a) {
  I512 r;
  uint64_t carry = 1;
  for (int i = 0; i < 8; ++i) {
    const u128 s = (u128)(~a.w[i]) + carry;
    r.w[i] = (uint64_t)s;
    carry = (uint64_t)(s >> 64);
  }
  return r;
}
TS_HD I512 sub(const I512& a, const I512& b) { return add(a, negate(b)); }
TS_HD int sign(const I512& a) {
  if (neg(a)) return -1;
  for (int i = 0; i < 8; ++i)
    if (a.w[i]) return 1;
  return 0;
}
// a * b for |a|, |b| < 2^255 (upper halves are sign extension).
TS_HD I512 mul(const I512& a, const I512& b) {
  const bool na = neg(a), nb = neg(b);
  const I512 ua = na ? negate(a) : a;
  const I512 ub = nb ? negate(b) : b;
  uint64_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < 4; ++i) {
    uint64_t carry = 0;
    for (int j = 0; j < 4; ++j) {
      const u128 p = (u128)ua.w[i] * ub.w[j] + r[i + j] + carry;
      r[i + j] = (uint64_t)p;
      carry = (uint64_t)(p >> 64);
    }
    r[i + 4] += carry;
  }
  I512 out;
  for (int i = 0; i < 8; ++i) out.w[i] = r[i];
  return (na != nb) ? negate(out) : out;
}

// exponent of the most / least significant set bit of a nonzero double
TS_HD void bit_range(double v, int& msb, int& lsb) {
  uint64_t bits;
  memcpy(&bits, &v, 8);
  const int e = (int)((bits >> 52) & 0x7FF);
  uint64_t m = bits & ((1ull << 52) - 1);
  if (e == 0) {  // subnormal
    int top = 63;
    while (!((m >> top) & 1)) --top;
    msb = -1074 + top;
    int low = 0;
    while (!((m >> low) & 1)) ++low;
    lsb = -1074 + low;
  } else {
    m |= 1ull << 52;
    msb = e - 1023;
    int low = 0;
    while (!((m >> low) & 1)) ++low;
    lsb = e - 1075 + low;
  }
}

// v * 2^-shift as an exact integer (caller guarantees exactness)
TS_HD i128 to_int(double v, int shift) {
  if (v == 0.0) return 0;
  uint64_t bits;
  memcpy(&bits, &v, 8);
  const int e = (int)((bits >> 52) & 0x7FF);
  uint64_t m = bits & ((1ull << 52) - 1);
  int ex;
  if (e == 0) ex = -1074;
  else { m |= 1ull << 52; ex = e - 1075; }
  const int s = ex - shift;  // v = m * 2^ex = (m << s) * 2^shift
  u128 mag = (u128)m;
  if (s >= 0) mag <<= s;
  else mag >>= -s;  // exact: shift <= lsb
  const i128 r = (i128)mag;
  return (bits >> 63) ? -r : r;
}

// Common scale for n doubles; false when the spread is too wide.
TS_HD bool common_shift(const double* v, int n, int& shift) {
  int hi = -100000, lo = 100000;
  bool any = false;
  for (int i = 0; i < n; ++i) {
    if (v[i] == 0.0) continue;
    int m, l;
    bit_range(v[i], m, l);
    hi = m > hi ? m : hi;
    lo = l < lo ? l : lo;
    any = true;
  }
  shift = any ? lo : 0;
  return !any || (hi - lo) <= 108;
}

TS_HD int orient_exact(double ax, double ay, double bx, double by, double cx,
                       double cy, bool* exact) {
  const double v[6] = {ax, ay, bx, by, cx, cy};
  int sh;
  if (!common_shift(v, 6, sh)) {
    *exact = false;
    const double d = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
    return d > 0 ? 1 : (d < 0 ? -1 : 0);
  }
  *exact = true;
  const i128 Ax = to_int(ax, sh), Ay = to_int(ay, sh);
  const i128 Bx = to_int(bx, sh), By = to_int(by, sh);
  const i128 Cx = to_int(cx, sh), Cy = to_int(cy, sh);
  const I512 l = mul(from_i128(Bx - Ax), from_i128(Cy - Ay));
  const I512 r = mul(from_i128(By - Ay), from_i128(Cx - Ax));
  return sign(sub(l, r));
}

// > 0 when c is left of a->b (counter-clockwise)
TS_HD int orient(double ax, double ay, double bx, double by, double cx,
                 double cy) {
  const double detl = (ax - cx) * (by - cy);
  const double detr = (ay - cy) * (bx - cx);
  const double det = detl - detr;
  const double sum = (detl < 0 ? -detl : detl) + (detr < 0 ? -detr : detr);
  const double bound = (3.0 + 16.0 * 1.1102230246251565e-16) *
                       1.1102230246251565e-16 * sum;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  bool ex;
  return orient_exact(ax, ay, bx, by, cx, cy, &ex);
}

TS_HD int incircle_exact(const double* p /* ax ay bx by cx cy dx dy */,
                         bool* exact) {
  int sh;
  if (!common_shift(p, 8, sh)) {
    *exact = false;
    return 0;
  }
  *exact = true;
  i128 q[8];
  for (int i = 0; i < 8; ++i) q[i] = to_int(p[i], sh);
  const I512 adx = from_i128(q[0] - q[6]), ady = from_i128(q[1] - q[7]);
  const I512 bdx = from_i128(q[2] - q[6]), bdy = from_i128(q[3] - q[7]);
  const I512 cdx = from_i128(q[4] - q[6]), cdy = from_i128(q[5] - q[7]);
  const I512 alift = add(mul(adx, adx), mul(ady, ady));
  const I512 blift = add(mul(bdx, bdx), mul(bdy, bdy));
  const I512 clift = add(mul(cdx, cdx), mul(cdy, cdy));
  const I512 bc = sub(mul(bdx, cdy), mul(cdx, bdy));
  const I512 ca = sub(mul(cdx, ady), mul(adx, cdy));
  const I512 ab = sub(mul(adx, bdy), mul(bdx, ady));
  const I512 det = add(add(mul(alift, bc), mul(blift, ca)), mul(clift, ab));
  return sign(det);
}

// > 0 when d lies strictly inside the circle through CCW a, b, c
TS_HD int incircle(double ax, double ay, double bx, double by, double cx,
                   double cy, double dx, double dy) {
  const double adx = ax - dx, ady = ay - dy;
  const double bdx = bx - dx, bdy = by - dy;
  const double cdx = cx - dx, cdy = cy - dy;
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double alift = adx * adx + ady * ady;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double blift = bdx * bdx + bdy * bdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double clift = cdx * cdx + cdy * cdy;
  const double det = alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) +
                     clift * (adxbdy - bdxady);
  const double perm =
      ((bdxcdy < 0 ? -bdxcdy : bdxcdy) + (cdxbdy < 0 ? -cdxbdy : cdxbdy)) * alift +
      ((cdxady < 0 ? -cdxady : cdxady) + (adxcdy < 0 ? -adxcdy : adxcdy)) * blift +
      ((adxbdy < 0 ? -adxbdy : adxbdy) + (bdxady < 0 ? -bdxady : bdxady)) * clift;
  const double bound = (10.0 + 96.0 * 1.1102230246251565e-16) *
                       1.1102230246251565e-16 * perm;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  const double p[8] = {ax, ay, bx, by, cx, cy, dx, dy};
  bool ex;
  const int s = incircle_exact(p, &ex);
  if (!ex) return det > 0 ? 1 : (det < 0 ? -1 : 0);
  return s;
}

}  // namespace pred
}  // namespace ts
