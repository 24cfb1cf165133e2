// Exact float32 polar quantization (HP-1 arithmetic), sm_100a.
//
// Reference semantics (polar_codec.py, all float32 numpy):
//   to_polar        :200-209  r = hypotf(x, y);  t = mod(atan2f(y, x) + pi, 2pi)
//   quantize_angle  :212-221  code = rint(t * fl32(2^(m-1)/pi)) mod 2^m   (half-even)
//   _quantize_radius_counted :267-278  raw = rint(r / s32); s32 == 0 -> 0; clamp to 2^n-1
//   quantize_subvectors :281-302  rcode == 0 -> angle = 2^(m-1); s16 == 0 -> both 0
//
// "Exact" here means the reference pipeline evaluated with a correctly rounded
// atan2f and glibc's hypotf (fl32(sqrt(fl64(x*x + y*y)))).  numpy's own float32
// arctan2 is a SIMD approximation (<= a few ulp), so a reference code may differ
// from ours only when the angle sits within ~1e-6 rad of a bin edge: the counted,
// admissible "ties" of the parity contract.
//
// Fast path.  Evaluating atan2 in double for every element would make the
// encoder FP64-bound, so the bin is decided geometrically: fold (x, y) into the
// first octant (m >= 3; quadrant for m = 2), then count the bin edges b_i below
// the point with one FMA each, D_i = mn - mx * tan(b_i).  A point farther than
// DELTA = 4e-6 rad from every edge gets the same code as the exact pipeline:
// the pipeline's total drift from the true angle is <= 1.0e-6 rad
//   (|pi_f32 - pi| = 8.7e-8, atan2 rounding 1.2e-7, t rounding 2.4e-7,
//    fl32(2^(m-1)/pi) relative 6e-8 -> 3.7e-7, product rounding 1.9e-7)
// and D_i's own float error is < 2e-7 r.  Points inside the band (about 1e-5
// of random inputs) take the exact double-precision path.  The radius uses the
// same scheme: a fast fp32 estimate of r/s, and the exact path only when the
// estimate lies within 2^-18 relative of a rounding boundary.
#pragma once

#include "common.cuh"
#include "angle_tables.h"

namespace pqb {

constexpr float kPiF = 3.14159274101257324219f;     // fl32(pi)
constexpr float kTwoPiF = 6.28318548202514648438f;  // fl32(2 pi) == 2 * fl32(pi)

// ------------------------------------------------------------ exact paths

// Steps 2-3 of the pipeline from the (correctly rounded) fp32 angle a.
PQB_DEV uint32_t angle_code_from_phi(float a, int m) {
  float t = __fadd_rn(a, kPiF);
  if (t >= kTwoPiF) t = 0.0f;  // np.mod(t, fl32(2 pi)); t <= 2 pi_f32 by construction
  const float u = __fmul_rn(t, kAngleScale[m]);
  return static_cast<uint32_t>(__float2int_rn(u)) & ((1u << m) - 1u);
}

PQB_DEV uint32_t angle_code_exact(float x, float y, int m) {
  return angle_code_from_phi(__double2float_rn(atan2(static_cast<double>(y), static_cast<double>(x))), m);
}

// fl32(sqrt(fl64(x^2 + y^2))): both squares are exact in double, one rounding
// in the sum, glibc's hypotf (sysdeps/ieee754/flt-32/e_hypotf.c) order.
PQB_DEV float radius_exact(float x, float y) {
  const double xd = x, yd = y;
  const double d2 = __fma_rn(xd, xd, __dmul_rn(yd, yd));
  return __double2float_rn(__dsqrt_rn(d2));
}

// rint(fl32(r / s)) as a float (may be +inf); s > 0.
PQB_DEV float radius_raw_exact(float x, float y, float s) {
  return rintf(__fdiv_rn(radius_exact(x, y), s));
}

// ------------------------------------------------------------- fast paths

// |v| in [2^-100, 2^100] as one unsigned compare on the float bits (false for
// 0, subnormals, huge values, Inf and NaN): the range where the fp32 edge tests
// below are provably accurate.
PQB_DEV bool in_safe_range(float v) {
  return (__float_as_uint(v) & 0x7fffffffu) - 0x0D800000u <= (0x71800000u - 0x0D800000u);
}
// Same for a value that is +0, positive or NaN (r2 = x*x + y*y): no abs mask
// needed (a sign-bit NaN lands far above the range).
PQB_DEV bool in_safe_range_nonneg(float v) { return __float_as_uint(v) - 0x0D800000u <= (0x71800000u - 0x0D800000u); }

// Angle code for angle_bits M; sets amb when the point is within DELTA of a bin
// edge (or outside the safe magnitude range) and the caller must use
// angle_code_exact.  Edge constants fold into FFMA/FMUL immediates.
template <int M>
PQB_DEV uint32_t angle_code_fast(float x, float y, bool& amb, const float* smem_tan,
                                 const float* smem_thr) {
  const float ax = fabsf(x), ay = fabsf(y);
  const uint32_t sx = __float_as_uint(x) >> 31, sy = __float_as_uint(y) >> 31;
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  // magnitude range: guaranteed by the caller's r2 check (r2 in [2^-100, 2^100]
  // => mx in [2^-51, 2^50], where every edge product below is a normal float)
  amb = false;
  if constexpr (M == 1) {
    // edges at phi = +-pi/2 (the y axis): code 1 iff x > 0
    amb |= !(ax > PQB_ANGLE_DELTA * (ax + ay));
    return sx ? 0u : 1u;
  } else {
    constexpr int H = 1 << (M - 1);
    int k;  // bin index within the quadrant, 0 .. 2^(M-2)
    if constexpr (M == 2) {
      const float dd = ay - ax;  // edge at pi/4; sign exact
      if (dd == 0.0f) {
        // exactly on the diagonal (frequent for bf16 keys): atan2f is
        // fl32(+-pi/4) or fl32(+-3pi/4), so finish the pipeline directly
        // instead of sending the whole group down the double-precision path
        return angle_code_from_phi(copysignf(sx ? 2.35619449615478515625f : 0.785398185253143310546875f, y), 2);
      }
      amb |= fabsf(dd) <= kQuadEdgeThr * (ax + ay);
      k = dd > 0.0f ? 1 : 0;
    } else {
      constexpr int NB = 1 << (M - 3);  // octant edges
      const float sum = mx + mn;
      int kk = 0;
      if constexpr (NB <= 4) {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const float di = fmaf(-mx, edge_tan(M, i), mn);
          kk += di > 0.0f ? 1 : 0;
          amb |= fabsf(di) <= edge_thr(M, i) * sum;
        }
      } else {
        // estimate psi = atan(mn/mx) to < step/4, then verify the two edges
        // around the estimated bin exactly.
        constexpr float kInvStep = static_cast<float>(1 << (M - 1)) / 3.14159265358979f;
        const float rho = mn * __frcp_rn(mx);
        // atan(rho) ~ rho*(pi/4 + 0.273*(1 - rho)), |err| < 4e-3 rad on [0, 1]
        const float psi = rho * fmaf(0.2732395f, 1.0f - rho, 0.78539816f);
        int ke = __float2int_rn(psi * kInvStep);
        ke = ke < 0 ? 0 : (ke > NB ? NB : ke);
        kk = ke;
        if (ke > 0) {  // edge below: b_{ke-1}
          const float di = fmaf(-mx, smem_tan[ke - 1], mn);
          kk -= di > 0.0f ? 0 : 1;
          amb |= fabsf(di) <= smem_thr[ke - 1] * sum;
        }
        if (ke < NB) {  // edge above: b_ke
          const float di = fmaf(-mx, smem_tan[ke], mn);
          kk += di > 0.0f ? 1 : 0;
          amb |= fabsf(di) <= smem_thr[ke] * sum;
        }
      }
      constexpr int Q = 1 << (M - 2);
      k = (ay > ax) ? (Q - kk) : kk;  // unfold the octant
    }
    // unfold the quadrant: code = (c_phi + H) mod 2H with c_phi the multiple of
    // the grid step nearest phi = atan2(y, x)
    const int base = sx ? (sy ? 0 : 2 * H) : H;
    const int c = (sx ^ sy) ? base - k : base + k;
    return static_cast<uint32_t>(c) & (2u * H - 1u);
  }
}

// Fast rint(r/s) (float; large values mean "clamped"), branch-free.  r is
// estimated as r2 * rsqrt(r2) (relative error < 2^-21 with the fp32 rounding of
// r2 and 1/s); amb when that estimate lies within 2^-18 (relative) of a
// half-integer or r2 is outside the safe range (zero, subnormal, huge, NaN).
PQB_DEV float rsqrt_approx(float v) {  // MUFU.RSQ; v is in the safe range when used
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

PQB_DEV float radius_raw_fast(float x, float y, float inv_s, bool& amb) {
  const float r2 = fmaf(x, x, y * y);
  amb = !in_safe_range_nonneg(r2);
  const float q = r2 * rsqrt_approx(r2) * inv_s;
  const float rq = rintf(q);
  amb |= fabsf(q - rq) >= fmaf(-0x1p-18f, q, 0.5f);
  return rq;
}

// Eight sub-vectors (one thread's channel group) with one divergent slow path:
// fast codes for all eight, then the exact pipeline only for the flagged ones.
// Returns the packed angle / radius chunks (code i at bits [b*i, b*(i+1))).
// live: bit i set when sub-vector i is a valid token with a non-zero scale;
// other positions produce (0, 0) (zero-scale rule, polar_codec.py:298-301).
template <int M>
PQB_DEV void encode8(const float (&x)[8], const float (&y)[8], const float (&s32)[8], const float (&inv)[8],
                     int n_bits, uint32_t live, unsigned long long& ca, unsigned long long& cr,
                     uint32_t& clamped, bool& bad, const float* smem_tan, const float* smem_thr) {
  const float top = static_cast<float>((1 << n_bits) - 1);
  float raw[8];
  uint32_t a[8];
  bool any_amb = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    bool ra, aa;
    raw[i] = radius_raw_fast(x[i], y[i], inv[i], ra);
    a[i] = angle_code_fast<M>(x[i], y[i], aa, smem_tan, smem_thr);
    any_amb |= ra | aa;
  }
  if (any_amb && live) {  // ~1e-5 of sub-vectors: the exact double-precision pipeline for
                          // this thread's eight (cheaper than tracking which one)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if ((live >> i) & 1u) {
        bad |= !(fabsf(x[i]) <= 3.40282347e38f && fabsf(y[i]) <= 3.40282347e38f);
        raw[i] = radius_raw_exact(x[i], y[i], s32[i]);
        a[i] = angle_code_exact(x[i], y[i], M);
      }
    }
  }
  uint32_t over = 0u;
  ca = 0ull;
  cr = 0ull;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    over |= static_cast<uint32_t>(raw[i] > top) << i;
    const uint32_t rc = static_cast<uint32_t>(fminf(raw[i], top));
    const uint32_t ac = rc == 0u ? (1u << (M - 1)) : a[i];  // canonical: origin's angle (polar_codec.py:297)
    ca |= static_cast<unsigned long long>(ac) << (M * i);
    cr |= static_cast<unsigned long long>(rc) << (n_bits * i);
  }
  clamped += __popc(over & live);
  // zero-scale channels and invalid tokens: both codes 0
  unsigned long long ka = 0ull, kr = 0ull;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if ((live >> i) & 1u) {
      ka |= ((1ull << M) - 1ull) << (M * i);
      kr |= ((1ull << n_bits) - 1ull) << (n_bits * i);
    }
  }
  ca &= ka;
  cr &= kr;
}

// Runtime-m variant: exact pipeline only (used by the generic / append paths).
PQB_DEV void encode_pair_exact(float x, float y, float s32, int m_bits, int n_bits,
                               uint32_t& acode, uint32_t& rcode, uint32_t& clamped) {
  if (s32 == 0.0f) {
    acode = 0u;
    rcode = 0u;
    return;
  }
  const float top = static_cast<float>((1 << n_bits) - 1);
  float raw = radius_raw_exact(x, y, s32);
  if (raw > top) {
    clamped += 1u;
    raw = top;
  }
  rcode = static_cast<uint32_t>(raw);
  if (rcode == 0u) {
    acode = 1u << (m_bits - 1);
    return;
  }
  acode = angle_code_exact(x, y, m_bits);
}

}  // namespace pqb
