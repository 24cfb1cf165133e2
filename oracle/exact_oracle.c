/*
 * exact_oracle.c -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * A plain-C restatement of the PolarQuant encoder / LUT scorer
 * (/root/reference/pkg/src/polarquant) with a *correctly rounded* float32
 * arctangent: atan2 is evaluated in double and rounded once to float, every
 * other step is the reference's float32 operation sequence:
 *
 *   to_polar                 polar_codec.py:200-209
 *   quantize_angle           polar_codec.py:212-221
 *   compute_radius_scales    polar_codec.py:236-251  (fp16 RNE, :77)
 *   _quantize_radius_counted polar_codec.py:267-278
 *   quantize_subvectors      polar_codec.py:281-302
 *   pack_stream              polar_codec.py:98-110
 *   build_query_lut/qk_scores lut_decode.py:86-104, 119-154
 *
 * It differs from the numpy reference only where numpy's SIMD float32 arctan2
 * is off by an ulp near a bin edge; the GPU kernels implement this same
 * definition, so GPU vs this oracle must agree bit-for-bit.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off: no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define PQO_HALF_SPLIT 1

static const float kPiF = 3.14159274101257324219f;
static const float kTwoPiF = 6.28318548202514648438f;

static uint32_t fbits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
static float bitsf(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* float32 -> float16, round to nearest even (numpy's astype(float16)). */
uint16_t pqo_f32_to_f16(float f) {
  const uint32_t x = fbits(f);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t absx = x & 0x7fffffffu;
  if (absx >= 0x7f800000u) return (uint16_t)(sign | (absx > 0x7f800000u ? 0x7e00u : 0x7c00u));
  if (absx >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* rounds to >= 65520 -> inf */
  if (absx < 0x38800000u) {                                   /* half subnormal / zero */
    const int e = (int)(absx >> 23);
    if (e < 102) return (uint16_t)sign;                        /* < 2^-25: rounds to 0 */
    const uint32_t mant = (absx & 0x7fffffu) | 0x800000u;
    const int shift = 126 - e; /* value = mant * 2^(e-150); half subnormal unit 2^-24 */
    const uint32_t q = mant >> shift;
    const uint32_t rem = mant & ((1u << shift) - 1u);
    const uint32_t halfway = 1u << (shift - 1);
    uint32_t r = q + ((rem > halfway || (rem == halfway && (q & 1u))) ? 1u : 0u);
    return (uint16_t)(sign | r);
  }
  uint32_t h = ((absx - 0x38000000u) >> 13);
  const uint32_t rem = absx & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1u;
  return (uint16_t)(sign | h);
}

float pqo_f16_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu, mant = h & 0x3ffu;
  if (e == 0) {
    if (mant == 0) return bitsf(sign);
    return (sign ? -1.0f : 1.0f) * ldexpf((float)mant, -24);
  }
  if (e == 31) return bitsf(sign | 0x7f800000u | (mant << 13));
  return bitsf(sign | ((e + 112u) << 23) | (mant << 13));
}

static void pair_at(const float* row, int half, int layout, int j, float* x, float* y) {
  if (layout == PQO_HALF_SPLIT) {
    *x = row[j];
    *y = row[j + half];
  } else {
    *x = row[2 * j];
    *y = row[2 * j + 1];
  }
}

static float radius32(float x, float y) {
  const double xd = x, yd = y;
  const double s = xd * xd + yd * yd; /* both squares exact; one rounding */
  return (float)sqrt(s);
}

static float angle_scale(int m) { return (float)((double)(1 << (m - 1)) / M_PI); }

static uint32_t angle_code(float x, float y, int m) {
  const float a = (float)atan2((double)y, (double)x);
  float t = a + kPiF;
  if (t >= kTwoPiF) t = 0.0f;
  const float u = t * angle_scale(m);
  return (uint32_t)(int64_t)rintf(u) & ((1u << m) - 1u);
}

/* scales_out[d/2] fp16 bits; returns nonzero if a scale is not finite. */
int pqo_scales(const float* keys, int64_t T, int d, int layout, int n, uint16_t* out) {
  const int half = d / 2;
  int bad = 0;
  for (int j = 0; j < half; ++j) {
    float top = 0.0f;
    for (int64_t t = 0; t < T; ++t) {
      float x, y;
      pair_at(keys + t * d, half, layout, j, &x, &y);
      const float r = radius32(x, y);
      if (r > top || r != r) top = r;
    }
    const float s = top / (float)((1 << n) - 1);
    out[j] = pqo_f32_to_f16(s);
    if ((out[j] & 0x7c00u) == 0x7c00u) bad = 1;
  }
  return bad;
}

/* angle/radius: [T][d/2] codes; returns the clamp count. */
int64_t pqo_encode(const float* keys, int64_t T, int d, int layout, int m, int n, const uint16_t* s16,
                   uint8_t* angle, uint8_t* radius) {
  const int half = d / 2;
  const float top = (float)((1 << n) - 1);
  int64_t clamps = 0;
  for (int64_t t = 0; t < T; ++t) {
    for (int j = 0; j < half; ++j) {
      float x, y;
      pair_at(keys + t * d, half, layout, j, &x, &y);
      const float s = pqo_f16_to_f32(s16[j]);
      uint32_t a = 0, rc = 0;
      if (s != 0.0f) {
        float raw = rintf(radius32(x, y) / s);
        if (raw > top) {
          ++clamps;
          raw = top;
        }
        rc = (uint32_t)raw;
        a = rc == 0 ? (1u << (m - 1)) : angle_code(x, y, m);
      }
      angle[t * half + j] = (uint8_t)a;
      radius[t * half + j] = (uint8_t)rc;
    }
  }
  return clamps;
}

/* LSB-first bit packing of `count` codes into out[(count*bits+7)/8]. */
void pqo_pack(const uint8_t* codes, int64_t count, int bits, uint8_t* out) {
  const int64_t nbytes = (count * bits + 7) / 8;
  memset(out, 0, (size_t)nbytes);
  for (int64_t i = 0; i < count; ++i)
    for (int b = 0; b < bits; ++b)
      if ((codes[i] >> b) & 1u) {
        const int64_t k = i * bits + b;
        out[k >> 3] |= (uint8_t)(1u << (k & 7));
      }
}

/* LUT scores of the quantized tokens (float32, channel-major, no FMA). */
void pqo_lut_scores(const float* q, const uint8_t* angle, const uint8_t* radius, int64_t T, int d,
                    const uint16_t* s16, int m, int n, int layout, float* out) {
  const int half = d / 2, L = 1 << m;
  float cs[256], sn[256];
  for (int a = 0; a < L; ++a) {
    const double g = M_PI * (double)a / (double)(1 << (m - 1)) - M_PI;
    cs[a] = (float)cos(g);
    sn[a] = (float)sin(g);
  }
  for (int64_t t = 0; t < T; ++t) out[t] = 0.0f;
  for (int j = 0; j < half; ++j) {
    float qx, qy;
    pair_at(q, half, layout, j, &qx, &qy);
    const float s = pqo_f16_to_f32(s16[j]);
    for (int64_t t = 0; t < T; ++t) {
      const uint8_t a = angle[t * half + j], r = radius[t * half + j];
      const float p1 = qx * cs[a];
      const float p2 = qy * sn[a];
      const float part = p1 + p2;
      const float rhat = s * (float)r;
      const float prod = part * rhat;
      out[t] = out[t] + prod;
    }
  }
  (void)n;
}
