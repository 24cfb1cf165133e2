// Element-wise reference API on the device (the functions polarquant exports
// besides the cache path) and the paged-store import of PQC1 streams.
//
//   to_polar        polar_codec.py:200-209   r = hypot(x, y), t = mod(atan2(y, x) + pi, 2 pi)
//   quantize_angle  polar_codec.py:212-221   rint(t * (2^(m-1) / pi)) mod 2^m  (half-even)
//   angle_grid      polar_codec.py:224-233   pi * a / 2^(m-1) - pi, float64
//   quantize_radius polar_codec.py:254-278   rint(r / s32), s32 == 0 -> 0, clamp to 2^n - 1
//   qk_scores_direct lut_decode.py:157-186   dequantize (polar_codec.py:305-316), then fp32 dots
//   import streams  polar_codec.py:415-446, kv_cache.py:369-397 (load_codes / load_snapshot)
//
// numpy evaluates these in the input's precision: float32 arrays in float32
// (the Python-float constants are cast to float32 first, NEP 50), float64
// arrays and Python scalars in float64.  Both are supported (PQB_F32 /
// PQB_F64); the float32 path is the one the encoder uses (polar_math.cuh).
#include "common.cuh"
#include "kernels.h"
#include "polar_math.cuh"

#include <algorithm>

namespace pqb {

constexpr double kPiAPI = 3.141592653589793115997963468544185161590576171875;  // == np.pi

PQB_DEV const uint8_t* page_base_a(const pqb_store& s, int64_t unit, int64_t page) {
  const int64_t pid = s.page_table ? static_cast<int64_t>(s.page_table[unit * s.max_pages + page])
                                   : unit * s.max_pages + page;
  return s.pool + pid * s.page_bytes;
}

// ------------------------------------------------------------ to_polar

__global__ void to_polar_f32_kernel(const float* x, const float* y, int64_t n, float* r, float* t) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float xv = x[i], yv = y[i];
    r[i] = radius_exact(xv, yv);  // glibc hypotf: fl32(sqrt(fl64(x^2 + y^2)))
    const float a = __double2float_rn(atan2(static_cast<double>(yv), static_cast<double>(xv)));
    float th = __fadd_rn(a, kPiF);
    if (th >= kTwoPiF) th = __fsub_rn(th, kTwoPiF);  // np.mod(., fl32(2 pi)); th <= 2 pi_f32
    t[i] = th;
  }
}

__global__ void to_polar_f64_kernel(const double* x, const double* y, int64_t n, double* r, double* t) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double xv = x[i], yv = y[i];
    r[i] = hypot(xv, yv);
    double th = __dadd_rn(atan2(yv, xv), kPiAPI);
    if (th >= 2.0 * kPiAPI) th = __dsub_rn(th, 2.0 * kPiAPI);  // np.mod(., 2 pi); th <= 2 pi
    t[i] = th;
  }
}

// -------------------------------------------------------- quantize_angle

// code = int64(rint(v)) mod 2^m; numpy's cast of a non-finite or out-of-range
// value yields INT64_MIN, whose residue is 0
PQB_DEV uint8_t angle_residue(double r, int m) {
  const int64_t k = (r >= -9.2e18 && r <= 9.2e18) ? static_cast<int64_t>(r) : INT64_MIN;
  return static_cast<uint8_t>(k & ((1ll << m) - 1));  // Python % for a power-of-two modulus
}

__global__ void quantize_angle_f32_kernel(const float* th, int64_t n, int m, uint8_t* out) {
  const float sc = kAngleScale[m];  // fl32(2^(m-1) / pi)
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = angle_residue(static_cast<double>(rintf(__fmul_rn(th[i], sc))), m);
}

__global__ void quantize_angle_f64_kernel(const double* th, int64_t n, int m, uint8_t* out) {
  const double sc = __ddiv_rn(static_cast<double>(1 << (m - 1)), kPiAPI);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = angle_residue(rint(__dmul_rn(th[i], sc)), m);
}

__global__ void angle_grid_kernel(int m, double* out) {
  const int a = threadIdx.x;
  if (a < (1 << m)) {
    const double hl = static_cast<double>(1 << (m - 1));
    out[a] = __dsub_rn(__ddiv_rn(__dmul_rn(kPiAPI, static_cast<double>(a)), hl), kPiAPI);
  }
}

// ------------------------------------------------------- quantize_radius

template <typename T>
PQB_DEV T div_rn(T a, T b);
template <>
PQB_DEV float div_rn<float>(float a, float b) { return __fdiv_rn(a, b); }
template <>
PQB_DEV double div_rn<double>(double a, double b) { return __ddiv_rn(a, b); }

template <typename T>
__global__ void quantize_radius_kernel(const T* r, const float* s32, int64_t n, int bits, uint8_t* out,
                                       unsigned long long* clamped) {
  const T top = static_cast<T>((1 << bits) - 1);
  unsigned cnt = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float s = s32[i];
    T raw = s == 0.0f ? T(0) : rint(div_rn<T>(r[i], static_cast<T>(s)));  // r / scale32 in r's precision
    cnt += raw > top;
    raw = raw > top ? top : raw;
    out[i] = raw >= T(0) ? static_cast<uint8_t>(raw) : uint8_t(0);  // clip; NaN -> 0
  }
  if (clamped != nullptr) {
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(clamped, static_cast<unsigned long long>(cnt));
  }
}

// ------------------------------------------------------------- import

// Scatter one contiguous reference stream (PQC1 payload, PolarCodes stream) into
// the unit's pages: the inverse of export_kernel (misc.cu).  The final byte's
// padding bits are stored as zero, since a later append ORs codes into them.
__global__ void import_kernel(pqb_store st, int64_t unit, int half, int b, int64_t region_off, int64_t T,
                              const uint8_t* in) {
  const int64_t bits = T * half * b;
  const int64_t nbytes = (bits + 7) / 8;
  const int64_t R = static_cast<int64_t>(st.page_tokens) * half * b / 8;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nbytes;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t page = k / R;
    uint8_t v = in[k];
    if (k == nbytes - 1 && (bits & 7)) v &= static_cast<uint8_t>((1u << (bits & 7)) - 1u);
    const_cast<uint8_t*>(page_base_a(st, unit, page))[region_off + (k - page * R)] = v;
  }
}

// ---------------------------------------------------- qk_scores_direct

// One warp per token.  Quantized tokens: dequantize every sub-vector exactly as
// dequantize_subvectors (rhat = fl(code * s32); x = fl(rhat cos_a), y = fl(rhat sin_a))
// and dot with q in fp32; residual tokens: fp32 dot with the stored row.
// The summation order (per-lane FMA chains, then a butterfly) differs from
// BLAS, as any two fp32 dot implementations do (lut_decode.py:157-186 only
// promises agreement with the LUT path within 1e-4 of the peak).
__global__ void scores_direct_kernel(pqb_cache c, int64_t unit, const void* q, int q_dtype, int64_t tokens,
                                     float* out) {
  __shared__ float cs[256], sn[256];
  const int m = c.angle_bits, n = c.radius_bits, half = c.d / 2;
  for (int a = threadIdx.x; a < (1 << m); a += blockDim.x) {
    const double hl = static_cast<double>(1 << (m - 1));
    const double g = __dsub_rn(__ddiv_rn(__dmul_rn(kPiAPI, static_cast<double>(a)), hl), kPiAPI);
    cs[a] = __double2float_rn(cos(g));
    sn[a] = __double2float_rn(sin(g));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int T = c.seq_lens[unit], Tq = c.quant_lens[unit];
  const int64_t P = c.store.page_tokens;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       t < tokens && t < T; t += warps) {
    float acc = 0.0f;
    if (t < Tq) {
      const int64_t page = t / P;
      const uint8_t* pb = page_base_a(c.store, unit, page);
      for (int j = lane; j < half; j += 32) {
        const int64_t f = (t - page * P) * half + j;
        const int64_t ab = f * m, rb = f * n;
        uint32_t av = pb[c.store.angle_off + (ab >> 3)], rv = pb[c.store.radius_off + (rb >> 3)];
        if ((ab & 7) + m > 8) av |= static_cast<uint32_t>(pb[c.store.angle_off + (ab >> 3) + 1]) << 8;
        if ((rb & 7) + n > 8) rv |= static_cast<uint32_t>(pb[c.store.radius_off + (rb >> 3) + 1]) << 8;
        const uint32_t a = (av >> (ab & 7)) & ((1u << m) - 1u), r = (rv >> (rb & 7)) & ((1u << n) - 1u);
        const float rhat = __fmul_rn(static_cast<float>(r), half_bits_to_f32(c.scales[unit * half + j]));
        const int ex = c.layout == PQB_HALF_SPLIT ? j : 2 * j;
        const int ey = c.layout == PQB_HALF_SPLIT ? j + half : 2 * j + 1;
        const float qx = q_dtype == PQB_F32 ? load1<PQB_F32>(q, ex) : (q_dtype == PQB_BF16 ? load1<PQB_BF16>(q, ex) : load1<PQB_F16>(q, ex));
        const float qy = q_dtype == PQB_F32 ? load1<PQB_F32>(q, ey) : (q_dtype == PQB_BF16 ? load1<PQB_BF16>(q, ey) : load1<PQB_F16>(q, ey));
        acc = fmaf(__fmul_rn(rhat, cs[a]), qx, acc);
        acc = fmaf(__fmul_rn(rhat, sn[a]), qy, acc);
      }
    } else if (c.res_cap > 0) {
      const float* kr = c.residual + (unit * c.res_cap + t % c.res_cap) * c.d;
      for (int e = lane; e < c.d; e += 32) {
        const float qe = q_dtype == PQB_F32 ? load1<PQB_F32>(q, e) : (q_dtype == PQB_BF16 ? load1<PQB_BF16>(q, e) : load1<PQB_F16>(q, e));
        acc = fmaf(kr[e], qe, acc);
      }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[t] = acc;
  }
}

// ------------------------------------------------------------ launchers

static unsigned grid_elems(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
}

int launch_to_polar(const void* x, const void* y, int dtype, int64_t n, void* r, void* t, cudaStream_t s) {
  if (n == 0) return PQB_OK;
  if (dtype == PQB_F64)
    to_polar_f64_kernel<<<grid_elems(n), 256, 0, s>>>(static_cast<const double*>(x), static_cast<const double*>(y),
                                                      n, static_cast<double*>(r), static_cast<double*>(t));
  else
    to_polar_f32_kernel<<<grid_elems(n), 256, 0, s>>>(static_cast<const float*>(x), static_cast<const float*>(y), n,
                                                      static_cast<float*>(r), static_cast<float*>(t));
  return PQB_OK;
}

int launch_quantize_angle(const void* theta, int dtype, int64_t n, int m, uint8_t* out, cudaStream_t s) {
  if (n == 0) return PQB_OK;
  if (dtype == PQB_F64)
    quantize_angle_f64_kernel<<<grid_elems(n), 256, 0, s>>>(static_cast<const double*>(theta), n, m, out);
  else
    quantize_angle_f32_kernel<<<grid_elems(n), 256, 0, s>>>(static_cast<const float*>(theta), n, m, out);
  return PQB_OK;
}

int launch_angle_grid(int m, double* out, cudaStream_t s) {
  angle_grid_kernel<<<1, 256, 0, s>>>(m, out);
  return PQB_OK;
}

int launch_quantize_radius(const void* radius, int dtype, const float* scale, int64_t n, int bits, uint8_t* out,
                           unsigned long long* clamped, cudaStream_t s) {
  if (n == 0) return PQB_OK;
  if (dtype == PQB_F64)
    quantize_radius_kernel<double><<<grid_elems(n), 256, 0, s>>>(static_cast<const double*>(radius), scale, n, bits,
                                                                 out, clamped);
  else
    quantize_radius_kernel<float><<<grid_elems(n), 256, 0, s>>>(static_cast<const float*>(radius), scale, n, bits,
                                                                out, clamped);
  return PQB_OK;
}

int launch_import(const pqb_store& st, int64_t unit, int d, int m, int n, int64_t T, const uint8_t* a,
                  const uint8_t* r, cudaStream_t s) {
  const int64_t half = d / 2;
  if (T == 0) return PQB_OK;
  if (a) import_kernel<<<grid_elems((T * half * m + 7) / 8), 256, 0, s>>>(st, unit, d / 2, m, st.angle_off, T, a);
  if (r) import_kernel<<<grid_elems((T * half * n + 7) / 8), 256, 0, s>>>(st, unit, d / 2, n, st.radius_off, T, r);
  return PQB_OK;
}

int launch_scores_direct(const pqb_cache& c, int64_t unit, const void* q, int q_dtype, int64_t tokens, float* out,
                         cudaStream_t s) {
  if (tokens == 0) return PQB_OK;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((tokens + 7) / 8, 148 * 8)));
  scores_direct_kernel<<<grid, 256, 0, s>>>(c, unit, q, q_dtype, tokens, out);
  return PQB_OK;
}

}  // namespace pqb
