// Accessor kernels for the reference API surface (tables, unpacked code views,
// stream export, value read-back, float64 softmax) and the seeded synthetic
// input generators used by tests and the benchmark.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace pqb {

constexpr double kPiD2 = 3.141592653589793115997963468544185161590576171875;

PQB_DEV const uint8_t* page_base_m(const pqb_store& s, int64_t unit, int64_t page) {
  const int64_t pid = s.page_table ? static_cast<int64_t>(s.page_table[unit * s.max_pages + page])
                                   : unit * s.max_pages + page;
  return s.pool + pid * s.page_bytes;
}

PQB_DEV void grid_cos_sin(int m, int a, float& c, float& s) {
  const double hl = static_cast<double>(1 << (m - 1));
  const double g = __dsub_rn(__ddiv_rn(__dmul_rn(kPiD2, static_cast<double>(a)), hl), kPiD2);
  c = __double2float_rn(cos(g));
  s = __double2float_rn(sin(g));
}

__global__ void angle_table_kernel(int m, float* c, float* s) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < (1 << m)) grid_cos_sin(m, a, c[a], s[a]);
}

// lut_decode.py:97-104: partial = qx[:,None]*cos + qy[:,None]*sin (no FMA)
__global__ void query_lut_kernel(const void* q, int q_dtype, int64_t n, int d, int layout, int m, float* out) {
  const int half = d / 2, L = 1 << m;
  const int64_t total = n * half * L;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int a = static_cast<int>(i % L);
    const int64_t rest = i / L;
    const int j = static_cast<int>(rest % half);
    const int64_t row = rest / half;
    const int ex = layout == PQB_HALF_SPLIT ? j : 2 * j;
    const int ey = layout == PQB_HALF_SPLIT ? j + half : 2 * j + 1;
    const int64_t qb = row * d;
    float qx, qy;
    if (q_dtype == PQB_F32) { qx = load1<PQB_F32>(q, qb + ex); qy = load1<PQB_F32>(q, qb + ey); }
    else if (q_dtype == PQB_BF16) { qx = load1<PQB_BF16>(q, qb + ex); qy = load1<PQB_BF16>(q, qb + ey); }
    else { qx = load1<PQB_F16>(q, qb + ex); qy = load1<PQB_F16>(q, qb + ey); }
    float c, s;
    grid_cos_sin(m, a, c, s);
    out[i] = __fadd_rn(__fmul_rn(qx, c), __fmul_rn(qy, s));
  }
}

// kv_cache.py:235-236: scales.as_compute()[:, None] * levels[None, :]
__global__ void radius_table_kernel(const uint16_t* scales, int64_t n_units, int half, int n_bits, float* out) {
  const int L = 1 << n_bits;
  const int64_t total = n_units * half * L;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i % L);
    out[i] = __fmul_rn(half_bits_to_f32(scales[i / L]), static_cast<float>(r));
  }
}

PQB_DEV uint32_t read_code_m(const uint8_t* region, int64_t flat, int b) {
  const int64_t bit = flat * b;
  const int64_t byte = bit >> 3;
  const int sh = static_cast<int>(bit & 7);
  uint32_t v = region[byte];
  if (sh + b > 8) v |= static_cast<uint32_t>(region[byte + 1]) << 8;
  return (v >> sh) & ((1u << b) - 1u);
}

__global__ void unpack_kernel(pqb_store st, int64_t unit, int half, int m, int n, int64_t T, uint8_t* ao,
                              uint8_t* ro) {
  const int64_t total = T * half;
  const int64_t P = st.page_tokens;
  for (int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; f < total;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = f / half;
    const int64_t page = t / P;
    const int64_t in_page_flat = f - page * P * half;
    const uint8_t* pb = page_base_m(st, unit, page);
    if (ao) ao[f] = static_cast<uint8_t>(read_code_m(pb + st.angle_off, in_page_flat, m));
    if (ro) ro[f] = static_cast<uint8_t>(read_code_m(pb + st.radius_off, in_page_flat, n));
  }
}

// Gather one stream: stream byte k lives in page k / R at offset k % R,
// R = page_tokens * half * b / 8 bytes per page.  The final byte keeps only the
// bits of the exported tokens (zero padding, polar_codec.py:103-104).
__global__ void export_kernel(pqb_store st, int64_t unit, int half, int b, int64_t region_off, int64_t T,
                              uint8_t* out) {
  const int64_t bits = T * half * b;
  const int64_t nbytes = (bits + 7) / 8;
  const int64_t R = static_cast<int64_t>(st.page_tokens) * half * b / 8;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nbytes;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t page = k / R;
    uint8_t v = page_base_m(st, unit, page)[region_off + (k - page * R)];
    if (k == nbytes - 1 && (bits & 7)) v &= static_cast<uint8_t>((1u << (bits & 7)) - 1u);
    out[k] = v;
  }
}

__global__ void read_values_kernel(pqb_store st, int64_t unit, int d, int64_t T, float* out) {
  const int64_t total = T * d;
  const int64_t P = st.page_tokens;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / d;
    const int e = static_cast<int>(i - t * d);
    const int64_t page = t / P;
    out[i] = load_value(st, page_base_m(st, unit, page), t - page * P, e, d);
  }
}

// lut_decode.py:200-206 in float64, one block.
__global__ void softmax_f64_kernel(const float* scores, int64_t n, double temperature, double* out) {
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double mx = -INFINITY;
  for (int64_t i = tid; i < n; i += blockDim.x) mx = fmax(mx, static_cast<double>(scores[i]) * temperature);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid < 32) {
    double v = tid < nw ? red[tid] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (tid == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  double sum = 0.0;
  for (int64_t i = tid; i < n; i += blockDim.x) {
    const double w = exp(static_cast<double>(scores[i]) * temperature - mx);
    out[i] = w;
    sum += w;
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  if (tid < 32) {
    double v = tid < nw ? red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (tid == 0) red[0] = v;
  }
  __syncthreads();
  const double total = red[0];
  for (int64_t i = tid; i < n; i += blockDim.x) out[i] = out[i] / total;
}

// ---------------------------------------------------------------- Philox4x32-10

PQB_DEV uint4 philox(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * ctr.x, hi0 = __umulhi(0xD2511F53u, ctr.x);
    const uint32_t lo1 = 0xCD9E8D57u * ctr.z, hi1 = __umulhi(0xCD9E8D57u, ctr.z);
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}

PQB_DEV float u01(uint32_t v) { return (static_cast<float>(v >> 8) + 0.5f) * (1.0f / 16777216.0f); }

PQB_DEV void store_any(void* out, int dt, int64_t i, float v) {
  if (dt == PQB_F32) static_cast<float*>(out)[i] = v;
  else if (dt == PQB_BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
  else static_cast<__half*>(out)[i] = __float2half_rn(v);
}

__global__ void synthetic_keys_kernel(uint64_t seed, int64_t T, int d, int layout, float mu, float sigma,
                                      uint64_t mask, float boost, void* out, int dt) {
  const int half = d / 2;
  const int64_t unit = blockIdx.y;
  const int64_t total = T * half;
  const uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 r = philox(make_uint4(static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32),
                                      static_cast<uint32_t>(unit), 0x5043u),
                           key);
    const int64_t t = i / half;
    const int j = static_cast<int>(i - t * half);
    const float mean = mu + ((j < 64 && ((mask >> j) & 1ull)) ? boost : 0.0f);
    const float z = sqrtf(-2.0f * logf(u01(r.x))) * cospif(2.0f * u01(r.y));
    const float rad = expf(mean + sigma * z);
    float sn, cs;
    sincospif(2.0f * u01(r.z), &sn, &cs);
    const int64_t rb = (unit * T + t) * d;
    const int ex = layout == PQB_HALF_SPLIT ? j : 2 * j;
    const int ey = layout == PQB_HALF_SPLIT ? j + half : 2 * j + 1;
    store_any(out, dt, rb + ex, rad * cs);
    store_any(out, dt, rb + ey, rad * sn);
  }
}

__global__ void synthetic_normal_kernel(uint64_t seed, int64_t count, void* out, int dt) {
  const uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; 4 * i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 r = philox(make_uint4(static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32), 0x4e4fu, 0u), key);
    const float m0 = sqrtf(-2.0f * logf(u01(r.x))), m1 = sqrtf(-2.0f * logf(u01(r.z)));
    float s0, c0, s1, c1;
    sincospif(2.0f * u01(r.y), &s0, &c0);
    sincospif(2.0f * u01(r.w), &s1, &c1);
    const float v[4] = {m0 * c0, m0 * s0, m1 * c1, m1 * s1};
    for (int k = 0; k < 4; ++k)
      if (4 * i + k < count) store_any(out, dt, 4 * i + k, v[k]);
  }
}

static unsigned grid_for(int64_t n) {
  return static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
}

int launch_angle_table(int m, float* c, float* s, cudaStream_t st) {
  angle_table_kernel<<<1, 256, 0, st>>>(m, c, s);
  return 0;
}
int launch_query_lut(const void* q, int q_dtype, int64_t n, int d, int layout, int m, float* out, cudaStream_t s) {
  const int64_t total = n * (d / 2) * (1 << m);
  if (total) query_lut_kernel<<<grid_for(total), 256, 0, s>>>(q, q_dtype, n, d, layout, m, out);
  return 0;
}
int launch_radius_table(const uint16_t* scales, int64_t n_units, int d, int n_bits, float* out, cudaStream_t s) {
  const int64_t total = n_units * (d / 2) * (1 << n_bits);
  if (total) radius_table_kernel<<<grid_for(total), 256, 0, s>>>(scales, n_units, d / 2, n_bits, out);
  return 0;
}
int launch_unpack(const pqb_store& st, int64_t unit, int d, int m, int n, int64_t T, uint8_t* a, uint8_t* r,
                  cudaStream_t s) {
  const int64_t total = T * (d / 2);
  if (total) unpack_kernel<<<grid_for(total), 256, 0, s>>>(st, unit, d / 2, m, n, T, a, r);
  return 0;
}
int launch_export(const pqb_store& st, int64_t unit, int d, int m, int n, int64_t T, uint8_t* a, uint8_t* r,
                  cudaStream_t s) {
  const int64_t half = d / 2;
  if (T == 0) return 0;
  if (a) export_kernel<<<grid_for((T * half * m + 7) / 8), 256, 0, s>>>(st, unit, d / 2, m, st.angle_off, T, a);
  if (r) export_kernel<<<grid_for((T * half * n + 7) / 8), 256, 0, s>>>(st, unit, d / 2, n, st.radius_off, T, r);
  return 0;
}
int launch_read_values(const pqb_store& st, int64_t unit, int d, int64_t T, float* out, cudaStream_t s) {
  if (T) read_values_kernel<<<grid_for(T * d), 256, 0, s>>>(st, unit, d, T, out);
  return 0;
}
int launch_softmax_f64(const float* scores, int64_t n, double temperature, double* out, cudaStream_t s) {
  softmax_f64_kernel<<<1, 1024, 0, s>>>(scores, n, temperature, out);
  return 0;
}
int launch_synthetic_keys(uint64_t seed, int64_t n_units, int64_t T, int d, int layout, float mu, float sigma,
                          uint64_t mask, float boost, void* out, int dtype, cudaStream_t s) {
  const int64_t per_unit = T * (d / 2);
  if (!per_unit || !n_units) return 0;
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((per_unit + 255) / 256, 1024)), static_cast<unsigned>(n_units));
  synthetic_keys_kernel<<<grid, 256, 0, s>>>(seed, T, d, layout, mu, sigma, mask, boost, out, dtype);
  return 0;
}
int launch_synthetic_normal(uint64_t seed, int64_t count, void* out, int dtype, cudaStream_t s) {
  if (count) synthetic_normal_kernel<<<grid_for((count + 3) / 4), 256, 0, s>>>(seed, count, out, dtype);
  return 0;
}

}  // namespace pqb

namespace pqb {

// dequantize_subvectors: rhat = fl(code * s); x = fl(rhat * cos[a]), y = fl(rhat * sin[a])
__global__ void dequantize_kernel(pqb_cache c, int64_t unit, int64_t T, float* out) {
  __shared__ float cs[256], sn[256];
  const int m = c.angle_bits, n = c.radius_bits, half = c.d / 2;
  for (int a = threadIdx.x; a < (1 << m); a += blockDim.x) grid_cos_sin(m, a, cs[a], sn[a]);
  __syncthreads();
  const int64_t total = T * half;
  const int64_t P = c.store.page_tokens;
  for (int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; f < total;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = f / half;
    const int j = static_cast<int>(f - t * half);
    const int64_t page = t / P;
    const uint8_t* pb = page_base_m(c.store, unit, page);
    const int64_t in_page = f - page * P * half;
    const uint32_t a = read_code_m(pb + c.store.angle_off, in_page, m);
    const uint32_t r = read_code_m(pb + c.store.radius_off, in_page, n);
    const float rhat = __fmul_rn(static_cast<float>(r), half_bits_to_f32(c.scales[unit * half + j]));
    const int ex = c.layout == PQB_HALF_SPLIT ? j : 2 * j;
    const int ey = c.layout == PQB_HALF_SPLIT ? j + half : 2 * j + 1;
    out[t * c.d + ex] = __fmul_rn(rhat, cs[a]);
    out[t * c.d + ey] = __fmul_rn(rhat, sn[a]);
  }
}

// _quantize_slices (baseline_quant.py:58-66) along a token row, then
// dequantize_uniform (:167): fl(fl(code * scale) + zp).  One warp per row.
__global__ void quantize_values_kernel(const void* vals, int dt, int64_t n, int d, int bits, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n) return;
  const float top = static_cast<float>((1 << bits) - 1);
  auto ld = [&](int e) {
    const int64_t i = row * d + e;
    return dt == PQB_F32 ? load1<PQB_F32>(vals, i) : (dt == PQB_BF16 ? load1<PQB_BF16>(vals, i) : load1<PQB_F16>(vals, i));
  };
  float mn = INFINITY, mx = -INFINITY;
  for (int e = lane; e < d; e += 32) {
    const float v = ld(e);
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const float scale = __fdiv_rn(__fsub_rn(mx, mn), top);
  for (int e = lane; e < d; e += 32) {
    float raw = scale == 0.0f ? 0.0f : rintf(__fdiv_rn(__fsub_rn(ld(e), mn), scale));
    raw = fminf(fmaxf(raw, 0.0f), top);
    out[row * d + e] = __fadd_rn(__fmul_rn(raw, scale), mn);
  }
}

int launch_dequantize(const pqb_cache& c, int64_t unit, int64_t T, float* out, cudaStream_t s) {
  const int64_t total = T * (c.d / 2);
  if (total) dequantize_kernel<<<grid_for(total), 256, 0, s>>>(c, unit, T, out);
  return 0;
}

// pqb_peer_wait: one thread bumps this layer's expected count, then spins
// (acquire, system scope) until every other rank's count has reached it.
__global__ void peer_wait_kernel(const uint32_t* flags, int n_peers, int rank, uint32_t* expect) {
  const uint32_t e = *expect + 1u;
  *expect = e;
  for (int k = 0; k < n_peers; ++k) {
    if (k == rank) continue;
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + k) : "memory");
      if (static_cast<int32_t>(v - e) >= 0) break;
      __nanosleep(100);
    }
  }
}

int launch_peer_wait(const uint32_t* flags, int n_peers, int rank, uint32_t* expect, cudaStream_t s) {
  peer_wait_kernel<<<1, 1, 0, s>>>(flags, n_peers, rank, expect);
  return 0;
}

int launch_quantize_values(const void* vals, int dt, int64_t n, int d, int bits, float* out, cudaStream_t s) {
  if (n) quantize_values_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(vals, dt, n, d, bits, out);
  return 0;
}

}  // namespace pqb

namespace pqb {

// pack_stream (polar_codec.py:98-110) of unpacked (T, d/2) code arrays of one
// unit, tokens [0, T), into the store: warp per 32 consecutive codes, b ballots.
__global__ void pack_codes_kernel(const uint8_t* __restrict__ ac, const uint8_t* __restrict__ rc, int64_t total,
                                  int half, int m, int n, pqb_store st, int64_t unit) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t P = st.page_tokens;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); 32 * g < total;
       g += warps) {
    const int64_t f = 32 * g + lane;
    const bool valid = f < total;
    const int64_t page = (32 * g) / (P * half);
    const int64_t g_in_page = g - page * P * half / 32;
    uint8_t* pb = const_cast<uint8_t*>(page_base_m(st, unit, page));
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const int b = pass == 0 ? m : n;
      const uint32_t code = valid ? ((pass == 0 ? ac[f] : rc[f]) & ((1u << b) - 1u)) : 0u;
      uint32_t* words = reinterpret_cast<uint32_t*>(pb + (pass == 0 ? st.angle_off : st.radius_off)) + g_in_page * b;
      for (int w = 0; w < b; ++w) {
        const int kb = 32 * w + lane;
        const uint32_t c = __shfl_sync(0xffffffffu, code, kb / b);
        const uint32_t word = __ballot_sync(0xffffffffu, (c >> (kb % b)) & 1u);
        if (lane == 0) words[w] = word;
      }
    }
  }
}

int launch_pack_codes(const uint8_t* a, const uint8_t* r, int64_t T, int d, int m, int n, const pqb_store& st,
                      int64_t unit, cudaStream_t s) {
  const int64_t total = T * (d / 2);
  if (total) pack_codes_kernel<<<grid_for((total + 31) / 32 * 32), 256, 0, s>>>(a, r, total, d / 2, m, n, st, unit);
  return 0;
}

}  // namespace pqb
