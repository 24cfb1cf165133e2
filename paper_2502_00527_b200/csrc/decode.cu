// HP-2: fused LUT decode attention (sm_100a).
//
//   reference  build_angle_table / build_query_lut   lut_decode.py:63-104
//              qk_scores (LUT gather x dequantized radius) lut_decode.py:119-154
//              _residual_scores (exact fp32 dots)     lut_decode.py:107-116
//              attention_weights (softmax)            lut_decode.py:189-206
//              softmax . V  -- not in the reference; restated over values() (kv_cache.py:247-259)
//
// One CTA = one (unit, split) pair: a unit is one (layer, sequence, kv head)
// with G query heads (GQA).  The CTA builds the unit's query lookup table
//   P[j][a][g] = fl(fl(qx_gj * cos_a) + fl(qy_gj * sin_a))       (fp32, in smem)
// and the radius table rhat[j][r] = fl(s_j * r), then 8 warps stream 32-token
// tiles of the paged cache.  Each warp owns a private 2-stage ring in shared
// memory fed by the TMA bulk-copy engine (cp.async.bulk + mbarrier complete_tx):
// per tile the angle codes (32*8m B), radius codes (32*8n B) and values (8 KB bf16).
//   scoring  lane = token: acc_g = fl(acc_g + fl(P[j][A_j][g] * rhat[j][R_j])) over
//            j = 0..63 in order -- the reference's exact float32 operation sequence,
//            so quantized-token scores are bit-identical to qk_scores.
//   softmax  warp-level online softmax (tile max via shuffles, exp2).
//   P.V      lane = 4 value dims: o[g][:] += p_g(t) * V[t][:] over the tile.
// Warps merge in shared memory; splits merge in a small LSE-combine kernel.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace pqb {

constexpr int kNW = 8;      // compute warps per CTA
constexpr int kStages = 2;  // TMA ring depth per warp
constexpr int kTile = 32;   // tokens per tile (one per lane)
constexpr float kLog2e = 1.4426950408889634f;
constexpr double kPiD = 3.141592653589793115997963468544185161590576171875;  // == np.pi

PQB_DEV const uint8_t* page_base_c(const pqb_store& s, int64_t unit, int64_t page) {
  const int64_t pid = s.page_table ? static_cast<int64_t>(__ldg(s.page_table + unit * s.max_pages + page))
                                   : unit * s.max_pages + page;
  return s.pool + pid * s.page_bytes;
}

// angle_grid (polar_codec.py:224-233) then cos/sin cast to fp32 (lut_decode.py:69-73).
PQB_DEV void angle_unit(int m, int a, float& c, float& s) {
  const double hl = static_cast<double>(1 << (m - 1));
  const double g = __dsub_rn(__ddiv_rn(__dmul_rn(kPiD, static_cast<double>(a)), hl), kPiD);
  c = __double2float_rn(cos(g));
  s = __double2float_rn(sin(g));
}

template <int DT>
PQB_DEV float ldq(const void* q, int64_t i) { return load1<DT>(q, i); }

PQB_DEV float load_q(const void* q, int dt, int64_t i) {
  return dt == PQB_F32 ? ldq<PQB_F32>(q, i) : (dt == PQB_BF16 ? ldq<PQB_BF16>(q, i) : ldq<PQB_F16>(q, i));
}

// code j of a token whose 64*B code bits are in w[] (little-endian stream bits)
template <int B>
PQB_DEV uint32_t code_at(const uint32_t* w, int j) {
  const int bit = j * B, wi = bit >> 5, sh = bit & 31;
  uint32_t v;
  if (sh + B <= 32) v = w[wi] >> sh;
  else v = __funnelshift_r(w[wi], w[wi + 1], sh);
  return v & ((1u << B) - 1u);
}

template <int G>
PQB_DEV void lds_g(const float* p, float (&v)[G]) {
  if constexpr (G == 1) {
    v[0] = p[0];
  } else if constexpr (G == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < G; i += 4) {
      const float4 t = *reinterpret_cast<const float4*>(p + i);
      v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
    }
  }
}

// ------------------------------------------------------------------ epilogue
// Merge the NW warps' (m, l, o) states of one CTA; o element (g, k) of lane L is
// value dim dim_of(L, k).  Writes either the normalized output (single split) or
// the split's partial state.
struct EpiArgs {
  void* out;
  int out_dtype;
  float* part_ml;  // [n_units][n_splits][G][2]
  float* part_o;   // [n_units][n_splits][G][d]
  int n_splits;
};

PQB_DEV void store_out(void* out, int dt, int64_t idx, float v) {
  if (dt == PQB_F32) static_cast<float*>(out)[idx] = v;
  else static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
}

// ------------------------------------------------------------------ fast kernel

template <int G, int M, int N>
struct FastCfg {
  static constexpr int kLutFloats = 64 * (1 << M) * G;
  static constexpr int kRtabFloats = 64 * (1 << N);
  static constexpr int kABytes = kTile * 8 * M;
  static constexpr int kRBytes = kTile * 8 * N;
  static constexpr int kVBytes = kTile * 128 * 2;
  static constexpr int kStageBytes = kABytes + kRBytes + kVBytes;
  static constexpr int kHeadBytes = (kLutFloats + kRtabFloats + G * 128 + 64) * 4;
  static constexpr int kWarpBytes = kStages * kStageBytes + kTile * G * 4 + 64;
  static constexpr int kSmem = kHeadBytes + kNW * kWarpBytes + 128;
};

template <int G, int M, int N>
__global__ void __launch_bounds__(kNW * 32, 1)
    decode_fast_kernel(const pqb_cache c, const void* __restrict__ q, int q_dtype, float sm_scale_log2,
                       float* __restrict__ scores, int64_t scores_ld, EpiArgs ep, int tiles_per_split) {
  using Cfg = FastCfg<G, M, N>;
  extern __shared__ __align__(128) uint8_t smem[];
  float* lut = reinterpret_cast<float*>(smem);             // [64][2^M][G]
  float* rtab = lut + Cfg::kLutFloats;                      // [64][2^N]
  float* q_s = rtab + Cfg::kRtabFloats;                     // [G][128]
  float* cs_s = q_s + G * 128;                              // cos[16] | sin[16] | spare
  uint8_t* warp_area = smem + Cfg::kHeadBytes;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t unit = blockIdx.y;
  const int split = blockIdx.x;
  const int T = c.seq_lens[unit], Tq = c.quant_lens[unit];
  const int n_tiles = (T + kTile - 1) / kTile;
  const int tile_lo = split * tiles_per_split;
  const int tile_hi = min(n_tiles, tile_lo + tiles_per_split);
  const bool want_out = ep.out != nullptr;

  uint8_t* my_area = warp_area + warp * Cfg::kWarpBytes;
  float* pbuf = reinterpret_cast<float*>(my_area + kStages * Cfg::kStageBytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(my_area + kStages * Cfg::kStageBytes + kTile * G * 4);

  // ---- per-CTA setup: query rows, angle/radius tables, LUT, barriers
  for (int i = tid; i < G * 128; i += blockDim.x) q_s[i] = load_q(q, q_dtype, unit * G * 128 + i);
  if (tid < (1 << M)) angle_unit(M, tid, cs_s[tid], cs_s[16 + tid]);
  for (int i = tid; i < Cfg::kRtabFloats; i += blockDim.x) {
    const int j = i >> N, r = i & ((1 << N) - 1);
    rtab[i] = __fmul_rn(half_bits_to_f32(c.scales[unit * 64 + j]), static_cast<float>(r));
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  for (int i = tid; i < Cfg::kLutFloats; i += blockDim.x) {
    const int g = i % G, a = (i / G) & ((1 << M) - 1), j = i / (G * (1 << M));
    const int ex = c.layout == PQB_HALF_SPLIT ? j : 2 * j;
    const int ey = c.layout == PQB_HALF_SPLIT ? j + 64 : 2 * j + 1;
    lut[i] = __fadd_rn(__fmul_rn(q_s[g * 128 + ex], cs_s[a]), __fmul_rn(q_s[g * 128 + ey], cs_s[16 + a]));
  }
  __syncthreads();

  // ---- TMA producer (lane 0 of each warp feeds its own ring)
  const int64_t P = c.store.page_tokens;
  auto issue = [&](int tile, int s) {
    uint8_t* st = my_area + s * Cfg::kStageBytes;
    const int64_t tok0 = static_cast<int64_t>(tile) * kTile;
    const int64_t page = tok0 / P, in_page = tok0 - page * P;
    const uint8_t* pb = page_base_c(c.store, unit, page);
    const uint32_t bytes = Cfg::kABytes + Cfg::kRBytes + (want_out ? Cfg::kVBytes : 0);
    mbar_arrive_expect_tx(bar + s, bytes);
    bulk_g2s(st, pb + c.store.angle_off + in_page * 8 * M, Cfg::kABytes, bar + s);
    bulk_g2s(st + Cfg::kABytes, pb + c.store.radius_off + in_page * 8 * N, Cfg::kRBytes, bar + s);
    if (want_out) bulk_g2s(st + Cfg::kABytes + Cfg::kRBytes, pb + c.store.value_off + in_page * 256, Cfg::kVBytes,
                           bar + s);
  };
  const int first = tile_lo + warp;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s)
      if (first + s * kNW < tile_hi) issue(first + s * kNW, s);
  }
  __syncwarp();

  float m_run[G], l_run[G], o[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m_run[g] = -INFINITY;
    l_run[g] = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) o[g][k] = 0.0f;
  }

  int k_iter = 0;
  for (int tile = first; tile < tile_hi; tile += kNW, ++k_iter) {
    const int s = k_iter % kStages;
    mbar_wait(bar + s, (k_iter / kStages) & 1);
    const uint8_t* st = my_area + s * Cfg::kStageBytes;
    const int tok = tile * kTile + lane;
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g] = 0.0f;
    if (tok < Tq) {
      uint32_t wa[2 * M + 1], wr[2 * N + 1];
      const uint2* pa = reinterpret_cast<const uint2*>(st + lane * 8 * M);
      const uint2* pr = reinterpret_cast<const uint2*>(st + Cfg::kABytes + lane * 8 * N);
#pragma unroll
      for (int i = 0; i < M; ++i) { const uint2 v = pa[i]; wa[2 * i] = v.x; wa[2 * i + 1] = v.y; }
#pragma unroll
      for (int i = 0; i < N; ++i) { const uint2 v = pr[i]; wr[2 * i] = v.x; wr[2 * i + 1] = v.y; }
      wa[2 * M] = 0u;
      wr[2 * N] = 0u;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const uint32_t a = code_at<M>(wa, j), r = code_at<N>(wr, j);
        const float rh = rtab[j * (1 << N) + r];
        float pv[G];
        lds_g<G>(lut + (j * (1 << M) + a) * G, pv);
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = __fadd_rn(acc[g], __fmul_rn(pv[g], rh));
      }
    } else if (tok < T) {  // residual window: exact fp32 dot (lut_decode.py:107-116)
      const float* kr = c.residual + (unit * c.res_cap + tok % c.res_cap) * 128;
      for (int e = 0; e < 128; ++e) {
        const float kv = kr[e];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = fmaf(kv, q_s[g * 128 + e], acc[g]);
      }
    }
    if (scores != nullptr && tok < T) {
#pragma unroll
      for (int g = 0; g < G; ++g) scores[(unit * G + g) * scores_ld + tok] = acc[g];
    }
    if (want_out) {
      float alpha[G], p[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float x = tok < T ? acc[g] * sm_scale_log2 : -INFINITY;
        const float mt = warp_max(x);
        const float mn = fmaxf(m_run[g], mt);
        alpha[g] = exp2f(m_run[g] - mn);
        p[g] = exp2f(x - mn);
        l_run[g] = fmaf(l_run[g], alpha[g], p[g]);
        m_run[g] = mn;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) pbuf[lane * G + g] = p[g];
      __syncwarp();
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int k = 0; k < 4; ++k) o[g][k] *= alpha[g];
      const int nvalid = min(kTile, T - tile * kTile);
      const uint8_t* vs = st + Cfg::kABytes + Cfg::kRBytes;
#pragma unroll 4
      for (int t = 0; t < nvalid; ++t) {
        const uint2 vv = *reinterpret_cast<const uint2*>(vs + t * 256 + lane * 8);
        const float v0 = __uint_as_float(vv.x << 16), v1 = __uint_as_float(vv.x & 0xffff0000u);
        const float v2 = __uint_as_float(vv.y << 16), v3 = __uint_as_float(vv.y & 0xffff0000u);
        float pt[G];
        lds_g<G>(pbuf + t * G, pt);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          o[g][0] = fmaf(pt[g], v0, o[g][0]);
          o[g][1] = fmaf(pt[g], v1, o[g][1]);
          o[g][2] = fmaf(pt[g], v2, o[g][2]);
          o[g][3] = fmaf(pt[g], v3, o[g][3]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      const int nt = tile + kStages * kNW;
      if (nt < tile_hi) {
        fence_proxy_async_smem();
        issue(nt, s);
      }
    }
  }
  if (!want_out) return;

  // ---- merge warps (stage memory is free: every issued copy was consumed)
#pragma unroll
  for (int g = 0; g < G; ++g) l_run[g] = warp_sum(l_run[g]);
  __syncthreads();
  float* red = reinterpret_cast<float*>(warp_area);  // [NW][G][4 + 128]: m, l, pad, o
  float* mine = red + warp * G * 132;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) { mine[g * 132] = m_run[g]; mine[g * 132 + 1] = l_run[g]; }
    *reinterpret_cast<float4*>(mine + g * 132 + 4 + 4 * lane) = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
  }
  __syncthreads();
  for (int i = tid; i < G * 128; i += blockDim.x) {
    const int g = i >> 7, e = i & 127;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kNW; ++w) mx = fmaxf(mx, red[(w * G + g) * 132]);
    float L = 0.0f, O = 0.0f;
    if (mx != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kNW; ++w) {
        const float* rw = red + (w * G + g) * 132;
        const float sc = exp2f(rw[0] - mx);
        L = fmaf(rw[1], sc, L);
        O = fmaf(rw[4 + e], sc, O);
      }
    }
    if (ep.n_splits == 1) {
      store_out(ep.out, ep.out_dtype, (unit * G + g) * 128 + e, O / L);
    } else {
      const int64_t slot = (unit * ep.n_splits + split) * G + g;
      ep.part_o[slot * 128 + e] = O;
      if (e == 0) { ep.part_ml[2 * slot] = mx; ep.part_ml[2 * slot + 1] = L; }
    }
  }
}

// ------------------------------------------------------------------ generic kernel
// Any even d <= 256, m/n in 1..8, G <= 8, V f32 or bf16; codes and values read
// straight from global memory.  Same float32 scoring sequence as the fast kernel.

constexpr int kGenMaxG = 8, kGenMaxDpl = 8;

PQB_DEV uint32_t read_code(const uint8_t* region, int64_t flat, int b) {
  const int64_t bit = flat * b;
  const int64_t byte = bit >> 3;
  const int sh = static_cast<int>(bit & 7);
  uint32_t v = region[byte];
  if (sh + b > 8) v |= static_cast<uint32_t>(region[byte + 1]) << 8;
  return (v >> sh) & ((1u << b) - 1u);
}

__global__ void __launch_bounds__(256)
    decode_generic_kernel(const pqb_cache c, int G, const void* __restrict__ q, int q_dtype, float sm_scale_log2,
                          float* __restrict__ scores, int64_t scores_ld, EpiArgs ep, int tiles_per_split) {
  extern __shared__ __align__(16) float gsm[];
  const int d = c.d, half = d / 2, m = c.angle_bits, n = c.radius_bits;
  float* q_s = gsm;                 // [G][d]
  float* cs_s = q_s + G * d;        // cos[256] sin[256]
  float* sc_s = cs_s + 512;         // scales [half]
  float* pbuf_all = sc_s + half;    // [NW][32][G]
  float* red = pbuf_all + kNW * kTile * G;  // [NW][G][2 + d]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t unit = blockIdx.y;
  const int split = blockIdx.x;
  const int T = c.seq_lens[unit], Tq = c.quant_lens[unit];
  const int n_tiles = (T + kTile - 1) / kTile;
  const int tile_lo = split * tiles_per_split;
  const int tile_hi = min(n_tiles, tile_lo + tiles_per_split);
  const bool want_out = ep.out != nullptr;
  for (int i = tid; i < G * d; i += blockDim.x) q_s[i] = load_q(q, q_dtype, unit * G * d + i);
  for (int a = tid; a < (1 << m); a += blockDim.x) angle_unit(m, a, cs_s[a], cs_s[256 + a]);
  for (int j = tid; j < half; j += blockDim.x) sc_s[j] = half_bits_to_f32(c.scales[unit * half + j]);
  __syncthreads();
  float* pbuf = pbuf_all + warp * kTile * G;
  const int dpl = (d + 31) / 32;
  const int vb = c.store.value_dtype == PQB_F32 ? 4 : 2;
  const int64_t P = c.store.page_tokens;
  const int64_t a_page_bytes = P * half * m / 8, r_page_bytes = P * half * n / 8;
  (void)a_page_bytes; (void)r_page_bytes;
  float m_run[kGenMaxG], l_run[kGenMaxG], o[kGenMaxG][kGenMaxDpl];
  for (int g = 0; g < kGenMaxG; ++g) {
    m_run[g] = -INFINITY; l_run[g] = 0.0f;
    for (int k = 0; k < kGenMaxDpl; ++k) o[g][k] = 0.0f;
  }
  for (int tile = tile_lo + warp; tile < tile_hi; tile += kNW) {
    const int tok = tile * kTile + lane;
    float acc[kGenMaxG];
    for (int g = 0; g < kGenMaxG; ++g) acc[g] = 0.0f;
    if (tok < Tq) {
      const int64_t page = tok / P, in_page = tok - page * P;
      const uint8_t* pb = page_base_c(c.store, unit, page);
      const uint8_t* ra = pb + c.store.angle_off;
      const uint8_t* rr = pb + c.store.radius_off;
      for (int j = 0; j < half; ++j) {
        const int64_t flat = in_page * half + j;
        const uint32_t a = read_code(ra, flat, m), r = read_code(rr, flat, n);
        const float rh = __fmul_rn(sc_s[j], static_cast<float>(r));
        const float ca = cs_s[a], sa = cs_s[256 + a];
        const int ex = c.layout == PQB_HALF_SPLIT ? j : 2 * j;
        const int ey = c.layout == PQB_HALF_SPLIT ? j + half : 2 * j + 1;
        for (int g = 0; g < G; ++g) {
          const float pv = __fadd_rn(__fmul_rn(q_s[g * d + ex], ca), __fmul_rn(q_s[g * d + ey], sa));
          acc[g] = __fadd_rn(acc[g], __fmul_rn(pv, rh));
        }
      }
    } else if (tok < T) {
      const float* kr = c.residual + (unit * c.res_cap + tok % c.res_cap) * d;
      for (int e = 0; e < d; ++e) {
        const float kv = kr[e];
        for (int g = 0; g < G; ++g) acc[g] = fmaf(kv, q_s[g * d + e], acc[g]);
      }
    }
    if (scores != nullptr && tok < T)
      for (int g = 0; g < G; ++g) scores[(unit * G + g) * scores_ld + tok] = acc[g];
    if (!want_out) continue;
    float alpha[kGenMaxG];
    for (int g = 0; g < G; ++g) {
      const float x = tok < T ? acc[g] * sm_scale_log2 : -INFINITY;
      const float mn = fmaxf(m_run[g], warp_max(x));
      alpha[g] = exp2f(m_run[g] - mn);
      const float p = exp2f(x - mn);
      l_run[g] = fmaf(l_run[g], alpha[g], p);
      m_run[g] = mn;
      pbuf[lane * G + g] = p;
    }
    __syncwarp();
    for (int g = 0; g < G; ++g)
      for (int k = 0; k < kGenMaxDpl; ++k) o[g][k] *= alpha[g];
    const int nvalid = min(kTile, T - tile * kTile);
    for (int t = 0; t < nvalid; ++t) {
      const int64_t ta = static_cast<int64_t>(tile) * kTile + t;
      const int64_t page = ta / P, in_page = ta - page * P;
      const uint8_t* vrow = page_base_c(c.store, unit, page) + c.store.value_off + in_page * d * vb;
      for (int k = 0; k < dpl; ++k) {
        const int e = lane + 32 * k;
        if (e < d) {
          const float v = vb == 4 ? reinterpret_cast<const float*>(vrow)[e]
                                  : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(vrow)[e]);
          for (int g = 0; g < G; ++g) o[g][k] = fmaf(pbuf[t * G + g], v, o[g][k]);
        }
      }
    }
    __syncwarp();
  }
  if (!want_out) return;
  for (int g = 0; g < G; ++g) l_run[g] = warp_sum(l_run[g]);
  float* mine = red + warp * G * (2 + d);
  for (int g = 0; g < G; ++g) {
    if (lane == 0) { mine[g * (2 + d)] = m_run[g]; mine[g * (2 + d) + 1] = l_run[g]; }
    for (int k = 0; k < dpl; ++k) {
      const int e = lane + 32 * k;
      if (e < d) mine[g * (2 + d) + 2 + e] = o[g][k];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * d; i += blockDim.x) {
    const int g = i / d, e = i - g * d;
    float mx = -INFINITY;
    for (int w = 0; w < kNW; ++w) mx = fmaxf(mx, red[(w * G + g) * (2 + d)]);
    float L = 0.0f, O = 0.0f;
    if (mx != -INFINITY) {
      for (int w = 0; w < kNW; ++w) {
        const float* rw = red + (w * G + g) * (2 + d);
        const float sc = exp2f(rw[0] - mx);
        L = fmaf(rw[1], sc, L);
        O = fmaf(rw[2 + e], sc, O);
      }
    }
    if (ep.n_splits == 1) {
      store_out(ep.out, ep.out_dtype, (unit * G + g) * d + e, O / L);
    } else {
      const int64_t slot = (unit * ep.n_splits + split) * G + g;
      ep.part_o[slot * d + e] = O;
      if (e == 0) { ep.part_ml[2 * slot] = mx; ep.part_ml[2 * slot + 1] = L; }
    }
  }
}

// LSE combine of split partials: out = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M)
__global__ void combine_kernel(const float* __restrict__ part_ml, const float* __restrict__ part_o, int n_splits,
                               int G, int d, void* out, int out_dtype) {
  const int64_t unit = blockIdx.x;
  for (int i = threadIdx.x; i < G * d; i += blockDim.x) {
    const int g = i / d, e = i - g * d;
    float mx = -INFINITY;
    for (int s = 0; s < n_splits; ++s) mx = fmaxf(mx, part_ml[2 * ((unit * n_splits + s) * G + g)]);
    float L = 0.0f, O = 0.0f;
    for (int s = 0; s < n_splits; ++s) {
      const int64_t slot = (unit * n_splits + s) * G + g;
      const float ms = part_ml[2 * slot];
      if (ms == -INFINITY) continue;
      const float sc = exp2f(ms - mx);
      L = fmaf(part_ml[2 * slot + 1], sc, L);
      O = fmaf(part_o[slot * d + e], sc, O);
    }
    store_out(out, out_dtype, (unit * G + g) * d + e, O / L);
  }
}

// ------------------------------------------------------------------ host side

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

static int max_splits(int max_tokens) {
  const int tiles = (max_tokens + kTile - 1) / kTile;
  return std::max(1, std::min(64, tiles / (2 * kNW)));
}

static int choose_splits(int64_t n_units, int max_tokens) {
  const int64_t want = (2 * static_cast<int64_t>(num_sms()) + n_units - 1) / n_units;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, max_splits(max_tokens))));
}

int decode_splits(int64_t n_units, int max_tokens) { return choose_splits(n_units, max_tokens); }

size_t decode_workspace_bytes(int64_t n_units, int group, int max_tokens, int d) {
  const int s = max_splits(max_tokens);
  return static_cast<size_t>(n_units) * s * group * (2 + d) * sizeof(float) + 256;
}

template <int G, int M, int N>
static int launch_fast(const DecodeArgs& a, const EpiArgs& ep, int splits, int tps, cudaStream_t s) {
  using Cfg = FastCfg<G, M, N>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(decode_fast_kernel<G, M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmem) != cudaSuccess) {
      set_error("cudaFuncSetAttribute(smem=%d) failed", Cfg::kSmem);
      return PQB_ECUDA;
    }
    attr_set = true;
  }
  dim3 grid(splits, static_cast<unsigned>(a.n_units));
  decode_fast_kernel<G, M, N><<<grid, kNW * 32, Cfg::kSmem, s>>>(*a.cache, a.q, a.q_dtype, a.sm_scale * kLog2e,
                                                                 a.scores, a.scores_ld, ep, tps);
  return PQB_OK;
}

template <int G>
static int dispatch_fast_mn(const DecodeArgs& a, const EpiArgs& ep, int splits, int tps, cudaStream_t s,
                            bool& handled) {
  handled = true;
  const int mn = a.cache->angle_bits * 10 + a.cache->radius_bits;
  switch (mn) {
    case 44: return launch_fast<G, 4, 4>(a, ep, splits, tps, s);
    case 32: return launch_fast<G, 3, 2>(a, ep, splits, tps, s);
    case 22: return launch_fast<G, 2, 2>(a, ep, splits, tps, s);
    case 42: return launch_fast<G, 4, 2>(a, ep, splits, tps, s);
    case 24: return launch_fast<G, 2, 4>(a, ep, splits, tps, s);
    case 34: return launch_fast<G, 3, 4>(a, ep, splits, tps, s);
    default: handled = false; return PQB_OK;
  }
}

int launch_decode(const DecodeArgs& a, cudaStream_t s) {
  const pqb_cache& c = *a.cache;
  const int splits = a.splits > 0 ? std::min(a.splits, max_splits(a.max_tokens)) : choose_splits(a.n_units, a.max_tokens);
  const int tiles = (a.max_tokens + kTile - 1) / kTile;
  const int tps = (tiles + splits - 1) / splits;
  EpiArgs ep;
  ep.out = a.out;
  ep.out_dtype = a.out_dtype;
  ep.n_splits = splits;
  ep.part_ml = static_cast<float*>(a.workspace);
  ep.part_o = ep.part_ml + static_cast<int64_t>(a.n_units) * splits * a.group * 2;
  if (splits > 1 && a.out != nullptr) {
    const size_t need = static_cast<size_t>(a.n_units) * splits * a.group * (2 + c.d) * sizeof(float);
    if (a.workspace == nullptr || a.workspace_bytes < need) {
      set_error("decode workspace too small: need %zu bytes, got %zu", need, a.workspace_bytes);
      return PQB_EINVAL;
    }
  }
  const bool fast_ok = c.d == 128 && (a.out == nullptr || c.store.value_dtype == PQB_BF16) &&
                       (a.group == 1 || a.group == 4 || a.group == 8) && c.store.page_tokens % kTile == 0 &&
                       (c.store.angle_off % 16 == 0) && (c.store.radius_off % 16 == 0) &&
                       (c.store.value_off % 16 == 0 || a.out == nullptr) && (c.store.page_bytes % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(c.store.pool) % 16 == 0);
  int rc = PQB_OK;
  bool handled = false;
  if (fast_ok && !(a.flags & PQB_DECODE_FORCE_GENERIC)) {
    if (a.group == 4) rc = dispatch_fast_mn<4>(a, ep, splits, tps, s, handled);
    else if (a.group == 8) rc = dispatch_fast_mn<8>(a, ep, splits, tps, s, handled);
    else rc = dispatch_fast_mn<1>(a, ep, splits, tps, s, handled);
    if (rc != PQB_OK) return rc;
  }
  if (!handled) {
    if (c.d > 256 || a.group > kGenMaxG) {
      set_error("decode: d=%d group=%d unsupported (d <= 256, group <= %d)", c.d, a.group, kGenMaxG);
      return PQB_EUNSUPPORTED;
    }
    const size_t shm = sizeof(float) * (a.group * c.d + 512 + c.d / 2 + kNW * kTile * a.group +
                                        kNW * a.group * (2 + c.d));
    static size_t attr = 0;
    if (shm > 48 * 1024 && shm > attr) {
      cudaFuncSetAttribute(decode_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shm));
      attr = shm;
    }
    dim3 grid(splits, static_cast<unsigned>(a.n_units));
    decode_generic_kernel<<<grid, kNW * 32, shm, s>>>(c, a.group, a.q, a.q_dtype, a.sm_scale * kLog2e, a.scores,
                                                      a.scores_ld, ep, tps);
  }
  if (splits > 1 && a.out != nullptr && !(a.flags & PQB_DECODE_NO_COMBINE)) {
    combine_kernel<<<static_cast<unsigned>(a.n_units), 256, 0, s>>>(ep.part_ml, ep.part_o, splits, a.group, c.d,
                                                                    a.out, a.out_dtype);
  }
  return PQB_OK;
}

}  // namespace pqb
