// HP-2: fused LUT decode attention (sm_100a).
//
//   reference  build_angle_table / build_query_lut    lut_decode.py:63-104
//              qk_scores (LUT gather x dequantized radius) lut_decode.py:119-154
//              _residual_scores (exact fp32 dots)      lut_decode.py:107-116
//              attention_weights (softmax)             lut_decode.py:189-206
//              softmax . V -- not in the reference; restated over values() (kv_cache.py:247-259)
//
// decode_fast_kernel<G, M, N, EXACT>  (d = 128, bf16 values; the hot kernel)
//   Persistent: one CTA per SM walks a balanced range of (unit, 32-token tile)
//   work items; a unit is one (layer, sequence, kv head) with G query heads.
//   Per unit segment the CTA builds the query lookup table in shared memory,
//       P[j][a][g] = fl(fl(qx_gj * cos_a) + fl(qy_gj * sin_a))      (lut_decode.py:97-104)
//   stored as float2 planes [j][g/2][a] (128-B rows: LDS.64 gathers are bank-
//   conflict free for any code pattern).  8 warps each own a private 2-stage ring
//   fed by the TMA bulk-copy engine (cp.async.bulk + mbarrier complete_tx): per
//   tile the angle codes, radius codes and the 8 KB bf16 value tile.
//   * scoring, lane = token.  Codes are masked into byte lanes once per word and
//     picked with one PRMT each; the radius becomes a float with PRMT + FADD
//     (magic 2^23).  EXACT: acc = fl(acc + fl(P * rhat)) in channel order -- the
//     reference's fp32 op sequence, bit-identical scores (qk_scores mode).
//     Fast (fused attention): LUT pre-scaled by s_j, acc = fma(P*s_j, r, acc).
//   * softmax: warp-level online softmax (tile max by shuffles, exp2).
//   * P.V on tensor cores: O^T[128 x 8] += V^T[128 x 32] . P^T[32 x 8] with
//     mma.sync m16n8k16 (bf16 in, fp32 accumulate).  V^T fragments come straight
//     from the tile with ldmatrix.trans (the page stores value rows XOR-swizzled,
//     value_offset(), so the 8 rows of a fragment hit 8 bank groups); P is split
//     into bf16 hi + lo (p - hi) so the product keeps ~2^-17 relative accuracy.
//   A CTA that covers a whole unit writes its output directly; otherwise it
//   writes a segment partial (m, l, o) and the last CTA to finish the unit
//   (atomic counter in the workspace) LSE-merges the partials -- one launch per
//   decode call.
#include "decode_common.cuh"

#include <cstdlib>
#include "kernels.h"

#include <algorithm>

namespace pqb {


// ------------------------------------------------------------------ fast kernel

template <int G, int M, int N, bool EXACT>
struct FastCfg {
  static constexpr int GP = G >= 2 ? G / 2 : 1;  // float2 planes
  static constexpr int kS = G >= 2 ? 3 : 2;      // log2(LUT entry bytes)
  static constexpr int kLutFloats = 64 * (1 << M) * G;
  static constexpr int kRtabFloats = EXACT ? 64 * (1 << N) : 0;
  static constexpr int kABytes = kTile * 8 * M;
  static constexpr int kRBytes = kTile * 8 * N;
  static constexpr int kVBytes = kTile * 256;
  static constexpr int kStageBytes = kABytes + kRBytes + kVBytes;
  static constexpr int kPBytes = 2 * 8 * kTile * 2;  // bf16 [hi/lo][8 queries][32 tokens]
  static constexpr int kHeadBytes = (kLutFloats + kRtabFloats + G * 128 + 64) * 4;
  static constexpr int kWarpBytes = kStages * kStageBytes + kPBytes;
  static constexpr int kSmem = kHeadBytes + kNW * kWarpBytes + 128;
  static_assert(kHeadBytes % 16 == 0 && kWarpBytes % 16 == 0, "alignment");
  static_assert(kNW * kStages * kStageBytes >= kNW * G * 132 * 4, "merge area");
};

template <int G, int M, int N, bool EXACT>
__global__ void __launch_bounds__(kNW * 32, 1)
    decode_fast_kernel(const pqb_cache c, const void* __restrict__ q, int q_dtype, float sm_scale_log2,
                       float* __restrict__ scores, int64_t scores_ld, EpiArgs ep, WorkSplit ws) {
  using Cfg = FastCfg<G, M, N, EXACT>;
  constexpr int GP = Cfg::GP;
  extern __shared__ __align__(128) uint8_t smem[];
  float* lut = reinterpret_cast<float*>(smem);  // [64][GP][2^M][2] (G>=2) or [64][2^M]
  float* rtab = lut + Cfg::kLutFloats;           // EXACT: [64][2^N]
  float* q_s = rtab + Cfg::kRtabFloats;          // [G][128]
  float* cs_s = q_s + G * 128;                   // cos[16] | sin[16] | spare
  uint8_t* warp_area = smem + Cfg::kHeadBytes;
  const uint8_t* lut_b = reinterpret_cast<const uint8_t*>(lut);
  const uint8_t* rtab_b = reinterpret_cast<const uint8_t*>(rtab);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool want_out = ep.out != nullptr;
  uint8_t* my_area = warp_area + warp * Cfg::kWarpBytes;
  uint8_t* pbuf = my_area + kStages * Cfg::kStageBytes;
  // mbarriers live outside the warp areas: the end-of-segment merge scratch
  // (red, G * 132 floats per warp) aliases the stage memory and, at G = 8,
  // would run over warp 0's barriers if they sat behind its stages
  __shared__ uint64_t s_bar[kNW][kStages];
  uint64_t* bar = s_bar[warp];
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  const int tpp = c.store.page_tokens / kTile;  // tiles per page
  const int64_t i_begin = static_cast<int64_t>(blockIdx.x) * ws.per_cta;
  const int64_t i_end = min(ws.items, i_begin + ws.per_cta);
  uint32_t k_iter = 0;  // per-warp ring position, continues across segments

  // lane constants for the tensor-core P.V
  const int qn = lane >> 2, t4 = lane & 3;  // fragment query column / pair
  // ldmatrix.trans row addresses in the grouped value layout (value_offset):
  // token 16 ks + 8 ((lane >> 4) & 1) + (lane & 7), chunk 2 mt + ((lane >> 3) & 1)
  const uint32_t ld_row = static_cast<uint32_t>(((lane >> 4) & 1) * 2048 + (lane & 7) * 128);
  const uint32_t ld_chunk = static_cast<uint32_t>((((lane >> 3) & 1) ^ (lane & 7)) << 4);

  for (int64_t seg = i_begin; seg < i_end;) {
    const int64_t unit = seg / ws.tiles_max;
    const int t_lo = static_cast<int>(seg - unit * ws.tiles_max);
    const int64_t seg_end = min(i_end, (unit + 1) * ws.tiles_max);
    seg = seg_end;
    const int T = c.seq_lens[unit], Tq = c.quant_lens[unit];
    const int n_tiles = (T + kTile - 1) / kTile;
    const int t_hi = min(static_cast<int>(seg_end - unit * ws.tiles_max), n_tiles);

    __syncthreads();  // previous segment finished with LUT / merge area
    const int first = t_lo + warp;
    // ---- unit setup: query rows, angle table, LUT (+ radius table)
    for (int i = tid; i < G * 128; i += blockDim.x) q_s[i] = load_q(q, q_dtype, unit * G * 128 + i);
    if (tid < (1 << M)) angle_unit(M, tid, cs_s[tid], cs_s[16 + tid]);
    if constexpr (EXACT) {
      for (int i = tid; i < Cfg::kRtabFloats; i += blockDim.x) {
        const int j = i >> N, r = i & ((1 << N) - 1);
        rtab[i] = __fmul_rn(half_bits_to_f32(c.scales[unit * 64 + j]), static_cast<float>(r));
      }
    }
    __syncthreads();
    for (int i = tid; i < Cfg::kLutFloats; i += blockDim.x) {
      // i = ((j*GP + gp) * 2^M + a) * 2 + h   (G >= 2)   |   j * 2^M + a   (G == 1)
      int j, a, g;
      if constexpr (G >= 2) {
        const int h = i & 1, rest = i >> 1;
        a = rest & ((1 << M) - 1);
        const int jg = rest >> M;
        j = jg / GP;
        g = (jg % GP) * 2 + h;
      } else {
        a = i & ((1 << M) - 1);
        j = i >> M;
        g = 0;
      }
      const int ex = c.layout == PQB_HALF_SPLIT ? j : 2 * j;
      const int ey = c.layout == PQB_HALF_SPLIT ? j + 64 : 2 * j + 1;
      float v = __fadd_rn(__fmul_rn(q_s[g * 128 + ex], cs_s[a]), __fmul_rn(q_s[g * 128 + ey], cs_s[16 + a]));
      if constexpr (!EXACT) v = __fmul_rn(v, half_bits_to_f32(c.scales[unit * 64 + j]));
      lut[i] = v;
    }
    __syncthreads();

    // ---- lane 0 fills this warp's ring with its first tiles (after the LUT
    // build: measured faster than overlapping it, scripts/ab_probe.sh)
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < kStages; ++s) {
        const int tile = first + s * kNW;
        if (tile < t_hi) {
          fence_proxy_async_smem();
          const uint32_t sl = (k_iter + s) % kStages;
          issue_tile<M, N>(my_area + sl * Cfg::kStageBytes, c.store, page_base_c(c.store, unit, tile / tpp), tile,
                           tpp, want_out, bar + sl);
        }
      }
    }
    float m_run[G], l_run[G];
    float d[8][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m_run[g] = -INFINITY;
      l_run[g] = 0.0f;
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int k = 0; k < 4; ++k) d[mt][k] = 0.0f;

    for (int tile = first; tile < t_hi; tile += kNW, ++k_iter) {
      const uint32_t s = k_iter % kStages;
      const int nt = tile + kStages * kNW;  // the tile this stage is refilled with
      mbar_wait(bar + s, (k_iter / kStages) & 1);
      const uint8_t* st = my_area + s * Cfg::kStageBytes;
      const int tok = tile * kTile + lane;
      float acc[G];
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g] = 0.0f;
      if (tok < Tq) {
        uint32_t wa[2 * M + 1], wr[2 * N + 1];
        load_token_codes<M>(st + lane * 8 * M, lane, wa);
        load_token_codes<N>(st + Cfg::kABytes + lane * 8 * N, lane, wr);
        wa[2 * M] = 0u;
        wr[2 * N] = 0u;
        CodeLanes<M, Cfg::kS> ca;
        ca.init(wa);
        if constexpr (EXACT) {
          CodeLanes<N, 2> cr;
          cr.init(wr);
#pragma unroll
          for (int j = 0; j < 64; ++j) {
            const uint32_t aoff = ca.get(wa, j);
            const float rh = *reinterpret_cast<const float*>(rtab_b + (j << (N + 2)) + cr.get(wr, j));
            float pv[G];
            if constexpr (G >= 2) {
#pragma unroll
              for (int gp = 0; gp < GP; ++gp) {
                const float2 t = *reinterpret_cast<const float2*>(lut_b + (((j * GP + gp) << M) << 3) + aoff);
                pv[2 * gp] = t.x;
                pv[2 * gp + 1] = t.y;
              }
            } else {
              pv[0] = *reinterpret_cast<const float*>(lut_b + ((j << M) << 2) + aoff);
            }
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = __fadd_rn(acc[g], __fmul_rn(pv[g], rh));
          }
        } else {
          CodeLanes<N, 0> cr;
          cr.init(wr);
#pragma unroll
          for (int j = 0; j < 64; ++j) {
            const uint32_t aoff = ca.get(wa, j);
            const float rf = cr.as_float(wr, j);
            if constexpr (G >= 2) {
#pragma unroll
              for (int gp = 0; gp < GP; ++gp) {
                const float2 t = *reinterpret_cast<const float2*>(lut_b + (((j * GP + gp) << M) << 3) + aoff);
                acc[2 * gp] = fmaf(t.x, rf, acc[2 * gp]);
                acc[2 * gp + 1] = fmaf(t.y, rf, acc[2 * gp + 1]);
              }
            } else {
              const float t = *reinterpret_cast<const float*>(lut_b + ((j << M) << 2) + aoff);
              acc[0] = fmaf(t, rf, acc[0]);
            }
          }
        }
      } else if (tok < T && c.res_cap > 0) {  // residual window: fp32 dot (lut_decode.py:107-116)
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
        // ---- online softmax (per query, warp-uniform running max)
        float alpha[G];
        bool rescale = false;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float x = tok < T ? acc[g] * sm_scale_log2 : -INFINITY;
          const float mn = fmaxf(m_run[g], warp_max(x));
          alpha[g] = exp2f(m_run[g] - mn);
          rescale |= mn != m_run[g];
          const float p = exp2f(x - mn);
          l_run[g] = fmaf(l_run[g], alpha[g], p);
          m_run[g] = mn;
          const __nv_bfloat16 hi = __float2bfloat16_rn(p);
          const __nv_bfloat16 lo = __float2bfloat16_rn(p - __bfloat162float(hi));
          reinterpret_cast<__nv_bfloat16*>(pbuf)[g * kTile + lane] = hi;
          reinterpret_cast<__nv_bfloat16*>(pbuf)[(8 + g) * kTile + lane] = lo;
        }
        if (rescale) {  // warp-uniform
          float a0 = 1.0f, a1 = 1.0f;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            if (g == 2 * t4) a0 = alpha[g];
            if (g == 2 * t4 + 1) a1 = alpha[g];
          }
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            d[mt][0] *= a0;
            d[mt][1] *= a1;
            d[mt][2] *= a0;
            d[mt][3] *= a1;
          }
        }
        __syncwarp();
        // ---- P.V on tensor cores: B = P^T fragments (hi, lo) for 2 k-steps
        uint32_t b[2][2][2];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int pl = 0; pl < 2; ++pl) {
            if (qn < G) {
              const uint32_t* row = reinterpret_cast<const uint32_t*>(pbuf + ((pl * 8 + qn) * kTile + 16 * ks) * 2);
              b[ks][pl][0] = row[t4];
              b[ks][pl][1] = row[t4 + 4];
            } else {
              b[ks][pl][0] = b[ks][pl][1] = 0u;
            }
          }
        const uint32_t vbase = smem_u32(st + Cfg::kABytes + Cfg::kRBytes) + ld_row;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_trans(vbase + ks * 4096 + (mt >> 2) * 1024 + (ld_chunk ^ ((mt & 3) << 5)), a0, a1, a2, a3);
            mma_bf16(d[mt], a0, a1, a2, a3, b[ks][0][0], b[ks][0][1]);
            mma_bf16(d[mt], a0, a1, a2, a3, b[ks][1][0], b[ks][1][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0 && nt < t_hi) {
        fence_proxy_async_smem();
        issue_tile<M, N>(my_area + s * Cfg::kStageBytes, c.store, page_base_c(c.store, unit, nt / tpp), nt, tpp,
                         want_out, bar + s);
      }
    }
    if (!want_out) continue;

    // ---- merge the warps of this segment (stage memory is idle now)
#pragma unroll
    for (int g = 0; g < G; ++g) l_run[g] = warp_sum(l_run[g]);
    __syncthreads();
    float* red = reinterpret_cast<float*>(warp_area);  // [NW][G][132]: m, l, pad, o[128]
    float* mine = red + warp * G * 132;
    if (lane == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        mine[g * 132] = m_run[g];
        mine[g * 132 + 1] = l_run[g];
      }
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int dim = 16 * mt + qn;
      if (2 * t4 < G) {
        mine[(2 * t4) * 132 + 4 + dim] = d[mt][0];
        mine[(2 * t4) * 132 + 4 + dim + 8] = d[mt][2];
      }
      if (2 * t4 + 1 < G) {
        mine[(2 * t4 + 1) * 132 + 4 + dim] = d[mt][1];
        mine[(2 * t4 + 1) * 132 + 4 + dim + 8] = d[mt][3];
      }
    }
    __shared__ int s_last;
    finish_segment<G>(ep, ws, unit, red, &s_last, tid, blockDim.x);
  }
}

// Stand-alone split merge after a DQ launch that wrote partials only
// (PQB_DECODE_MERGE_KERNEL): one CTA per (unit, query), thread = output
// element, launched with programmatic dependent launch so its CTAs are
// resident and waiting when the decode grid drains.  Same LSE merge as
// merge_slots (one element per thread instead of G * 128 / nthreads).
__global__ void __launch_bounds__(128) merge_split_kernel(EpiArgs ep, WorkSplit ws) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t unit = blockIdx.x / ep.group;
  const int g = static_cast<int>(blockIdx.x - unit * ep.group), e = threadIdx.x;
  const int nseg = static_cast<int>(last_cta(ws, unit) - first_cta(ws, unit) + 1);
  constexpr int kB = 8;
  float mx = -INFINITY, L = 0.0f, O = 0.0f;
  for (int s0 = 0; s0 < nseg; s0 += kB) {
    float ms[kB], ls[kB], os[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const bool ok = s0 + k < nseg;
      const int64_t sl = (unit * ep.slots + min(s0 + k, nseg - 1)) * ep.group + g;
      const float m = __ldcg(ep.part_ml + 2 * sl), l = __ldcg(ep.part_ml + 2 * sl + 1);
      const float o = __ldcg(ep.part_o + sl * 128 + e);
      ms[k] = ok ? m : -INFINITY;
      ls[k] = ok ? l : 0.0f;
      os[k] = ok ? o : 0.0f;
    }
    float bm = mx;
#pragma unroll
    for (int k = 0; k < kB; ++k) bm = fmaxf(bm, ms[k]);
    if (bm == -INFINITY) continue;
    const float r = exp2f(mx - bm);
    L *= r;
    O *= r;
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      if (ms[k] == -INFINITY) continue;
      const float sc = exp2f(ms[k] - bm);
      L = fmaf(ls[k], sc, L);
      O = fmaf(os[k], sc, O);
    }
    mx = bm;
  }
  emit(ep, unit, g, e, O / L);
}

static int launch_merge_split(const EpiArgs& ep, const WorkSplit& ws, int64_t n_units, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n_units * ep.group));
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, merge_split_kernel, ep, ws) != cudaSuccess) {
    set_error("merge_split launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return PQB_ECUDA;
  }
  return PQB_OK;
}

// ------------------------------------------------------------------ generic kernel
// Any even d <= 256, m/n in 1..8, G <= 8, V f32 or bf16; codes and values read
// straight from global memory.  Exact fp32 scoring sequence (as EXACT above).

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
  const int64_t P = c.store.page_tokens;
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
    } else if (tok < T && c.res_cap > 0) {
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
      const uint8_t* pg = page_base_c(c.store, unit, page);
      for (int k = 0; k < dpl; ++k) {
        const int e = lane + 32 * k;
        if (e < d) {
          const float v = load_value(c.store, pg, in_page, e, d);
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
    if (ep.slots == 1) {
      store_out(ep.out, ep.out_dtype, (unit * G + g) * d + e, O / L);
    } else {
      const int64_t slot = (unit * ep.slots + split) * G + g;
      ep.part_o[slot * d + e] = O;
      if (e == 0) { ep.part_ml[2 * slot] = mx; ep.part_ml[2 * slot + 1] = L; }
    }
  }
}

// LSE combine of generic-kernel split partials.
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

static int num_sms() { return device_sms(); }

constexpr int kMaxCtas = 256;  // bound used to size the partial-slot workspace

static int tiles_of(int max_tokens) { return (max_tokens + kTile - 1) / kTile; }

// generic kernel: (unit, split) grid
static int max_splits(int max_tokens) { return std::max(1, std::min(64, tiles_of(max_tokens) / (2 * kNW))); }

static int choose_splits(int64_t n_units, int max_tokens) {
  const int64_t want = (2 * static_cast<int64_t>(num_sms()) + n_units - 1) / n_units;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, max_splits(max_tokens))));
}

// fast kernel: persistent split over units x tiles
static WorkSplit make_split(int64_t n_units, int max_tokens, int ctas) {
  WorkSplit w;
  w.balanced = 0;
  w.n_cta = 0;
  w.cluster = 0;
  w.tiles_max = tiles_of(max_tokens);
  w.items = n_units * w.tiles_max;
  const int64_t c = std::max<int64_t>(1, std::min<int64_t>(ctas, w.items));
  w.per_cta = (w.items + c - 1) / c;
  // Short launches (few tiles per CTA): cut every unit into the same number k
  // of CTA ranges so no CTA straddles two units -- a straddling CTA pays a
  // second unit setup and adds a merge segment, which dominates when a CTA
  // only has a handful of tiles (configs[0]: 12.6 vs 18.9 us per launch,
  // scripts/small_probe.py).
  if (w.per_cta <= 64 && w.tiles_max >= 2 * w.per_cta) {
    const int64_t k = w.tiles_max / w.per_cta;
    w.per_cta = (w.tiles_max + k - 1) / k;
  }
  return w;
}

static int fast_slots(int64_t n_units, int max_tokens) {
  // CTAs touching one unit <= ceil(tiles_max / per_cta) + 1 with per_cta >= items / kMaxCtas;
  // a balanced split's ranges are >= per_cta / 2 (make_split_balanced), hence 2x + 2
  const int tm = tiles_of(max_tokens);
  const int64_t per_min = std::max<int64_t>(1, (n_units * tm) / kMaxCtas);
  return static_cast<int>(std::min<int64_t>(tm, 2 * ((tm + per_min - 1) / per_min) + 2));
}

// Segment cost in tiles for the DQ kernel's balanced split: a CTA range that
// crosses into a second unit pays a second unit setup and a merge epilogue
// (launch traces: ~4-8 us, i.e. ~20-35 tiles at one CTA's share of HBM), so it
// gets that many fewer tiles and CTAs finish together.  PQB_SPLIT_COST
// overrides (0: uniform ranges).
static int split_cost() {
  static const int c = [] {
    const char* e = std::getenv("PQB_SPLIT_COST");
    return e ? std::atoi(e) : 24;
  }();
  return c;
}

// Greedy balanced ranges: CTA ranges of budget B tiles, minus `cost` per unit
// segment; a range that would cross a unit boundary with less than its second
// segment's cost left stops at the boundary.  B is the smallest budget whose
// greedy cover needs no more than `ctas` CTAs.  Uniform ranges are kept when
// the cost is small against a CTA's share (short launches, many segments) or
// the item space does not fit the table.
static WorkSplit make_split_balanced(int64_t n_units, int max_tokens, int ctas) {
  WorkSplit w = make_split(n_units, max_tokens, ctas);
  const int cost = split_cost();
  const int64_t tm = w.tiles_max, items = w.items;
  if (cost <= 0 || ctas > kSplitMaxCtas || w.per_cta < 8 * cost || items >= (int64_t(1) << 31)) return w;
  auto cover = [&](int64_t B, int32_t* starts) -> int {
    int64_t s = 0;
    int c = 0;
    while (s < items && c <= ctas) {
      if (starts && c < ctas) starts[c] = static_cast<int32_t>(s);
      const int64_t bnd = (s / tm + 1) * tm;
      int64_t e = s + (B - cost);
      if (e > bnd) {
        const int64_t e2 = s + (B - 2 * cost);
        e = e2 > bnd ? e2 : bnd;
      }
      s = std::min(e, items);
      ++c;
    }
    return c;
  };
  int64_t lo = w.per_cta / 2 + 2 * cost, hi = w.per_cta + 2 * cost;  // hi always covers in <= ctas
  if (cover(lo, nullptr) <= ctas) hi = lo;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (cover(mid, nullptr) <= ctas) hi = mid;
    else lo = mid;
  }
  const int n = cover(hi, w.starts);
  if (n > ctas) return w;
  w.starts[n] = static_cast<int32_t>(items);
  w.n_cta = n;
  w.balanced = 1;
  w.per_cta = hi;
  return w;
}

int decode_splits(int64_t n_units, int max_tokens) { return choose_splits(n_units, max_tokens); }

// workspace: [counters: n_units ints, 256-B rounded][partials: n_units * slots * G * (2 + d) floats]
// The counter region sits at a fixed offset for a given n_units, is zero before
// the first call and is left zeroed by every fused call.
// one counter per unit (split merge) + the grid-done counter of peer mode
static size_t counter_bytes(int64_t n_units) {
  return (static_cast<size_t>(n_units + 1) * sizeof(int) + 255) / 256 * 256;
}

static size_t partial_bytes(int64_t n_units, int group, int max_tokens, int d) {
  const int s = std::max(max_splits(max_tokens), fast_slots(n_units, max_tokens));
  return static_cast<size_t>(n_units) * s * group * (2 + d) * sizeof(float);
}

size_t decode_workspace_bytes(int64_t n_units, int group, int max_tokens, int d) {
  return counter_bytes(n_units) + partial_bytes(n_units, group, max_tokens, d) + 256;
}

// Work split + epilogue arguments shared by the LUT and DQ fast kernels.
static int fast_setup(const DecodeArgs& a, EpiArgs& ep, WorkSplit& ws, int& grid, bool balanced = false) {
  static const int ctas_env = [] {  // PQB_DQ_CTAS: persistent-grid CTA count override (A/B of grid sizes)
    const char* e = std::getenv("PQB_DQ_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  const int ctas = a.splits > 0 ? std::min(a.splits, kMaxCtas)
                                : std::min(ctas_env > 0 ? ctas_env : num_sms(), kMaxCtas);
  ws = balanced ? make_split_balanced(a.n_units, a.max_tokens, ctas) : make_split(a.n_units, a.max_tokens, ctas);
  grid = ws.balanced ? ws.n_cta : static_cast<int>((ws.items + ws.per_cta - 1) / ws.per_cta);
  ep.out = a.out;
  ep.out_dtype = a.out_dtype;
  ep.slots = fast_slots(a.n_units, a.max_tokens);
  ep.counters = static_cast<int*>(a.workspace);
  ep.part_ml = reinterpret_cast<float*>(static_cast<uint8_t*>(a.workspace) + counter_bytes(a.n_units));
  ep.part_o = ep.part_ml + a.n_units * ep.slots * a.group * 2;
  ep.merge = !(a.flags & PQB_DECODE_NO_COMBINE);
  ep.group = a.group;
  ep.peer_mode = a.peer != nullptr;
  if (a.peer) ep.peer = *a.peer;
  if (a.out != nullptr) {
    const size_t need = decode_workspace_bytes(a.n_units, a.group, a.max_tokens, 128);
    if (a.workspace == nullptr || a.workspace_bytes < need) {
      set_error("decode workspace too small: need %zu bytes, got %zu", need, a.workspace_bytes);
      return PQB_EINVAL;
    }
  }
  return PQB_OK;
}

template <int G, int M, int N, bool EXACT>
static int launch_fast(const DecodeArgs& a, cudaStream_t s) {
  using Cfg = FastCfg<G, M, N, EXACT>;
  static std::atomic<uint64_t> attr_done{0};
  const int arc = once_per_device(attr_done, [] {
    if (cudaFuncSetAttribute(decode_fast_kernel<G, M, N, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmem) != cudaSuccess) {
      set_error("cudaFuncSetAttribute(smem=%d) failed", Cfg::kSmem);
      return PQB_ECUDA;
    }
    return PQB_OK;
  });
  if (arc != PQB_OK) return arc;
  EpiArgs ep;
  WorkSplit ws;
  int grid = 0;
  const int rc = fast_setup(a, ep, ws, grid);
  if (rc != PQB_OK) return rc;
  decode_fast_kernel<G, M, N, EXACT><<<grid, kNW * 32, Cfg::kSmem, s>>>(
      *a.cache, a.q, a.q_dtype, a.sm_scale * kLog2e, a.scores, a.scores_ld, ep, ws);
  return PQB_OK;
}

// Scoring variant for the fused (output-only) call.  G in {4, 8}: the product-
// table gather + tensor-core contraction of decode_dq.cu (A/B on B200,
// configs[1] launch: 0.87 vs 0.80 of HBM peak at G = 4, 0.66 vs 0.45 at G = 8;
// the LUT gather is shared-memory bound).  Scores requested, G = 1 or
// PQB_DECODE_LUT: the LUT kernel (bit-exact qk_scores sequence).
// Scores-only calls with PQB_DECODE_DQ (G in {4, 8}) take the DQ kernel's
// scores mode: qk_scores within the stated tolerance instead of bit-identical.
static bool use_dq(const DecodeArgs& a) {
  if (a.group != 4 && a.group != 8) return false;
  if (a.scores != nullptr) return a.out == nullptr && (a.flags & PQB_DECODE_DQ) && !(a.flags & PQB_DECODE_LUT);
  if (a.out == nullptr || (a.flags & PQB_DECODE_LUT)) return false;
  return true;
}

// Partials only in the decode grid and the split merge in a separate PDL launch
// (one CTA per (unit, query), all in parallel) instead of the last CTA of each
// unit merging G x 128 outputs serially in the launch's tail, when units are
// cut into many segments (> 8: configs[0] 11.8 -> 9.8 us per launch,
// profiles/r01/small_launch.md) or for G = 8 from 16K tokens (configs[3] +2.5%,
// scripts/g8_scaling.py); G = 4 long launches and short G = 8 ones measured
// equal or slightly slower.  PQB_DECODE_MERGE_KERNEL forces it.
static bool separate_merge(int flags, int group, int max_tokens, const WorkSplit& ws) {
  const int64_t seg_max = (ws.tiles_max + ws.per_cta - 1) / ws.per_cta + 1;
  if (flags & PQB_DECODE_MERGE_INKERNEL) return false;
  return (flags & PQB_DECODE_MERGE_KERNEL) || seg_max > 8 || (group == 8 && max_tokens >= 16384);
}

// Thread-block-cluster path of the DQ kernel: when the units of a launch fill
// the GPU with k = 2, 4 or 8 CTAs each (n_units * k >= 80 % of the SMs, no
// more than the SMs), each unit is cut into k equal ranges run by one cluster,
// and the split merge goes through distributed shared memory (finish_cluster):
// no CTA straddles two units, no partials in global memory, no merge launch.
// configs[3] (32 units of G = 8): k = 4.  0 when the call or the device
// (resident clusters) does not qualify.
static int dq_cluster_size(int64_t n_units, int group, int max_tokens, int flags, const pqb_cache* c,
                           bool peer, bool scores) {
  (void)peer;  // peer mode works too: finish_cluster stores through emit(), peer_publish runs after it
  if ((group != 4 && group != 8) || scores) return 0;
  if (flags & (PQB_DECODE_MERGE_KERNEL | PQB_DECODE_MERGE_INKERNEL | PQB_DECODE_NO_CLUSTER |
               PQB_DECODE_LUT | PQB_DECODE_DQ_LINEAR | PQB_DECODE_PROBE_MEM | PQB_DECODE_PROBE_COMPUTE))
    return 0;
  if (c != nullptr && (c->angle_bits != 4 || c->radius_bits != 4 || c->store.value_dtype != PQB_BF16)) return 0;
  const int sms = num_sms(), tm = tiles_of(max_tokens);
  static const int min_fill = [] {  // percent of the SMs the clusters must fill (PQB_CLUSTER_MIN_FILL, A/B)
    const char* e = std::getenv("PQB_CLUSTER_MIN_FILL");
    return e ? std::atoi(e) : 80;
  }();
  for (int k : {8, 4, 2}) {
    // short launches (<= 32 tiles per CTA: latency-bound, e.g. configs[0]) take the
    // cluster path from 40 % of the SMs: one launch instead of decode + merge
    // (configs[0] 14.4-15.6 -> 12.7 us per single-layer graph, scripts/small_cluster_probe.py)
    const int fill = tm / k <= 32 ? std::min(min_fill, 40) : min_fill;
    if (n_units * k > sms || n_units * k * 100 < static_cast<int64_t>(sms) * fill || tm % k != 0 || tm / k < kNW)
      continue;
    if (dq_prmt::dq_cluster_capacity(group, 44, PQB_BF16, k) < n_units) return 0;
    return k;
  }
  return 0;
}

int decode_launch_count(int64_t n_units, int group, int max_tokens, int flags, int angle_bits, int radius_bits,
                       int value_dtype) {
  if (group != 4 && group != 8) return 1;
  pqb_cache probe = {};  // only the fields dq_cluster_size reads
  probe.angle_bits = angle_bits;
  probe.radius_bits = radius_bits;
  probe.store.value_dtype = value_dtype;
  if (dq_cluster_size(n_units, group, max_tokens, flags, &probe, false, false) > 1) return 1;
  const WorkSplit ws = make_split_balanced(n_units, max_tokens, std::min(num_sms(), kMaxCtas));
  return (flags & PQB_DECODE_NO_COMBINE) || !separate_merge(flags, group, max_tokens, ws) ? 1 : 2;
}

int decode_split_starts(int64_t n_units, int max_tokens, int ctas, int32_t* starts) {
  if (n_units <= 0 || max_tokens <= 0 || ctas <= 0 || ctas > kMaxCtas) return -1;
  const WorkSplit w = make_split_balanced(n_units, max_tokens, ctas);
  if (!w.balanced) return 0;
  for (int c = 0; c <= w.n_cta; ++c) starts[c] = w.starts[c];
  return w.n_cta;
}

static std::atomic<int> g_dq_layout{0};
int decode_dq_layout() { return g_dq_layout.load(std::memory_order_relaxed); }

static int launch_dq_path(const DecodeArgs& a, cudaStream_t s, bool& handled) {
  EpiArgs ep;
  WorkSplit ws;
  int grid = 0;
  const int cl = a.splits > 0 || a.out == nullptr
                     ? 0
                     : dq_cluster_size(a.n_units, a.group, a.max_tokens, a.flags, a.cache, a.peer != nullptr,
                                       a.scores != nullptr);
  const int rc = fast_setup(a, ep, ws, grid, true);
  if (rc != PQB_OK) {
    handled = true;
    return rc;
  }
  if (cl > 1) {  // aligned split: cluster u = unit u, CTA rank r = tiles [r tm / k, (r + 1) tm / k)
    ws.balanced = 0;
    ws.cluster = cl;
    ws.per_cta = ws.tiles_max / cl;
    grid = static_cast<int>(a.n_units * cl);
    ep.merge = !(a.flags & PQB_DECODE_NO_COMBINE);  // NO_COMBINE: the CTA partials only (kernel-only timing)
    const int rc2 = dq_prmt::launch_decode_dq(a, ep, ws, grid, s, handled);
    if (rc2 == PQB_OK && handled) g_dq_layout.store(1, std::memory_order_relaxed);
    if (rc2 != kDqLayoutUnavailable) return rc2;
    ws.cluster = 0;  // (the layout check failed: the non-cluster path below)
    DecodeArgs b = a;
    b.flags |= PQB_DECODE_NO_CLUSTER;
    return launch_dq_path(b, s, handled);
  }
  const bool sep = ep.merge && a.out != nullptr && a.peer == nullptr &&
                   separate_merge(a.flags, a.group, a.max_tokens, ws);
  if (sep) ep.merge = false;
  int rc2 = (a.flags & PQB_DECODE_DQ_LINEAR) ? kDqLayoutUnavailable : dq_prmt::launch_decode_dq(a, ep, ws, grid, s, handled);
  int layout = 1;
  if (rc2 == kDqLayoutUnavailable) {
    rc2 = dq_lin::launch_decode_dq(a, ep, ws, grid, s, handled);
    layout = 2;
  }
  if (rc2 == PQB_OK && handled) g_dq_layout.store(layout, std::memory_order_relaxed);
  if (rc2 != PQB_OK || !handled || !sep) return rc2;
  return launch_merge_split(ep, ws, a.n_units, s);
}

template <int G, bool EXACT>
static int dispatch_fast_mn(const DecodeArgs& a, cudaStream_t s, bool& handled) {
  handled = true;
  switch (a.cache->angle_bits * 10 + a.cache->radius_bits) {
    case 44: return launch_fast<G, 4, 4, EXACT>(a, s);
    case 32: return launch_fast<G, 3, 2, EXACT>(a, s);
    case 22: return launch_fast<G, 2, 2, EXACT>(a, s);
    case 42: return launch_fast<G, 4, 2, EXACT>(a, s);
    case 24: return launch_fast<G, 2, 4, EXACT>(a, s);
    case 34: return launch_fast<G, 3, 4, EXACT>(a, s);
    default: handled = false; return PQB_OK;
  }
}

template <bool EXACT>
static int dispatch_fast(const DecodeArgs& a, cudaStream_t s, bool& handled) {
  if (a.group == 4) return dispatch_fast_mn<4, EXACT>(a, s, handled);
  if (a.group == 8) return dispatch_fast_mn<8, EXACT>(a, s, handled);
  return dispatch_fast_mn<1, EXACT>(a, s, handled);
}

int launch_decode(const DecodeArgs& a, cudaStream_t s) {
  const pqb_cache& c = *a.cache;
  const bool vq = vq_bits(c.store.value_dtype) && a.out != nullptr;  // quantized values: DQ kernel or generic
  const bool f32v = c.store.value_dtype == PQB_F32 && a.out != nullptr;  // fp32 values: DQ kernel or generic
  const bool fast_ok = c.d == 128 && (a.out == nullptr || c.store.value_dtype == PQB_BF16 || vq || f32v) &&
                       (a.group == 1 || a.group == 4 || a.group == 8) && c.store.page_tokens % kTile == 0 &&
                       (c.store.angle_off % 16 == 0) && (c.store.radius_off % 16 == 0) &&
                       (c.store.value_off % 16 == 0 || a.out == nullptr) && (c.store.page_bytes % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(c.store.pool) % 16 == 0);
  bool handled = false;
  if (fast_ok && !(a.flags & PQB_DECODE_FORCE_GENERIC) && use_dq(a)) {
    const int rc = launch_dq_path(a, s, handled);
    if (rc != PQB_OK) return rc;
  }
  if (a.peer != nullptr && !handled) {
    set_error("peer-gather decode needs the DQ kernel (group 4 or 8, d = 128, a fast-path store and bit widths)");
    return PQB_EUNSUPPORTED;
  }
  if (fast_ok && !handled && !vq && !f32v && !(a.flags & PQB_DECODE_FORCE_GENERIC)) {
    // scores requested -> the bit-exact scoring sequence; fused-only -> FMA form
    const int rc = a.scores != nullptr ? dispatch_fast<true>(a, s, handled) : dispatch_fast<false>(a, s, handled);
    if (rc != PQB_OK) return rc;
  }
  if (handled) return PQB_OK;
  if (c.d > 256 || a.group > kGenMaxG) {
    set_error("decode: d=%d group=%d unsupported (d <= 256, group <= %d)", c.d, a.group, kGenMaxG);
    return PQB_EUNSUPPORTED;
  }
  const int splits = a.splits > 0 ? std::min(a.splits, max_splits(a.max_tokens)) : choose_splits(a.n_units, a.max_tokens);
  const int tps = (tiles_of(a.max_tokens) + splits - 1) / splits;
  EpiArgs ep;
  ep.out = a.out;
  ep.out_dtype = a.out_dtype;
  ep.group = a.group;
  ep.peer_mode = false;
  ep.slots = splits;
  // partials after the (untouched) counter region of the fast path
  ep.part_ml = reinterpret_cast<float*>(static_cast<uint8_t*>(a.workspace) + counter_bytes(a.n_units));
  ep.part_o = ep.part_ml + a.n_units * splits * a.group * 2;
  ep.counters = nullptr;
  ep.merge = false;
  if (splits > 1 && a.out != nullptr) {
    const size_t need = counter_bytes(a.n_units) +
                        static_cast<size_t>(a.n_units) * splits * a.group * (2 + c.d) * sizeof(float);
    if (a.workspace == nullptr || a.workspace_bytes < need) {
      set_error("decode workspace too small: need %zu bytes, got %zu", need, a.workspace_bytes);
      return PQB_EINVAL;
    }
  }
  const size_t shm = sizeof(float) * (a.group * c.d + 512 + c.d / 2 + kNW * kTile * a.group +
                                      kNW * a.group * (2 + c.d));
  static std::atomic<size_t> attr[64];  // largest opt-in set so far, per device
  if (shm > 48 * 1024) {
    std::atomic<size_t>& cur = attr[current_device() & 63];
    if (shm > cur.load(std::memory_order_acquire)) {
      if (cudaFuncSetAttribute(decode_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(shm)) != cudaSuccess) {
        set_error("cudaFuncSetAttribute(smem=%zu) failed", shm);
        return PQB_ECUDA;
      }
      size_t seen = cur.load(std::memory_order_acquire);
      while (seen < shm && !cur.compare_exchange_weak(seen, shm, std::memory_order_acq_rel)) {
      }
    }
  }
  dim3 grid(splits, static_cast<unsigned>(a.n_units));
  decode_generic_kernel<<<grid, kNW * 32, shm, s>>>(c, a.group, a.q, a.q_dtype, a.sm_scale * kLog2e, a.scores,
                                                    a.scores_ld, ep, tps);
  if (splits > 1 && a.out != nullptr && !(a.flags & PQB_DECODE_NO_COMBINE))
    combine_kernel<<<static_cast<unsigned>(a.n_units), 256, 0, s>>>(ep.part_ml, ep.part_o, splits, a.group, c.d,
                                                                    a.out, a.out_dtype);
  return PQB_OK;
}

}  // namespace pqb
