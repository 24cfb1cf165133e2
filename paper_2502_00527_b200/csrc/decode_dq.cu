// HP-2, dequantize-then-contract variant (sm_100a): decode_dq_kernel<G, M, N>.
//
//   reference  qk_scores_direct (dequantize, then dot)   lut_decode.py:157-186
//              decode_keys (rhat * (cos, sin)[A])        polar_codec.py:305-316
//              _residual_scores (exact fp32 dots)        lut_decode.py:107-116
//              softmax . V restated over values()        kv_cache.py:247-259
//
// Why a second kernel.  The LUT kernel (decode.cu) gathers G*4 bytes of table
// per (token, channel pair) from shared memory: 1 KB per token at G = 4 and
// 2 KB at G = 8, against 320 B of HBM per token.  At G = 8 that gather alone
// needs ~50 TB/s of shared-memory bandwidth for an HBM-rate kernel (the SMs
// deliver ~36), so the 70B shape is capped near 60% of HBM by construction.
// Here the per-(token, pair) shared-memory traffic is one 8-byte angle-table
// entry, independent of G, and the G-query contraction S^T = K^ . Q'^T runs on
// the tensor cores (it is a genuine dense [32 x 128] x [128 x G] product per
// tile once the keys are dequantized).
//
// Numerics (fast / fused path only; scores-only calls use the bit-exact LUT
// kernel).  K-order is pair-major (x_j, y_j) for both layouts (a contraction
// is order-free; Q' is laid out to match).  Per unit
//     Q'[g][2j + c] = q[g][e_c(j)] * s_j * 2^e         (s_j = fp16 scale, 2^e
//                                                       puts max|Q'| in [2^14, 2^15))
// split into fp16 hi + lo (22 significant bits).  The key side needs no
// arithmetic at all: a per-CTA product table holds, for every (angle code a,
// radius code r), the dequantized pair  (r cos_a, r sin_a)  split into fp16
// hi + lo halves (22 bits):
//     PT[(a << N) | r] = { half2(x_hi, y_hi), half2(x_lo, y_lo) }
// and one 8-byte gather per (token, pair) yields both MMA A-fragment registers.
// The table is replicated 16 times with copy k in bank slot k, so lane L reads
// copy L % 16 and every LDS.64 is bank-conflict free whatever the codes
// (2^(M+N) * 128 B: 32 KB at m = n = 4).  MMAs (m16n8k16 f16, fp32 accumulate):
//     G = 8:  K_hi.Q_hi + K_lo.Q_hi + K_hi.Q_lo          (dropped K_lo.Q_lo ~ 2^-22)
//     G = 4:  the 8 MMA columns hold Q_hi | Q_lo, so K_hi, K_lo x [Q_hi | Q_lo]
//             is complete; columns q and q + 4 are summed after.
// Per-element relative error ~2^-22 before the tensor cores' fp32 accumulation,
// i.e. scores agree with the fp32 LUT sequence to ~1e-6 of sum |q_i k_i| --
// far inside the reference's LUT == dequant tolerance (test_lut_decode.py:107-108).
//
// Tile flow per warp (32 tokens, same TMA ring / persistent split / epilogue as
// the LUT kernel): lane (g, t4) dequantizes tokens {g, g+8, g+16, g+24} x pairs
// {4i + t4} straight into MMA A-fragment registers; C = S^T[token][query] feeds
// a register online softmax (3 shuffles per query pair); P (bf16 hi/lo) goes
// through 1 KB of shared memory and comes back as P^T B-fragments with one
// ldmatrix.trans each; P.V as in the LUT kernel.
#include "decode_common.cuh"
#include "kernels.h"

#include <algorithm>

namespace pqb {

template <int G, int M, int N>
struct DqCfg {
  static constexpr int kABytes = kTile * 8 * M;
  static constexpr int kRBytes = kTile * 8 * N;
  static constexpr int kVBytes = kTile * 256;
  static constexpr int kStageBytes = kABytes + kRBytes + kVBytes;
  static constexpr int kPBytes = 2 * kTile * 16;             // bf16 [hi/lo][32 tokens][8 queries]; fp32 [32][8] residual scratch
  static constexpr int kTabBytes = 128 << (M + N);          // product table, 16 bank-slot copies
  static constexpr int kFragBytes = 8 * 32 * 16;             // Q' B-fragments [ks][lane] uint4
  static constexpr int kHeadBytes = kTabBytes + kFragBytes + G * 128 * 4 + 128 + 8 * (1 << M);
  static constexpr int kWarpBytes = kStages * kStageBytes + kPBytes + 64;
  static constexpr int kSmem = kHeadBytes + kNW * kWarpBytes + 128;
  static_assert(kHeadBytes % 16 == 0 && kWarpBytes % 16 == 0, "alignment");
  static_assert(kNW * kStages * kStageBytes >= kNW * G * 132 * 4, "merge area");
};

PQB_DEV uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
PQB_DEV __half2 bits_h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

PQB_DEV void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Code i of the lane's pair set {4i + t4} from the row pre-shifted by t4*B bits:
// it sits at bit 4iB (never straddles a word for B in {2, 3, 4}).
template <int B>
PQB_DEV uint32_t dq_code(const uint32_t* ws, int i) {
  const int bit = 4 * i * B;
  return (ws[bit >> 5] >> (bit & 31)) & ((1u << B) - 1u);
}

// Product-table indices (a << N) | r of codes i and i + 1 (i even).
template <int M, int N>
PQB_DEV void dq_index2(const uint32_t* wa, const uint32_t* wr, int i, uint32_t& i0, uint32_t& i1) {
  if constexpr (M == 4 && N == 4) {
    // codes i, i+1 at bits 0 and 16 of word i/2 in both streams
    const uint32_t v = ((wa[i >> 1] << 4) & 0x00F000F0u) | (wr[i >> 1] & 0x000F000Fu);
    i0 = v & 0xFFu;
    i1 = v >> 16;
  } else {
    i0 = (dq_code<M>(wa, i) << N) | dq_code<N>(wr, i);
    i1 = (dq_code<M>(wa, i + 1) << N) | dq_code<N>(wr, i + 1);
  }
}

template <int G, int M, int N>
__global__ void __launch_bounds__(kNW * 32, 1)
    decode_dq_kernel(const pqb_cache c, const void* __restrict__ q, int q_dtype, float sm_scale_log2, EpiArgs ep,
                     WorkSplit ws) {
  using Cfg = DqCfg<G, M, N>;
  static_assert(G == 4 || G == 8, "G");
  extern __shared__ __align__(128) uint8_t smem[];
  uint2* ptab = reinterpret_cast<uint2*>(smem);                                   // [2^(M+N)][16]
  uint4* qfrag = reinterpret_cast<uint4*>(smem + Cfg::kTabBytes);                    // [8][32]
  float* q_s = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(qfrag) + Cfg::kFragBytes);  // [G][128]
  int* s_misc = reinterpret_cast<int*>(q_s + G * 128);  // [0] max|Q'| bits, [1] merge flag
  float2* cs_s = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(s_misc) + 128);  // [2^M] (cos, sin)
  uint8_t* warp_area = smem + Cfg::kHeadBytes;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* my_area = warp_area + warp * Cfg::kWarpBytes;
  uint8_t* pbuf = my_area + kStages * Cfg::kStageBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(pbuf + Cfg::kPBytes);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  // product table (once per CTA): PT[(a << N) | r][copy] = (r cos_a, r sin_a) as fp16 hi + lo
  if (tid < (1 << M)) {
    float cf, sf;
    angle_unit(M, tid, cf, sf);
    cs_s[tid] = make_float2(cf, sf);
  }
  __syncthreads();
  for (int i = tid; i < (16 << (M + N)); i += blockDim.x) {
    const int e = i >> 4, a = e >> N, r = e & ((1 << N) - 1);
    const float2 cs = cs_s[a];
    const double x = static_cast<double>(r) * cs.x, y = static_cast<double>(r) * cs.y;  // exact products
    const __half xh = __float2half_rn(static_cast<float>(x)), yh = __float2half_rn(static_cast<float>(y));
    ptab[i] = make_uint2(h2_bits(__halves2half2(xh, yh)),
                         h2_bits(__halves2half2(__float2half_rn(static_cast<float>(x - __half2float(xh))),
                                                __float2half_rn(static_cast<float>(y - __half2float(yh))))));
  }
  const uint8_t* ptab_l = smem + ((threadIdx.x & 15) << 3);  // this lane's bank-slot copy
  const int tpp = c.store.page_tokens / kTile;  // tiles per page
  const int64_t i_begin = static_cast<int64_t>(blockIdx.x) * ws.per_cta;
  const int64_t i_end = min(ws.items, i_begin + ws.per_cta);
  uint32_t k_iter = 0;

  const int g8 = lane >> 2, t4 = lane & 3;  // fragment group / thread-in-group
  const uint32_t ld_row = static_cast<uint32_t>((((lane >> 4) & 1) * 8 + (lane & 7)) * 256);
  const uint32_t ld_chunk = static_cast<uint32_t>((((lane >> 3) & 1) ^ (lane & 7)) << 4);

  for (int64_t seg = i_begin; seg < i_end;) {
    const int64_t unit = seg / ws.tiles_max;
    const int t_lo = static_cast<int>(seg - unit * ws.tiles_max);
    const int64_t seg_end = min(i_end, (unit + 1) * ws.tiles_max);
    seg = seg_end;
    const int T = c.seq_lens[unit], Tq = c.quant_lens[unit];
    const int n_tiles = (T + kTile - 1) / kTile;
    const int t_hi = min(static_cast<int>(seg_end - unit * ws.tiles_max), n_tiles);

    __syncthreads();  // previous segment is done with q_s / qfrag / merge area
    const int first = t_lo + warp;
    // ---- unit setup: q rows, max |q * s|, then the Q' hi/lo B-fragments
    if (tid == 0) s_misc[0] = 0;
    for (int i = tid; i < G * 128; i += blockDim.x) q_s[i] = load_q(q, q_dtype, unit * G * 128 + i);
    __syncthreads();
    {
      float mx = 0.0f;
      for (int i = tid; i < G * 128; i += blockDim.x) {
        const int e = i & 127;
        const int j = c.layout == PQB_HALF_SPLIT ? (e & 63) : (e >> 1);
        mx = fmaxf(mx, fabsf(q_s[i] * half_bits_to_f32(c.scales[unit * 64 + j])));
      }
      mx = warp_max(mx);
      if (lane == 0) atomicMax(s_misc, __float_as_int(mx));  // non-negative floats order as ints
    }
    __syncthreads();
    const float qmax = __int_as_float(s_misc[0]);
    // 2^e * qmax in [2^14, 2^15)
    const int e_sc = (qmax > 0.0f && qmax < INFINITY)
                         ? max(-90, min(90, 14 - (static_cast<int>((__float_as_uint(qmax) >> 23) & 0xff) - 127)))
                         : 0;
    for (int i = tid; i < 8 * 32; i += blockDim.x) {
      const int ks = i >> 5, ln = i & 31, n = ln >> 2, t = ln & 3;
      uint32_t w[4];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int j = 8 * ks + t + 4 * hh;
        const float sj = half_bits_to_f32(c.scales[unit * 64 + j]);
        const int ex = c.layout == PQB_HALF_SPLIT ? j : 2 * j;
        const int ey = c.layout == PQB_HALF_SPLIT ? j + 64 : 2 * j + 1;
        const int g = G == 8 ? n : (n & 3);
        const float vx = ldexpf(q_s[g * 128 + ex] * sj, e_sc), vy = ldexpf(q_s[g * 128 + ey] * sj, e_sc);
        const __half hx = __float2half_rn(vx), hy = __float2half_rn(vy);
        const __half lx = __float2half_rn(vx - __half2float(hx)), ly = __float2half_rn(vy - __half2float(hy));
        if constexpr (G == 8) {
          w[hh] = h2_bits(__halves2half2(hx, hy));
          w[2 + hh] = h2_bits(__halves2half2(lx, ly));
        } else {  // columns 0-3: Q_hi, 4-7: Q_lo
          w[hh] = n < 4 ? h2_bits(__halves2half2(hx, hy)) : h2_bits(__halves2half2(lx, ly));
          w[2 + hh] = 0u;
        }
      }
      qfrag[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncthreads();
    uint32_t bq[8][4];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint4 v = qfrag[ks * 32 + lane];
      bq[ks][0] = v.x;
      bq[ks][1] = v.y;
      bq[ks][2] = v.z;
      bq[ks][3] = v.w;
    }
    const float xscale = ldexpf(sm_scale_log2, -e_sc);

    // ---- lane 0 fills this warp's ring with its first tiles (after the setup:
    // measured faster than overlapping it, scripts/ab_probe.sh)
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < kStages; ++s) {
        const int tile = first + s * kNW;
        if (tile < t_hi) {
          fence_proxy_async_smem();
          const uint32_t sl = (k_iter + s) % kStages;
          issue_tile<M, N>(my_area + sl * Cfg::kStageBytes, c.store, page_base_c(c.store, unit, tile / tpp), tile,
                           tpp, true, bar + sl);
        }
      }
    }
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};
    float d[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int k = 0; k < 4; ++k) d[mt][k] = 0.0f;

    for (int tile = first; tile < t_hi; tile += kNW, ++k_iter) {
      const uint32_t s = k_iter % kStages;
      const int nt = tile + kStages * kNW;  // the tile this stage is refilled with
      mbar_wait(bar + s, (k_iter / kStages) & 1);
      const uint8_t* st = my_area + s * Cfg::kStageBytes;
      const int tok0 = tile * kTile;

      // ---- S^T = K^ . Q'^T on the tensor cores, two 16-token m-tiles
      float sc[2][4], sc2[2][4];  // two MMA accumulation chains per m-tile, summed after
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int k = 0; k < 4; ++k) sc[mt][k] = sc2[mt][k] = 0.0f;
        uint32_t wa[2][2 * M + 1], wr[2][2 * N + 1];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 16 * mt + g8 + 8 * h;
          const uint32_t* ra = reinterpret_cast<const uint32_t*>(st + r * 8 * M);
          const uint32_t* rr = reinterpret_cast<const uint32_t*>(st + Cfg::kABytes + r * 8 * N);
          if constexpr (M % 2 == 0) {
#pragma unroll
            for (int k = 0; k < 2 * M; k += 4) {
              const uint4 v = *reinterpret_cast<const uint4*>(ra + k);
              wa[h][k] = v.x; wa[h][k + 1] = v.y; wa[h][k + 2] = v.z; wa[h][k + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int k = 0; k < 2 * M; k += 2) {
              const uint2 v = *reinterpret_cast<const uint2*>(ra + k);
              wa[h][k] = v.x; wa[h][k + 1] = v.y;
            }
          }
          if constexpr (N % 2 == 0) {
#pragma unroll
            for (int k = 0; k < 2 * N; k += 4) {
              const uint4 v = *reinterpret_cast<const uint4*>(rr + k);
              wr[h][k] = v.x; wr[h][k + 1] = v.y; wr[h][k + 2] = v.z; wr[h][k + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int k = 0; k < 2 * N; k += 2) {
              const uint2 v = *reinterpret_cast<const uint2*>(rr + k);
              wr[h][k] = v.x; wr[h][k + 1] = v.y;
            }
          }
          wa[h][2 * M] = 0u;
          wr[h][2 * N] = 0u;
          const bool live = tok0 + r < Tq;  // residual / past-the-end rows: radius 0 => key 0
          // pre-shift so code (4i + t4) sits at bit 4iB
#pragma unroll
          for (int k = 0; k < 2 * M; ++k) wa[h][k] = __funnelshift_r(wa[h][k], wa[h][k + 1], t4 * M);
#pragma unroll
          for (int k = 0; k < 2 * N; ++k) wr[h][k] = live ? __funnelshift_r(wr[h][k], wr[h][k + 1], t4 * N) : 0u;
        }
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t ahi[4], alo[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            // pairs i = 2ks (a0 / a1: k 2t4..) and 2ks + 1 (a2 / a3: k 2t4 + 8..)
            uint32_t e0, e1;
            dq_index2<M, N>(wa[h], wr[h], 2 * ks, e0, e1);
            const uint2 t0 = *reinterpret_cast<const uint2*>(ptab_l + (e0 << 7));
            const uint2 t1 = *reinterpret_cast<const uint2*>(ptab_l + (e1 << 7));
            ahi[h] = t0.x;
            alo[h] = t0.y;
            ahi[2 + h] = t1.x;
            alo[2 + h] = t1.y;
          }
          mma_f16(sc[mt], ahi[0], ahi[1], ahi[2], ahi[3], bq[ks][0], bq[ks][1]);
          mma_f16(sc2[mt], alo[0], alo[1], alo[2], alo[3], bq[ks][0], bq[ks][1]);
          if constexpr (G == 8) mma_f16(sc2[mt], ahi[0], ahi[1], ahi[2], ahi[3], bq[ks][2], bq[ks][3]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) sc[mt][k] += sc2[mt][k];
      }
      if constexpr (G == 4) {  // fold columns q (hi) and q + 4 (lo): lanes t4 and t4 ^ 2
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int k = 0; k < 4; ++k) sc[mt][k] += __shfl_xor_sync(0xffffffffu, sc[mt][k], 2);
      }
      // ---- residual window (fp32 keys): exact dots, lane = token (rare tiles)
      if (tok0 + kTile > Tq && Tq < T) {
        float* rbuf = reinterpret_cast<float*>(pbuf);  // [32][8], scaled like C
        const int tok = tok0 + lane;
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.0f;
        if (tok >= Tq && tok < T) {
          const float* kr = c.residual + (unit * c.res_cap + tok % c.res_cap) * 128;
          for (int e = 0; e < 128; ++e) {
            const float kv = kr[e];
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = fmaf(kv, q_s[g * 128 + e], acc[g]);
          }
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) rbuf[lane * 8 + g] = g < G ? ldexpf(acc[g], e_sc) : 0.0f;
        __syncwarp();
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = 16 * mt + g8 + 8 * (k >> 1), col = 2 * t4 + (k & 1);
            if (tok0 + r >= Tq && col < G) sc[mt][k] += rbuf[r * 8 + col];
          }
        __syncwarp();
      }
      // ---- online softmax: lane holds queries 2t4, 2t4+1 for tokens {g8, g8+8} + 16mt
      float alpha[2];
      bool rescale = false;
#pragma unroll
      for (int cq = 0; cq < 2; ++cq) {
        float x[4];
        float mx = -INFINITY;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int mt = v >> 1, h = v & 1;
          const int r = 16 * mt + g8 + 8 * h;
          x[v] = tok0 + r < T ? sc[mt][2 * h + cq] * xscale : -INFINITY;
          mx = fmaxf(mx, x[v]);
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float mn = fmaxf(m_run[cq], mx);
        alpha[cq] = exp2f(m_run[cq] - mn);
        rescale |= mn != m_run[cq];
        m_run[cq] = mn;
        float ls = 0.0f;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float p = exp2f(x[v] - mn);
          ls += p;
          sc[v >> 1][2 * (v & 1) + cq] = p;
        }
        l_run[cq] = fmaf(l_run[cq], alpha[cq], ls);
      }
      // P -> pbuf [hi/lo][token][8 queries] bf16 (queries >= G stay zero)
      const bool qvalid = 2 * t4 < G;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int mt = v >> 1, h = v & 1;
        const int r = 16 * mt + g8 + 8 * h;
        const float p0 = qvalid ? sc[mt][2 * h] : 0.0f, p1 = qvalid ? sc[mt][2 * h + 1] : 0.0f;
        const __nv_bfloat162 hi = __floats2bfloat162_rn(p0, p1);
        const float2 hf = __bfloat1622float2(hi);
        const __nv_bfloat162 lo = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
        *reinterpret_cast<__nv_bfloat162*>(pbuf + r * 16 + 4 * t4) = hi;
        *reinterpret_cast<__nv_bfloat162*>(pbuf + kTile * 16 + r * 16 + 4 * t4) = lo;
      }
      if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          d[mt][0] *= alpha[0];
          d[mt][1] *= alpha[1];
          d[mt][2] *= alpha[0];
          d[mt][3] *= alpha[1];
        }
      }
      __syncwarp();
      // ---- P.V on tensor cores (as decode_fast_kernel): P^T fragments via ldmatrix.trans
      uint32_t b[2][2][2];  // [pl][ks][reg]
      {
        const uint32_t pb0 = smem_u32(pbuf) + lane * 16;
        ldsm_x4_trans(pb0, b[0][0][0], b[0][0][1], b[0][1][0], b[0][1][1]);
        ldsm_x4_trans(pb0 + kTile * 16, b[1][0][0], b[1][0][1], b[1][1][0], b[1][1][1]);
      }
      const uint32_t vbase = smem_u32(st + Cfg::kABytes + Cfg::kRBytes) + ld_row;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4_trans(vbase + ks * 16 * 256 + (ld_chunk ^ (mt << 5)), a0, a1, a2, a3);
          mma_bf16(d[mt], a0, a1, a2, a3, b[0][ks][0], b[0][ks][1]);
          mma_bf16(d[mt], a0, a1, a2, a3, b[1][ks][0], b[1][ks][1]);
        }
      }
      __syncwarp();
      if (lane == 0 && nt < t_hi) {
        fence_proxy_async_smem();
        issue_tile<M, N>(my_area + s * Cfg::kStageBytes, c.store, page_base_c(c.store, unit, nt / tpp), nt, tpp,
                         true, bar + s);
      }
    }

    // ---- segment epilogue: per-warp (m, l, o) -> shared, then the common merge
#pragma unroll
    for (int cq = 0; cq < 2; ++cq) {
      l_run[cq] += __shfl_xor_sync(0xffffffffu, l_run[cq], 4);
      l_run[cq] += __shfl_xor_sync(0xffffffffu, l_run[cq], 8);
      l_run[cq] += __shfl_xor_sync(0xffffffffu, l_run[cq], 16);
    }
    __syncthreads();
    float* red = reinterpret_cast<float*>(warp_area);
    float* mine = red + warp * G * 132;
    if (g8 == 0) {
#pragma unroll
      for (int cq = 0; cq < 2; ++cq) {
        const int qq = 2 * t4 + cq;
        if (qq < G) {
          mine[qq * 132] = m_run[cq];
          mine[qq * 132 + 1] = l_run[cq];
        }
      }
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int dim = 16 * mt + g8;
      if (2 * t4 < G) {
        mine[(2 * t4) * 132 + 4 + dim] = d[mt][0];
        mine[(2 * t4) * 132 + 4 + dim + 8] = d[mt][2];
        mine[(2 * t4 + 1) * 132 + 4 + dim] = d[mt][1];
        mine[(2 * t4 + 1) * 132 + 4 + dim + 8] = d[mt][3];
      }
    }
    finish_segment<G>(ep, ws, unit, red, s_misc + 1, tid, blockDim.x);
  }
}

// ------------------------------------------------------------------ host side

template <int G, int M, int N>
static int launch_dq(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s) {
  using Cfg = DqCfg<G, M, N>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(decode_dq_kernel<G, M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem) !=
        cudaSuccess) {
      set_error("cudaFuncSetAttribute(smem=%d) failed", Cfg::kSmem);
      return PQB_ECUDA;
    }
    attr_set = true;
  }
  decode_dq_kernel<G, M, N><<<grid, kNW * 32, Cfg::kSmem, s>>>(*a.cache, a.q, a.q_dtype, a.sm_scale * kLog2e, ep, ws);
  return PQB_OK;
}

template <int G>
static int dispatch_dq_mn(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s,
                          bool& handled) {
  handled = true;
  switch (a.cache->angle_bits * 10 + a.cache->radius_bits) {
    case 44: return launch_dq<G, 4, 4>(a, ep, ws, grid, s);
    case 32: return launch_dq<G, 3, 2>(a, ep, ws, grid, s);
    case 22: return launch_dq<G, 2, 2>(a, ep, ws, grid, s);
    case 42: return launch_dq<G, 4, 2>(a, ep, ws, grid, s);
    case 24: return launch_dq<G, 2, 4>(a, ep, ws, grid, s);
    case 34: return launch_dq<G, 3, 4>(a, ep, ws, grid, s);
    default: handled = false; return PQB_OK;
  }
}

int launch_decode_dq(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s,
                     bool& handled) {
  handled = false;
  if (a.group == 8) return dispatch_dq_mn<8>(a, ep, ws, grid, s, handled);
  if (a.group == 4) return dispatch_dq_mn<4>(a, ep, ws, grid, s, handled);
  return PQB_OK;
}

}  // namespace pqb
