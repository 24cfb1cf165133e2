// HP-1 K2, persistent TMA-fed encoder for the common shapes (sm_100a):
// encode_fast_kernel<DT, LAYOUT, M, N>.
//
//   reference  quantize_subvectors (polar_codec.py:281-302), pack_stream (:98-110),
//              PackedKVCache._encode_block (kv_cache.py:191-197)
//
// Same arithmetic contract as encode_v8 (polar_math.cuh): a fast fp32 decision
// per sub-vector pair, and the exact double-precision pipeline for a thread's
// eight pairs whenever one of them lies within the ambiguity band of an angle
// edge or a radius rounding boundary.  What changes is the cost per pair
// (encode_v8 measured 78 instructions per pair, ALU-pipe bound,
// profiles/r01/ncu_encode_fast.json):
//   * m, n are compile-time: codes pack into 32-bit words with constant shifts;
//     for m = 4 / n = 4 a thread's eight codes are exactly one stream word.
//   * the octant fold works on s = |x| + |y| and a = ||x| - |y||:
//       sign(mn - mx tan b) = sign(s - a (1 + tan b) / (1 - tan b)),
//     one FFMA per edge with an immediate; the ambiguity test of all pairs and
//     edges folds into one running maximum.
//   * the radius code is taken from the float bits (magic-number add) and
//     packed with IMADs; clamp events are counted with saturating adds.
//   * keys arrive through per-warp rings of TMA bulk copies (4 KB stages), the
//     grid is persistent (one 16-warp CTA per SM) and warps take 512-token
//     (unit, chunk) items round-robin; no CTA-wide barrier in the loop, so the
//     rare exact-path lane stalls only its own warp.
// Requirements (checked by the launcher, else encode_v8): d = 128, dense
// 16-byte aligned rows, page_tokens % 16 == 0, start token % 16 == 0,
// m in {2, 3, 4}, n in {2, 3, 4}.
#include "kernels.h"
#include "polar_math.cuh"

#include <algorithm>

namespace pqb {

namespace {

#ifndef PQB_EF_WARPS
#define PQB_EF_WARPS 16
#endif
constexpr int kEfWarps = PQB_EF_WARPS;  // warps per CTA (one CTA per SM)
constexpr int kEfStages = 3;     // ring depth per warp
constexpr int kEfItemTok = 512;  // tokens per work item (one unit)
constexpr int kEfAlign = 16;     // start token / page alignment the kernel needs

template <int DT>
struct EfCfg {
  static constexpr int kRowBytes = 128 * DType<DT>::kBytes;
  static constexpr int kStageBytes = 4096;                  // per-warp stage
  static constexpr int kStageTok = kStageBytes / kRowBytes;  // 16 (2-byte keys) or 8 (fp32)
  static constexpr int kSmem = kEfWarps * kEfStages * kStageBytes;
};

// Octant-fold constants of angle_bits M (M >= 3): edge i at b_i, t = tan(b_i):
//   K_i = (1 + t) / (1 - t),  e_i = s - a K_i  (sign of mn - mx t),
//   band: |mn - mx t| <= thr_i (mx + mn)  <=>  |e_i| <= 2 thr_i / (1 - t) s.
// The band constant is inflated by 1% (covers the fp32 rounding of s, a, K_i
// and the FFMA, <= 1e-6 s; polar_math.cuh has the pipeline's error budget).
__host__ __device__ constexpr float ef_k(int m, int i) { return (1.0f + edge_tan(m, i)) / (1.0f - edge_tan(m, i)); }
__host__ __device__ constexpr float ef_band(int m, int i) { return 2.02f * edge_thr(m, i) / (1.0f - edge_tan(m, i)); }
template <int M>
__host__ __device__ constexpr float ef_band_max() {
  float b = 0.0f;
  for (int i = 0; i < (1 << (M - 3)); ++i) b = ef_band(M, i) > b ? ef_band(M, i) : b;
  return b;
}

// Exact |x| == |y| at m = 2 (frequent with bf16 keys): atan2f is fl32(+-pi/4)
// or fl32(+-3pi/4); the reference pipeline's code for each sign pattern.
PQB_DEV uint32_t ef_m2_diag(float x, float y) {
  const uint32_t sx = __float_as_uint(x) >> 31;
  return angle_code_from_phi(copysignf(sx ? 2.35619449615478515625f : 0.785398185253143310546875f, y), 2);
}

// Fast codes of one pair.  Returns the angle code (before the canonical
// origin rule) and the rounded radius ratio rq; `worst` collects the
// ambiguity metric (>= 0: inside a band), `rok` the magnitude-range check.
// Octant-table index of a pair (m >= 3): the sign bits of x, y, |x| - |y| and
// of the NB edge tests e_i, appended with funnel shifts (one SHF each).  The
// table (ef_build_octant_table) maps it to the angle code.
template <int M>
__host__ __device__ constexpr int ef_index_bits() { return M == 2 ? 4 : 3 + (1 << (M - 3)); }

template <int M>
PQB_DEV uint32_t ef_angle(float x, float y, float& worst, const uint8_t* tab) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float s = ax + ay, dif = ax - ay, a = fabsf(dif);
  if constexpr (M == 2) {
    // the only edge is the diagonal (swap bit).  An exact tie |x| == |y|
    // (frequent with bf16 keys) is a fourth index bit: t = a - 2^-100 < 0 iff
    // a == 0 (nonzero a >= 2^-75 in the safe magnitude range); ties are exact,
    // so they are excluded from the band.
    const float t = a - 0x1p-100f;
    uint32_t idx = __funnelshift_l(__float_as_uint(x), 0u, 1);
    idx = __funnelshift_l(__float_as_uint(y), idx, 1);
    idx = __funnelshift_l(__float_as_uint(dif), idx, 1);
    idx = __funnelshift_l(__float_as_uint(t), idx, 1);
    worst = fmaxf(worst, fminf(fmaf(kQuadEdgeThr * 1.01f, s, -a), t));
    return tab[idx];
  } else {
    constexpr int NB = 1 << (M - 3);
    uint32_t idx = __funnelshift_l(__float_as_uint(x), 0u, 1);
    idx = __funnelshift_l(__float_as_uint(y), idx, 1);
    idx = __funnelshift_l(__float_as_uint(dif), idx, 1);
    float mn_e = INFINITY;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const float e = fmaf(-a, ef_k(M, i), s);
      idx = __funnelshift_l(__float_as_uint(e), idx, 1);
      mn_e = fminf(mn_e, fabsf(e));
    }
    worst = fmaxf(worst, fmaf(ef_band_max<M>(), s, -mn_e));
    return tab[idx];
  }
}

// Table of ef_angle (m >= 3): index = sx sy swap sign(e_0) .. sign(e_NB-1).
// kk = edges the folded point lies above = NB - #(negative e_i); unfold as in
// polar_math.cuh angle_code_fast.  (Non-monotone sign patterns cannot occur
// outside the ambiguity band, which takes the exact path.)
template <int M>
PQB_DEV void ef_build_octant_table(uint8_t* tab, int tid, int nthreads) {
  if constexpr (M == 2) {  // index = sx sy swap tie
    for (int i = tid; i < 16; i += nthreads) {
      const int sx = (i >> 3) & 1, sy = (i >> 2) & 1, swap = (i >> 1) & 1, tie = i & 1;
      uint32_t c;
      if (tie) {
        c = ef_m2_diag(sx ? -1.0f : 1.0f, sy ? -1.0f : 1.0f);
      } else {
        const int base = sx ? (sy ? 0 : 4) : 2;
        c = static_cast<uint32_t>((sx ^ sy) ? base - swap : base + swap) & 3u;
      }
      tab[i] = static_cast<uint8_t>(c);
    }
  } else {
    constexpr int NB = 1 << (M - 3), Q = 1 << (M - 2), H = 2 * Q;
    for (int i = tid; i < (1 << ef_index_bits<M>()); i += nthreads) {
      const int sx = (i >> (NB + 2)) & 1, sy = (i >> (NB + 1)) & 1, swap = (i >> NB) & 1;
      const int kk = NB - __popc(i & ((1 << NB) - 1));
      const int k0 = swap ? Q - kk : kk;
      const int base = sx ? (sy ? 0 : 2 * H) : H;
      const int c = (sx ^ sy) ? base - k0 : base + k0;
      tab[i] = static_cast<uint8_t>(c & (2 * H - 1));
    }
  }
}

// Packed fp32x2 arithmetic (FFMA2 / FMUL2 on sm_100a): two sub-vector pairs per
// instruction, IEEE round-to-nearest per lane.
struct F2 {
  float x, y;
};
PQB_DEV F2 ffma2(F2 a, F2 b, F2 c) {
  F2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
PQB_DEV F2 fadd2(F2 a, F2 b) {
  F2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
PQB_DEV F2 fmul2(F2 a, F2 b) {
  F2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// ef_angle of two pairs with the fp32 arithmetic packed (FADD2 / FFMA2 take the
// |.| and -|.| operand modifiers and broadcast immediates, so |x| +- |y|, the
// edge tests and the band term cost one instruction per two pairs); every
// lane value is the IEEE result of the scalar form, so codes and flags are
// those of ef_angle (which ef_pair_flag re-evaluates).
template <int M>
PQB_DEV void ef_angle2(float x0, float x1, float y0, float y1, float& worst, const uint8_t* tab, uint32_t& c0,
                       uint32_t& c1) {
  const F2 ax{fabsf(x0), fabsf(x1)}, ay{fabsf(y0), fabsf(y1)};
  const F2 s = fadd2(ax, ay);
  const F2 dif = fadd2(ax, F2{-ay.x, -ay.y});
  const F2 a{fabsf(dif.x), fabsf(dif.y)};
  uint32_t i0 = __funnelshift_l(__float_as_uint(x0), 0u, 1), i1 = __funnelshift_l(__float_as_uint(x1), 0u, 1);
  i0 = __funnelshift_l(__float_as_uint(y0), i0, 1);
  i1 = __funnelshift_l(__float_as_uint(y1), i1, 1);
  i0 = __funnelshift_l(__float_as_uint(dif.x), i0, 1);
  i1 = __funnelshift_l(__float_as_uint(dif.y), i1, 1);
  if constexpr (M == 2) {
    const F2 t = fadd2(a, F2{-0x1p-100f, -0x1p-100f});
    i0 = __funnelshift_l(__float_as_uint(t.x), i0, 1);
    i1 = __funnelshift_l(__float_as_uint(t.y), i1, 1);
    const F2 b = ffma2(F2{kQuadEdgeThr * 1.01f, kQuadEdgeThr * 1.01f}, s, F2{-a.x, -a.y});
    worst = fmaxf(worst, fmaxf(fminf(b.x, t.x), fminf(b.y, t.y)));
  } else {
    constexpr int NB = 1 << (M - 3);
    F2 mn{INFINITY, INFINITY};
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const F2 e = ffma2(F2{-a.x, -a.y}, F2{ef_k(M, i), ef_k(M, i)}, s);
      i0 = __funnelshift_l(__float_as_uint(e.x), i0, 1);
      i1 = __funnelshift_l(__float_as_uint(e.y), i1, 1);
      mn.x = fminf(mn.x, fabsf(e.x));
      mn.y = fminf(mn.y, fabsf(e.y));
    }
    const F2 w = ffma2(F2{ef_band_max<M>(), ef_band_max<M>()}, s, F2{-mn.x, -mn.y});
    worst = fmaxf(worst, fmaxf(w.x, w.y));
  }
  c0 = tab[i0];
  c1 = tab[i1];
}

// rint(r / s) of two pairs (fast estimate, polar_math.cuh radius_raw_fast),
// returned biased: t = rq + 1.5 * 2^23 (the packer takes the code from t's low
// mantissa bits).  q + 1.5 * 2^23 rounds q to the nearest integer, ties to
// even, exactly as rintf for 0 <= q < 2^22; two packed adds replace two FRND
// and the packer's per-code add.
// Band: |q - rq| >= 0.5 - 2^-18 q, tested as dq^2 >= 0.25 - 2^-18 q (a
// superset: (0.5 - e)^2 >= 0.25 - e), so worst_r collects dq^2 + 2^-18 q - 0.25.
constexpr float kRqBias = 12582912.0f;  // 1.5 * 2^23
PQB_DEV void ef_radius2(F2 x, F2 y, F2 inv, float& t0, float& t1, float& worst_r, bool& rok) {
  const F2 r2 = ffma2(x, x, fmul2(y, y));
  rok &= in_safe_range_nonneg(r2.x) & in_safe_range_nonneg(r2.y);
  const F2 q = fmul2(fmul2(r2, F2{rsqrt_approx(r2.x), rsqrt_approx(r2.y)}), inv);
  const F2 t = fadd2(q, F2{kRqBias, kRqBias});               // rq + bias
  const F2 rq = fadd2(t, F2{-kRqBias, -kRqBias});            // exact
  const F2 dq = ffma2(rq, F2{-1.0f, -1.0f}, q);  // exact
  const F2 m = ffma2(dq, dq, ffma2(q, F2{0x1p-18f, 0x1p-18f}, F2{-0.25f, -0.25f}));
  worst_r = fmaxf(worst_r, fmaxf(m.x, m.y));
  t0 = t.x;
  t1 = t.y;
}

// Does pair (x, y) sit in an ambiguity band (or outside the safe magnitude
// range)?  Exactly the fast path's arithmetic (FFMA2 / FMUL2 lanes are IEEE
// single operations), so it flags the same pairs the combined metric did.
template <int M>
PQB_DEV bool ef_pair_flag(float x, float y, float inv, const uint8_t* tab) {
  const float r2 = fmaf(x, x, y * y);
  const bool rok = in_safe_range_nonneg(r2);
  const float q = (r2 * rsqrt_approx(r2)) * inv;
  const float rq = rintf(q);
  const float dq = fmaf(rq, -1.0f, q);
  const float m = fmaf(dq, dq, fmaf(q, 0x1p-18f, -0.25f));
  float w = -1.0f;
  (void)ef_angle<M>(x, y, w, tab);
  return !rok || !(fmaxf(w, m) < 0.0f);
}

// Word w (0 <= w < 2B) of a token row of B-bit codes when lane-in-row j holds
// codes 8j .. 8j+7 as chunk c (8B bits).  Shuffles stay inside the row's 8 lanes.
template <int B>
PQB_DEV uint32_t ef_row_word(uint32_t c, int j) {
  if constexpr (B == 4) {
    return c;
  } else if constexpr (B == 2) {
    const uint32_t hi = __shfl_sync(0xffffffffu, c, 2 * j + 1, 8);
    const uint32_t lo = __shfl_sync(0xffffffffu, c, 2 * j, 8);
    return lo | (hi << 16);
  } else {  // B == 3: 24-bit chunks; word j spans chunks a, a + 1
    const int bit = 32 * j, a = bit / 24, o = bit - 24 * a;
    const uint32_t c0 = __shfl_sync(0xffffffffu, c, a & 7, 8);
    const uint32_t c1 = __shfl_sync(0xffffffffu, c, (a + 1) & 7, 8);
    return (c0 >> o) | (c1 << (24 - o));
  }
}

struct EfArgs {
  const void* keys;
  int64_t T;
  int64_t unit_stride;  // elements
  int64_t n_units;
  int64_t items, chunks_per_unit;
  const uint16_t* scales;
  pqb_store st;
  int64_t tok0;  // absolute position of call-token 0 (multiple of 16)
  unsigned long long* clamp_counts;
  int32_t* flags;
};

// Eight codes of B bits per lane of a token row -> the 32-bit chunk, with the
// canonical forms applied.  rt = radius codes biased by 1.5 * 2^23 (ef_radius2).
// Shared by the fast and the exact path.
template <int M, int N>
PQB_DEV void ef_pack(const uint32_t (&ac)[8], const float (&rt)[8], uint32_t keep_a, uint32_t keep_r,
                     float& clamps, uint32_t& ca, uint32_t& cr) {
  constexpr float kTopB = kRqBias + static_cast<float>((1 << N) - 1);
  constexpr uint32_t kMagic = 0x4B400000u;  // bits of 1.5 * 2^23: f + 1.5*2^23 carries int(f) in the low bits
  // sum over the 8 fields of kMagic << (N * i), mod 2^32 (removed after packing)
  constexpr uint32_t kMagicSum = [] {
    uint32_t t = 0;
    for (int i = 0; i < 8; ++i) t += kMagic << (N * i);
    return t;
  }();
  ca = 0u;
  cr = 0u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    clamps += __saturatef(rt[i] - kTopB);  // 1 iff rq >= top + 1 (integers)
    const float rc = fminf(rt[i], kTopB);   // clamped code + bias (exact)
    cr += __float_as_uint(rc) << (N * i);
    if constexpr (M == N) {
      ca += ac[i] << (M * i);
    } else {
      const uint32_t a = rc == kRqBias ? (1u << (M - 1)) : ac[i];  // polar_codec.py:297
      ca += a << (M * i);
    }
  }
  cr -= kMagicSum;
  if constexpr (M == N) {
    // canonical origin angle (polar_codec.py:297) on whole words: fields whose
    // radius code is 0 get angle 2^(M-1)
    constexpr uint32_t kLow = M == 4 ? 0x11111111u : (M == 3 ? 0x00249249u : 0x00005555u);
    uint32_t t = cr | (cr >> 1);
    if constexpr (M >= 3) t |= cr >> 2;
    if constexpr (M == 4) t |= cr >> 3;
    const uint32_t z = (t & kLow) ^ kLow;  // bit 0 of each zero field
    ca = (ca & ~(z * ((1u << M) - 1u))) | (z << (M - 1));
  }
  ca &= keep_a;  // zero-scale channels: both codes 0 (polar_codec.py:298-301)
  cr &= keep_r;
}

// Warp-level persistent kernel.  Warp gw (of W = grid * kEfWarps) encodes items
// gw, gw + W, ...; an item is kEfItemTok consecutive tokens of one unit, read as
// stages of kEfStageTok tokens through the warp's own ring of TMA bulk copies
// (lane 0 produces; no CTA-wide barrier, so a lane on the exact path delays
// only its own warp).  Lane = (row r = lane / 8 of the 4 rows an iteration
// covers, channel group cg = lane % 8).
template <int DT, int LAYOUT, int M, int N>
__global__ void __launch_bounds__(kEfWarps * 32, 1) encode_fast_kernel(const EfArgs p) {
  using Cfg = EfCfg<DT>;
  constexpr int kStageTok = Cfg::kStageTok;
  constexpr int kStagesPerItem = kEfItemTok / kStageTok;
  extern __shared__ __align__(128) uint8_t esm[];
  __shared__ uint64_t bars_all[kEfWarps][kEfStages];
  __shared__ uint8_t octant_tab[64];
  ef_build_octant_table<M>(octant_tab, threadIdx.x, blockDim.x);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 3, cg = lane & 7;
  uint64_t* bars = bars_all[warp];
  uint8_t* ring = esm + warp * (kEfStages * Cfg::kStageBytes);
  const int64_t W = static_cast<int64_t>(gridDim.x) * kEfWarps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kEfWarps + warp;
  const int64_t my_items = p.items > gw ? (p.items - gw + W - 1) / W : 0;
  const int n_stage = static_cast<int>(my_items * kStagesPerItem);  // < 2^31 stages per warp
  if (lane == 0) {
    for (int s = 0; s < kEfStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncwarp();

  // Stage g of this warp = stage g % S of item gw + (g / S) * W; stages past the
  // unit's end are empty.  Incremental cursors: one 64-bit division per item.
  struct Cursor {
    int64_t item, unit, t_item;
    int st;
  };
  auto cursor_item = [&](Cursor& c) {
    c.unit = c.item / p.chunks_per_unit;
    c.t_item = (c.item - c.unit * p.chunks_per_unit) * kEfItemTok;
  };
  auto cursor_next = [&](Cursor& c) {
    if (++c.st == kStagesPerItem) {
      c.st = 0;
      c.item += W;
      cursor_item(c);
    }
  };
  auto stage_rows = [&](const Cursor& c) {
    const int64_t left = p.T - (c.t_item + c.st * kStageTok);
    return left <= 0 ? 0 : (left < kStageTok ? static_cast<int>(left) : kStageTok);
  };
  Cursor pc{gw, 0, 0, 0};  // producer (lane 0)
  cursor_item(pc);
  int p_slot = 0;  // ring slot of the next issue (counters, not divisions: 3 stages)
  auto issue_next = [&]() {
    const int slot = p_slot;
    const int rows = stage_rows(pc);
    if (rows == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + slot)) : "memory");
    } else {
      const uint32_t bytes = static_cast<uint32_t>(rows) * Cfg::kRowBytes;
      mbar_arrive_expect_tx(bars + slot, bytes);
      const uint8_t* src = static_cast<const uint8_t*>(p.keys) +
                           (pc.unit * p.unit_stride + (pc.t_item + pc.st * kStageTok) * 128) *
                               static_cast<int64_t>(DType<DT>::kBytes);
      bulk_g2s(ring + slot * Cfg::kStageBytes, src, bytes, bars + slot);
    }
    p_slot = p_slot + 1 == kEfStages ? 0 : p_slot + 1;
    cursor_next(pc);
  };
  if (lane == 0)
    for (int g = 0; g < kEfStages && g < n_stage; ++g) issue_next();

  int64_t cur_unit = -1;
  float s32[8], inv[8];
  uint32_t keep_a = 0u, keep_r = 0u;  // fields of channels with a non-zero scale
  float clamps = 0.0f;
  bool bad = false;
  auto flush_clamps = [&]() {
    if (cur_unit >= 0 && p.clamp_counts) {
      unsigned int c = static_cast<unsigned int>(clamps);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0 && c) atomicAdd(p.clamp_counts + cur_unit, static_cast<unsigned long long>(c));
    }
    clamps = 0.0f;
  };

  Cursor cc{gw, 0, 0, 0};  // consumer
  cursor_item(cc);
  int64_t pg = 0;  // page of the stage's first token, and its row in the page
  int in_pg0 = 0;
  int slot = 0;
  uint32_t phase = 0;
  for (int g = 0; g < n_stage; ++g, cursor_next(cc)) {
    const int64_t unit = cc.unit, t0 = cc.t_item + cc.st * kStageTok;
    const int rows = stage_rows(cc);
    if (cc.st == 0) {
      const int64_t tok = p.tok0 + t0;
      pg = tok / p.st.page_tokens;
      in_pg0 = static_cast<int>(tok - pg * p.st.page_tokens);
    } else {
      in_pg0 += kStageTok;
      if (in_pg0 == p.st.page_tokens) {
        in_pg0 = 0;
        ++pg;
      }
    }
    if (unit != cur_unit) {  // warp-uniform: flush the clamp count, load this unit's scales
      flush_clamps();
      cur_unit = unit;
      const uint4 sv = __ldg(reinterpret_cast<const uint4*>(p.scales + unit * 64 + 8 * cg));
      const uint32_t w[4] = {sv.x, sv.y, sv.z, sv.w};
      keep_a = keep_r = 0u;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        s32[2 * i] = half_bits_to_f32(static_cast<uint16_t>(w[i] & 0xffffu));
        s32[2 * i + 1] = half_bits_to_f32(static_cast<uint16_t>(w[i] >> 16));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        inv[i] = s32[i] > 0.0f ? __frcp_rn(s32[i]) : 0.0f;
        if (s32[i] > 0.0f) {
          keep_a |= ((1u << M) - 1u) << (M * i);
          keep_r |= ((1u << N) - 1u) << (N * i);
        }
      }
    }
    mbar_wait(bars + slot, phase);
    const int64_t pid = p.st.page_table ? static_cast<int64_t>(__ldg(p.st.page_table + unit * p.st.max_pages + pg))
                                        : unit * p.st.max_pages + pg;
    uint8_t* pb = p.st.pool + pid * p.st.page_bytes;
#pragma unroll 1
    for (int it = 0; it < kStageTok / 4; ++it) {
      const int row = 4 * it + r;
      const bool valid = row < rows;
      uint32_t ca = 0u, cr = 0u;
      float x[8], y[8], rq[8];
      uint32_t ac[8];
      bool need = false;
      if (valid) {
        const uint8_t* rp = ring + slot * Cfg::kStageBytes + row * Cfg::kRowBytes;
        if constexpr (LAYOUT == PQB_HALF_SPLIT) {
          load8s<DT>(rp, 8 * cg, x);
          load8s<DT>(rp, 64 + 8 * cg, y);
        } else {
          float v0[8], v1[8];
          load8s<DT>(rp, 16 * cg, v0);
          load8s<DT>(rp, 16 * cg + 8, v1);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            x[i] = v0[2 * i]; y[i] = v0[2 * i + 1];
            x[4 + i] = v1[2 * i]; y[4 + i] = v1[2 * i + 1];
          }
        }
        float worst = -1.0f, worst_r = -1.0f;
        bool rok = true;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          ef_radius2(F2{x[i], x[i + 1]}, F2{y[i], y[i + 1]}, F2{inv[i], inv[i + 1]}, rq[i], rq[i + 1], worst_r, rok);
          ef_angle2<M>(x[i], x[i + 1], y[i], y[i + 1], worst, octant_tab, ac[i], ac[i + 1]);
        }
        need = !(fmaxf(worst, worst_r) < 0.0f) || !rok;
        if (!need) ef_pack<M, N>(ac, rq, keep_a, keep_r, clamps, ca, cr);
      }
      if (__any_sync(0xffffffffu, need)) {
        // rare (~2% of warp iterations): the exact double-precision pipeline,
        // per pair slot, only for slots some lane flagged (the flags are the
        // fast path's own metrics recomputed bit-identically); zero-scale
        // channels are masked in ef_pack and need no exact work
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const bool f = need && ef_pair_flag<M>(x[i], y[i], inv[i], octant_tab);
          if (__any_sync(0xffffffffu, f)) {
            if (f && s32[i] > 0.0f) {
              bad |= !(fabsf(x[i]) <= 3.40282347e38f && fabsf(y[i]) <= 3.40282347e38f);
              rq[i] = radius_raw_exact(x[i], y[i], s32[i]) + kRqBias;  // biased like ef_radius2
              ac[i] = angle_code_exact(x[i], y[i], M);
            }
          }
        }
        if (need) ef_pack<M, N>(ac, rq, keep_a, keep_r, clamps, ca, cr);
      }
      // ---- the row's 2M angle words and 2N radius words (a stage never
      // straddles a page).  Row-word shuffles run on all lanes.
      const uint32_t wa = ef_row_word<M>(ca, cg), wr = ef_row_word<N>(cr, cg);
      if (valid) {
        const int in_pg = in_pg0 + row;
        if (cg < 2 * M) reinterpret_cast<uint32_t*>(pb + p.st.angle_off + in_pg * 8 * M)[cg] = wa;
        if (cg < 2 * N) reinterpret_cast<uint32_t*>(pb + p.st.radius_off + in_pg * 8 * N)[cg] = wr;
      }
    }
    __syncwarp();  // every lane is done with this slot
    if (lane == 0 && g + kEfStages < n_stage) {
      fence_proxy_async_smem();
      issue_next();
    }
    if (++slot == kEfStages) {
      slot = 0;
      phase ^= 1u;
    }
  }
  flush_clamps();
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.flags, PQB_FLAG_NONFINITE);
}

int ef_num_sms() {
  return device_sms();
}

template <int DT, int LAYOUT, int M, int N>
void launch_ef(const EfArgs& p, cudaStream_t s) {
  using Cfg = EfCfg<DT>;
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    return cudaFuncSetAttribute(encode_fast_kernel<DT, LAYOUT, M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                Cfg::kSmem) == cudaSuccess ? PQB_OK : PQB_ECUDA;
  });
  const int64_t grid = std::min<int64_t>((p.items + kEfWarps - 1) / kEfWarps, ef_num_sms());
  encode_fast_kernel<DT, LAYOUT, M, N><<<static_cast<unsigned>(grid), kEfWarps * 32, Cfg::kSmem, s>>>(p);
}

template <int DT, int LAYOUT>
bool dispatch_ef_mn(const EfArgs& p, int m, int n, cudaStream_t s) {
  switch (m * 10 + n) {
    case 44: launch_ef<DT, LAYOUT, 4, 4>(p, s); return true;
    case 42: launch_ef<DT, LAYOUT, 4, 2>(p, s); return true;
    case 43: launch_ef<DT, LAYOUT, 4, 3>(p, s); return true;
    case 34: launch_ef<DT, LAYOUT, 3, 4>(p, s); return true;
    case 32: launch_ef<DT, LAYOUT, 3, 2>(p, s); return true;
    case 33: launch_ef<DT, LAYOUT, 3, 3>(p, s); return true;
    case 24: launch_ef<DT, LAYOUT, 2, 4>(p, s); return true;
    case 22: launch_ef<DT, LAYOUT, 2, 2>(p, s); return true;
    case 23: launch_ef<DT, LAYOUT, 2, 3>(p, s); return true;
    default: return false;
  }
}

}  // namespace

// The persistent fast encoder when the call qualifies; false -> caller uses encode_v8.
bool launch_encode_fast(const EncodeArgs& a, cudaStream_t s) {
  const pqb_store& st = *a.store;
  const int eb = a.key_dtype == PQB_F32 ? 4 : 2;
  const bool ok = a.vector_ok && a.d == 128 && a.tok_stride == 128 && a.tok_offset == nullptr &&
                  a.tok_offset_const % kEfAlign == 0 && st.page_tokens % kEfAlign == 0 &&
                  reinterpret_cast<uintptr_t>(a.keys) % 16 == 0 && (a.unit_stride * eb) % 16 == 0 &&
                  reinterpret_cast<uintptr_t>(a.scales) % 16 == 0 && a.angle_bits >= 2 && a.angle_bits <= 4 &&
                  a.radius_bits >= 2 && a.radius_bits <= 4 && st.angle_off % 4 == 0 && st.radius_off % 4 == 0 &&
                  st.page_bytes % 4 == 0 && reinterpret_cast<uintptr_t>(st.pool) % 4 == 0;
  if (!ok || a.tokens == 0 || a.n_units == 0) return false;
  EfArgs p;
  p.keys = a.keys;
  p.T = a.tokens;
  p.unit_stride = a.unit_stride;
  p.n_units = a.n_units;
  p.chunks_per_unit = (a.tokens + kEfItemTok - 1) / kEfItemTok;
  p.items = a.n_units * p.chunks_per_unit;
  p.scales = a.scales;
  p.st = st;
  p.tok0 = a.tok_offset_const;
  p.clamp_counts = a.clamp_counts;
  p.flags = a.flags;
  const int m = a.angle_bits, n = a.radius_bits;
  switch (a.key_dtype * 2 + a.layout) {
    case PQB_F32 * 2 + PQB_ADJACENT: return dispatch_ef_mn<PQB_F32, PQB_ADJACENT>(p, m, n, s);
    case PQB_F32 * 2 + PQB_HALF_SPLIT: return dispatch_ef_mn<PQB_F32, PQB_HALF_SPLIT>(p, m, n, s);
    case PQB_BF16 * 2 + PQB_ADJACENT: return dispatch_ef_mn<PQB_BF16, PQB_ADJACENT>(p, m, n, s);
    case PQB_BF16 * 2 + PQB_HALF_SPLIT: return dispatch_ef_mn<PQB_BF16, PQB_HALF_SPLIT>(p, m, n, s);
    case PQB_F16 * 2 + PQB_ADJACENT: return dispatch_ef_mn<PQB_F16, PQB_ADJACENT>(p, m, n, s);
    default: return dispatch_ef_mn<PQB_F16, PQB_HALF_SPLIT>(p, m, n, s);
  }
}

}  // namespace pqb
