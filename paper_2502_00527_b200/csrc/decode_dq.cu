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

// the product-table layout (see kPtTabAbs below); before DqCfg, which sizes by it.
// The library carries both builds: this file (PRMT table, namespace dq_prmt)
// and decode_dq_lin.cu (the same source with the linear layout, dq_lin), the
// runtime fallback when the shared window is laid out other than measured.
#ifndef PQB_DQ_PRMT_TAB
#define PQB_DQ_PRMT_TAB 1
#endif
#if PQB_DQ_PRMT_TAB
#define PQB_DQ_NS dq_prmt
#else
#define PQB_DQ_NS dq_lin
#endif

namespace pqb {
namespace PQB_DQ_NS {

// Warp specialisation: a fourth warpgroup of producers (warp kNW + j fills the
// rings of compute warps j and j + 4, which share its SM sub-partition) takes
// the TMA issue code off the compute warps; registers are rebalanced with
// setmaxnreg (compute warps 232, producers 40: 2 x 128 x 232 + 128 x 40 <= 64K).
// PQB_DQ_WS=0 builds the previous layout (lane 0 of each compute warp issues).
// mbarrier waits with a suspend-time hint (common.cuh mbar_wait_sleep) for the
// producers' empty-slot waits and the compute warps' full-slot waits
#ifndef PQB_DQ_SLEEP_PROD
#define PQB_DQ_SLEEP_PROD 1
#endif
#ifndef PQB_DQ_PHI_BF16  // G = 8 bf16 values with bf16 outputs: the kDqBf16P instances (A/B: 0 keeps hi + lo)
#define PQB_DQ_PHI_BF16 1
#endif
#ifndef PQB_DQ_PHI_BF16_G4  // the same at G = 4: P_lo is free in the MMA there, but its computation and
                            // packing shuffles are not (configs[1] +1.5 %, scripts/gpu_g4phi_ab.sh)
#define PQB_DQ_PHI_BF16_G4 1
#endif
#ifndef PQB_DQ_FULL_TILE  // softmax of a tile wholly inside the sequence without per-token bound tests
                          // (configs[1] sustained +0.8 %, value unchanged: scripts/gpu_bench_ab.sh)
#define PQB_DQ_FULL_TILE 1
#endif
#ifndef PQB_DQ_TWO_CHAINS  // two MMA accumulation chains per n-block in the QK block (m4n4, bf16 values);
                           // with the bf16-P instances one chain measures better (configs[3] 0.886 -> 0.897,
                           // configs[1] value +1 %, sustained equal: scripts/gpu_abcd.sh)
#define PQB_DQ_TWO_CHAINS 0
#endif
#ifndef PQB_DQ_SLEEP_CONS
#define PQB_DQ_SLEEP_CONS 1
#endif
#ifndef PQB_DQ_WS
#define PQB_DQ_WS 1
#endif
#ifndef PQB_DQ_CONS_REGS
#define PQB_DQ_CONS_REGS 232
#define PQB_DQ_PROD_REGS 40
#endif
// setmaxnreg.inc blocks until the CTA's own pool (168 x 384 allocated at launch)
// has the registers the producers released: two compute warpgroups may grow by
// no more than the producer warpgroup shrinks, or the kernel deadlocks (240/32
// does: 2 x 72 > 136).
static_assert(2 * (PQB_DQ_CONS_REGS - 168) <= 168 - PQB_DQ_PROD_REGS, "setmaxnreg budget exceeds the CTA pool");
constexpr bool kDqWs = PQB_DQ_WS != 0;
constexpr int kDqThreads = kDqWs ? (kNW + 4) * 32 : kNW * 32;
constexpr int kConsThreads = kNW * 32;
static_assert(!kDqWs || kNW == 8, "producer j serves compute warps j and j + 4");

// Value-cache treatments (template parameter VQ): the page's value region as
// the decode kernel streams it.
constexpr int kValBf16 = 0;  // bf16 rows, tensor-core P.V (hi/lo P)
constexpr int kValVq4 = 1;   // PQB_VQ4: 4-bit per-token codes + (zp, scale), tensor-core P.V
constexpr int kValF32 = 2;   // PQB_F32: the reference's default fp32 rows (kv_cache.py:8-9, :209), CUDA-core P.V
constexpr int kValVq2 = 3;   // PQB_VQ2: 2-bit codes, as kValVq4
constexpr int kValVq8 = 4;   // PQB_VQ8: 8-bit codes as two nibble planes, two MMAs per fragment
constexpr bool val_is_vq(int v) { return v == kValVq4 || v == kValVq2 || v == kValVq8; }
constexpr int val_vq_bits(int v) { return v == kValVq2 ? 2 : v == kValVq8 ? 8 : 4; }

template <int G, int M, int N, int VQ = 0>
struct DqCfg {
  static constexpr int kABytes = kTile * 8 * M;
  static constexpr int kRBytes = kTile * 8 * N;
  // bf16 value rows, 2 KB of fragment-order 4-bit codes + 32 (zp, scale), or fp32 rows
  static constexpr int kVqCodeBytes = 512 * val_vq_bits(VQ);  // a tile's value codes (quantized modes)
  static constexpr int kVBytes = val_is_vq(VQ) ? kVqCodeBytes + kTile * 8 : VQ == kValF32 ? kTile * 512 : kTile * 256;
  static constexpr int kStageBytes = kABytes + kRBytes + kVBytes;
  // stages per compute warp: fp32 rows make an 18 KB stage, so one per warp
  // (8 in flight per SM, double the bytes of the bf16 ring's 16 x 10 KB)
  static constexpr int kSt = VQ == kValF32 ? 1 : kStages;
  static constexpr int kPBytes = kTile * 8 * 4;              // fp32 [32 tokens][8 queries] residual-dot scratch
  static constexpr int kTabBytes = 128 << (M + N);          // product table, 16 bank-slot copies
  static constexpr int kFragBytes = 16 * 32 * 16;            // Q' A-fragments [ks][lane] uint4 (hi, lo, hi, lo)
  static constexpr int kHeadBytes = kTabBytes + kFragBytes + G * 128 * 4 + 128 + 8 * (1 << M);
  static constexpr int kWarpBytes = kSt * kStageBytes + kPBytes;
#if PQB_DQ_PRMT_TAB
  // the whole opt-in budget minus the 256 B of static barriers; the kernel
  // checks that its stages fit around the table
  static constexpr int kSmem = 232448 - 256;
#else
  static constexpr int kSmem = kHeadBytes + kNW * kWarpBytes + 128;
#endif
  static constexpr bool kPacked = G <= 4;  // P.V: columns 0-3 carry P_hi, 4-7 P_lo
  static_assert(kHeadBytes % 16 == 0 && kWarpBytes % 16 == 0, "alignment");
  static_assert(kNW * kSt * kStageBytes >= kNW * G * 132 * 4, "merge area");
};

// PQB_DQ_UMMA=1 (A/B build): P.V of the G = 4 bf16-value kernel on the 5th-
// generation tensor cores instead of mma.sync.  The four compute warps of a
// warpgroup score their tiles as before and share one online-softmax reference
// max (exchanged through shared memory, raised lazily: only when a tile max
// exceeds it by more than 2^8, so P <= 256); each warp writes its P^T (bf16 hi
// | lo columns) as K-major core matrices, and one elected thread issues
//   O^T[128 dims x 8] += V^T[128 x 128 tokens] . P^T[128 x 8]
// as 8 tcgen05.mma (M 128, N 8, K 16) straight from the warps' TMA-filled value
// stages (the grouped value layout is the 128-byte-swizzled MN-major
// canonical form), accumulating in tensor memory.  A stage is released once
// the MMAs reading it commit (next round); O is read back with tcgen05.ld at
// the end of the segment and rescaled there when the reference max rises.
#ifndef PQB_DQ_UMMA
#define PQB_DQ_UMMA 0
#endif
constexpr int kGapUmmaB = 164;    // 64 slots: P^T core matrices [wg][parity][warp][chunk]
constexpr int kGapUmmaMisc = 228;  // tile maxes, row sums, stage addresses, mbarriers, TMEM base
constexpr float kUmmaTau = 8.0f;
#ifndef PQB_DQ_UMMA_RELEASE
#define PQB_DQ_UMMA_RELEASE 1  // the issuing lane waits for the round's MMAs and releases the 4 stages at once
#endif   // lazy max: rescale only when a tile max exceeds the reference by > 2^8

// PQB_DQ_TRACE=1 (probe builds only): consumer thread 0 of every CTA stamps
// %globaltimer at the launch phases into pqb_dq_trace[cta][32] (read back by
// pqb_debug_dq_trace; scripts/trace_probe.py): [0] entry, [1] after the grid
// dependency wait, per segment k < 6: [2+4k] unit setup done, [3+4k] tile loop
// done, [4+4k] epilogue (incl. a last-CTA merge) done, [5+4k] unit; [31] exit.
#ifndef PQB_DQ_TRACE
#define PQB_DQ_TRACE 0
#endif
#if PQB_DQ_TRACE
__device__ unsigned long long pqb_dq_trace[1024 * 32];
PQB_DEV void trace_stamp(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  pqb_dq_trace[blockIdx.x * 32 + slot] = t;
}
#define DQ_TRACE(cond, slot) \
  do {                       \
    if (cond) trace_stamp(slot); \
  } while (0)
#else
#define DQ_TRACE(cond, slot) \
  do {                       \
  } while (0)
#endif

PQB_DEV uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// PQB_DQ_PRMT_TAB=1 (default; A/B +1.3% G = 4, +2.9% G = 8, all decode tests
// green; 0 builds the previous layout): the product table sits at shared-window
// address 0x10000 in 256 slots of 256 B (slot e's first 128 B = entry e's 16
// bank-slot copies), so one PRMT composes a gather address from the index
// byte, the lane's copy offset and the table base (no add); the slots' second
// halves hold the small buffers (GapArr), the stages sit before and after the
// table (scripts/micro/smem_base.cu: 1 KB reserved, static from 0x400).
constexpr uint32_t kPtTabAbs = 0x10000;
template <typename T>
struct GapArr {
  static constexpr int kPer = 128 / sizeof(T);
  uint8_t* tab;
  int g0;
  PQB_DEV T& operator[](int i) const { return reinterpret_cast<T*>(tab + (g0 + i / kPer) * 256 + 128)[i % kPer]; }
};
constexpr int kGapQfrag = 0, kGapQ = 64, kGapRbuf = 96, kGapMisc = 160, kGapCs = 161, kGapScale = 162;

PQB_DEV void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Lane t4 owns channel pairs [16 t4, 16 t4 + 16) of every token; k-step ks
// contracts pair 16 t4 + dq_pair(ks).  For m = n = 4 the order follows the
// nibble fusion below (even pairs of a word, then odd); for m = 3, n = 2 the
// SWAR byte spread (byte b of word j = pair 4b + j, k-step 4j + b); else ks.
template <int M, int N>
PQB_DEV constexpr int dq_pair(int ks) {
  return (M == 4 && N == 4) ? ((ks >> 2) & 1) + 2 * (ks & 3) + 8 * (ks >> 3)
         : (M == 3 && N == 2 && PQB_DQ_PRMT_TAB) ? 4 * (ks & 3) + (ks >> 2)
                                                 : ks;
}

// B bits starting at bit b of the little-endian word array x (b compile-time
// after unrolling).
template <int B>
PQB_DEV uint32_t bits_at(const uint32_t* x, int b) {
  const int w = b >> 5, s = b & 31;
  const uint32_t v = (s + B <= 32) ? (x[w] >> s) : __funnelshift_r(x[w], x[w + 1], s);
  return v & ((1u << B) - 1u);
}

// The lane's 16 codes of B bits (stream bits [16 t4 B, 16 t4 B + 16 B) of the
// token row), right-aligned into x[0..].  16 t4 B is a multiple of 16 bits.
template <int B>
PQB_DEV void load_lane_codes(const uint8_t* row, int t4, uint32_t (&x)[(B + 1) / 2 + 1]) {
  constexpr int kW = (B + 1) / 2 + 1;
  const int bit0 = 16 * t4 * B;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row) + (bit0 >> 5);
  if constexpr (B % 2 == 0) {  // word aligned
#pragma unroll
    for (int k = 0; k < B / 2; ++k) x[k] = w[k];
    x[kW - 1] = 0u;
  } else {
    uint32_t r[kW];
#pragma unroll
    for (int k = 0; k < kW; ++k) r[k] = w[k];
    const int sh = bit0 & 31;  // 0 or 16
#pragma unroll
    for (int k = 0; k < kW - 1; ++k) x[k] = __funnelshift_r(r[k], r[k + 1], sh);
    x[kW - 1] = 0u;
  }
}

// Product-table indices idx = (a << N) | r of the lane's 16 pairs of one token.
// For m = n = 4 they stay packed: byte k of w[q] is the index of k-step 4q + k
// (w = e0, o0, e1, o1 with e = (a_even << 4) | r_even, o = (a_odd << 4) | r_odd);
// otherwise w[ks] is the index itself.  live = false (a residual or past-the-end
// token) forces radius code 0, i.e. the zero key.
template <int M, int N>
struct DqIdx {
  static constexpr bool kFused = M == 4 && N == 4;
  static constexpr bool kSwar = M == 3 && N == 2 && PQB_DQ_PRMT_TAB;  // byte-spread indices, PRMT addressing
  uint32_t w[kFused || kSwar ? 4 : 16];
  PQB_DEV void load(const uint8_t* arow, const uint8_t* rrow, int t4, bool live) {
    if constexpr (kFused) {
      const uint2 a = *reinterpret_cast<const uint2*>(arow + 8 * t4);
      uint2 r = *reinterpret_cast<const uint2*>(rrow + 8 * t4);
      if (!live) r = make_uint2(0u, 0u);
      w[0] = ((a.x << 4) & 0xF0F0F0F0u) | (r.x & 0x0F0F0F0Fu);
      w[1] = (a.x & 0xF0F0F0F0u) | ((r.x >> 4) & 0x0F0F0F0Fu);
      w[2] = ((a.y << 4) & 0xF0F0F0F0u) | (r.y & 0x0F0F0F0Fu);
      w[3] = (a.y & 0xF0F0F0F0u) | ((r.y >> 4) & 0x0F0F0F0Fu);
    } else if constexpr (kSwar) {
      // 16 pairs: angle a_k at bits 3k of 48, radius r_k at bits 2k of 32; byte b
      // of w[j] = (a_{4b+j} << 2) | r_{4b+j}
      uint32_t xa[3];
      load_lane_codes<3>(arow, t4, xa);  // bits 0..47 valid (xa[1] bits 16+ belong to the next lane)
      uint32_t R = reinterpret_cast<const uint32_t*>(rrow)[t4];
      if (!live) R = 0u;
      const uint32_t E = R & 0x33333333u, O = (R >> 2) & 0x33333333u;  // r_{2i} / r_{2i+1} in nibble i
      const uint32_t rw[4] = {E & 0x0F0F0F0Fu, O & 0x0F0F0F0Fu, (E >> 4) & 0x0F0F0F0Fu, (O >> 4) & 0x0F0F0F0Fu};
      // 12-bit groups g_b = a_{4b..4b+3}: P0 = g0 | g2 << 16, P1 = g1 | g3 << 16 (stray
      // bits land at 12-15 / 28-31, outside every field mask below)
      const uint32_t t24 = __funnelshift_r(xa[0], xa[1], 24);
      const uint32_t P0 = (xa[0] & 0xFFFu) | ((t24 << 16) & 0x0FFF0000u);
      const uint32_t P1 = ((xa[0] >> 12) & 0xFFFu) | ((xa[1] << 12) & 0x0FFF0000u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t lo = (P0 >> (3 * j)) & 0x00070007u;                                   // bytes 0, 2
        const uint32_t hi = (j < 3 ? (P1 << (8 - 3 * j)) : (P1 >> 1)) & 0x07000700u;        // bytes 1, 3
        w[j] = ((lo | hi) << 2) | rw[j];
      }
    } else {
      uint32_t xa[(M + 1) / 2 + 1], xr[(N + 1) / 2 + 1];
      load_lane_codes<M>(arow, t4, xa);
      load_lane_codes<N>(rrow, t4, xr);
      if (!live) {
#pragma unroll
        for (int k = 0; k < (N + 1) / 2 + 1; ++k) xr[k] = 0u;
      }
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) w[ks] = (bits_at<M>(xa, ks * M) << N) | bits_at<N>(xr, ks * N);
    }
  }
  // shared address of the k-step ks entry in the lane's table copy
  PQB_DEV uint32_t addr(uint32_t tab, int ks) const {
#if PQB_DQ_PRMT_TAB
    // tab = kPtTabAbs | lane copy offset: the absolute address in one PRMT
    if constexpr (kFused || kSwar) return __byte_perm(w[ks >> 2], tab, 0x7604u | ((ks & 3) << 4));
    else return tab + (w[ks] << 8);
#else
    if constexpr (kFused) return tab + (__byte_perm(w[ks >> 2], 0u, 0x4440u | (ks & 3)) << 7);
    else return tab + (w[ks] << 7);
#endif
  }
};

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp, results below 2^-126 flush to 0;
// exp2f's range fix-up would add three instructions per call)
PQB_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

PQB_DEV uint2 lds_u2(uint32_t addr) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
// PROBE: 0 = the kernel; kDqBf16P = the kernel with bf16-P P.V (G = 4 / 8, bf16 outputs);
// kDqScores = scores-only mode (qk_scores within the
// stated tolerance, lut_decode.py:119-154: the QK contraction of the fused
// kernel, the raw fp32 score rows stored, no softmax / values; only the code
// bytes are streamed).  Diagnostics (flags PQB_DECODE_PROBE_*): 1 = memory only
// (tiles stream through the ring, no compute); 2 = compute only (every tile is
// re-read from the unit's first page, i.e. from L2).
// VQ: PQB_VQ4 value pages (kv_cache.py:199-209 quantize_values): the P.V MMA
// takes the 4-bit codes as exact bf16 integers (A) against P * scale (B, hi/lo),
// and the zero points join as sum_t p_t zp_t per query:
//   o = sum_t p_t (c_t s_t + z_t) = [codes] . (p s) + sum_t p_t z_t.
constexpr int kDqScores = 3;
constexpr int kDqBf16P = 4;  // the kernel with bf16-P P.V (G = 4 / 8, bf16 values, bf16 outputs)

template <int M, int N, int VQ, bool CODES_ONLY = false>
PQB_DEV void issue_tile_dq(uint8_t* st, const pqb_store& s, const uint8_t* pb, int tin, uint64_t* bar) {
  // tin: tile index within the page (tokens tin * 32 ...)
  constexpr uint32_t kA = kTile * 8 * M, kR = kTile * 8 * N;
  const int in_page = tin * kTile;
  if constexpr (CODES_ONLY) {
    mbar_arrive_expect_tx(bar, kA + kR);
    bulk_g2s(st, pb + s.angle_off + in_page * 8 * M, kA, bar);
    bulk_g2s(st + kA, pb + s.radius_off + in_page * 8 * N, kR, bar);
  } else if constexpr (VQ == kValBf16 || VQ == kValF32) {
    constexpr uint32_t kRow = VQ == kValF32 ? 512 : 256, kV = kTile * kRow;
    mbar_arrive_expect_tx(bar, kA + kR + kV);
    bulk_g2s(st, pb + s.angle_off + in_page * 8 * M, kA, bar);
    bulk_g2s(st + kA, pb + s.radius_off + in_page * 8 * N, kR, bar);
    bulk_g2s(st + kA + kR, pb + s.value_off + static_cast<int64_t>(in_page) * kRow, kV, bar);
  } else {
    constexpr uint32_t kC = 512 * val_vq_bits(VQ);
    mbar_arrive_expect_tx(bar, kA + kR + kC + kTile * 8);
    bulk_g2s(st, pb + s.angle_off + in_page * 8 * M, kA, bar);
    bulk_g2s(st + kA, pb + s.radius_off + in_page * 8 * N, kR, bar);
    bulk_g2s(st + kA + kR, pb + s.value_off + static_cast<int64_t>(tin) * kC, kC, bar);
    bulk_g2s(st + kA + kR + kC, pb + s.value_off + static_cast<int64_t>(s.page_tokens) * (kC / kTile) + in_page * 8,
             kTile * 8, bar);
  }
}

// Lane 0's cursor over this warp's tiles (first, first + kNW, ...): page and
// tile-in-page advanced incrementally (a division per segment, not per tile).
struct TileCursor {
  int tile, pg, tin;
  PQB_DEV void init(int t, int tpp) {
    tile = t;
    pg = t / tpp;
    tin = t - pg * tpp;
  }
  PQB_DEV void next(int dpg, int dtin, int tpp) {
    tile += kNW;
    pg += dpg;
    tin += dtin;
    if (tin >= tpp) {
      tin -= tpp;
      ++pg;
    }
  }
};

// ---- thread-block cluster: the split merge of a unit's K CTAs through
// distributed shared memory (decode_dq_kernel CL > 1).
PQB_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
PQB_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
PQB_DEV float ld_dsmem(const float* local, uint32_t rank) {  // the same smem offset in CTA `rank` of the cluster
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// End of the single segment of a cluster CTA (aligned split: the K CTAs of a
// cluster cut one unit into K equal ranges).  The CTA merges its warps into
// cpart[g][130] (m, l, o[128]; the arithmetic of finish_segment), then, after
// a cluster barrier, CTA rank r LSE-merges the K partials of dims
// [r 128 / K, (r + 1) 128 / K) read from its peers' shared memory, in rank
// order (merge_slots' arithmetic: outputs bit-identical to the global-slot
// merge of the same split), and stores the output.  No partials in global
// memory, no counter, no merge launch.  A second cluster barrier keeps every
// CTA's partial alive until its peers have read it.  Callers: all consumer
// threads (the producers only join the two cluster barriers).
template <int G, int K>
PQB_DEV void finish_cluster(const EpiArgs& ep, int64_t unit, const float* red, float* cpart, int tid, int nthreads) {
  static_assert(K >= 2 && K <= 8 && 128 % K == 0, "cluster size");
  named_sync(1, nthreads);
  for (int i = tid; i < G * 128; i += nthreads) {
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
    cpart[g * 130 + 2 + e] = O;
    if (e == 0) {
      cpart[g * 130] = mx;
      cpart[g * 130 + 1] = L;
    }
  }
  cluster_sync_all();
  constexpr int kSlice = 128 / K;
  const int e0 = static_cast<int>(cluster_rank()) * kSlice;
  for (int i = tid; ep.merge && i < G * kSlice; i += nthreads) {  // (!merge: PQB_DECODE_NO_COMBINE timing)
    const int g = i / kSlice, e = e0 + i % kSlice;
    float ms[K], ls[K], os[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      ms[k] = ld_dsmem(cpart + g * 130, k);
      ls[k] = ld_dsmem(cpart + g * 130 + 1, k);
      os[k] = ld_dsmem(cpart + g * 130 + 2 + e, k);
    }
    float mx = -INFINITY, L = 0.0f, O = 0.0f;
    float bm = mx;
#pragma unroll
    for (int k = 0; k < K; ++k) bm = fmaxf(bm, ms[k]);
    if (bm != -INFINITY) {
      const float r = exp2f(mx - bm);
      L *= r;
      O *= r;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (ms[k] == -INFINITY) continue;
        const float sc = exp2f(ms[k] - bm);
        L = fmaf(ls[k], sc, L);
        O = fmaf(os[k], sc, O);
      }
    }
    emit(ep, unit, g, e, O / L);
  }
  cluster_sync_all();
}

template <int G, int M, int N, int PROBE = 0, int VQ = 0, int CL = 0>
__global__ void __launch_bounds__(kDqThreads, 1)
    decode_dq_kernel(const pqb_cache c, const void* __restrict__ q, int q_dtype, float sm_scale_log2, EpiArgs ep,
                     WorkSplit ws, float* __restrict__ scores, int64_t scores_ld) {
  using Cfg = DqCfg<G, M, N, VQ>;
  constexpr int kSt = Cfg::kSt;
  constexpr bool kVq4 = val_is_vq(VQ), kVf32 = VQ == kValF32;  // kVq4: any quantized value mode
  constexpr int kVqB = val_vq_bits(VQ);
  constexpr float kVqMid = kVqB == 8 ? 128.0f : kVqB == 4 ? 7.0f : 1.0f;  // ~ half the code range
  constexpr bool kScores = PROBE == kDqScores;
  // bf16 outputs (bf16 values): P.V on bf16 P without its lo part -- at G = 8 one
  // MMA per k-step instead of two, at G = 4 (P_lo rides in the hi MMA's spare
  // columns) no P_lo conversion and packing shuffles; |dO| <= 2^-9 sum_t p_t |v_t|,
  // at the output's own bf16 rounding
  constexpr bool kPhiOnly = PROBE == kDqBf16P;
  static_assert(!kPhiOnly || (VQ == kValBf16 && (G == 8 || G == 4)), "bf16-P instance: G = 4 / 8, bf16 values");
  constexpr bool kFused = M == 4 && N == 4;
  constexpr bool kPacked = Cfg::kPacked;
  // (m = n = 4: the codes take 2 KB of the 10 KB stage, so value tiles stay 1 KB aligned)
  constexpr bool kUmma = PQB_DQ_UMMA && PQB_DQ_PRMT_TAB && VQ == kValBf16 && G == 4 && M == 4 && N == 4 && PROBE == 0;
  static_assert(G == 1 || G == 2 || G == 4 || G == 8, "G");
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  DQ_TRACE(tid == 0, 0);
#if PQB_DQ_PRMT_TAB
  // (in a cluster launch CTA rank r's shared window starts at r << 24, scripts/micro/smem_base_cluster.cu;
  // the PRMT-composed gather address keeps that top byte)
  const uint32_t tab_abs = (smem_u32(smem) & 0xFF000000u) | kPtTabAbs;
  const int tab_off = static_cast<int>(tab_abs - smem_u32(smem));  // dynamic offset of the table
  // UMMA: value tiles 1 KB aligned (the 128-byte swizzle pattern is taken from address bits 7-9)
  const int st_pad = kUmma ? static_cast<int>((1024u - (smem_u32(smem) & 1023u)) & 1023u) : 0;
  const int n_before = (tab_off - st_pad) / Cfg::kStageBytes;          // stages before the table
  uint8_t* const tabp = smem + tab_off;
  uint2* ptab = reinterpret_cast<uint2*>(tabp);  // entry e at slot e (e * 32 uint2)
  const GapArr<uint4> qfrag{tabp, kGapQfrag};
  const GapArr<float> q_s{tabp, kGapQ};
  int* s_misc = reinterpret_cast<int*>(tabp + kGapMisc * 256 + 128);
  float2* cs_s = reinterpret_cast<float2*>(tabp + kGapCs * 256 + 128);
  const GapArr<float> s_scale{tabp, kGapScale};  // 64 floats: two gaps
  auto stage_ptr = [&](int i) -> uint8_t* {
    return smem + (i < n_before ? st_pad + i * Cfg::kStageBytes : tab_off + 65536 + (i - n_before) * Cfg::kStageBytes);
  };
  uint8_t* warp_area = smem;  // merge scratch aliases the first stages (all before the table)
  if (tid == 0 && (tab_off < 0 || n_before * Cfg::kStageBytes < kNW * G * 132 * 4 ||
                   tab_off + 65536 + (kNW * kSt - n_before) * Cfg::kStageBytes > Cfg::kSmem))
    __trap();  // shared-window layout other than measured: the table cannot sit at kPtTabAbs
  const GapArr<float> rbuf{tabp, kGapRbuf + 8 * (warp < kNW ? warp : 0)};
  uint8_t* const um_b = tabp + kGapUmmaB * 256 + 128;      // P^T core matrix k at um_b + 256 k
  float* const um_max = reinterpret_cast<float*>(tabp + kGapUmmaMisc * 256 + 128);        // [2][4][4]
  float* const um_l = reinterpret_cast<float*>(tabp + (kGapUmmaMisc + 1) * 256 + 128);    // [2][4][4]
  uint32_t* const um_va = reinterpret_cast<uint32_t*>(tabp + (kGapUmmaMisc + 2) * 256 + 128);  // [2][4]
  uint64_t* const um_bar = reinterpret_cast<uint64_t*>(um_va + 16);  // [2][2] (um_va: [2][4] addresses, [2][4] stages)
  uint32_t* const um_tmem = reinterpret_cast<uint32_t*>(um_bar + 4);
#else
  uint8_t* const um_b = smem;  // (the UMMA variant needs the PRMT layout's gap slots)
  float* const um_max = nullptr;
  float* const um_l = nullptr;
  uint32_t* const um_va = nullptr;
  uint64_t* const um_bar = nullptr;
  uint32_t* const um_tmem = nullptr;
  uint2* ptab = reinterpret_cast<uint2*>(smem);                                   // [2^(M+N)][16]
  uint4* qfrag = reinterpret_cast<uint4*>(smem + Cfg::kTabBytes);                    // [16][32]
  float* q_s = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(qfrag) + Cfg::kFragBytes);  // [G][128]
  int* s_misc = reinterpret_cast<int*>(q_s + G * 128);  // [0] max|Q'| bits, [1] merge flag
  float2* cs_s = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(s_misc) + 128);  // [2^M] (cos, sin)
  uint8_t* warp_area = smem + Cfg::kHeadBytes;
  auto stage_ptr = [&](int i) -> uint8_t* {
    return warp_area + (i / kSt) * Cfg::kWarpBytes + (i % kSt) * Cfg::kStageBytes;
  };
  float* rbuf = reinterpret_cast<float*>(warp_area + (warp < kNW ? warp : 0) * Cfg::kWarpBytes +
                                         kSt * Cfg::kStageBytes);  // [32][8]
#endif
  // mbarriers live outside the warp areas: the end-of-segment merge scratch
  // (red, G * 132 floats per warp) aliases the stage memory and, at G = 8,
  // would run over warp 0's barriers if they sat behind its stages
  __shared__ uint64_t s_bar[kNW][kStages];    // stage full (TMA transaction count)
  __shared__ uint64_t s_empty[kNW][kStages];  // stage released by its compute warp (WS)
#if !PQB_DQ_PRMT_TAB
  __shared__ float s_scale[64];  // the current unit's radius scales
#endif
  uint64_t* bar = s_bar[warp < kNW ? warp : 0];
  if (lane == 0 && warp < kNW) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar + s, 1);
      mbar_init(&s_empty[warp][s], 1);
    }
    fence_mbar_init();
  }
  if constexpr (kUmma) {  // MMA-completion barriers and 32 columns of tensor memory (2 x 8 used)
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mbar_init(um_bar + k, 1);
      fence_mbar_init();
    }
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(um_tmem))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
  }
  // product table (once per CTA): PT[(a << N) | r][copy] = (r cos_a, r sin_a) as fp16 hi + lo
  if (tid == 0) s_misc[0] = 0;
  if (tid < (1 << M)) {
    float cf, sf;
    angle_unit(M, tid, cf, sf);
    cs_s[tid] = make_float2(cf, sf);
  }
  __syncthreads();
  // one entry per thread, its 16 bank-slot copies as 8 x 16-byte stores
  for (int e = tid; e < (1 << (M + N)); e += blockDim.x) {
    const int a = e >> N, r = e & ((1 << N) - 1);
    const float2 cs = cs_s[a];
    const double x = static_cast<double>(r) * cs.x, y = static_cast<double>(r) * cs.y;  // exact products
    const __half xh = __float2half_rn(static_cast<float>(x)), yh = __float2half_rn(static_cast<float>(y));
    const uint32_t hi = h2_bits(__halves2half2(xh, yh));
    const uint32_t lo = h2_bits(__halves2half2(__float2half_rn(static_cast<float>(x - __half2float(xh))),
                                               __float2half_rn(static_cast<float>(y - __half2float(yh)))));
    uint4* dst = reinterpret_cast<uint4*>(ptab + e * (PQB_DQ_PRMT_TAB ? 32 : 16));
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[k] = make_uint4(hi, lo, hi, lo);
  }
  if constexpr (kDqWs) __syncthreads();  // producers helped build the table
  uint32_t tmem_base = 0;
  if constexpr (kUmma) {
    tc_fence_after();
    tmem_base = *um_tmem;
  }
  uint32_t u_round = 0;  // UMMA: this warpgroup's P.V rounds so far (mbarrier phases)
#if PQB_DQ_PRMT_TAB
  const uint32_t ptab_l = tab_abs | ((lane & 15) << 3);  // this lane's bank-slot copy
#else
  const uint32_t ptab_l = smem_u32(smem) + ((lane & 15) << 3);  // this lane's bank-slot copy
#endif
  // Programmatic dependent launch: everything above uses constants only; the
  // cache, q and the outputs may belong to the previous kernel in the stream.
  // Let the next launch start its own prologue as SMs drain, then wait for
  // this grid's predecessors to complete.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  DQ_TRACE(tid == 0, 1);
  const int tpp = c.store.page_tokens / kTile;  // tiles per page
  const int dpg = kNW / tpp, dtin = kNW - (kNW / tpp) * tpp;  // cursor step of kNW tiles
  const int64_t i_begin = cta_begin(ws, blockIdx.x);
  const int64_t i_end = cta_end(ws, blockIdx.x);
  uint32_t k_iter = 0;
  int n_seg_tr = 0;  // PQB_DQ_TRACE: segment index
  (void)n_seg_tr;

  if constexpr (kDqWs) {
    if (warp >= kNW) {  // ---- producer warpgroup
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PQB_DQ_PROD_REGS) : "memory");
      const int w0 = warp - kNW, w1 = w0 + 4;
      uint32_t it0 = 0, it1 = 0;
      bool first_seg = true;
      for (int64_t seg = i_begin; seg < i_end;) {
        const int64_t unit = seg / ws.tiles_max;
        const int t_lo = static_cast<int>(seg - unit * ws.tiles_max);
        const int64_t seg_end = min(i_end, (unit + 1) * ws.tiles_max);
        seg = seg_end;
        const int n_tiles = (c.seq_lens[unit] + kTile - 1) / kTile;
        const int t_hi = min(static_cast<int>(seg_end - unit * ws.tiles_max), n_tiles);
        // the previous segment's merge scratch aliases the stages
        if (!first_seg) named_sync(2, kDqThreads);
        first_seg = false;
        if (lane == 0) {
          TileCursor c0, c1;
          c0.init(t_lo + w0, tpp);
          c1.init(t_lo + w1, tpp);
          // the page base of each cursor's next tile is loaded one issue ahead (the
          // page-table read is a dependent global load; its latency then overlaps
          // the wait for the stage instead of following it)
          auto page_of = [&](const TileCursor& cu) {
            return page_base_c(c.store, unit, PROBE == 2 ? 0 : (cu.tile < t_hi ? cu.pg : 0));
          };
          auto issue = [&](int w, uint32_t it, const TileCursor& cu, const uint8_t* pb) {
            const uint32_t s = it % kSt;
            // the ring starts empty: the first kSt fills need no release
            if (it >= kSt) {
              if constexpr (PQB_DQ_SLEEP_PROD) mbar_wait_sleep(&s_empty[w][s], ((it / kSt) & 1) ^ 1);
              else mbar_wait(&s_empty[w][s], ((it / kSt) & 1) ^ 1);
            }
            fence_proxy_async_smem();
            issue_tile_dq<M, N, VQ, kScores>(stage_ptr(w * kSt + s), c.store, pb, PROBE == 2 ? 0 : cu.tin,
                                             &s_bar[w][s]);
          };
          const uint8_t* pb0 = page_of(c0);
          const uint8_t* pb1 = page_of(c1);
          while (c0.tile < t_hi) {  // c1 runs 4 tiles behind c0's stream position, never past it
            TileCursor n0 = c0;
            n0.next(dpg, dtin, tpp);
            const uint8_t* nb0 = page_of(n0);
            issue(w0, it0++, c0, pb0);
            c0 = n0;
            pb0 = nb0;
            if (c1.tile < t_hi) {
              TileCursor n1 = c1;
              n1.next(dpg, dtin, tpp);
              const uint8_t* nb1 = page_of(n1);
              issue(w1, it1++, c1, pb1);
              c1 = n1;
              pb1 = nb1;
            }
          }
        }
        __syncwarp();
      }
      if constexpr (CL > 1) {  // the consumers' two cluster barriers (finish_cluster), before their arrive on 2
        cluster_sync_all();
        cluster_sync_all();
      }
      if (!first_seg) named_sync(2, kDqThreads);
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(PQB_DQ_CONS_REGS) : "memory");
  }

  const int g8 = lane >> 2, t4 = lane & 3;  // fragment group / thread-in-group
  // ldmatrix.trans row addresses in the grouped value layout (value_offset):
  // token 16 ks + 8 ((lane >> 4) & 1) + (lane & 7), chunk 2 mt + ((lane >> 3) & 1)
  const uint32_t ld_row = static_cast<uint32_t>(((lane >> 4) & 1) * 2048 + (lane & 7) * 128);
  const uint32_t ld_chunk = static_cast<uint32_t>((((lane >> 3) & 1) ^ (lane & 7)) << 4);
  // P.V output columns 2 t4, 2 t4 + 1 belong to queries qc0, qc1 (packed: col & 3)
  const int qc0 = kPacked ? ((2 * t4) & 3) : 2 * t4, qc1 = qc0 + 1;

  for (int64_t seg = i_begin; seg < i_end;) {
    const int64_t unit = seg / ws.tiles_max;
    const int t_lo = static_cast<int>(seg - unit * ws.tiles_max);
    const int64_t seg_end = min(i_end, (unit + 1) * ws.tiles_max);
    seg = seg_end;
    const int T = c.seq_lens[unit], Tq = c.quant_lens[unit];
    const int n_tiles = (T + kTile - 1) / kTile;
    const int t_hi = min(static_cast<int>(seg_end - unit * ws.tiles_max), n_tiles);

    named_sync(1, kConsThreads);  // previous segment is done with q_s / qfrag / merge area
    const int first = t_lo + warp;
    // ---- unit setup: q rows, max |q * s|, then the Q' hi/lo A-fragments
    // one round of independent global loads: the G query rows and the 64 scales
    // (s_misc[0] is zero here: prologue / reset after the previous fragments)
    {
      constexpr int kQPer = G * 128 / kConsThreads;
      static_assert(kQPer * kConsThreads == G * 128, "q rows per thread");
      float qv[kQPer];
#pragma unroll
      for (int k = 0; k < kQPer; ++k) qv[k] = load_q(q, q_dtype, unit * G * 128 + tid + k * kConsThreads);
      const float sc = tid < 64 ? half_bits_to_f32(c.scales[unit * 64 + tid]) : 0.0f;
#pragma unroll
      for (int k = 0; k < kQPer; ++k) q_s[tid + k * kConsThreads] = qv[k];
      if (tid < 64) s_scale[tid] = sc;
    }
    named_sync(1, kConsThreads);
    {
      float mx = 0.0f;
#pragma unroll
      for (int k = 0; k < G * 128 / kConsThreads; ++k) {
        const int i = tid + k * kConsThreads, e = i & 127;
        const int j = c.layout == PQB_HALF_SPLIT ? (e & 63) : (e >> 1);
        mx = fmaxf(mx, fabsf(q_s[i] * s_scale[j]));
      }
      mx = warp_max(mx);
      if (lane == 0) atomicMax(s_misc, __float_as_int(mx));  // non-negative floats order as ints
    }
    named_sync(1, kConsThreads);
    const float qmax = __int_as_float(s_misc[0]);
    // 2^e * qmax in [2^14, 2^15)
    const int e_sc = (qmax > 0.0f && qmax < INFINITY)
                         ? max(-90, min(90, 14 - (static_cast<int>((__float_as_uint(qmax) >> 23) & 0xff) - 127)))
                         : 0;
    // A-fragment rows: g < 8 -> Q'_hi of query g, 8 + g -> Q'_lo of query g (zero for g >= G)
    for (int i = tid; i < 16 * 32; i += kConsThreads) {
      const int ks = i >> 5, ln = i & 31, g = ln >> 2, t = ln & 3;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (g < G) {
        const int j = 16 * t + dq_pair<M, N>(ks);
        const float sj = s_scale[j];
        const int ex = c.layout == PQB_HALF_SPLIT ? j : 2 * j;
        const int ey = c.layout == PQB_HALF_SPLIT ? j + 64 : 2 * j + 1;
        const float vx = ldexpf(q_s[g * 128 + ex] * sj, e_sc), vy = ldexpf(q_s[g * 128 + ey] * sj, e_sc);
        const __half hx = __float2half_rn(vx), hy = __float2half_rn(vy);
        const __half lx = __float2half_rn(vx - __half2float(hx)), ly = __float2half_rn(vy - __half2float(hy));
        const uint32_t hb = h2_bits(__halves2half2(hx, hy)), lb = h2_bits(__halves2half2(lx, ly));
        v = make_uint4(hb, lb, hb, lb);  // a2 / a3 (k + 8) repeat a0 / a1: they multiply K_lo
      }
      qfrag[i] = v;
    }
    named_sync(1, kConsThreads);
    if (tid == 0) s_misc[0] = 0;  // all have read qmax; the next atomicMax is >= 2 barriers later
    // (the k + 8 half repeats (hi, lo); loading it as its own registers measured
    // 1.5-6% faster than passing aq[ks][0..1] twice: the compiler schedules the
    // QK block differently)
    uint32_t aq[16][4];
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      const uint4 v = qfrag[ks * 32 + lane];
      aq[ks][0] = v.x;
      aq[ks][1] = v.y;
      aq[ks][2] = v.z;
      aq[ks][3] = v.w;
    }
    const float xscale = ldexpf(sm_scale_log2, -e_sc);
    DQ_TRACE(tid == 0 && n_seg_tr < 6, 2 + 4 * n_seg_tr);
#if PQB_DQ_TRACE
    if (tid == 0 && n_seg_tr < 6) pqb_dq_trace[blockIdx.x * 32 + 5 + 4 * n_seg_tr] = unit;
#endif

    // S = Q' . K^T of one tile (+ the residual window's exact dots): lane (g8, t4)
    // gets query g8 at tokens 8 nb + 2 t4 + j in x[nb][j], unscaled
    auto tile_scores = [&](const uint8_t* st, int tok0, float (&x)[4][2]) {
      // ---- S = Q' . K^T on the tensor cores: n-block nb = tokens 8 nb .. 8 nb + 7;
      // this lane gathers the keys of token 8 nb + g8 (B column g8).
      float sc[4][4];
      {
        DqIdx<M, N> ix[4];
        float sc2[4][4];  // second accumulation chain per n-block (odd k-steps): 8 independent MMA chains
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          const int r = 8 * nb + g8;
          ix[nb].load(st + r * 8 * M, st + Cfg::kABytes + r * 8 * N, t4, tok0 + r < Tq);
#pragma unroll
          for (int k = 0; k < 4; ++k) sc[nb][k] = sc2[nb][k] = 0.0f;
        }
        // m = n = 4 with bf16 values: two chains per n-block measured +1% G = 4, +3% G = 8
        // before the bf16-P instances and worse since (PQB_DQ_TWO_CHAINS, off); the other
        // instances always measured better with one (m3n2 -6%, 4-bit values -1.5%)
        constexpr bool kTwoChains = PQB_DQ_TWO_CHAINS && kFused && !kVq4;
#pragma unroll
        for (int ks = 0; ks < 16; ks += 2) {
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) {
            const uint2 t = lds_u2(ix[nb].addr(ptab_l, ks));
            mma_f16(sc[nb], aq[ks][0], aq[ks][1], aq[ks][2], aq[ks][3], t.x, t.y);
          }
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) {
            const uint2 t = lds_u2(ix[nb].addr(ptab_l, ks + 1));
            mma_f16(kTwoChains ? sc2[nb] : sc[nb], aq[ks + 1][0], aq[ks + 1][1], aq[ks + 1][2], aq[ks + 1][3], t.x,
                    t.y);
          }
        }
        if constexpr (kTwoChains) {
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int k = 0; k < 4; ++k) sc[nb][k] += sc2[nb][k];
        }
      }
      // lane (g8, t4): query g8, tokens 8 nb + 2 t4 + j  (hi row + lo row)
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        x[nb][0] = sc[nb][0] + sc[nb][2];
        x[nb][1] = sc[nb][1] + sc[nb][3];
      }
      // ---- residual window (fp32 keys): exact dots, lane = token (rare tiles)
      if (tok0 + kTile > Tq && Tq < T) {
        const int tok = tok0 + lane;
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.0f;
        if (tok >= Tq && tok < T && c.res_cap > 0) {  // (res_cap = 0 implies Tq = T)
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
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r = 8 * nb + 2 * t4 + j;
            if (tok0 + r >= Tq) x[nb][j] += rbuf[r * 8 + g8];
          }
        __syncwarp();
      }
    };

    // ---- lane 0 fills this warp's ring with its first tiles
    TileCursor cur;
    cur.init(first, tpp);
    if (!kDqWs && lane == 0) {
#pragma unroll
      for (int s = 0; s < kSt; ++s) {
        if (cur.tile < t_hi) {
          fence_proxy_async_smem();
          const uint32_t sl = (k_iter + s) % kSt;
          issue_tile_dq<M, N, VQ, kScores>(stage_ptr(warp * kSt + sl), c.store,
                                  page_base_c(c.store, unit, PROBE == 2 ? 0 : cur.pg), PROBE == 2 ? 0 : cur.tin,
                                  bar + sl);
        }
        cur.next(dpg, dtin, tpp);
      }
    }
    float m_run = -INFINITY, l_run = 0.0f;  // query g8 (lanes g8 < G)
    float z_run = 0.0f;                     // VQ: sum_t p_t zp_t of query g8 (lane partial)
    float d[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int k = 0; k < 4; ++k) d[mt][k] = 0.0f;
    float o[G][4];  // fp32 values: output dims 4 lane .. 4 lane + 3 of every query
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int k = 0; k < 4; ++k) o[g][k] = 0.0f;

    if constexpr (kUmma) {
      // ---- P.V on tcgen05, warpgroup-synchronous rounds (PQB_DQ_UMMA, see top)
      const int wg = warp >> 2, wq = warp & 3;
      const int t_wg = t_lo + 4 * wg;  // round k: warp wq of the group takes tile t_wg + wq + 8 k
      const int n_rounds = t_hi > t_wg ? (t_hi - t_wg + 7) / 8 : 0;
      const uint32_t tcol = tmem_base + 8 * wg;                    // D: lanes = dims, 8 columns
      const uint32_t tq = tcol + (static_cast<uint32_t>(32 * wq) << 16);  // this warp's quarter of D
      constexpr uint32_t kIdesc = umma_idesc_bf16(128, 8, 1);
      int pend = -1;  // stage of this warp's previous tile, released once its MMAs commit
      bool first_mma = true;
      for (int k = 0; k < n_rounds; ++k, ++u_round) {
        const int tile = t_wg + wq + 8 * k;
        const bool has = tile < t_hi;
        const int tok0 = tile * kTile;
        uint32_t s = 0;
        const uint8_t* st = nullptr;
        float x[4][2];
        if (has) {
          s = k_iter % kSt;
          if constexpr (PQB_DQ_SLEEP_CONS) mbar_wait_sleep(bar + s, (k_iter / kSt) & 1);
      else mbar_wait(bar + s, (k_iter / kSt) & 1);
          st = stage_ptr(warp * kSt + s);
          tile_scores(st, tok0, x);
        }
        float mx = -INFINITY;
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            x[nb][j] = has && tok0 + 8 * nb + 2 * t4 + j < T ? x[nb][j] * xscale : -INFINITY;
            mx = fmaxf(mx, x[nb][j]);
          }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        if (t4 == 0 && g8 < G) um_max[(wg * 4 + wq) * 4 + g8] = mx;
        named_sync(3 + wg, 128);
        const int gq = g8 < G ? g8 : 0;
        const float mt = fmaxf(fmaxf(um_max[(wg * 4 + 0) * 4 + gq], um_max[(wg * 4 + 1) * 4 + gq]),
                               fmaxf(um_max[(wg * 4 + 2) * 4 + gq], um_max[(wg * 4 + 3) * 4 + gq]));
        if (k > 0) {  // the previous round's MMAs: its stages and P^T buffer are free after this
          mbar_wait(um_bar + wg * 2 + ((u_round - 1) & 1), ((u_round - 1) >> 1) & 1);
          tc_fence_after();
        }
        if (pend >= 0) {
          if (!PQB_DQ_UMMA_RELEASE && lane == 0) mbar_arrive(&s_empty[warp][pend]);
          pend = -1;
        }
        // lazy reference max: raised only when the tile max exceeds it by more than 2^tau
        const bool upd = g8 < G && mt > m_run + kUmmaTau;
        const float m_new = upd ? mt : m_run;
        const float alpha = upd ? fast_exp2(m_run - m_new) : 1.0f;
        if (k > 0 && __any_sync(0xffffffffu, upd)) {  // rescale the accumulated O (columns q, q + 4: query q)
          float v[8];
          tmem_ld8(tq, v);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) v[cc] *= __shfl_sync(0xffffffffu, alpha, (cc & 3) * 4);
          tmem_st8(tq, v);
        }
        l_run *= alpha;
        m_run = m_new;
        float ls = 0.0f;
        uint8_t* bbuf = um_b + ((wg * 2 + (u_round & 1)) * 16 + wq * 4) * 256;  // this warp's 4 core matrices
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          const float p0 = fast_exp2(x[nb][0] - m_run), p1 = fast_exp2(x[nb][1] - m_run);
          ls += p0 + p1;
          const __nv_bfloat162 hi = __floats2bfloat162_rn(p0, p1);
          const float2 hf = __bfloat1622float2(hi);
          const __nv_bfloat162 lo = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
          if (g8 < G) {  // core matrix nb (tokens 8 nb ..): row g8 = P_hi of query g8, row 4 + g8 = P_lo
            *reinterpret_cast<__nv_bfloat162*>(bbuf + nb * 256 + g8 * 16 + t4 * 4) = hi;
            *reinterpret_cast<__nv_bfloat162*>(bbuf + nb * 256 + (4 + g8) * 16 + t4 * 4) = lo;
          }
        }
        l_run += ls;
        fence_proxy_async_smem();  // P^T (generic stores) -> the tensor core's async proxy
        if (lane == 0) {
          um_va[wg * 4 + wq] = has ? smem_u32(st + Cfg::kABytes + Cfg::kRBytes) : 0u;
          um_va[8 + wg * 4 + wq] = s;
        }
        tc_fence_before();
        named_sync(3 + wg, 128);
        if (wq == 0 && lane == 0) {
          tc_fence_after();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t va = um_va[wg * 4 + i];
            if (va == 0u) continue;
            const uint32_t bb = smem_u32(um_b + ((wg * 2 + (u_round & 1)) * 16 + i * 4) * 256);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              // A = V^T: MN-major, 128-byte swizzle, dims 64-127 at +1 KB, token groups at +2 KB;
              // B = P^T: K-major core matrices, tokens 16 h + 8 .. at +256 B
              umma_bf16(tcol, umma_smem_desc(va + h * 4096, 1024, 2048, 2), umma_smem_desc(bb + h * 512, 256, 256, 0),
                        kIdesc, !first_mma);
              first_mma = false;
            }
          }
          umma_commit(um_bar + wg * 2 + (u_round & 1));
          if (PQB_DQ_UMMA_RELEASE) {  // the stages are free once the MMAs reading them are done
            mbar_wait(um_bar + wg * 2 + (u_round & 1), (u_round >> 1) & 1);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (um_va[wg * 4 + i] != 0u) mbar_arrive(&s_empty[4 * wg + i][um_va[8 + wg * 4 + i]]);
          }
        }
        __syncwarp();
        if (has) {
          pend = static_cast<int>(s);
          ++k_iter;
        }
      }
      // ---- segment end: the last round's MMAs, then O^T back from tensor memory
      float ov[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (n_rounds > 0) {
        mbar_wait(um_bar + wg * 2 + ((u_round - 1) & 1), ((u_round - 1) >> 1) & 1);
        tc_fence_after();
        tmem_ld8(tq, ov);
      }
      if (!PQB_DQ_UMMA_RELEASE && pend >= 0 && lane == 0) mbar_arrive(&s_empty[warp][pend]);
      l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
      l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
      if (t4 == 0 && g8 < G) um_l[(wg * 4 + wq) * 4 + g8] = l_run;
      tc_fence_before();
      named_sync(1, kConsThreads);  // every warp is past its last stage read and MMA
      float* red = reinterpret_cast<float*>(warp_area);
      // the group's partial goes in warp slot 4 wg (dims 32 wq + lane from each warp); slots
      // 4 wg + 1 .. 3 stay empty (m = -inf)
      float* grp = red + (4 * wg) * G * 132;
#pragma unroll
      for (int g = 0; g < G; ++g) grp[g * 132 + 4 + 32 * wq + lane] = ov[g] + ov[G + g];
      const float mg = __shfl_sync(0xffffffffu, m_run, (lane & 3) * 4);  // query lane's reference max
      if (lane < G) {
        float* mine = red + warp * G * 132;
        if (wq == 0) {
          mine[lane * 132] = mg;
          mine[lane * 132 + 1] = um_l[(wg * 4 + 0) * 4 + lane] + um_l[(wg * 4 + 1) * 4 + lane] +
                                 um_l[(wg * 4 + 2) * 4 + lane] + um_l[(wg * 4 + 3) * 4 + lane];
        } else {
          mine[lane * 132] = -INFINITY;
          mine[lane * 132 + 1] = 0.0f;
        }
      }
      if (wq != 0) {  // the empty slots' accumulators must be finite (the merge weighs them by 0)
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int k = 0; k < 4; ++k) red[(warp * G + g) * 132 + 4 + 32 * k + lane] = 0.0f;
      }
      finish_segment<G>(ep, ws, unit, red, s_misc + 1, tid, kConsThreads);
      if constexpr (kDqWs) named_arrive(2, kDqThreads);  // producers may refill the stages
      ++n_seg_tr;
      continue;
    }
    for (int tile = first; tile < t_hi; tile += kNW, ++k_iter) {
      const uint32_t s = k_iter % kSt;
      const int nt = tile + kSt * kNW;  // the tile this stage is refilled with
      if constexpr (PQB_DQ_SLEEP_CONS) mbar_wait_sleep(bar + s, (k_iter / kSt) & 1);
      else mbar_wait(bar + s, (k_iter / kSt) & 1);
      const uint8_t* st = stage_ptr(warp * kSt + s);
      const int tok0 = tile * kTile;
      if constexpr (PROBE == 1) {
        __syncwarp();
        if (kDqWs) {
          if (lane == 0) mbar_arrive(&s_empty[warp][s]);
        } else if (lane == 0) {
          if (nt < t_hi) {
            fence_proxy_async_smem();
            issue_tile_dq<M, N, VQ, kScores>(stage_ptr(warp * kSt + s), c.store, page_base_c(c.store, unit, cur.pg), cur.tin,
                                    bar + s);
          }
          cur.next(dpg, dtin, tpp);
        }
        continue;
      }

      float x[4][2];
      tile_scores(st, tok0, x);
      if constexpr (kScores) {  // raw scores: x = S * 2^e_sc (exact rescale), tokens 8 nb + 2 t4 + j
        if (g8 < G) {
          const float inv_sc = ldexpf(1.0f, -e_sc);
          float* row = scores + (unit * G + g8) * scores_ld;
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) {
            const int tok = tok0 + 8 * nb + 2 * t4;
            const float v0 = x[nb][0] * inv_sc, v1 = x[nb][1] * inv_sc;
            if (tok + 1 < T && (scores_ld & 1) == 0) {
              __stcs(reinterpret_cast<float2*>(row + tok), make_float2(v0, v1));
            } else {
              if (tok < T) row[tok] = v0;
              if (tok + 1 < T) row[tok + 1] = v1;
            }
          }
        }
        __syncwarp();
        if (kDqWs) {
          if (lane == 0) mbar_arrive(&s_empty[warp][s]);
        } else if (lane == 0) {
          if (nt < t_hi) {
            fence_proxy_async_smem();
            issue_tile_dq<M, N, VQ, kScores>(stage_ptr(warp * kSt + s), c.store, page_base_c(c.store, unit, cur.pg),
                                             cur.tin, bar + s);
          }
          cur.next(dpg, dtin, tpp);
        }
        continue;
      }
      // ---- online softmax (query g8; the four t4 lanes share it)
      float mx = -INFINITY;
      if (PQB_DQ_FULL_TILE && tok0 + kTile <= T) {  // whole tile inside the sequence: no bound tests
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            x[nb][j] *= xscale;
            mx = fmaxf(mx, x[nb][j]);
          }
      } else {
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            x[nb][j] = tok0 + 8 * nb + 2 * t4 + j < T ? x[nb][j] * xscale : -INFINITY;
            mx = fmaxf(mx, x[nb][j]);
          }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mn = fmaxf(m_run, mx);
      const float alpha = fast_exp2(m_run - mn);
      const bool rescale = mn != m_run;
      m_run = mn;
      if constexpr (kVf32) {
        // ---- fp32 values (the reference's default cache): P.V on the CUDA
        // cores in full fp32.  P goes through the warp's [32 tokens][8] buffer;
        // lane L owns output dims 4L .. 4L + 3 and reads each fp32 value row
        // with one conflict-free LDS.128 (512 B per row = 4 wavefronts) and the
        // row's G probabilities as broadcast LDS.128s.
        float ls = 0.0f;
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          const float p0 = fast_exp2(x[nb][0] - mn), p1 = fast_exp2(x[nb][1] - mn);
          ls += p0 + p1;
          if (g8 < G) {
            rbuf[(8 * nb + 2 * t4) * 8 + g8] = p0;
            rbuf[(8 * nb + 2 * t4 + 1) * 8 + g8] = p1;
          }
        }
        l_run = fmaf(l_run, alpha, ls);
        if (__any_sync(0xffffffffu, rescale && g8 < G)) {
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float ag = __shfl_sync(0xffffffffu, alpha, g * 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) o[g][k] *= ag;
          }
        }
        __syncwarp();
        const float4* vrow = reinterpret_cast<const float4*>(st + Cfg::kABytes + Cfg::kRBytes) + lane;
#pragma unroll 8
        for (int t = 0; t < kTile; ++t) {
          const float4 v = vrow[t * 32];
#pragma unroll
          for (int g4 = 0; g4 < G; g4 += 4) {
            const float4 pv = *reinterpret_cast<const float4*>(&rbuf[t * 8 + g4]);
            const float pg[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
            for (int k = 0; k < 4 && g4 + k < G; ++k) {
              o[g4 + k][0] = fmaf(pg[k], v.x, o[g4 + k][0]);
              o[g4 + k][1] = fmaf(pg[k], v.y, o[g4 + k][1]);
              o[g4 + k][2] = fmaf(pg[k], v.z, o[g4 + k][2]);
              o[g4 + k][3] = fmaf(pg[k], v.w, o[g4 + k][3]);
            }
          }
        }
      } else {
      float ls = 0.0f, zs = 0.0f;
      uint32_t phi[4], plo[4];  // bf16x2 (tokens 8 nb + 2 t4, +1)
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        float p0 = fast_exp2(x[nb][0] - mn), p1 = fast_exp2(x[nb][1] - mn);
        ls += p0 + p1;
        if constexpr (kVq4) {  // (zp, scale) of tokens 8 nb + 2 t4, +1
          const float4 zsv =
              reinterpret_cast<const float4*>(st + Cfg::kABytes + Cfg::kRBytes + Cfg::kVqCodeBytes)[4 * nb + t4];
          // centred split: c s + zp = (c - K) s + (zp + K s), K = kVqMid; the MMA
          // takes c - K (via the tile bias below), the row midpoints go here,
          // so neither sum carries the rows' common offset
          zs = fmaf(p0, fmaf(kVqMid, zsv.y, zsv.x), fmaf(p1, fmaf(kVqMid, zsv.w, zsv.z), zs));
          p0 *= zsv.y;
          p1 *= zsv.w;
        }
        const __nv_bfloat162 hi = __floats2bfloat162_rn(p0, p1);
        phi[nb] = *reinterpret_cast<const uint32_t*>(&hi);
        if constexpr (!kPhiOnly) {
          const float2 hf = __bfloat1622float2(hi);
          const __nv_bfloat162 lo = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
          plo[nb] = *reinterpret_cast<const uint32_t*>(&lo);
        }
      }
      l_run = fmaf(l_run, alpha, ls);
      if constexpr (kVq4) z_run = fmaf(z_run, alpha, zs);
      if (__any_sync(0xffffffffu, rescale && g8 < G)) {
        const float a0 = __shfl_sync(0xffffffffu, alpha, qc0 * 4), a1 = __shfl_sync(0xffffffffu, alpha, qc1 * 4);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          d[mt][0] *= a0;
          d[mt][1] *= a1;
          d[mt][2] *= a0;
          d[mt][3] *= a1;
        }
      }
      if constexpr (kPacked && kPhiOnly) {  // columns 4..7 (lanes 16..31) stay zero
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) phi[nb] = lane < 16 ? phi[nb] : 0u;
      } else if constexpr (kPacked) {  // columns 4..7 (lanes 16..31) take P_lo of query g8 - 4
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, plo[nb], 16);
          phi[nb] = lane < 16 ? phi[nb] : o;
        }
      }
      // ---- P.V on tensor cores: O^T[128 x 8] += V^T[128 x 32] . P^T[32 x 8];
      // the P^T B-fragments are the score registers (k-step ks = n-blocks 2ks, 2ks+1)
      if constexpr (kVq4) {
        // A fragments straight from the code words: nibble -> bf16 (128 + c) by
        // OR-ing into the bit pattern of 128.0.  The 128 * sum(B) this adds is
        // removed from the accumulators after every tile, by one more MMA per
        // k-step with A = -128 against the same B fragments (exactly the
        // per-column sums of the bf16 hi + lo values consumed), together with
        // the centring offset K.  Removing the offset only at the end let the
        // accumulators carry 128 x the result across all tiles (measured
        // 9e-4 (4-bit) .. 3e-3 (2-bit) relative error at 32K tokens).
        // 2-bit codes: 16 bits per fragment, byte-spread by one PRMT so each
        // register's two codes land at bits 2k / 16 + 2k.  8-bit codes: two
        // nibble planes; the high plane as bf16 (2048 + 16 h) (exact: [2048,
        // 4096) has spacing 16), so A_lo + A_hi = 2176 + c and both MMAs share
        // one accumulator (the tile bias below is 2176 sum(B) instead of 128).
        const uint32_t* vw = reinterpret_cast<const uint32_t*>(st + Cfg::kABytes + Cfg::kRBytes);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            uint32_t a[4];
            if constexpr (kVqB == 2) {
              const uint32_t w = __byte_perm(vw[mt * 32 + lane], 0u, ks ? 0x4342u : 0x4140u);
#pragma unroll
              for (int k = 0; k < 4; ++k) a[k] = ((w >> (2 * k)) & 0x00030003u) | 0x43004300u;
            } else {
              const uint32_t w = kVqB == 8 ? vw[2 * ((mt * 2 + ks) * 32 + lane)] : vw[(mt * 2 + ks) * 32 + lane];
#pragma unroll
              for (int k = 0; k < 4; ++k) a[k] = ((w >> (4 * k)) & 0x000F000Fu) | 0x43004300u;
            }
            mma_bf16(d[mt], a[0], a[1], a[2], a[3], phi[2 * ks], phi[2 * ks + 1]);
            if constexpr (!kPacked) mma_bf16(d[mt], a[0], a[1], a[2], a[3], plo[2 * ks], plo[2 * ks + 1]);
            if constexpr (kVqB == 8) {
              const uint32_t wh = vw[2 * ((mt * 2 + ks) * 32 + lane) + 1];
#pragma unroll
              for (int k = 0; k < 4; ++k) a[k] = ((wh >> (4 * k)) & 0x000F000Fu) | 0x45004500u;
              mma_bf16(d[mt], a[0], a[1], a[2], a[3], phi[2 * ks], phi[2 * ks + 1]);
              if constexpr (!kPacked) mma_bf16(d[mt], a[0], a[1], a[2], a[3], plo[2 * ks], plo[2 * ks + 1]);
            }
          }
        }
        {  // the tile's bias: -(offset + K) * sum_t B[t][col] (every row alike), added to every dim block
          // bf16 -(2176 + 128) / -(128 + 7) / -(128 + 1), all exact
          constexpr uint32_t kNegBias = kVqB == 8 ? 0xC510C510u : kVqB == 4 ? 0xC307C307u : 0xC301C301u;
          float bias[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            mma_bf16(bias, kNegBias, kNegBias, kNegBias, kNegBias, phi[2 * ks], phi[2 * ks + 1]);
            if constexpr (!kPacked) mma_bf16(bias, kNegBias, kNegBias, kNegBias, kNegBias, plo[2 * ks], plo[2 * ks + 1]);
          }
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            d[mt][0] += bias[0];
            d[mt][1] += bias[1];
            d[mt][2] += bias[2];
            d[mt][3] += bias[3];
          }
        }
      } else {
        const uint32_t vbase = smem_u32(st + Cfg::kABytes + Cfg::kRBytes) + ld_row;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_trans(vbase + ks * 4096 + (mt >> 2) * 1024 + (ld_chunk ^ ((mt & 3) << 5)), a0, a1, a2, a3);
            mma_bf16(d[mt], a0, a1, a2, a3, phi[2 * ks], phi[2 * ks + 1]);
            if constexpr (!kPacked && !kPhiOnly) mma_bf16(d[mt], a0, a1, a2, a3, plo[2 * ks], plo[2 * ks + 1]);
          }
        }
      }
      }  // bf16 / 4-bit values
      __syncwarp();
      if (kDqWs) {
        if (lane == 0) mbar_arrive(&s_empty[warp][s]);
      } else if (lane == 0) {
        if (nt < t_hi) {
          fence_proxy_async_smem();
          issue_tile_dq<M, N, VQ, kScores>(stage_ptr(warp * kSt + s), c.store,
                                  page_base_c(c.store, unit, PROBE == 2 ? 0 : cur.pg), PROBE == 2 ? 0 : cur.tin,
                                  bar + s);
        }
        cur.next(dpg, dtin, tpp);
      }
    }

    if constexpr (kScores) {  // scores-only: nothing to merge
      if constexpr (kDqWs) named_arrive(2, kDqThreads);
      continue;
    }
    // ---- segment epilogue: per-warp (m, l, o) -> shared, then the common merge
    DQ_TRACE(tid == 0 && n_seg_tr < 6, 3 + 4 * n_seg_tr);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    if constexpr (kPacked && !kVf32) {  // O = columns q (P_hi) + q + 4 (P_lo): lanes t4, t4 ^ 2
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int k = 0; k < 4; ++k) d[mt][k] += __shfl_xor_sync(0xffffffffu, d[mt][k], 2);
    }
    if constexpr (kVq4) {  // + sum_t p_t zp_t of the column's query
      z_run += __shfl_xor_sync(0xffffffffu, z_run, 1);
      z_run += __shfl_xor_sync(0xffffffffu, z_run, 2);
      const float z0 = __shfl_sync(0xffffffffu, z_run, qc0 * 4), z1 = __shfl_sync(0xffffffffu, z_run, qc1 * 4);
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        d[mt][0] += z0;
        d[mt][1] += z1;
        d[mt][2] += z0;
        d[mt][3] += z1;
      }
    }
    named_sync(1, kConsThreads);  // every warp is past its last stage read
    float* red = reinterpret_cast<float*>(warp_area);
    float* mine = red + warp * G * 132;
    if (t4 == 0 && g8 < G) {
      mine[g8 * 132] = m_run;
      mine[g8 * 132 + 1] = l_run;
    }
    if constexpr (kVf32) {
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int k = 0; k < 4; ++k) mine[g * 132 + 4 + 4 * lane + k] = o[g][k];
    } else if (qc0 < G && (!kPacked || t4 < 2)) {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int dim = 16 * mt + g8;
        mine[qc0 * 132 + 4 + dim] = d[mt][0];
        mine[qc0 * 132 + 4 + dim + 8] = d[mt][2];
        if (qc1 < G) {
          mine[qc1 * 132 + 4 + dim] = d[mt][1];
          mine[qc1 * 132 + 4 + dim + 8] = d[mt][3];
        }
      }
    }
    if constexpr (CL > 1) {
      // one segment per CTA; its merge area sits after the warps' red rows, before the table
      finish_cluster<G, CL>(ep, unit, red, red + kNW * G * 132, tid, kConsThreads);
    } else {
      finish_segment<G>(ep, ws, unit, red, s_misc + 1, tid, kConsThreads);
    }
    if constexpr (kDqWs) named_arrive(2, kDqThreads);  // producers may refill the stages
    DQ_TRACE(tid == 0 && n_seg_tr < 6, 4 + 4 * n_seg_tr);
    ++n_seg_tr;
  }
  peer_publish(ep, ep.counters + ws.items / ws.tiles_max, tid, kConsThreads);
  if constexpr (kUmma) {
    tc_fence_before();
    named_sync(1, kConsThreads);
    if (warp == 0) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem_base) : "memory");
    }
  }
  DQ_TRACE(tid == 0, 31);
#if PQB_DQ_TRACE
  if (tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    pqb_dq_trace[blockIdx.x * 32 + 30] = smid;
    pqb_dq_trace[blockIdx.x * 32 + 29] = static_cast<unsigned long long>(i_end - i_begin);
  }
#endif
}

// ------------------------------------------------------------------ host side

// once per device and instance: the shared-memory opt-in (and, for the PRMT
// build, the check that the table lands at kPtTabAbs with the stages around it)
template <int G, int M, int N, int PROBE, int VQ, int CL>
static int dq_prepare() {
  using Cfg = DqCfg<G, M, N, VQ>;
  static std::atomic<uint64_t> attr_done{0};
  return once_per_device(attr_done, [] {
#if PQB_DQ_PRMT_TAB
    {
      cudaFuncAttributes fa;
      int reserved = 0;
      cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, current_device());
      if (cudaFuncGetAttributes(&fa, decode_dq_kernel<G, M, N, PROBE, VQ, CL>) != cudaSuccess) {
        set_error("cudaFuncGetAttributes failed");
        return PQB_ECUDA;
      }
      // static bytes as reported may include the reserved block; dynamic memory starts after both
      const int stat = static_cast<int>(fa.sharedSizeBytes) >= reserved ? static_cast<int>(fa.sharedSizeBytes) - reserved
                                                                         : static_cast<int>(fa.sharedSizeBytes);
      const int dyn0 = reserved + ((stat + 127) / 128) * 128;
      const int tab_off = static_cast<int>(kPtTabAbs) - dyn0;
      const int n_before = tab_off / Cfg::kStageBytes;
      // (cluster instances: the CTA's merge partial follows the warps' rows)
      const int merge_bytes = kNW * G * 132 * 4 + (CL > 1 ? G * 130 * 4 : 0);
      if (tab_off < 0 || n_before * Cfg::kStageBytes < merge_bytes ||
          tab_off + 65536 + (kNW * Cfg::kSt - n_before) * Cfg::kStageBytes > Cfg::kSmem ||
          stat + Cfg::kSmem > 232448)
        return kDqLayoutUnavailable;  // the caller falls back to the linear-layout build
    }
#endif
    if (cudaFuncSetAttribute(decode_dq_kernel<G, M, N, PROBE, VQ, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmem) != cudaSuccess) {
      set_error("cudaFuncSetAttribute(smem=%d) failed", Cfg::kSmem);
      return PQB_ECUDA;
    }
    return PQB_OK;
  });
}

template <int G, int M, int N, int PROBE = 0, int VQ = 0, int CL = 0>
static int launch_dq(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s) {
  using Cfg = DqCfg<G, M, N, VQ>;
  const int arc = dq_prepare<G, M, N, PROBE, VQ, CL>();
  if (arc != PQB_OK) return arc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDqThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CL > 1 ? CL : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CL > 1 ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, decode_dq_kernel<G, M, N, PROBE, VQ, CL>, *a.cache, a.q, a.q_dtype,
                         a.sm_scale * kLog2e, ep, ws, a.scores, a.scores_ld) != cudaSuccess) {
    set_error("decode_dq launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return PQB_ECUDA;
  }
  return PQB_OK;
}

// Clusters of CL CTAs of this instance that can be resident at once (0: not
// available), cached per device.
template <int G, int M, int N, int VQ, int CL>
static int cluster_capacity() {
  static std::atomic<int> cache[64];
  std::atomic<int>& slot = cache[current_device() & 63];
  int n = slot.load(std::memory_order_relaxed);
  if (n != 0) return n > 0 ? n : 0;
  using Cfg = DqCfg<G, M, N, VQ>;
  n = -1;
  if (dq_prepare<G, M, N, 0, VQ, CL>() == PQB_OK) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * 64);
    cfg.blockDim = dim3(kDqThreads);
    cfg.dynamicSmemBytes = Cfg::kSmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, decode_dq_kernel<G, M, N, 0, VQ, CL>, &cfg) == cudaSuccess && c > 0) n = c;
    else (void)cudaGetLastError();
  }
  slot.store(n, std::memory_order_relaxed);
  return n > 0 ? n : 0;
}

// bf16 values: the bf16-P instance for G = 4 / 8 launches with bf16 outputs
// (configs[3]: layer step 0.866 -> 0.886 of the copy peak, scripts/g8_rate.py;
// configs[1]: +1.5 % value and sustained at the power cap, scripts/gpu_g4phi_ab.sh)
template <int G, int M, int N, int CL = 0>
static int launch_bf16v(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s) {
  if constexpr ((G == 8 || (G == 4 && PQB_DQ_PHI_BF16_G4)) && PQB_DQ_PHI_BF16) {
    if (ep.out_dtype == PQB_BF16) return launch_dq<G, M, N, kDqBf16P, 0, CL>(a, ep, ws, grid, s);
  }
  return launch_dq<G, M, N, 0, 0, CL>(a, ep, ws, grid, s);
}

template <int G>
static int dispatch_dq_mn(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s,
                          bool& handled) {
  handled = true;
  const int mn = a.cache->angle_bits * 10 + a.cache->radius_bits;
  if (a.out == nullptr) {  // scores-only (the caller checked a.scores)
    switch (mn) {
      case 44: return launch_dq<G, 4, 4, kDqScores>(a, ep, ws, grid, s);
      case 32: return launch_dq<G, 3, 2, kDqScores>(a, ep, ws, grid, s);
      case 22: return launch_dq<G, 2, 2, kDqScores>(a, ep, ws, grid, s);
      case 42: return launch_dq<G, 4, 2, kDqScores>(a, ep, ws, grid, s);
      case 24: return launch_dq<G, 2, 4, kDqScores>(a, ep, ws, grid, s);
      case 34: return launch_dq<G, 3, 4, kDqScores>(a, ep, ws, grid, s);
      default: handled = false; return PQB_OK;
    }
  }
  if (a.cache->store.value_dtype == PQB_VQ4) {
    switch (mn) {
      case 44: return launch_dq<G, 4, 4, 0, kValVq4>(a, ep, ws, grid, s);
      case 32: return launch_dq<G, 3, 2, 0, kValVq4>(a, ep, ws, grid, s);
      case 22: return launch_dq<G, 2, 2, 0, kValVq4>(a, ep, ws, grid, s);
      case 42: return launch_dq<G, 4, 2, 0, kValVq4>(a, ep, ws, grid, s);
      case 24: return launch_dq<G, 2, 4, 0, kValVq4>(a, ep, ws, grid, s);
      case 34: return launch_dq<G, 3, 4, 0, kValVq4>(a, ep, ws, grid, s);
      default: handled = false; return PQB_OK;
    }
  }
  if (a.cache->store.value_dtype == PQB_VQ2 || a.cache->store.value_dtype == PQB_VQ8) {
    const bool b8 = a.cache->store.value_dtype == PQB_VQ8;
    switch (mn) {  // the configs' shapes; other (m, n) take the generic kernel
      case 44: return b8 ? launch_dq<G, 4, 4, 0, kValVq8>(a, ep, ws, grid, s) : launch_dq<G, 4, 4, 0, kValVq2>(a, ep, ws, grid, s);
      case 32: return b8 ? launch_dq<G, 3, 2, 0, kValVq8>(a, ep, ws, grid, s) : launch_dq<G, 3, 2, 0, kValVq2>(a, ep, ws, grid, s);
      default: handled = false; return PQB_OK;
    }
  }
  if (a.cache->store.value_dtype == PQB_F32) {
    switch (mn) {
      case 44: return launch_dq<G, 4, 4, 0, kValF32>(a, ep, ws, grid, s);
      case 32: return launch_dq<G, 3, 2, 0, kValF32>(a, ep, ws, grid, s);
      case 22: return launch_dq<G, 2, 2, 0, kValF32>(a, ep, ws, grid, s);
      case 42: return launch_dq<G, 4, 2, 0, kValF32>(a, ep, ws, grid, s);
      case 24: return launch_dq<G, 2, 4, 0, kValF32>(a, ep, ws, grid, s);
      case 34: return launch_dq<G, 3, 4, 0, kValF32>(a, ep, ws, grid, s);
      default: handled = false; return PQB_OK;
    }
  }
  if (ws.cluster > 1 && mn == 44) {  // aligned split, merge through distributed shared memory
    switch (ws.cluster) {
      case 2: return launch_bf16v<G, 4, 4, 2>(a, ep, ws, grid, s);
      case 4: return launch_bf16v<G, 4, 4, 4>(a, ep, ws, grid, s);
      case 8: return launch_bf16v<G, 4, 4, 8>(a, ep, ws, grid, s);
      default: break;
    }
  }
  if (mn == 44 && (a.flags & PQB_DECODE_PROBE_MEM)) return launch_dq<G, 4, 4, 1>(a, ep, ws, grid, s);
  if (mn == 44 && (a.flags & PQB_DECODE_PROBE_COMPUTE)) return launch_dq<G, 4, 4, 2>(a, ep, ws, grid, s);
  switch (mn) {
    case 44: return launch_bf16v<G, 4, 4>(a, ep, ws, grid, s);
    case 32: return launch_bf16v<G, 3, 2>(a, ep, ws, grid, s);
    case 22: return launch_bf16v<G, 2, 2>(a, ep, ws, grid, s);
    case 42: return launch_bf16v<G, 4, 2>(a, ep, ws, grid, s);
    case 24: return launch_bf16v<G, 2, 4>(a, ep, ws, grid, s);
    case 34: return launch_bf16v<G, 3, 4>(a, ep, ws, grid, s);
    default: handled = false; return PQB_OK;
  }
}

#if PQB_DQ_TRACE && PQB_DQ_PRMT_TAB
extern "C" int pqb_debug_dq_trace(void* host, int n_ctas) {
  return cudaMemcpyFromSymbol(host, pqb_dq_trace, sizeof(unsigned long long) * 32 * std::min(n_ctas, 1024)) ==
                 cudaSuccess ? 0 : -1;
}
#endif

int dq_cluster_capacity(int group, int mn, int value_dtype, int cl) {
  if (mn != 44 || value_dtype != PQB_BF16) return 0;
  if (group == 8) return cl == 2 ? cluster_capacity<8, 4, 4, 0, 2>() : cl == 4 ? cluster_capacity<8, 4, 4, 0, 4>()
                                                                   : cl == 8 ? cluster_capacity<8, 4, 4, 0, 8>() : 0;
  if (group == 4) return cl == 2 ? cluster_capacity<4, 4, 4, 0, 2>() : cl == 4 ? cluster_capacity<4, 4, 4, 0, 4>()
                                                                   : cl == 8 ? cluster_capacity<4, 4, 4, 0, 8>() : 0;
  return 0;
}

int launch_decode_dq(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s,
                     bool& handled) {
  handled = false;
  if (a.group == 8) return dispatch_dq_mn<8>(a, ep, ws, grid, s, handled);
  if (a.group == 4) return dispatch_dq_mn<4>(a, ep, ws, grid, s, handled);
  return PQB_OK;
}

}  // namespace PQB_DQ_NS
}  // namespace pqb
