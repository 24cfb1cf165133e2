// Shared pieces of the decode kernels (LUT: decode.cu, dequant + tensor-core
// scoring: decode_dq.cu): constants, code extraction, mma helpers, the
// persistent work split and the segment epilogue (warp merge, direct output or
// partial + last-CTA merge).
#pragma once

#include "common.cuh"

namespace pqb {

constexpr int kNW = 8;      // compute warps per CTA
constexpr int kStages = 2;  // TMA ring depth per warp
constexpr int kTile = 32;   // tokens per tile (one per lane)
constexpr float kLog2e = 1.4426950408889634f;
constexpr double kPiD = 3.141592653589793115997963468544185161590576171875;  // == np.pi
constexpr uint32_t kMagic = 0x4B000000u;  // 2^23 as float bits

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

PQB_DEV float load_q(const void* q, int dt, int64_t i) {
  return dt == PQB_F32 ? load1<PQB_F32>(q, i) : (dt == PQB_BF16 ? load1<PQB_BF16>(q, i) : load1<PQB_F16>(q, i));
}

PQB_DEV uint32_t shift_lr(uint32_t x, int s) { return s >= 0 ? (x >> s) : (x << (-s)); }

// ---- code extraction.  A token's 64 codes of B bits are 2B words (stream
// bits, LSB first).  For B in {2, 4} the codes are first masked into byte lanes
// (scaled by 2^S); afterwards each code is one PRMT.

template <int B, int S>
struct CodeLanes {
  static constexpr int kMasked = (B == 4 || B == 2) ? 16 : 1;
  uint32_t mw[kMasked];
  PQB_DEV void init(const uint32_t* w) {
    if constexpr (B == 4) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mw[2 * i] = shift_lr(w[i], -S) & (0x0F0F0F0Fu << S);         // even codes: byte k = code 2k
        mw[2 * i + 1] = shift_lr(w[i], 4 - S) & (0x0F0F0F0Fu << S);  // odd codes
      }
    } else if constexpr (B == 2) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int r = 0; r < 4; ++r) mw[4 * i + r] = shift_lr(w[i], 2 * r - S) & (0x03030303u << S);
    }
  }
  // code j << S, as a register usable as an address offset
  PQB_DEV uint32_t get(const uint32_t* w, int j) const {
    if constexpr (B == 4) {
      return __byte_perm(mw[2 * (j >> 3) + (j & 1)], 0u, 0x4440u | ((j & 7) >> 1));
    } else if constexpr (B == 2) {
      return __byte_perm(mw[4 * (j >> 4) + (j & 3)], 0u, 0x4440u | ((j & 15) >> 2));
    } else {
      const int bit = j * B, wi = bit >> 5, sh = bit & 31;
      uint32_t v;
      if (sh + B <= 32) v = shift_lr(w[wi], sh - S);
      else v = __funnelshift_r(w[wi], w[wi + 1], sh) << S;
      return v & (((1u << B) - 1u) << S);
    }
  }
  // float(code j), exact (requires S == 0)
  PQB_DEV float as_float(const uint32_t* w, int j) const {
    uint32_t bits;
    if constexpr (B == 4) {
      bits = __byte_perm(mw[2 * (j >> 3) + (j & 1)], kMagic, 0x7650u | ((j & 7) >> 1));
    } else if constexpr (B == 2) {
      bits = __byte_perm(mw[4 * (j >> 4) + (j & 3)], kMagic, 0x7650u | ((j & 15) >> 2));
    } else {
      bits = get(w, j) | kMagic;
    }
    return __uint_as_float(bits) - 8388608.0f;
  }
};

// A token's 8B code bytes from the stage (lane-strided rows of 8B bytes).  For
// B = 4 (32-byte rows) the two 16-byte halves are read in lane-dependent order
// so a quarter-warp's LDS.128 touches 8 distinct bank groups (no 2-way conflict).
template <int B>
PQB_DEV void load_token_codes(const uint8_t* row, int lane, uint32_t* w) {
  if constexpr (B == 4) {
    const uint32_t sw = (lane >> 2) & 1u;
    const uint4 v0 = *reinterpret_cast<const uint4*>(row + (sw << 4));
    const uint4 v1 = *reinterpret_cast<const uint4*>(row + ((sw ^ 1u) << 4));
    const uint4 lo = sw ? v1 : v0, hi = sw ? v0 : v1;
    w[0] = lo.x; w[1] = lo.y; w[2] = lo.z; w[3] = lo.w;
    w[4] = hi.x; w[5] = hi.y; w[6] = hi.z; w[7] = hi.w;
  } else {
    const uint2* p = reinterpret_cast<const uint2*>(row);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const uint2 v = p[i];
      w[2 * i] = v.x;
      w[2 * i + 1] = v.y;
    }
  }
}

// ---- tensor-core helpers

PQB_DEV void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

PQB_DEV void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---- tcgen05 (5th-generation tensor cores, accumulators in tensor memory).
// Shared-memory matrix descriptor (sm_100 format): start address, leading /
// stride byte offsets (16-byte units), version 1 at bits 46-47, layout type at
// bits 61-63 (0 none, 2 = 128-byte swizzle).
PQB_DEV uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46) |
         (static_cast<uint64_t>(layout) << 61);
}
// Instruction descriptor, kind::f16: fp32 accumulate, bf16 A and B, A major
// (0 K, 1 MN), B K-major, N and M.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int m, int n, int a_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn_major) << 15) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
PQB_DEV void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate))
      : "memory");
}
// arrive on the mbarrier once every tcgen05 operation this thread issued is done
PQB_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
PQB_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
PQB_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 32 lanes (the warp's quarter) x 8 consecutive fp32 columns
PQB_DEV void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}
PQB_DEV void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---- TMA producer.  One tile = angle codes (32 * 8M B), radius codes (32 * 8N B)
// and optionally the bf16 value rows (8 KB) of 32 consecutive tokens of one page
// (tpp = tiles per page).  The caller resolves the page base (page-table load)
// one tile ahead so its latency is off the issue path.
template <int M, int N>
PQB_DEV void issue_tile(uint8_t* st, const pqb_store& s, const uint8_t* pb, int tile, int tpp, bool with_v,
                        uint64_t* bar) {
  constexpr uint32_t kA = kTile * 8 * M, kR = kTile * 8 * N, kV = kTile * 256;
  const int in_page = (tile % tpp) * kTile;
  mbar_arrive_expect_tx(bar, kA + kR + (with_v ? kV : 0u));
  bulk_g2s(st, pb + s.angle_off + in_page * 8 * M, kA, bar);
  bulk_g2s(st + kA, pb + s.radius_off + in_page * 8 * N, kR, bar);
  if (with_v) bulk_g2s(st + kA + kR, pb + s.value_off + static_cast<int64_t>(in_page) * 256, kV, bar);
}

// ------------------------------------------------------------------ epilogue

struct EpiArgs {
  void* out;
  int out_dtype;
  float* part_ml;  // [n_units][slots][G][2]
  float* part_o;   // [n_units][slots][G][d]
  int* counters;   // [n_units] finished-segment counts (zero between calls)
  int slots;       // partial slots per unit
  bool merge;      // fast kernel: last CTA of a unit merges (else leave partials)
  bool peer_mode;  // outputs go to every peer's gathered buffer (pqb_decode_attn_peer)
  int group;       // queries per unit (peer-mode destination index)
  pqb_peer_out peer;
};

PQB_DEV void store_out(void* out, int dt, int64_t idx, float v) {
  if (dt == PQB_F32) static_cast<float*>(out)[idx] = v;
  else static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
}

// Output element (unit, query g, dim e): the local [unit][G][128] array, or in
// peer mode row (sequence, q head) of every peer's gathered [B][Hq][128] buffer.
PQB_DEV void emit(const EpiArgs& ep, int64_t unit, int g, int e, float v) {
  if (!ep.peer_mode) {
    store_out(ep.out, ep.out_dtype, (unit * ep.group + g) * 128 + e, v);
    return;
  }
  const int64_t b = ep.peer.batch0 + unit / ep.peer.kv_local;
  const int64_t hq = (ep.peer.head0 + unit % ep.peer.kv_local) * ep.group + g;
  const int64_t idx = (b * ep.peer.q_heads + hq) * 128 + e;
  for (int k = 0; k < ep.peer.n_peers; ++k) store_out(ep.peer.out[k], ep.peer.out_dtype, idx, v);
}

// Peer mode, end of the kernel: once every CTA has stored its outputs (each
// fences at system scope before counting itself done), the last one increments
// flags[rank] in every peer's flag array (release, system scope).  grid_done
// lives in the workspace counter region and is left zeroed.  Caller: the
// nthreads threads that stored outputs (named barrier 1).
PQB_DEV void peer_publish(const EpiArgs& ep, int* grid_done, int tid, int nthreads) {
  if (!ep.peer_mode) return;
  __threadfence_system();
  named_sync(1, nthreads);
  if (tid == 0 && atomicAdd(grid_done, 1) == static_cast<int>(gridDim.x) - 1) {
    __threadfence_system();
    for (int k = 0; k < ep.peer.n_peers; ++k)
      asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(ep.peer.flags[k] + ep.peer.rank) : "memory");
    *grid_done = 0;
  }
}

// Persistent work split: items = n_units * tiles_max, CTA c owns
// [c*per_cta, min(items, (c+1)*per_cta)).  The slot of (unit u, CTA c) is
// c - first_cta(u).
// Cost-balanced split (DQ kernel, host make_split_balanced): CTA c owns
// [starts[c], starts[c + 1]); a CTA whose range crosses into a second unit is
// given fewer tiles (each unit segment costs a setup and a merge epilogue).
constexpr int kSplitMaxCtas = 256;
struct WorkSplit {
  int64_t items, per_cta;
  int tiles_max;
  int balanced;  // 0: uniform per_cta ranges
  int n_cta;     // CTAs of the decode launch (balanced)
  int cluster;   // DQ: CTAs per thread-block cluster (> 1: aligned split, merge through DSMEM)
  int32_t starts[kSplitMaxCtas + 1];
};

PQB_DEV int64_t cta_begin(const WorkSplit& w, int64_t c) { return w.balanced ? w.starts[c] : c * w.per_cta; }
PQB_DEV int64_t cta_end(const WorkSplit& w, int64_t c) {
  return w.balanced ? w.starts[c + 1] : min(w.items, (c + 1) * w.per_cta);
}
// the CTA whose range holds item i (balanced: the last c with starts[c] <= i)
PQB_DEV int64_t cta_of(const WorkSplit& w, int64_t i) {
  if (!w.balanced) return i / w.per_cta;
  int lo = 0, hi = w.n_cta;  // invariant: starts[lo] <= i < starts[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (w.starts[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}
PQB_DEV int64_t first_cta(const WorkSplit& w, int64_t unit) { return cta_of(w, unit * w.tiles_max); }
PQB_DEV int64_t last_cta(const WorkSplit& w, int64_t unit) { return cta_of(w, (unit + 1) * w.tiles_max - 1); }

// LSE merge of a unit's segment partials: out = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M).
// It runs in the tail of the launch (the last CTA of a unit), so its L2 reads
// are issued together: up to 8 segments in one batch of independent loads.
PQB_DEV void merge_slots(const EpiArgs& ep, int64_t unit, int nseg, int G, int tid, int nthreads) {
  constexpr int kB = 8;
  for (int i = tid; i < G * 128; i += nthreads) {
    const int g = i >> 7, e = i & 127;
    float mx = -INFINITY, L = 0.0f, O = 0.0f;
    for (int s0 = 0; s0 < nseg; s0 += kB) {
      float ms[kB], ls[kB], os[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {  // slots past nseg re-read the last one (in bounds) and are masked
        const bool ok = s0 + k < nseg;
        const int64_t sl = (unit * ep.slots + min(s0 + k, nseg - 1)) * G + g;
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
      const float r = exp2f(mx - bm);  // rescale what was merged so far (0 when mx = -inf)
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
}

// End of a unit segment.  Every warp has written, for each query g, its running
// max, its row sum and its 128 output accumulators into red[warp][g][132]
// (m, l, pad, pad, o[128]).  Merge the warps; a CTA covering the whole unit
// stores the output, otherwise it writes a partial slot and the last CTA to
// finish the unit LSE-merges the slots.  Caller: the nthreads threads
// (tid < nthreads) that wrote red, after the red writes; it synchronises them
// on named barrier 1.
template <int G>
PQB_DEV void finish_segment(const EpiArgs& ep, const WorkSplit& ws, int64_t unit, const float* red, int* s_flag,
                            int tid, int nthreads) {
  named_sync(1, nthreads);
  const int64_t c_first = first_cta(ws, unit);
  const int nseg = static_cast<int>(last_cta(ws, unit) - c_first + 1);
  const bool direct = nseg == 1;
  const int64_t slot = (unit * ep.slots + (blockIdx.x - c_first)) * G;
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
    if (direct && ep.merge) {
      emit(ep, unit, g, e, O / L);
    } else {
      ep.part_o[(slot + g) * 128 + e] = O;
      if (e == 0) {
        ep.part_ml[2 * (slot + g)] = mx;
        ep.part_ml[2 * (slot + g) + 1] = L;
      }
    }
  }
  if (direct || !ep.merge) return;
  __threadfence();
  named_sync(1, nthreads);
  if (tid == 0) *s_flag = atomicAdd(ep.counters + unit, 1) == nseg - 1;
  named_sync(1, nthreads);
  if (*s_flag) {
    __threadfence();
    merge_slots(ep, unit, nseg, G, tid, nthreads);
    if (tid == 0) ep.counters[unit] = 0;  // leave the workspace zeroed for the next call
  }
}

struct DecodeArgs;
// decode_dq.cu: dequantize + tensor-core scoring variant of the fused kernel
// (G in {4, 8}).  handled = false when (m, n) has no instance.  Two builds:
// dq_prmt (product table at a fixed shared-window address, the default) returns
// kDqLayoutUnavailable when this device's shared window is laid out so the
// table cannot sit there; dq_lin (decode_dq_lin.cu, linear layout) always runs.
constexpr int kDqLayoutUnavailable = -1;
namespace dq_prmt {
int launch_decode_dq(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s,
                     bool& handled);
int dq_cluster_capacity(int group, int mn, int value_dtype, int cl);
}
namespace dq_lin {
int launch_decode_dq(const DecodeArgs& a, const EpiArgs& ep, const WorkSplit& ws, int grid, cudaStream_t s,
                     bool& handled);
int dq_cluster_capacity(int group, int mn, int value_dtype, int cl);
}

}  // namespace pqb
