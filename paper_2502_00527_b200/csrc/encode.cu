// HP-1: key-cache encoder kernels (sm_100a).
//
//   K1 radius_max_*      per-(unit, sub-channel) max of fl64(x^2 + y^2)
//                        -> compute_radius_scales (polar_codec.py:236-251)
//   K1' scales_finalize  fp16( fl32(sqrt(max)) / (2^n - 1) )   (polar_codec.py:250-251, 77-81)
//   K2 encode_v8 / encode_generic
//                        quantize_subvectors + pack_stream + _encode_block
//                        (polar_codec.py:281-302, 98-110; kv_cache.py:191-197)
//   store_values / store_residual / append
//                        kv_cache.py:175-176, 179-189, 199-209
//
// Memory layout: keys are read with 128-bit loads, one thread per 8 consecutive
// sub-channels of a token (x-half and y-half for HALF_SPLIT, one 8-pair run for
// ADJACENT).  A warp therefore owns 256 consecutive codes = a contiguous 32*b-byte
// span of each stream; the lanes assemble whole 32-bit words with warp shuffles
// and write them with coalesced 32-bit stores straight into the paged store.
#include "polar_math.cuh"
#include "kernels.h"

#include <cstdlib>
#include <cstring>

#include <algorithm>

namespace pqb {

PQB_DEV uint8_t* page_base(const pqb_store& s, int64_t unit, int64_t page) {
  const int64_t pid = s.page_table ? static_cast<int64_t>(__ldg(s.page_table + unit * s.max_pages + page))
                                   : unit * s.max_pages + page;
  return s.pool + pid * s.page_bytes;
}

// Monotone map of a non-negative double to uint64 for atomicMax.
PQB_DEV unsigned long long dbits(double v) { return static_cast<unsigned long long>(__double_as_longlong(v)); }

PQB_DEV bool finite2(float x, float y) { return fabsf(x) <= 3.40282347e38f && fabsf(y) <= 3.40282347e38f; }

// ------------------------------------------------------------------ K1

// The exact per-channel maximum of d2 = fl64(x^2 + y^2) needs double precision
// only for candidates: f = fl32(x*x + fl32(y*y)) is within 2^-23 (relative) of
// d2, so any element whose d2 could be the maximum has f >= (running max of f)
// * (1 - 2^-20).  Only those take the double path; for random data that is a
// vanishing fraction after the first few tokens.  A token row's eight channels
// share one branch.  NaN/Inf inputs always become candidates (their f bits
// compare above any finite threshold) and propagate through the integer max
// of the double bits into the scale, where finalize flags them.
template <int DT, int LAYOUT>
__global__ void __launch_bounds__(256) radius_max_v8_kernel(const void* __restrict__ keys, int64_t T,
                                                            int half, int64_t unit_stride,
                                                            int64_t tok_stride, int64_t chunk,
                                                            unsigned long long* __restrict__ maxsq,
                                                            int32_t* __restrict__ flags) {
  __shared__ unsigned long long s_red[8][256];  // [channel-in-group][thread]
  const int unit = blockIdx.y;
  const int tpr = half >> 3;  // threads per token row
  const int rows = 256 / tpr;
  const int cg = threadIdx.x % tpr, row = threadIdx.x / tpr;
  const int64_t t_begin = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t t_end = min(T, t_begin + chunk);
  const int64_t ubase = static_cast<int64_t>(unit) * unit_stride;
  unsigned long long dmax[8];  // exact max of d2 (double bits; non-negative -> integer order)
  uint32_t thr[8];             // candidate threshold on f bits (f >= 0: integer order; NaN sorts high)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    dmax[i] = 0ull;
    thr[i] = 0u;
  }
  auto load_row = [&](int64_t t, float (&x)[8], float (&y)[8]) {
    const int64_t rb = ubase + t * tok_stride;
    if constexpr (LAYOUT == PQB_HALF_SPLIT) {
      load8<DT>(keys, rb + 8 * cg, x);
      load8<DT>(keys, rb + half + 8 * cg, y);
    } else {
      float v0[8], v1[8];
      load8<DT>(keys, rb + 16 * cg, v0);
      load8<DT>(keys, rb + 16 * cg + 8, v1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[i] = v0[2 * i]; y[i] = v0[2 * i + 1];
        x[4 + i] = v1[2 * i]; y[4 + i] = v1[2 * i + 1];
      }
    }
  };
  auto consider = [&](const float (&x)[8], const float (&y)[8]) {
    float f[8];
    bool cand = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      f[i] = fmaf(x[i], x[i], y[i] * y[i]);
      cand |= __float_as_uint(f[i]) >= thr[i];
    }
    if (cand) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (__float_as_uint(f[i]) >= thr[i]) {
          const double xd = x[i], yd = y[i];
          const unsigned long long db = dbits(__fma_rn(xd, xd, __dmul_rn(yd, yd)));
          dmax[i] = db > dmax[i] ? db : dmax[i];
          const uint32_t nt = __float_as_uint(f[i] * (1.0f - 0x1p-20f));
          thr[i] = f[i] <= 3.40282347e38f ? (nt > thr[i] ? nt : thr[i]) : 0u;  // non-finite: all candidates
        }
      }
    }
  };
  // four token rows per iteration: all loads issued before any use
  int64_t t = t_begin + row;
  for (; t + 3 * rows < t_end; t += 4 * rows) {
    float x0[8], y0[8], x1[8], y1[8], x2[8], y2[8], x3[8], y3[8];
    load_row(t, x0, y0);
    load_row(t + rows, x1, y1);
    load_row(t + 2 * rows, x2, y2);
    load_row(t + 3 * rows, x3, y3);
    consider(x0, y0);
    consider(x1, y1);
    consider(x2, y2);
    consider(x3, y3);
  }
  for (; t < t_end; t += rows) {
    float x0[8], y0[8];
    load_row(t, x0, y0);
    consider(x0, y0);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) s_red[i][threadIdx.x] = dmax[i];
  __syncthreads();
  for (int c = threadIdx.x; c < half; c += 256) {
    const int g = c >> 3, i = c & 7;
    unsigned long long m = 0ull;
    for (int r = 0; r < rows; ++r) {
      const unsigned long long v = s_red[i][r * tpr + g];
      m = v > m ? v : m;
    }
    if (m) atomicMax(maxsq + static_cast<int64_t>(unit) * half + c, m);
  }
}

// Threshold seed for the dense pass: the exact max of d2 over every 64th token
// row of each unit (1/64 of the bytes), atomically max-ed into maxsq.  The
// dense pass starts its candidate thresholds at fl32(seed) * (1 - 2^-20)
// instead of 0: an element whose d2 can reach the final max has
// f >= d2 (1 - 2^-23) >= seed (1 - 2^-23) > that threshold, so exactness is
// unchanged, while the early-row candidate flood (at warp level, nearly
// every iteration took the double-precision branch) disappears.
constexpr int kSeedStride = 64;

template <int DT, int LAYOUT>
__global__ void __launch_bounds__(256) radius_seed_kernel(const void* __restrict__ keys, int64_t T, int half,
                                                          int64_t unit_stride, unsigned long long* __restrict__ maxsq) {
  const int unit = blockIdx.y;
  const int tpr = half >> 3;
  const int rows = 256 / tpr;
  const int cg = threadIdx.x % tpr, row = threadIdx.x / tpr;
  unsigned long long dmax[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  const int64_t n_samples = (T + kSeedStride - 1) / kSeedStride;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * rows + row; s < n_samples; s += static_cast<int64_t>(gridDim.x) * rows) {
    const int64_t rb = static_cast<int64_t>(unit) * unit_stride + s * kSeedStride * 2 * half;
    float x[8], y[8];
    if constexpr (LAYOUT == PQB_HALF_SPLIT) {
      load8<DT>(keys, rb + 8 * cg, x);
      load8<DT>(keys, rb + half + 8 * cg, y);
    } else {
      float v0[8], v1[8];
      load8<DT>(keys, rb + 16 * cg, v0);
      load8<DT>(keys, rb + 16 * cg + 8, v1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[i] = v0[2 * i]; y[i] = v0[2 * i + 1];
        x[4 + i] = v1[2 * i]; y[4 + i] = v1[2 * i + 1];
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double xd = x[i], yd = y[i];
      const unsigned long long db = dbits(__fma_rn(xd, xd, __dmul_rn(yd, yd)));
      dmax[i] = db > dmax[i] ? db : dmax[i];
    }
  }
  __shared__ unsigned long long s_red[8][256];  // block max first: one atomic per (block, channel)
#pragma unroll
  for (int i = 0; i < 8; ++i) s_red[i][threadIdx.x] = dmax[i];
  __syncthreads();
  for (int c = threadIdx.x; c < half; c += 256) {
    const int g = c >> 3, i = c & 7;
    unsigned long long m = 0ull;
    for (int r = 0; r < rows; ++r) m = s_red[i][r * tpr + g] > m ? s_red[i][r * tpr + g] : m;
    if (m) atomicMax(maxsq + static_cast<int64_t>(unit) * half + c, m);
  }
}

// Same reduction for dense rows (tok_stride == d) fed by the TMA bulk-copy
// engine: a 4-stage ring of 16 KB row blocks per CTA keeps ~64 KB per CTA in
// flight independent of register pressure; threads read their 8-channel
// slices from shared memory.
constexpr int kRmaxStages = 4;
constexpr int kRmaxStageBytes = 16384;

template <int DT, int LAYOUT>
__global__ void __launch_bounds__(256) radius_max_tma_kernel(const void* __restrict__ keys, int64_t T, int half,
                                                             int64_t unit_stride, int64_t chunk,
                                                             unsigned long long* __restrict__ maxsq) {
  extern __shared__ __align__(128) uint8_t rsm[];
  __shared__ uint64_t bars[kRmaxStages];
  constexpr int EB = DType<DT>::kBytes;
  const int unit = blockIdx.y;
  const int d = 2 * half;
  const int row_bytes = d * EB;
  const int rows_per_stage = kRmaxStageBytes / row_bytes;
  const int tpr = half >> 3;
  const int rows = 256 / tpr;
  const int cg = threadIdx.x % tpr, row = threadIdx.x / tpr;
  const int64_t t_begin = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t t_end = min(T, t_begin + chunk);
  const int n_stages = static_cast<int>((t_end - t_begin + rows_per_stage - 1) / rows_per_stage);
  const uint8_t* src = static_cast<const uint8_t*>(keys) + (static_cast<int64_t>(unit) * unit_stride + t_begin * d) * EB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRmaxStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int64_t r0 = static_cast<int64_t>(k) * rows_per_stage;
    const int64_t left = (t_end - t_begin) - r0;
    const int nr = left < rows_per_stage ? static_cast<int>(left) : rows_per_stage;
    const int slot = k % kRmaxStages;
    mbar_arrive_expect_tx(bars + slot, nr * row_bytes);
    bulk_g2s(rsm + slot * kRmaxStageBytes, src + r0 * row_bytes, nr * row_bytes, bars + slot);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < kRmaxStages && k < n_stages; ++k) issue(k);
  unsigned long long dmax[8];
  uint32_t thr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {  // seeded by radius_seed_kernel (exact d2 of sampled rows)
    dmax[i] = 0ull;
    const double seed = __longlong_as_double(static_cast<long long>(
        __ldcg(maxsq + static_cast<int64_t>(unit) * half + 8 * cg + i)));
    const float sf = __double2float_rd(seed) * (1.0f - 0x1p-20f);
    thr[i] = sf <= 3.40282347e38f ? __float_as_uint(sf) : 0u;  // NaN / Inf seed: every element a candidate
  }
  for (int k = 0; k < n_stages; ++k) {
    const int slot = k % kRmaxStages;
    mbar_wait(bars + slot, (k / kRmaxStages) & 1);
    const int64_t left = (t_end - t_begin) - static_cast<int64_t>(k) * rows_per_stage;
    const int nr = left < rows_per_stage ? static_cast<int>(left) : rows_per_stage;
    const uint8_t* st = rsm + slot * kRmaxStageBytes;
    for (int r = row; r < nr; r += rows) {
      float x[8], y[8];
      const void* rp = st + r * row_bytes;
      if constexpr (LAYOUT == PQB_HALF_SPLIT) {
        load8s<DT>(rp, 8 * cg, x);
        load8s<DT>(rp, half + 8 * cg, y);
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
      float f[8];
      bool cand = false;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        f[i] = fmaf(x[i], x[i], y[i] * y[i]);
        cand |= __float_as_uint(f[i]) >= thr[i];
      }
      if (cand) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (__float_as_uint(f[i]) >= thr[i]) {
            const double xd = x[i], yd = y[i];
            const unsigned long long db = dbits(__fma_rn(xd, xd, __dmul_rn(yd, yd)));
            dmax[i] = db > dmax[i] ? db : dmax[i];
            const uint32_t nt = __float_as_uint(f[i] * (1.0f - 0x1p-20f));
            thr[i] = f[i] <= 3.40282347e38f ? (nt > thr[i] ? nt : thr[i]) : 0u;
          }
        }
      }
    }
    __syncthreads();  // every thread is done with this slot
    if (threadIdx.x == 0 && k + kRmaxStages < n_stages) {
      fence_proxy_async_smem();
      issue(k + kRmaxStages);
    }
  }
  // block reduction of the per-thread maxima (reuse stage memory)
  unsigned long long* red = reinterpret_cast<unsigned long long*>(rsm);  // [8][256]
#pragma unroll
  for (int i = 0; i < 8; ++i) red[i * 256 + threadIdx.x] = dmax[i];
  __syncthreads();
  for (int c = threadIdx.x; c < half; c += 256) {
    const int g = c >> 3, i = c & 7;
    unsigned long long m = 0ull;
    for (int r = 0; r < rows; ++r) {
      const unsigned long long v = red[i * 256 + r * tpr + g];
      m = v > m ? v : m;
    }
    if (m) atomicMax(maxsq + static_cast<int64_t>(unit) * half + c, m);
  }
}

// Any even d / layout / stride / alignment; one element pair per thread step.
template <int DT>
__global__ void __launch_bounds__(256) radius_max_generic_kernel(const void* __restrict__ keys, int64_t T,
                                                                 int half, int layout,
                                                                 int64_t unit_stride, int64_t tok_stride,
                                                                 int64_t chunk,
                                                                 unsigned long long* __restrict__ maxsq,
                                                                 int32_t* __restrict__ flags) {
  extern __shared__ unsigned long long s_max[];  // [half]
  const int unit = blockIdx.y;
  for (int c = threadIdx.x; c < half; c += blockDim.x) s_max[c] = 0ull;
  __syncthreads();
  const int64_t f_begin = static_cast<int64_t>(blockIdx.x) * chunk * half;
  const int64_t f_end = min(T * half, f_begin + chunk * half);
  const int64_t ubase = static_cast<int64_t>(unit) * unit_stride;
  bool bad = false;
  for (int64_t f = f_begin + threadIdx.x; f < f_end; f += blockDim.x) {
    const int64_t t = f / half;
    const int j = static_cast<int>(f - t * half);
    const int64_t rb = ubase + t * tok_stride;
    const int64_t ex = layout == PQB_HALF_SPLIT ? j : 2 * j;
    const int64_t ey = layout == PQB_HALF_SPLIT ? j + half : 2 * j + 1;
    const float x = load1<DT>(keys, rb + ex), y = load1<DT>(keys, rb + ey);
    bad |= !finite2(x, y);
    const double xd = x, yd = y;
    const double d2 = __fma_rn(xd, xd, __dmul_rn(yd, yd));
    if (d2 > 0.0) atomicMax(s_max + j, dbits(d2));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, PQB_FLAG_NONFINITE);
  __syncthreads();
  for (int c = threadIdx.x; c < half; c += blockDim.x)
    if (s_max[c]) atomicMax(maxsq + static_cast<int64_t>(unit) * half + c, s_max[c]);
}

__global__ void scales_finalize_kernel(const unsigned long long* __restrict__ maxsq, int64_t count,
                                       int n_bits, uint16_t* __restrict__ scales,
                                       int32_t* __restrict__ flags) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double d2 = __longlong_as_double(static_cast<long long>(maxsq[i]));
  if (!(d2 <= 1.79769313486231570815e308)) atomicOr(flags, PQB_FLAG_NONFINITE);  // NaN/Inf keys
  const float top = __double2float_rn(__dsqrt_rn(d2));                 // radius.max(axis=0), fp32
  const float s = __fdiv_rn(top, static_cast<float>((1 << n_bits) - 1));  // fp32 / int
  const __half h = __float2half_rn(s);                                  // ChannelScales -> fp16
  if (__hisinf(h) || __hisnan(h)) atomicOr(flags, PQB_FLAG_SCALE_OVERFLOW);
  scales[i] = __half_as_ushort(h);
}

// ------------------------------------------------------------------ K2

// Word `w` of the bit string formed by concatenating the lanes' `cb`-bit chunks
// (cb = 8*b, lane order).  Warp-collective: every lane must call with the same
// `cb`; lanes pass their own w (only lanes with w < 8*b use the result).
PQB_DEV uint32_t warp_word(unsigned long long chunk, int cb, int nch, int w) {
  const int bit = 32 * w;
  const int c0 = bit / cb;
  const int o = bit - c0 * cb;
  unsigned long long v = 0ull;
  int have = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < nch) {  // warp-uniform
      const unsigned long long cv = __shfl_sync(0xffffffffu, chunk, (c0 + k) & 31);
      if (k == 0) {
        v = cv >> o;
        have = cb - o;
      } else if (have < 32 && c0 + k < 32) {
        v |= cv << have;
        have += cb;
      }
    }
  }
  return static_cast<uint32_t>(v);
}

PQB_DEV int chunks_per_word(int b) { return b == 1 ? 4 : (b == 2 ? 2 : ((b == 4 || b == 8) ? 1 : 2)); }

template <int DT, int LAYOUT, int M>
__global__ void __launch_bounds__(256) encode_v8_kernel(const void* __restrict__ keys, int64_t T, int half,
                                                        int64_t unit_stride, int64_t tok_stride,
                                                        int64_t chunk, int n_bits,
                                                        const uint16_t* __restrict__ scales, pqb_store st,
                                                        const int32_t* __restrict__ tok_offset,
                                                        int64_t tok_offset_const,
                                                        unsigned long long* __restrict__ clamp_counts,
                                                        int32_t* __restrict__ flags) {
  __shared__ float s_tan[32], s_thr[32];
  __shared__ unsigned int s_clamp;
  if (threadIdx.x < 32) {
    s_tan[threadIdx.x] = kEdgeTan[M][threadIdx.x];
    s_thr[threadIdx.x] = kEdgeThr[M][threadIdx.x];
  }
  if (threadIdx.x == 0) s_clamp = 0u;
  __syncthreads();
  const int unit = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int tpr = half >> 3;
  const int rows = 256 / tpr;
  const int cg = threadIdx.x % tpr, row = threadIdx.x / tpr;
  const int warp_row0 = (threadIdx.x >> 5) * (32 / tpr);
  const int64_t off = (tok_offset ? static_cast<int64_t>(tok_offset[unit]) : 0) + tok_offset_const;
  const int64_t t_begin = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t t_end = min(T, t_begin + chunk);
  const int64_t ubase = static_cast<int64_t>(unit) * unit_stride;

  float s32[8], inv[8];
  {
    const uint4 sv = __ldg(reinterpret_cast<const uint4*>(scales + static_cast<int64_t>(unit) * half + 8 * cg));
    const uint32_t w[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      s32[2 * i] = half_bits_to_f32(static_cast<uint16_t>(w[i] & 0xffffu));
      s32[2 * i + 1] = half_bits_to_f32(static_cast<uint16_t>(w[i] >> 16));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) inv[i] = s32[i] > 0.0f ? __frcp_rn(s32[i]) : 0.0f;
  }
  uint32_t nz_mask = 0u;  // channels with a non-zero scale
#pragma unroll
  for (int i = 0; i < 8; ++i) nz_mask |= static_cast<uint32_t>(s32[i] > 0.0f) << i;
  const int wpt_a = half * M / 32, wpt_r = half * n_bits / 32;  // 32-bit words per token
  const int cb_a = 8 * M, cb_r = 8 * n_bits;
  const int nch_a = chunks_per_word(M), nch_r = chunks_per_word(n_bits);
  // words this lane stores per pass: w = lane + 32*k; token / word-in-token are lane constants
  const int tw_a0 = lane / wpt_a, wi_a0 = lane - tw_a0 * wpt_a;
  const int tw_a1 = (lane + 32) / wpt_a, wi_a1 = lane + 32 - tw_a1 * wpt_a;
  const int tw_r0 = lane / wpt_r, wi_r0 = lane - tw_r0 * wpt_r;
  const int tw_r1 = (lane + 32) / wpt_r, wi_r1 = lane + 32 - tw_r1 * wpt_r;
  // page position of the block-iteration's first token (rows <= page_tokens:
  // one iteration crosses at most one page boundary)
  const int P = st.page_tokens;
  int64_t pg = (off + t_begin) / P;
  int in_pg = static_cast<int>(off + t_begin - pg * P);
  uint32_t clamps = 0;
  bool bad = false;

  for (int64_t base = t_begin; base < t_end; base += rows) {
    const int64_t t = base + row;
    const bool valid = t < t_end;
    float x[8], y[8];
    if (valid) {
      const int64_t rb = ubase + t * tok_stride;
      if constexpr (LAYOUT == PQB_HALF_SPLIT) {
        load8<DT>(keys, rb + 8 * cg, x);
        load8<DT>(keys, rb + half + 8 * cg, y);
      } else {
        float v0[8], v1[8];
        load8<DT>(keys, rb + 16 * cg, v0);
        load8<DT>(keys, rb + 16 * cg + 8, v1);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          x[i] = v0[2 * i]; y[i] = v0[2 * i + 1];
          x[4 + i] = v1[2 * i]; y[4 + i] = v1[2 * i + 1];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = y[i] = 0.0f;
    }
    unsigned long long ca, cr;
    encode8<M>(x, y, s32, inv, n_bits, valid ? nz_mask : 0u, ca, cr, clamps, bad, s_tan, s_thr);
    // pages of this iteration (uniform): pg, and pg+1 if the rows cross into it
    const uint8_t* pb0 = page_base(st, unit, pg);
    const uint8_t* pb1 = (in_pg + rows > P && base + (P - in_pg) < t_end) ? page_base(st, unit, pg + 1) : pb0;
    // ---- assemble and store the warp's 8*M angle words and 8*n radius words
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const int b = pass == 0 ? M : n_bits;
      const int cb = pass == 0 ? cb_a : cb_r;
      const int nch = pass == 0 ? nch_a : nch_r;
      const int wpt = pass == 0 ? wpt_a : wpt_r;
      const int64_t region = pass == 0 ? st.angle_off : st.radius_off;
      const unsigned long long chunk_bits = pass == 0 ? ca : cr;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (32 * k >= 8 * b) break;  // warp-uniform
        const int w = 32 * k + lane;
        const uint32_t word = warp_word(chunk_bits, cb, nch, w);
        const int tw = pass == 0 ? (k ? tw_a1 : tw_a0) : (k ? tw_r1 : tw_r0);
        const int wi = pass == 0 ? (k ? wi_a1 : wi_a0) : (k ? wi_r1 : wi_r0);
        if (w < 8 * b && base + warp_row0 + tw < t_end) {
          int in_w = in_pg + warp_row0 + tw;
          const uint8_t* pb = pb0;
          if (in_w >= P) {
            in_w -= P;
            pb = pb1;
          }
          *reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(pb) + region + (static_cast<int64_t>(in_w) * wpt + wi) * 4) =
              word;
        }
      }
    }
    in_pg += rows;
    while (in_pg >= P) {
      in_pg -= P;
      ++pg;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, PQB_FLAG_NONFINITE);
  if (clamp_counts) {
    unsigned int c = clamps;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0 && c) atomicAdd(&s_clamp, c);
    __syncthreads();
    if (threadIdx.x == 0 && s_clamp) atomicAdd(clamp_counts + unit, static_cast<unsigned long long>(s_clamp));
  }
}

// Generic encoder: any even d, any layout/stride, runtime bits, exact path.
// Each warp owns 32 consecutive (absolute) flat codes; their b*32 bits are
// b whole words of the stream.  Words not fully covered by this call's tokens
// are merged with atomicOr (fresh pages are zero).
struct GenericSrc {
  const void* keys;  // [unit][t][d] with strides (elements)
  int dtype;
  int64_t unit_stride, tok_stride;
};

template <int DT>
PQB_DEV float ld_any(const void* p, int64_t off) { return load1<DT>(p, off); }

PQB_DEV float load_elem(const GenericSrc& s, int64_t off) {
  switch (s.dtype) {
    case PQB_F32: return ld_any<PQB_F32>(s.keys, off);
    case PQB_BF16: return ld_any<PQB_BF16>(s.keys, off);
    default: return ld_any<PQB_F16>(s.keys, off);
  }
}

// Encode flat codes [32*g, 32*g + 32) of `unit` whose token range of this call
// is [tok0, tok0 + T) (absolute).  Keys of call-token t at src row t.
PQB_DEV void encode_group_exact(const GenericSrc& src, int64_t unit, int64_t g, int64_t tok0, int64_t T,
                                int half, int layout, int m_bits, int n_bits, const float* s32_row,
                                const pqb_store& st, uint32_t& clamps, bool& bad) {
  const int lane = threadIdx.x & 31;
  const int64_t f = 32 * g + lane;
  const int64_t t_abs = f / half;
  const int j = static_cast<int>(f - t_abs * half);
  const int64_t t_call = t_abs - tok0;
  const bool valid = t_call >= 0 && t_call < T;
  uint32_t a = 0u, r = 0u;
  if (valid) {
    const int64_t rb = unit * src.unit_stride + t_call * src.tok_stride;
    const int64_t ex = layout == PQB_HALF_SPLIT ? j : 2 * j;
    const int64_t ey = layout == PQB_HALF_SPLIT ? j + half : 2 * j + 1;
    const float x = load_elem(src, rb + ex), y = load_elem(src, rb + ey);
    bad |= !finite2(x, y);
    encode_pair_exact(x, y, s32_row[j], m_bits, n_bits, a, r, clamps);
  }
  const unsigned vmask = __ballot_sync(0xffffffffu, valid);
  if (vmask == 0u) return;
  const int64_t page_tok = st.page_tokens;
  const int64_t page = (32 * g) / (page_tok * half);
  const int64_t g_in_page = g - page * page_tok * half / 32;
  uint8_t* pbase = page_base(st, unit, page);
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int b = pass == 0 ? m_bits : n_bits;
    const uint32_t code = pass == 0 ? a : r;
    uint32_t* words = reinterpret_cast<uint32_t*>(pbase + (pass == 0 ? st.angle_off : st.radius_off)) +
                      g_in_page * b;
    for (int w = 0; w < b; ++w) {
      const int kb = 32 * w + lane;  // my bit in word w
      const uint32_t c = __shfl_sync(0xffffffffu, code, kb / b);
      const uint32_t word = __ballot_sync(0xffffffffu, (c >> (kb % b)) & 1u);
      // lanes (codes) touching word w: [32w/b, (32w+31)/b]
      const int lo = (32 * w) / b, hi = (32 * w + 31) / b;
      const unsigned need = (hi >= 31 ? 0xffffffffu : ((2u << hi) - 1u)) & ~((1u << lo) - 1u);
      if (lane == 0) {
        if ((vmask & need) == need) words[w] = word;
        else if (vmask & need) atomicOr(words + w, word);
      }
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(256) encode_generic_kernel(GenericSrc src, int64_t T, int half, int layout,
                                                             int m_bits, int n_bits,
                                                             const uint16_t* __restrict__ scales, pqb_store st,
                                                             const int32_t* __restrict__ tok_offset,
                                                             int64_t tok_offset_const, int64_t groups_per_block,
                                                             unsigned long long* __restrict__ clamp_counts,
                                                             int32_t* __restrict__ flags) {
  extern __shared__ float s_scale[];  // [half]
  const int64_t unit = blockIdx.y;
  for (int c = threadIdx.x; c < half; c += blockDim.x)
    s_scale[c] = half_bits_to_f32(scales[unit * half + c]);
  __syncthreads();
  const int64_t tok0 = (tok_offset ? static_cast<int64_t>(tok_offset[unit]) : 0) + tok_offset_const;
  const int64_t f_lo = tok0 * half, f_hi = (tok0 + T) * half;
  const int64_t g_lo = f_lo / 32, g_hi = (f_hi + 31) / 32;
  const int64_t gb = g_lo + static_cast<int64_t>(blockIdx.x) * groups_per_block;
  const int64_t ge = min(g_hi, gb + groups_per_block);
  uint32_t clamps = 0;
  bool bad = false;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int64_t g = gb + warp; g < ge; g += nwarps)
    encode_group_exact(src, unit, g, tok0, T, half, layout, m_bits, n_bits, s_scale, st, clamps, bad);
  const int lane = threadIdx.x & 31;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, PQB_FLAG_NONFINITE);
  if (clamp_counts) {
    unsigned int c = clamps;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0 && c) atomicAdd(clamp_counts + unit, static_cast<unsigned long long>(c));
  }
}

// ------------------------------------------------------------- values

// d = 128 bf16 pages: one thread per (token, 16-byte chunk) -> one 128-bit
// store at the chunk's swizzled slot (value_offset()).
template <int DT>
__global__ void store_values_v8_kernel(const void* __restrict__ vals, int64_t T, int64_t unit_stride,
                                       int64_t tok_stride, pqb_store st, int64_t tok_offset_const) {
  const int64_t unit = blockIdx.y;
  const int64_t n = T * 16;
  const int P = st.page_tokens;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i >> 4;
    const int c = static_cast<int>(i & 15);
    uint4 w = make_uint4(0u, 0u, 0u, 0u);
    if (vals) {
      float v[8];
      load8<DT>(vals, unit * unit_stride + t * tok_stride + 8 * c, v);
      uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
        wp[k] = *reinterpret_cast<const uint32_t*>(&b);
      }
    }
    const int64_t ta = tok_offset_const + t;
    const int64_t page = ta / P;
    const int64_t tp = ta - page * P;
    uint8_t* dst = page_base(st, unit, page) + st.value_off + value_offset_bf16_128(tp, 8 * c);
    *reinterpret_cast<uint4*>(dst) = w;
  }
}


__global__ void store_values_kernel(const void* __restrict__ vals, int src_dtype, int64_t T, int d,
                                    int64_t unit_stride, int64_t tok_stride, pqb_store st,
                                    const int32_t* __restrict__ tok_offset, int64_t tok_offset_const) {
  const int64_t unit = blockIdx.y;
  const int64_t off = (tok_offset ? static_cast<int64_t>(tok_offset[unit]) : 0) + tok_offset_const;
  const int64_t n = T * d;
  const int vbytes = st.value_dtype == PQB_F32 ? 4 : 2;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / d;
    const int e = static_cast<int>(i - t * d);
    float v = 0.0f;
    if (vals) {
      const int64_t so = unit * unit_stride + t * tok_stride + e;
      v = src_dtype == PQB_F32 ? load1<PQB_F32>(vals, so)
                               : (src_dtype == PQB_BF16 ? load1<PQB_BF16>(vals, so) : load1<PQB_F16>(vals, so));
    }
    const int64_t ta = off + t;
    const int64_t page = ta / st.page_tokens;
    uint8_t* p = page_base(st, unit, page) + st.value_off +
                 value_offset(ta - page * st.page_tokens, e, d, st.value_dtype);
    if (vbytes == 4) *reinterpret_cast<float*>(p) = v;
    else *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
  }
}

// PQB_VQ{2,4,8} pages: _quantize_slices along each token row (baseline_quant.py:58-66:
// zp = min, scale = fl(fl(max - zp) / (2^b - 1)), code = rint(fl(fl(v - zp) / scale))
// clipped to [0, 2^b - 1], scale == 0 -> 0), written in the fragment order of
// vq_pos().  One CTA per (32-token tile, unit); tile starts are 32-aligned.
__global__ void __launch_bounds__(256) store_values_vq_kernel(const void* __restrict__ vals, int src_dtype,
                                                               int64_t T, int64_t unit_stride, int64_t tok_stride,
                                                               pqb_store st, int64_t tok_offset_const,
                                                               int32_t* __restrict__ flags) {
  __shared__ uint8_t codes[32][132];
  __shared__ float2 params[32];
  const int bits = vq_bits(st.value_dtype);
  const float top = static_cast<float>((1 << bits) - 1);
  const int64_t unit = blockIdx.y;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool bad = false;
  for (int r = warp; r < 32; r += 8) {  // token rows: warp-wide min / max, then codes
    const int64_t t = t0 + r;
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = 0.0f;
      if (vals && t < T) {
        const int64_t so = unit * unit_stride + t * tok_stride + lane + 32 * k;
        v[k] = src_dtype == PQB_F32 ? load1<PQB_F32>(vals, so)
                                    : (src_dtype == PQB_BF16 ? load1<PQB_BF16>(vals, so) : load1<PQB_F16>(vals, so));
      }
      bad |= !(fabsf(v[k]) <= 3.40282347e38f);
    }
    float mn = fminf(fminf(v[0], v[1]), fminf(v[2], v[3])), mx = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const float scale = __fdiv_rn(__fsub_rn(mx, mn), top);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float raw = scale == 0.0f ? 0.0f : rintf(__fdiv_rn(__fsub_rn(v[k], mn), scale));
      raw = fminf(fmaxf(raw, 0.0f), top);
      codes[r][lane + 32 * k] = t < T ? static_cast<uint8_t>(raw) : 0;
    }
    if (lane == 0) params[r] = t < T ? make_float2(mn, scale) : make_float2(0.0f, 0.0f);
  }
  __syncthreads();
  const int64_t ta = tok_offset_const + t0;
  const int64_t page = ta / st.page_tokens;
  const int64_t tp = ta - page * st.page_tokens;  // multiple of 32
  uint8_t* pb = page_base(st, unit, page);
  uint32_t* wout = reinterpret_cast<uint32_t*>(pb + st.value_off + (tp >> 5) * vq_tile_bytes(bits));
  // one thread per (dim block, token block, lane) chunk of 8 codes: its words
  // (b = 4: one, b = 8: two, b = 2: one half word) in vq_pos() order
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    const int blk = i >> 5, mt = blk >> 1, ks = blk & 1, ln = i & 31, g = ln >> 2, tq = ln & 3;
    uint32_t lo = 0u, hi = 0u, two = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int t = 16 * ks + 2 * tq + c + 8 * (k >> 1), e = 16 * mt + g + 8 * (k & 1);
        const uint32_t code = codes[t][e];
        lo |= (code & 15u) << (4 * k + 16 * c);
        hi |= (code >> 4) << (4 * k + 16 * c);
        two |= code << (8 * c + 2 * k);
      }
    if (bits == 4) {
      wout[i] = lo;
    } else if (bits == 8) {
      reinterpret_cast<uint2*>(wout)[i] = make_uint2(lo, hi);
    } else {  // b = 2: blocks 2j, 2j + 1 share word j * 32 + lane (low / high half)
      reinterpret_cast<uint16_t*>(wout)[2 * ((blk >> 1) * 32 + ln) + (blk & 1)] = static_cast<uint16_t>(two);
    }
  }
  if (threadIdx.x < 32) reinterpret_cast<float2*>(pb + vq_params_off(st))[tp + threadIdx.x] = params[threadIdx.x];
  if (bad && flags) atomicOr(flags, PQB_FLAG_NONFINITE);
}

__global__ void store_residual_kernel(const void* __restrict__ keys, int src_dtype, int64_t T, int d,
                                      int64_t unit_stride, int64_t tok_stride, float* __restrict__ ring,
                                      int res_cap, int64_t tok_offset_const, int32_t* __restrict__ flags) {
  const int64_t unit = blockIdx.y;
  const int64_t n = T * d;
  bool bad = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / d;
    const int e = static_cast<int>(i - t * d);
    const int64_t so = unit * unit_stride + t * tok_stride + e;
    const float v = src_dtype == PQB_F32 ? load1<PQB_F32>(keys, so)
                                         : (src_dtype == PQB_BF16 ? load1<PQB_BF16>(keys, so) : load1<PQB_F16>(keys, so));
    bad |= !(fabsf(v) <= 3.40282347e38f);
    const int64_t slot = (tok_offset_const + t) % res_cap;
    ring[(unit * res_cap + slot) * d + e] = v;
  }
  if (bad) atomicOr(flags, PQB_FLAG_NONFINITE);
}

// ----------------------------------------------------------------- K5

// One token's value row into a PQB_VQ{2,4,8} page (append): quantize as
// store_values_vq_kernel, OR the code bits into the tile's words (pages start
// zeroed and every token slot is written once).  red: >= 2 * 32 floats of
// shared scratch.  Caller: the whole block (d = 128 threads or more).
__device__ void append_value_vq(const pqb_cache& c, int64_t unit, int64_t T, const void* vals, int val_dtype,
                                 float* red, bool& bad) {
  const int e = threadIdx.x, lane = e & 31, warp = e >> 5, nw = (blockDim.x + 31) >> 5;
  float v = 0.0f;
  if (e < 128 && vals) {
    const int64_t ko = unit * 128 + e;
    v = val_dtype == PQB_F32 ? load1<PQB_F32>(vals, ko)
                             : (val_dtype == PQB_BF16 ? load1<PQB_BF16>(vals, ko) : load1<PQB_F16>(vals, ko));
  }
  if (e < 128) bad |= !(fabsf(v) <= 3.40282347e38f);
  float mn = e < 128 ? v : INFINITY, mx = e < 128 ? v : -INFINITY;
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    red[warp] = mn;
    red[32 + warp] = mx;
  }
  __syncthreads();
  mn = INFINITY;
  mx = -INFINITY;
  for (int w = 0; w < nw; ++w) {
    mn = fminf(mn, red[w]);
    mx = fmaxf(mx, red[32 + w]);
  }
  const int vb = vq_bits(c.store.value_dtype);
  const float top = static_cast<float>((1 << vb) - 1);
  const float scale = __fdiv_rn(__fsub_rn(mx, mn), top);
  const int64_t page = T / c.store.page_tokens, tp = T - page * c.store.page_tokens;
  uint8_t* pb = page_base(c.store, unit, page);
  if (e < 128) {
    float raw = scale == 0.0f ? 0.0f : rintf(__fdiv_rn(__fsub_rn(v, mn), scale));
    raw = fminf(fmaxf(raw, 0.0f), top);
    int w, sh;
    vq_pos(vb, static_cast<int>(tp & 31), e, w, sh);
    const uint32_t code = static_cast<uint32_t>(raw);
    unsigned int* words = reinterpret_cast<unsigned int*>(pb + c.store.value_off + (tp >> 5) * vq_tile_bytes(vb));
    const uint32_t b0 = (vb == 8 ? (code & 15u) : code) << sh;
    if (b0) atomicOr(words + w, b0);
    if (vb == 8 && (code >> 4)) atomicOr(words + w + 1, (code >> 4) << sh);
  }
  if (e == 0) reinterpret_cast<float2*>(pb + vq_params_off(c.store))[tp] = make_float2(mn, scale);
  __syncthreads();
}

// One block per unit.  kv_cache.py:179-189 with the residual deque as a ring.
__global__ void __launch_bounds__(256) append_kernel(pqb_cache c, const void* __restrict__ keys, int key_dtype,
                                                     const void* __restrict__ vals, int val_dtype,
                                                     unsigned long long* __restrict__ clamp_counts,
                                                     int32_t* __restrict__ flags) {
  extern __shared__ float s_scale[];  // [half]
  const int64_t unit = blockIdx.x;
  const int d = c.d, half = d / 2;
  for (int j = threadIdx.x; j < half; j += blockDim.x) s_scale[j] = half_bits_to_f32(c.scales[unit * half + j]);
  const int64_t T = c.seq_lens[unit], Tq = c.quant_lens[unit];
  __syncthreads();
  const bool flush = (T - Tq) >= c.res_cap;  // after the push the FIFO exceeds residual_len
  uint32_t clamps = 0;
  bool bad = false;
  if (flush) {
    GenericSrc src;
    if (c.res_cap == 0) {
      src.keys = keys; src.dtype = key_dtype; src.unit_stride = d; src.tok_stride = d;
    } else {  // oldest residual key: token Tq lives in slot Tq % res_cap
      src.keys = c.residual + (unit * c.res_cap + Tq % c.res_cap) * d;
      src.dtype = PQB_F32; src.unit_stride = 0; src.tok_stride = d;
    }
    const int64_t g_lo = (Tq * half) / 32, g_hi = ((Tq + 1) * half + 31) / 32;
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int64_t g = g_lo + warp; g < g_hi; g += nwarps)
      encode_group_exact(src, unit, g, Tq, 1, half, c.layout, c.angle_bits, c.radius_bits, s_scale, c.store,
                         clamps, bad);
  }
  __syncthreads();  // the flushed slot is read before it is overwritten
  if (vq_bits(c.store.value_dtype)) append_value_vq(c, unit, T, vals, val_dtype, s_scale + half, bad);
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    const int64_t ko = unit * d + e;
    const float kv = key_dtype == PQB_F32 ? load1<PQB_F32>(keys, ko)
                                          : (key_dtype == PQB_BF16 ? load1<PQB_BF16>(keys, ko) : load1<PQB_F16>(keys, ko));
    bad |= !(fabsf(kv) <= 3.40282347e38f);
    if (c.res_cap > 0) c.residual[(unit * c.res_cap + T % c.res_cap) * d + e] = kv;
    if (c.store.value_off >= 0 && !vq_bits(c.store.value_dtype)) {
      float v = 0.0f;
      if (vals)
        v = val_dtype == PQB_F32 ? load1<PQB_F32>(vals, ko)
                                 : (val_dtype == PQB_BF16 ? load1<PQB_BF16>(vals, ko) : load1<PQB_F16>(vals, ko));
      const int64_t page = T / c.store.page_tokens;
      uint8_t* p = page_base(c.store, unit, page) + c.store.value_off +
                   value_offset(T - page * c.store.page_tokens, e, d, c.store.value_dtype);
      if (c.store.value_dtype == PQB_F32) *reinterpret_cast<float*>(p) = v;
      else *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
    }
  }
  if (bad) atomicOr(flags, PQB_FLAG_NONFINITE);
  const int lane = threadIdx.x & 31;
  unsigned int cl = clamps;
  for (int o = 16; o > 0; o >>= 1) cl += __shfl_xor_sync(0xffffffffu, cl, o);
  if (lane == 0 && cl && clamp_counts) atomicAdd(clamp_counts + unit, static_cast<unsigned long long>(cl));
  __syncthreads();
  if (threadIdx.x == 0) {
    c.seq_lens[unit] = static_cast<int32_t>(T + 1);
    if (flush) c.quant_lens[unit] = static_cast<int32_t>(Tq + 1);
  }
}

// ------------------------------------------------------------ launchers

template <int DT, int LAYOUT>
static void launch_rmax_v8(const RadiusScalesArgs& a, int64_t chunk, dim3 grid, cudaStream_t s) {
  radius_max_v8_kernel<DT, LAYOUT><<<grid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.tok_stride,
                                                        chunk, a.maxsq_ws, a.flags);
}

template <int DT, int LAYOUT>
static void launch_rmax_tma(const RadiusScalesArgs& a, int64_t chunk, dim3 grid, size_t shm, cudaStream_t s) {
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [shm] {
    return cudaFuncSetAttribute(radius_max_tma_kernel<DT, LAYOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(shm)) == cudaSuccess ? PQB_OK : PQB_ECUDA;
  });
  radius_max_tma_kernel<DT, LAYOUT><<<grid, 256, shm, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, chunk,
                                                           a.maxsq_ws);
}

int launch_radius_scales(const RadiusScalesArgs& a, cudaStream_t s) {
  const int half = a.d / 2;
  cudaMemsetAsync(a.maxsq_ws, 0, sizeof(unsigned long long) * a.n_units * half, s);
  const int64_t chunk = 4096;
  dim3 grid(static_cast<unsigned>((a.tokens + chunk - 1) / chunk), static_cast<unsigned>(a.n_units));
  const int eb = a.key_dtype == PQB_F32 ? 4 : 2;
  const bool dense = a.vector_ok && a.tok_stride == a.d && (static_cast<int64_t>(a.d) * eb) % 16 == 0 &&
                     kRmaxStageBytes % (a.d * eb) == 0 && (a.unit_stride * eb) % 16 == 0;
  if (dense) {
    const size_t shm = kRmaxStages * kRmaxStageBytes;
    const int64_t n_samples = (a.tokens + kSeedStride - 1) / kSeedStride;
    dim3 sgrid(static_cast<unsigned>(std::min<int64_t>((n_samples * (a.d / 16) + 255) / 256, 8)),
               static_cast<unsigned>(a.n_units));
    switch (a.key_dtype * 2 + a.layout) {
      case PQB_F32 * 2 + PQB_ADJACENT: radius_seed_kernel<PQB_F32, PQB_ADJACENT><<<sgrid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.maxsq_ws); break;
      case PQB_F32 * 2 + PQB_HALF_SPLIT: radius_seed_kernel<PQB_F32, PQB_HALF_SPLIT><<<sgrid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.maxsq_ws); break;
      case PQB_BF16 * 2 + PQB_ADJACENT: radius_seed_kernel<PQB_BF16, PQB_ADJACENT><<<sgrid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.maxsq_ws); break;
      case PQB_BF16 * 2 + PQB_HALF_SPLIT: radius_seed_kernel<PQB_BF16, PQB_HALF_SPLIT><<<sgrid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.maxsq_ws); break;
      case PQB_F16 * 2 + PQB_ADJACENT: radius_seed_kernel<PQB_F16, PQB_ADJACENT><<<sgrid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.maxsq_ws); break;
      default: radius_seed_kernel<PQB_F16, PQB_HALF_SPLIT><<<sgrid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.maxsq_ws); break;
    }
    switch (a.key_dtype * 2 + a.layout) {
      case PQB_F32 * 2 + PQB_ADJACENT: launch_rmax_tma<PQB_F32, PQB_ADJACENT>(a, chunk, grid, shm, s); break;
      case PQB_F32 * 2 + PQB_HALF_SPLIT: launch_rmax_tma<PQB_F32, PQB_HALF_SPLIT>(a, chunk, grid, shm, s); break;
      case PQB_BF16 * 2 + PQB_ADJACENT: launch_rmax_tma<PQB_BF16, PQB_ADJACENT>(a, chunk, grid, shm, s); break;
      case PQB_BF16 * 2 + PQB_HALF_SPLIT: launch_rmax_tma<PQB_BF16, PQB_HALF_SPLIT>(a, chunk, grid, shm, s); break;
      case PQB_F16 * 2 + PQB_ADJACENT: launch_rmax_tma<PQB_F16, PQB_ADJACENT>(a, chunk, grid, shm, s); break;
      default: launch_rmax_tma<PQB_F16, PQB_HALF_SPLIT>(a, chunk, grid, shm, s); break;
    }
  } else if (a.vector_ok) {
    switch (a.key_dtype * 2 + a.layout) {
      case PQB_F32 * 2 + PQB_ADJACENT: launch_rmax_v8<PQB_F32, PQB_ADJACENT>(a, chunk, grid, s); break;
      case PQB_F32 * 2 + PQB_HALF_SPLIT: launch_rmax_v8<PQB_F32, PQB_HALF_SPLIT>(a, chunk, grid, s); break;
      case PQB_BF16 * 2 + PQB_ADJACENT: launch_rmax_v8<PQB_BF16, PQB_ADJACENT>(a, chunk, grid, s); break;
      case PQB_BF16 * 2 + PQB_HALF_SPLIT: launch_rmax_v8<PQB_BF16, PQB_HALF_SPLIT>(a, chunk, grid, s); break;
      case PQB_F16 * 2 + PQB_ADJACENT: launch_rmax_v8<PQB_F16, PQB_ADJACENT>(a, chunk, grid, s); break;
      default: launch_rmax_v8<PQB_F16, PQB_HALF_SPLIT>(a, chunk, grid, s); break;
    }
  } else {
    const size_t shm = sizeof(unsigned long long) * half;
    switch (a.key_dtype) {
      case PQB_F32:
        radius_max_generic_kernel<PQB_F32><<<grid, 256, shm, s>>>(a.keys, a.tokens, half, a.layout, a.unit_stride,
                                                                   a.tok_stride, chunk, a.maxsq_ws, a.flags);
        break;
      case PQB_BF16:
        radius_max_generic_kernel<PQB_BF16><<<grid, 256, shm, s>>>(a.keys, a.tokens, half, a.layout, a.unit_stride,
                                                                    a.tok_stride, chunk, a.maxsq_ws, a.flags);
        break;
      default:
        radius_max_generic_kernel<PQB_F16><<<grid, 256, shm, s>>>(a.keys, a.tokens, half, a.layout, a.unit_stride,
                                                                   a.tok_stride, chunk, a.maxsq_ws, a.flags);
        break;
    }
  }
  const int64_t count = a.n_units * half;
  scales_finalize_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(a.maxsq_ws, count, a.radius_bits,
                                                                                   a.scales_out, a.flags);
  return 0;
}

template <int DT, int LAYOUT, int M>
static void launch_enc_v8(const EncodeArgs& a, int64_t chunk, dim3 grid, cudaStream_t s) {
  encode_v8_kernel<DT, LAYOUT, M><<<grid, 256, 0, s>>>(a.keys, a.tokens, a.d / 2, a.unit_stride, a.tok_stride,
                                                       chunk, a.radius_bits, a.scales, *a.store, a.tok_offset,
                                                       a.tok_offset_const, a.clamp_counts, a.flags);
}

template <int DT, int LAYOUT>
static void dispatch_m(const EncodeArgs& a, int64_t chunk, dim3 grid, cudaStream_t s) {
  switch (a.angle_bits) {
    case 1: launch_enc_v8<DT, LAYOUT, 1>(a, chunk, grid, s); break;
    case 2: launch_enc_v8<DT, LAYOUT, 2>(a, chunk, grid, s); break;
    case 3: launch_enc_v8<DT, LAYOUT, 3>(a, chunk, grid, s); break;
    case 4: launch_enc_v8<DT, LAYOUT, 4>(a, chunk, grid, s); break;
    case 5: launch_enc_v8<DT, LAYOUT, 5>(a, chunk, grid, s); break;
    case 6: launch_enc_v8<DT, LAYOUT, 6>(a, chunk, grid, s); break;
    case 7: launch_enc_v8<DT, LAYOUT, 7>(a, chunk, grid, s); break;
    default: launch_enc_v8<DT, LAYOUT, 8>(a, chunk, grid, s); break;
  }
}

int launch_encode(const EncodeArgs& a, cudaStream_t s) {
  const int half = a.d / 2;
  if (a.tokens == 0) return 0;
  // PQB_ENCODE_KERNEL=v8 forces the per-call-grid kernel below (A/B and parity tests)
  const char* kern = std::getenv("PQB_ENCODE_KERNEL");
  if (!(kern && std::strcmp(kern, "v8") == 0) && launch_encode_fast(a, s)) return 0;
  if (a.vector_ok) {
    const int64_t chunk = 2048;
    dim3 grid(static_cast<unsigned>((a.tokens + chunk - 1) / chunk), static_cast<unsigned>(a.n_units));
    switch (a.key_dtype * 2 + a.layout) {
      case PQB_F32 * 2 + PQB_ADJACENT: dispatch_m<PQB_F32, PQB_ADJACENT>(a, chunk, grid, s); break;
      case PQB_F32 * 2 + PQB_HALF_SPLIT: dispatch_m<PQB_F32, PQB_HALF_SPLIT>(a, chunk, grid, s); break;
      case PQB_BF16 * 2 + PQB_ADJACENT: dispatch_m<PQB_BF16, PQB_ADJACENT>(a, chunk, grid, s); break;
      case PQB_BF16 * 2 + PQB_HALF_SPLIT: dispatch_m<PQB_BF16, PQB_HALF_SPLIT>(a, chunk, grid, s); break;
      case PQB_F16 * 2 + PQB_ADJACENT: dispatch_m<PQB_F16, PQB_ADJACENT>(a, chunk, grid, s); break;
      default: dispatch_m<PQB_F16, PQB_HALF_SPLIT>(a, chunk, grid, s); break;
    }
  } else {
    GenericSrc src{a.keys, a.key_dtype, a.unit_stride, a.tok_stride};
    // groups spanned by one unit's call (upper bound, offsets are per unit)
    const int64_t groups = (a.tokens * half) / 32 + 2;
    const int64_t gpb = 64;
    dim3 grid(static_cast<unsigned>((groups + gpb - 1) / gpb), static_cast<unsigned>(a.n_units));
    const size_t shm = sizeof(float) * half;
    switch (a.key_dtype) {
      case PQB_F32:
        encode_generic_kernel<PQB_F32><<<grid, 256, shm, s>>>(src, a.tokens, half, a.layout, a.angle_bits,
                                                               a.radius_bits, a.scales, *a.store, a.tok_offset,
                                                               a.tok_offset_const, gpb, a.clamp_counts, a.flags);
        break;
      case PQB_BF16:
        encode_generic_kernel<PQB_BF16><<<grid, 256, shm, s>>>(src, a.tokens, half, a.layout, a.angle_bits,
                                                                a.radius_bits, a.scales, *a.store, a.tok_offset,
                                                                a.tok_offset_const, gpb, a.clamp_counts, a.flags);
        break;
      default:
        encode_generic_kernel<PQB_F16><<<grid, 256, shm, s>>>(src, a.tokens, half, a.layout, a.angle_bits,
                                                               a.radius_bits, a.scales, *a.store, a.tok_offset,
                                                               a.tok_offset_const, gpb, a.clamp_counts, a.flags);
        break;
    }
  }
  return 0;
}

int launch_store_values(const void* vals, int dtype, int64_t n_units, int64_t T, int d, int64_t us, int64_t ts,
                        const pqb_store& st, const int32_t* tok_offset, int64_t tok_offset_const, cudaStream_t s,
                        int32_t* flags) {
  if (T == 0) return 0;
  if (st.value_dtype == PQB_VQ4 || st.value_dtype == PQB_VQ2 || st.value_dtype == PQB_VQ8) {
    dim3 grid(static_cast<unsigned>((T + 31) / 32), static_cast<unsigned>(n_units));
    store_values_vq_kernel<<<grid, 256, 0, s>>>(vals, dtype, T, us, ts, st, tok_offset_const, flags);
    return 0;
  }
  const int eb = dtype == PQB_F32 ? 4 : 2;
  const bool vec = d == 128 && st.value_dtype == PQB_BF16 && tok_offset == nullptr && st.value_off % 16 == 0 &&
                   st.page_bytes % 16 == 0 && (vals == nullptr || (reinterpret_cast<uintptr_t>(vals) % 16 == 0 &&
                                                                   (us * eb) % 16 == 0 && (ts * eb) % 16 == 0));
  if (vec) {
    const int64_t n = T * 16;
    dim3 grid(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4096)), static_cast<unsigned>(n_units));
    if (dtype == PQB_F32) store_values_v8_kernel<PQB_F32><<<grid, 256, 0, s>>>(vals, T, us, ts, st, tok_offset_const);
    else if (dtype == PQB_F16) store_values_v8_kernel<PQB_F16><<<grid, 256, 0, s>>>(vals, T, us, ts, st, tok_offset_const);
    else store_values_v8_kernel<PQB_BF16><<<grid, 256, 0, s>>>(vals, T, us, ts, st, tok_offset_const);
    return 0;
  }
  const int64_t n = T * d;
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4096)), static_cast<unsigned>(n_units));
  store_values_kernel<<<grid, 256, 0, s>>>(vals, dtype, T, d, us, ts, st, tok_offset, tok_offset_const);
  return 0;
}

int launch_store_residual(const pqb_cache& c, const void* keys, int dtype, int64_t n_units, int64_t T, int64_t us,
                          int64_t ts, int64_t tok_offset_const, int32_t* flags, cudaStream_t s) {
  if (T == 0) return 0;
  const int64_t n = T * c.d;
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4096)), static_cast<unsigned>(n_units));
  store_residual_kernel<<<grid, 256, 0, s>>>(keys, dtype, T, c.d, us, ts, c.residual, c.res_cap, tok_offset_const,
                                              flags);
  return 0;
}

int launch_append(const pqb_cache& c, int64_t n_units, const void* keys, int key_dtype, const void* vals,
                  int val_dtype, unsigned long long* clamp_counts, int32_t* flags, cudaStream_t s) {
  const size_t shm = sizeof(float) * (c.d / 2 + 64);
  append_kernel<<<static_cast<unsigned>(n_units), 128, shm, s>>>(c, keys, key_dtype, vals, val_dtype, clamp_counts,
                                                                  flags);
  return 0;
}

}  // namespace pqb
