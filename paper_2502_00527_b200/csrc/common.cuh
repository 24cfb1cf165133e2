// Shared device helpers for the PolarQuant B200 kernels (sm_100a only).
//
// Nothing here is PolarQuant-specific: element loads for the three key dtypes,
// mbarrier / cp.async.bulk (TMA bulk-copy engine) wrappers, warp reductions.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <atomic>

#include "../../include/pqb200.h"

#define PQB_DEV __device__ __forceinline__

namespace pqb {

// ------------------------------------------------------- host: per device
// One-time setup per device ordinal (kernel attributes, SM counts), safe for
// concurrent callers and for one process driving several GPUs: a bit per
// device, set after the setup succeeded (a race at worst repeats an
// idempotent cudaFuncSetAttribute).
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

template <typename F>
inline int once_per_device(std::atomic<uint64_t>& done, F&& setup) {
  const uint64_t bit = 1ull << (current_device() & 63);
  if (done.load(std::memory_order_acquire) & bit) return PQB_OK;
  const int rc = setup();
  if (rc == PQB_OK) done.fetch_or(bit, std::memory_order_acq_rel);
  return rc;
}

// SM count of the current device (148 on B200), cached per device.
inline int device_sms() {
  static std::atomic<int> cache[64];
  const int dev = current_device();
  int n = cache[dev & 63].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

constexpr int kWarp = 32;

// ----------------------------------------------------------------- dtypes

template <int DT> struct DType;
template <> struct DType<PQB_F32>  { using T = float;          static constexpr int kBytes = 4; };
template <> struct DType<PQB_BF16> { using T = __nv_bfloat16;  static constexpr int kBytes = 2; };
template <> struct DType<PQB_F16>  { using T = __half;         static constexpr int kBytes = 2; };

PQB_DEV float to_f32(float v) { return v; }
PQB_DEV float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
PQB_DEV float to_f32(__half v) { return __half2float(v); }

// Load 8 consecutive elements (16-byte aligned for 2-byte types, 32-byte for f32)
// and widen to f32.  Widening is exact for every supported dtype.
template <int DT>
PQB_DEV void load8(const void* base, int64_t elem_off, float (&out)[8]) {
  if constexpr (DT == PQB_F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + elem_off);
    float4 a = __ldg(p), b = __ldg(p + 1);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(
        static_cast<const typename DType<DT>::T*>(base) + elem_off);
    uint4 w = __ldg(p);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (DT == PQB_BF16) {
        out[2 * i] = __uint_as_float(ws[i] << 16);
        out[2 * i + 1] = __uint_as_float(ws[i] & 0xffff0000u);
      } else {
        __half2 h = *reinterpret_cast<const __half2*>(&ws[i]);
        float2 f = __half22float2(h);
        out[2 * i] = f.x;
        out[2 * i + 1] = f.y;
      }
    }
  }
}

// 8 consecutive elements from shared memory (16-byte aligned), widened to f32.
template <int DT>
PQB_DEV void load8s(const void* base, int elem_off, float (&out)[8]) {
  if constexpr (DT == PQB_F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + elem_off);
    const float4 a = p[0], b = p[1];
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  } else {
    const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const typename DType<DT>::T*>(base) + elem_off);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (DT == PQB_BF16) {
        out[2 * i] = __uint_as_float(ws[i] << 16);
        out[2 * i + 1] = __uint_as_float(ws[i] & 0xffff0000u);
      } else {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ws[i]));
        out[2 * i] = f.x;
        out[2 * i + 1] = f.y;
      }
    }
  }
}

template <int DT>
PQB_DEV float load1(const void* base, int64_t elem_off) {
  return to_f32(static_cast<const typename DType<DT>::T*>(base)[elem_off]);
}

PQB_DEV float half_bits_to_f32(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// Byte offset of value element (token t of a page, dim e) inside the page's
// value region.  bf16 rows of d = 128 are stored in 2 KB groups of 8 tokens:
// [dims 0-63 of the 8 tokens][dims 64-127], 128 B per token and half, the
// 16-byte chunks XOR-swizzled by (t & 7).  A linear bulk copy of a tile then
// lands in shared memory in the conflict-free layout ldmatrix.trans needs (8
// rows of the same logical chunk hit 8 different bank groups), and each 1 KB
// half-group is exactly the canonical 128-byte-swizzled MN-major atom a
// tcgen05 shared-memory descriptor reads (dims contiguous, 8 tokens).  Other
// shapes are linear.
PQB_DEV int64_t value_offset_bf16_128(int64_t t, int e) {
  return ((t >> 3) << 11) + ((e >> 6) << 10) + ((t & 7) << 7) + ((((e >> 3) & 7) ^ static_cast<int>(t & 7)) << 4) +
         ((e & 7) << 1);
}
PQB_DEV int64_t value_offset(int64_t t, int e, int d, int value_dtype) {
  if (value_dtype == PQB_F32) return (t * d + e) * 4;
  if (d == 128) return value_offset_bf16_128(t, e);
  return (t * d + e) * 2;
}

// Per-token uniform value codes of b in {2, 4, 8} bits (PQB_VQ2 / PQB_VQ4 /
// PQB_VQ8; quantize_uniform PER_TOKEN, baseline_quant.py:58-110), d = 128.
// A 32-token tile's 4096 codes (512 b bytes) are stored in m16n8k16
// A-fragment order of V^T (rows = dims, cols = tokens), so the decode kernel
// turns code words straight into MMA registers.  Lane = 4 g + t of dim block
// mt and token block ks owns 8 codes: register a_k (k = 0..3) low half
// (token 2t + 8 (k >> 1), dim g + 8 (k & 1)), high half (token + 1, same dim).
//   b = 4: word (mt * 2 + ks) * 32 + lane; a_k low at bits 4k, high at 16 + 4k.
//   b = 8: word pair 2 ((mt * 2 + ks) * 32 + lane) + {0, 1}: the low nibbles,
//          then the high nibbles, each in the b = 4 arrangement.
//   b = 2: word ((mt * 2 + ks) >> 1) * 32 + lane, half h = (mt * 2 + ks) & 1:
//          a_k low at bits 16 h + 2k, high at 16 h + 8 + 2k.
// After the codes, fp32 (zp, scale) per token: [page_tokens][2].
__host__ __device__ __forceinline__ int vq_bits(int value_dtype) {
  return value_dtype == PQB_VQ4 ? 4 : value_dtype == PQB_VQ2 ? 2 : value_dtype == PQB_VQ8 ? 8 : 0;
}
__host__ __device__ __forceinline__ int vq_tile_bytes(int bits) { return 512 * bits; }

// Word index and bit shift of code (token t_in_tile, dim e); for b = 8 the
// low nibble's position (the high nibble sits in word + 1 at the same shift).
PQB_DEV void vq_pos(int bits, int t_in_tile, int e, int& word, int& shift) {
  const int ks = t_in_tile >> 4, tt = t_in_tile & 15, mt = e >> 4, ee = e & 15;
  const int k = (ee >> 3) + 2 * (tt >> 3);
  const int ln = (ee & 7) * 4 + ((tt & 7) >> 1), c = tt & 1, blk = mt * 2 + ks;
  if (bits == 2) {
    word = (blk >> 1) * 32 + ln;
    shift = 16 * (blk & 1) + 8 * c + 2 * k;
  } else if (bits == 8) {
    word = 2 * (blk * 32 + ln);
    shift = 4 * k + 16 * c;
  } else {
    word = blk * 32 + ln;
    shift = 4 * k + 16 * c;
  }
}
PQB_DEV void vq4_pos(int t_in_tile, int e, int& word, int& shift) { vq_pos(4, t_in_tile, e, word, shift); }

PQB_DEV int64_t vq_params_off(const pqb_store& st) {
  return st.value_off + static_cast<int64_t>(st.page_tokens) * 16 * vq_bits(st.value_dtype);
}
PQB_DEV int64_t vq4_params_off(const pqb_store& st) { return vq_params_off(st); }

// Code of (token t_in_tile, dim e) from a tile's words.
PQB_DEV uint32_t vq_code(int bits, const uint32_t* tile_words, int t_in_tile, int e) {
  int w, sh;
  vq_pos(bits, t_in_tile, e, w, sh);
  if (bits == 8) return ((tile_words[w] >> sh) & 15u) | (((tile_words[w + 1] >> sh) & 15u) << 4);
  return (tile_words[w] >> sh) & ((1u << bits) - 1u);
}

// Value (token t of the page, element e) of any value store, as fp32
// (quantized: dequantize_uniform's fl(fl(code * scale) + zp), baseline_quant.py:143-167).
PQB_DEV float load_value(const pqb_store& st, const uint8_t* page, int64_t t, int e, int d) {
  const int vb = vq_bits(st.value_dtype);
  if (vb) {
    const uint32_t* words = reinterpret_cast<const uint32_t*>(page + st.value_off + (t >> 5) * vq_tile_bytes(vb));
    const uint32_t code = vq_code(vb, words, static_cast<int>(t & 31), e);
    const float2 zs = reinterpret_cast<const float2*>(page + vq_params_off(st))[t];
    return __fadd_rn(__fmul_rn(static_cast<float>(code), zs.y), zs.x);
  }
  const uint8_t* vp = page + st.value_off + value_offset(t, e, d, st.value_dtype);
  return st.value_dtype == PQB_F32 ? *reinterpret_cast<const float*>(vp)
                                   : __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(vp));
}

// ---------------------------------------------------------------- warp ops

PQB_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
PQB_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
PQB_DEV unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------- mbarrier + bulk copy
// cp.async.bulk (SASS UBLKCP) moves a contiguous byte range global->shared on
// the TMA engine and signals an mbarrier with the byte count on completion.

PQB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

PQB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

PQB_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

PQB_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

PQB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

#ifndef PQB_MBAR_SLEEP_NS
#define PQB_MBAR_SLEEP_NS 20000
#endif

PQB_DEV bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

PQB_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}

// try_wait with a suspend-time hint: the thread sleeps in the barrier unit
// until the phase completes (or the hint, in ns, expires) instead of spinning
// through try_wait / branch / yield -- a spinning producer lane otherwise
// takes issue slots (and power) from the compute warps of its sub-partition.
PQB_DEV bool mbar_try_wait_sleep(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "r"(PQB_MBAR_SLEEP_NS)
      : "memory");
  return ok != 0;
}
PQB_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait_sleep(bar, phase)) {
  }
}

PQB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Named CTA barriers (id 0 is __syncthreads): nthreads, a multiple of 32, of
// the CTA take part; arrive does not wait.
PQB_DEV void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
PQB_DEV void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

PQB_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Streaming-data hint: bulk copy with an L2 evict-first policy.
PQB_DEV void bulk_g2s_evict_first(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                  uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

PQB_DEV uint64_t make_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

}  // namespace pqb
