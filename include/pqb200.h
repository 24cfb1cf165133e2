/*
 * pqb200.h — C ABI of libpqb200.so, the B200 (sm_100a) PolarQuant hot path.
 *
 * This is the drop-in boundary for the two hot paths of the PolarQuant reference
 * (pure Python/numpy, /root/reference/pkg/src/polarquant):
 *
 *   HP-1  key-cache encoder      polar_codec.py:236-251 (compute_radius_scales)
 *                                polar_codec.py:281-302 (quantize_subvectors)
 *                                polar_codec.py:98-110  (pack_stream)
 *                                polar_codec.py:319-344 (encode_keys)
 *                                kv_cache.py:152-209    (PackedKVCache.prefill/_encode_block/_store_values)
 *                                kv_cache.py:179-189    (PackedKVCache.append)
 *   HP-2  LUT decode attention   lut_decode.py:63-104   (build_angle_table / build_query_lut)
 *                                lut_decode.py:119-154  (qk_scores)
 *                                lut_decode.py:189-206  (attention_weights)   + softmax.V (not in reference)
 *
 * Conventions (every entry point):
 *   - returns PQB_OK (0) or a PQB_E* status; a thread-local message is available
 *     from pqb_last_error().  The Python host layer maps PQB_EINVAL/PQB_EUNSUPPORTED
 *     to ValueError and PQB_ESTATE/PQB_ECUDA to RuntimeError, as the reference raises.
 *   - all pointers except the pqb_store / pqb_cache descriptors themselves (which
 *     live in host memory) are DEVICE pointers owned by the caller;
 *   - work is enqueued on `stream`; no call synchronizes or allocates device memory;
 *   - inputs are never modified; device-side error flags (`flags`, int32) are
 *     OR-ed with PQB_FLAG_* bits so the host can check them lazily.
 *
 * Code-stream format (identical to the reference stream, polar_codec.py:98-110):
 *   code i of a unit (flat index i = token*(d/2) + channel) occupies stream bits
 *   [i*b, (i+1)*b); stream bit k lives in byte k/8 at bit position k%8 (LSB first).
 *   Angle and radius codes are two separate streams.  A paged store splits each
 *   stream into pages of `page_tokens` tokens: page p of a unit holds stream bytes
 *   [p*page_tokens*(d/2)*b/8, (p+1)*page_tokens*(d/2)*b/8).  Concatenating a unit's
 *   pages in page-table order therefore reproduces PolarCodes.angle_stream /
 *   radius_stream byte for byte (up to the final partial byte's zero padding).
 */
#ifndef PQB200_H_
#define PQB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQB_ABI_VERSION 1

/* status codes */
#define PQB_OK 0
#define PQB_EINVAL 1        /* bad argument (shape, bits, dtype, pointer)        -> ValueError   */
#define PQB_ESTATE 2        /* cache state misuse                                -> RuntimeError */
#define PQB_ECUDA 3         /* CUDA launch / runtime failure                     -> RuntimeError */
#define PQB_EUNSUPPORTED 4  /* valid in the reference, not supported on this path -> ValueError  */

/* device-side flag bits (int32 flags[0]) */
#define PQB_FLAG_NONFINITE 1      /* a key was NaN/Inf (polar_codec.py:340-341, kv_cache.py:168-169) */
#define PQB_FLAG_SCALE_OVERFLOW 2 /* a radius scale overflowed fp16 (polar_codec.py:80-81)          */

/* element dtypes */
#define PQB_F32 0
#define PQB_BF16 1
#define PQB_F16 2
#define PQB_F64 3 /* element-wise reference API only (to_polar / quantize_angle / quantize_radius) */
/* pqb_store.value_dtype only: 4-bit per-token uniform value codes
 * (quantize_uniform PER_TOKEN, baseline_quant.py:58-110; the reference's
 * PackedKVCache(quantize_values=True, value_bits=4), kv_cache.py:199-209).
 * Value region of a page (d = 128): [page_tokens/32 tiles][2048 B codes in
 * MMA-fragment order, see INTEGRATION.md] then [page_tokens][zp, scale] fp32.
 * Read back: fl(fl(code * scale) + zp) (dequantize_uniform, :143-167). */
#define PQB_VQ4 16
/* The same with 2-bit and 8-bit codes (value_bits 2 / 8): a tile's codes take
 * 512 * bits bytes, then [page_tokens][zp, scale]. */
#define PQB_VQ2 17
#define PQB_VQ8 18

/* pairing layouts: same numeric values as PairingLayout (tensor_core.py:41-50) */
#define PQB_ADJACENT 0
#define PQB_HALF_SPLIT 1

typedef struct CUstream_st* pqb_stream_t; /* == cudaStream_t */

/*
 * A paged code/value store.  Page `p` of unit `u` lives at
 *   pool + page_bytes * (page_table ? page_table[u*max_pages + p] : u*max_pages + p)
 * and holds, at the given byte offsets, `page_tokens` tokens of angle codes,
 * radius codes and (optionally) values [page_tokens][d] of `value_dtype`.
 * page_tokens must be a multiple of 32; offsets and page_bytes multiples of 16.
 */
typedef struct pqb_store {
  uint8_t* pool;
  int64_t page_bytes;
  int64_t angle_off;
  int64_t radius_off;
  int64_t value_off; /* -1: the store holds no values */
  const int32_t* page_table;
  int32_t max_pages;
  int32_t page_tokens;
  int32_t value_dtype; /* PQB_F32, PQB_BF16, PQB_VQ2, PQB_VQ4 or PQB_VQ8 */
  int32_t reserved;
} pqb_store;

/*
 * Batched PackedKVCache state (kv_cache.py:85-289) for n_units independent
 * (layer, sequence, kv-head) units.  Tokens [0, quant_lens[u]) are polar codes in
 * the store; tokens [quant_lens[u], seq_lens[u]) are full-precision keys in the
 * residual ring (slot = token % res_cap), exactly the reference's residual FIFO.
 */
typedef struct pqb_cache {
  pqb_store store;
  int32_t d;
  int32_t angle_bits;
  int32_t radius_bits;
  int32_t layout;
  uint16_t* scales;  /* [n_units][d/2] fp16 bit patterns (ChannelScales, polar_codec.py:66-90) */
  int32_t* seq_lens; /* [n_units] */
  int32_t* quant_lens;
  float* residual;   /* [n_units][res_cap][d] or NULL when res_cap == 0 */
  int32_t res_cap;
  int32_t reserved;
} pqb_cache;

int pqb_abi_version(void);
const char* pqb_last_error(void);
/* Number of visible CUDA devices (0 on a host without a GPU); never fails. */
int pqb_device_count(void);

/* ---------------------------------------------------------------- HP-1 ----
 * K1: per-(unit, sub-channel) radius scales.  Replaces compute_radius_scales
 * (polar_codec.py:236-251): s_j = fp16( fp32(max_t hypot(x_tj, y_tj)) / (2^n - 1) ).
 * keys[u][t][e] is at keys + u*unit_stride + t*tok_stride + e (elements).
 * maxsq_ws: n_units*d/2 uint64 scratch (this call zeroes it).
 * scales_out: [n_units][d/2] fp16 bits.  flags: device int32[1].
 */
int pqb_radius_scales(const void* keys, int key_dtype, int64_t n_units, int64_t tokens, int d,
                      int64_t unit_stride, int64_t tok_stride, int layout, int radius_bits,
                      unsigned long long* maxsq_ws, uint16_t* scales_out, int32_t* flags,
                      pqb_stream_t stream);

/*
 * K2: quantize + bit-pack `tokens` tokens per unit into the store, starting at
 * token index tok_offset[u] (device array, may be NULL) + tok_offset_const.
 * Replaces quantize_subvectors + pack_stream (polar_codec.py:281-302, 98-110) and
 * PackedKVCache._encode_block (kv_cache.py:191-197).  Target code bits must be
 * zero (fresh pages): partial words are merged with atomicOr.
 * clamp_counts: [n_units] uint64 (may be NULL) += radii clamped from above
 * (polar_codec.py:276).  scales: [n_units][d/2] fp16 bits.
 */
int pqb_encode(const void* keys, int key_dtype, int64_t n_units, int64_t tokens, int d,
               int64_t unit_stride, int64_t tok_stride, int layout, int angle_bits,
               int radius_bits, const uint16_t* scales, const pqb_store* store,
               const int32_t* tok_offset, int64_t tok_offset_const,
               unsigned long long* clamp_counts, int32_t* flags, pqb_stream_t stream);

/* Store values [n_units][tokens][d] (NULL => zeros, kv_cache.py:200-201) into the
 * store's value region, converting to store->value_dtype. */
int pqb_store_values(const void* values, int value_dtype, int64_t n_units, int64_t tokens, int d,
                     int64_t unit_stride, int64_t tok_stride, const pqb_store* store,
                     const int32_t* tok_offset, int64_t tok_offset_const, pqb_stream_t stream);
/* Same, with a device flag word: non-finite values are OR-ed in as
 * PQB_FLAG_NONFINITE (quantize_uniform raises on them, baseline_quant.py:88-89;
 * checked for PQB_VQ4 stores). */
int pqb_store_values_ex(const void* values, int value_dtype, int64_t n_units, int64_t tokens, int d,
                        int64_t unit_stride, int64_t tok_stride, const pqb_store* store, const int32_t* tok_offset,
                        int64_t tok_offset_const, int32_t* flags, pqb_stream_t stream);

/* Write full-precision keys [n_units][tokens][d] into the residual ring at
 * token indices tok_offset_const + t (prefill's residual tail, kv_cache.py:175-176). */
int pqb_store_residual(const pqb_cache* cache, const void* keys, int key_dtype, int64_t n_units,
                       int64_t tokens, int64_t unit_stride, int64_t tok_stride,
                       int64_t tok_offset_const, int32_t* flags, pqb_stream_t stream);

/*
 * K5: one streaming append per unit (kv_cache.py:179-189): the new key enters the
 * residual ring; if the ring overflows, its oldest key is encoded with the frozen
 * scales at token index quant_lens[u]; the value is stored at token seq_lens[u];
 * seq_lens / quant_lens advance on device.  keys/values: [n_units][d].
 */
int pqb_append(const pqb_cache* cache, int64_t n_units, const void* keys, int key_dtype,
               const void* values, int value_dtype, unsigned long long* clamp_counts,
               int32_t* flags, pqb_stream_t stream);

/* ---------------------------------------------------------------- HP-2 ----
 * Fused LUT decode attention over a batched cache.  Query rows q[u][g][d]
 * (group = G query heads sharing KV unit u, GQA hq = h*G + g).
 *   scores = LUT scores exactly as qk_scores (lut_decode.py:119-154): for quantized
 *            tokens sum_j fl(P[g][j][A_tj] * rhat_j[R_tj]) accumulated in channel
 *            order in fp32 (bit-identical to the reference), then fp32 dots
 *            against the residual keys (lut_decode.py:107-116).
 *   out    = softmax(scores * sm_scale) . V   (online softmax, fp32 state).
 * out [n_units][G][d] (out_dtype PQB_F32/PQB_BF16) may be NULL (scores-only mode);
 * scores [n_units][G][scores_ld] fp32 may be NULL.  max_tokens >= max_u seq_lens[u]
 * (host bound used to size the split over tokens).
 */
size_t pqb_decode_workspace_bytes(int64_t n_units, int group, int max_tokens, int d);
int pqb_decode_attn(const pqb_cache* cache, int64_t n_units, int group, const void* q,
                    int q_dtype, float sm_scale, int max_tokens, void* out, int out_dtype,
                    float* scores, int64_t scores_ld, void* workspace, size_t workspace_bytes,
                    pqb_stream_t stream);

/* Extended form: flags = PQB_DECODE_* bits; splits > 0 overrides the automatic
 * split over tokens (clamped to what the workspace sizing allows). */
#define PQB_DECODE_FORCE_GENERIC 1 /* use the runtime-shape kernel (testing)          */
#define PQB_DECODE_NO_COMBINE 2    /* leave split partials in the workspace (timing) */
#define PQB_DECODE_DQ 4            /* fused call: product-table + tensor-core scoring (default, G 4/8);
                                      scores-only call (out NULL), G 4/8: the same contraction writes
                                      the score rows, within 1e-4 max(1, peak) of qk_scores instead of
                                      bit-identical (no softmax, no value bytes)                       */
#define PQB_DECODE_LUT 8           /* fused call: LUT-gather scoring (default for scores / G = 1)     */
#define PQB_DECODE_MERGE_KERNEL 256 /* DQ fused call: split merge in a separate PDL launch instead of
                                       the last CTA of each unit (default for G = 8 from 16K tokens and
                                       when units are cut into more than 8 segments)                 */
#define PQB_DECODE_NO_CLUSTER 2048 /* DQ fused call: no thread-block-cluster (DSMEM merge) path (A/B) */
#define PQB_DECODE_MERGE_INKERNEL 1024 /* DQ fused call: last-CTA split merge inside the decode launch (A/B) */
#define PQB_DECODE_DQ_LINEAR 512   /* DQ kernel: the linear shared-memory layout build (the automatic
                                       fallback when the default table placement does not fit)        */
#define PQB_DECODE_PROBE_MEM 64    /* diagnostics, m4n4 DQ only: stream tiles, skip all compute      */
#define PQB_DECODE_PROBE_COMPUTE 128 /* diagnostics, m4n4 DQ only: compute on L2-resident tiles      */
int pqb_decode_attn_ex(const pqb_cache* cache, int64_t n_units, int group, const void* q,
                       int q_dtype, float sm_scale, int max_tokens, void* out, int out_dtype,
                       float* scores, int64_t scores_ld, void* workspace, size_t workspace_bytes,
                       int flags, int splits, pqb_stream_t stream);
/* Split count the automatic policy picks (for workspace sizing / reporting). */
/*
 * Head-output gather fused into the decode epilogue (KV-head-sharded layers,
 * SURVEY 8(e); replaces the per-layer NCCL all-gather of [B, Hq, d]): every
 * output row is stored straight into each peer's gathered buffer
 * [batch][q_heads][128] through peer pointers (NVLink P2P / CUDA IPC), and the
 * grid's last CTA then increments flags[rank] in every peer's flag array
 * (fence + release add, system scope; counting, so CUDA-graph replays work).  Unit u of the call is
 * (sequence batch0 + u / kv_local, kv head head0 + u % kv_local); query g of it
 * is head (head0 + u % kv_local) * group + g.  DQ kernel only (group 4 or 8,
 * d = 128); the workspace is the same as pqb_decode_attn's.
 */
#define PQB_MAX_PEERS 8
typedef struct pqb_peer_out {
  void* out[PQB_MAX_PEERS];       /* peer k's gathered buffer of this layer (out[rank]: local) */
  uint32_t* flags[PQB_MAX_PEERS]; /* peer k's flag array [n_peers] of this layer */
  int32_t n_peers, rank;
  int32_t batch0, head0, kv_local, q_heads;
  int32_t out_dtype;              /* PQB_F32 or PQB_BF16 */
  int32_t reserved;
} pqb_peer_out;
int pqb_decode_attn_peer(const pqb_cache* cache, int64_t n_units, int group, const void* q, int q_dtype,
                         float sm_scale, int max_tokens, const pqb_peer_out* peer, void* workspace,
                         size_t workspace_bytes, pqb_stream_t stream);
/* Enqueue on `stream`: ++*expect (device counter of this layer), then wait until
 * flags[k] >= *expect for every k != rank (acquire loads, system scope).  After
 * it the layer's gathered buffer is complete. */
int pqb_peer_wait(const uint32_t* flags, int n_peers, int rank, uint32_t* expect, pqb_stream_t stream);
/* Peer-visible buffers for pqb_peer_out (one process per GPU).  The owner
 * allocates with pqb_ipc_alloc on `device` (cudaMalloc, zero-filled, so the
 * handle names the allocation's base) and sends the PQB_IPC_HANDLE_BYTES
 * handle to the other ranks; each of them maps it with pqb_ipc_open into ITS
 * OWN device's address space (peer access enabled on first use), so the
 * decode kernel running on that device can store into it over NVLink.
 * pqb_ipc_close unmaps an opened buffer; pqb_ipc_free releases an owned one
 * (after every importer has closed it).  pqb_peer_access reports whether
 * `device` can reach `peer_device` (1) or not (0). */
#define PQB_IPC_HANDLE_BYTES 64
int pqb_ipc_alloc(int device, size_t bytes, void** ptr, void* handle);
int pqb_ipc_open(int device, const void* handle, void** ptr);
int pqb_ipc_close(int device, void* ptr);
int pqb_ipc_free(int device, void* ptr);
int pqb_peer_access(int device, int peer_device, int* can_access);

int pqb_decode_splits(int64_t n_units, int max_tokens);
/* Kernels one fused DQ decode call (group 4 or 8, out != NULL, no peers) enqueues
 * for this shape and flags: 1, or 2 when the split merge runs as its own launch. */
int pqb_decode_launches(int64_t n_units, int group, int max_tokens, int flags);
/* The same for a store of angle_bits / radius_bits codes and value_dtype
 * values (pqb_store.value_dtype): the thread-block-cluster path (one launch)
 * needs m = n = 4 with bf16 values; pqb_decode_launches assumes that store. */
int pqb_decode_launches_ex(int64_t n_units, int group, int max_tokens, int flags, int angle_bits, int radius_bits,
                           int value_dtype);
/* Shared-memory layout the last fused DQ launch in this process used: 0 none
 * yet, 1 the product table at its fixed shared-window address (the fast
 * build), 2 the linear-layout fallback (a device whose shared window is laid
 * out other than measured).  Diagnostics: tests and the bench assert 1. */
int pqb_decode_dq_layout(void);
/* Host-side view of the DQ kernel's cost-balanced persistent split for
 * n_units units of max_tokens tokens on at most `ctas` CTAs: writes the CTA
 * range starts (in 32-token tiles of the unit-major item space, n + 1 values
 * with starts[n] = n_units * tiles) to starts (capacity >= ctas + 1) and
 * returns n, the CTA count; 0 when the split is uniform (per_cta = ceil(items /
 * ctas)).  No device needed (tests of the host logic). */
int pqb_decode_split_starts(int64_t n_units, int max_tokens, int ctas, int32_t* starts);

/* ------------------------------------------------------------ accessors ----
 * Tables and views the reference API exposes (all computed on the device). */
/* build_angle_table (lut_decode.py:63-74): cos/sin of angle_grid (polar_codec.py:224-233), fp32 */
int pqb_angle_table(int angle_bits, float* cos_out, float* sin_out, pqb_stream_t stream);
/* build_query_lut (lut_decode.py:86-104): out[n][d/2][2^m] = qx*cos + qy*sin, fp32 */
int pqb_query_lut(const void* q, int q_dtype, int64_t n, int d, int layout, int angle_bits,
                  float* out, pqb_stream_t stream);
/* PackedKVCache.radius_table (kv_cache.py:228-237): out[u][d/2][2^n] = s32_j * code */
int pqb_radius_table(const uint16_t* scales, int64_t n_units, int d, int radius_bits, float* out,
                     pqb_stream_t stream);
/* Unpack codes tokens [0, tokens) of one unit to uint8 (T, d/2) arrays
 * (PackedKVCache.code_arrays, kv_cache.py:213-221; PolarCodes.angle_codes, polar_codec.py:182-194). */
int pqb_unpack_codes(const pqb_store* store, int64_t unit, int d, int angle_bits, int radius_bits,
                     int64_t tokens, uint8_t* angle_out, uint8_t* radius_out, pqb_stream_t stream);
/* pack_stream (polar_codec.py:98-110) of unpacked uint8 code arrays [tokens][d/2]
 * (low b bits of each entry) into unit `unit` of a fresh store (PolarCodes.from_arrays). */
int pqb_pack_codes(const uint8_t* angle_codes, const uint8_t* radius_codes, int64_t tokens, int d,
                   int angle_bits, int radius_bits, const pqb_store* store, int64_t unit,
                   pqb_stream_t stream);
/* Gather a unit's pages into the two contiguous reference streams (PolarCodes, PQC1 payload). */
int pqb_export_streams(const pqb_store* store, int64_t unit, int d, int angle_bits,
                       int radius_bits, int64_t tokens, uint8_t* angle_stream,
                       uint8_t* radius_stream, pqb_stream_t stream);
/* Read values of one unit back as fp32 [tokens][d] (PackedKVCache.values, kv_cache.py:247-259). */
int pqb_read_values(const pqb_store* store, int64_t unit, int d, int64_t tokens, float* out,
                    pqb_stream_t stream);
/* Dequantize the quantized tokens [0, tokens) of one unit to fp32 keys [tokens][d]
 * (PackedKVCache.decode_quantized kv_cache.py:239-245 via dequantize_subvectors
 * polar_codec.py:305-316 + merge_pairs tensor_core.py:72-84), bit-identical. */
int pqb_dequantize(const pqb_cache* cache, int64_t unit, int64_t tokens, float* out, pqb_stream_t stream);
/* Per-token uniform b-bit quantize -> dequantize of value rows [n][d]
 * (quantize_uniform PER_TOKEN baseline_quant.py:58-110 then dequantize_uniform
 * :143-167, the PackedKVCache(quantize_values=True) path kv_cache.py:206-207,256). */
int pqb_quantize_values(const void* values, int dtype, int64_t n, int d, int bits, float* out,
                        pqb_stream_t stream);
/* attention_weights (lut_decode.py:189-206): float64 softmax of scores*temperature. */
int pqb_softmax_f64(const float* scores, int64_t n, double temperature, double* out,
                    pqb_stream_t stream);

/* ------------------------------------------------- element-wise API ----
 * The reference's array-level functions (polarquant.__init__:38-51), evaluated
 * in the input's precision like numpy: dtype PQB_F32 (float32 arithmetic, the
 * Python-float constants rounded to float32 first) or PQB_F64.  Operands are
 * contiguous device arrays of n elements (the host broadcasts). */
/* to_polar (polar_codec.py:200-209): r = hypot(x, y) (float32: glibc hypotf's
 * fl32(sqrt(fl64(x^2 + y^2)))), t = mod(atan2(y, x) + pi, 2 pi) with a correctly
 * rounded float32 atan2 (numpy's SIMD arctan2 may differ by a few ulp). */
int pqb_to_polar(const void* x, const void* y, int dtype, int64_t n, void* radius_out, void* theta_out,
                 pqb_stream_t stream);
/* quantize_angle (polar_codec.py:212-221): uint8(int64(rint(t * 2^(m-1)/pi)) mod 2^m). */
int pqb_quantize_angle(const void* theta, int dtype, int64_t n, int angle_bits, uint8_t* out, pqb_stream_t stream);
/* angle_grid (polar_codec.py:224-233): pi * a / 2^(m-1) - pi, float64 [2^m]. */
int pqb_angle_grid(int angle_bits, double* out, pqb_stream_t stream);
/* quantize_radius / _quantize_radius_counted (polar_codec.py:254-278): rint(r / s)
 * in r's precision (s already float32), 0 where s == 0, clipped to [0, 2^n - 1];
 * clamped (nullable) += entries clamped from above. */
int pqb_quantize_radius(const void* radius, int dtype, const float* scale, int64_t n, int radius_bits, uint8_t* out,
                        unsigned long long* clamped, pqb_stream_t stream);
/* qk_scores_direct (lut_decode.py:157-186): the dequantized keys of unit `unit`
 * (bit-identical to pqb_dequantize) dotted with q [d] in fp32, then the residual
 * keys; out[t] for t < min(tokens, seq_lens[unit]). */
int pqb_scores_direct(const pqb_cache* cache, int64_t unit, const void* q, int q_dtype, int64_t tokens, float* out,
                      pqb_stream_t stream);
/* Scatter two contiguous reference streams of `tokens` tokens (PolarCodes /
 * PQC1 payload, load_codes polar_codec.py:415-446, load_snapshot kv_cache.py:369-397)
 * into unit `unit`'s pages: the inverse of pqb_export_streams.  Target pages
 * must be zero past the imported bits (fresh), so later appends can OR codes in. */
int pqb_import_streams(const pqb_store* store, int64_t unit, int d, int angle_bits, int radius_bits, int64_t tokens,
                       const uint8_t* angle_stream, const uint8_t* radius_stream, pqb_stream_t stream);

/* ------------------------------------------------------------ synthetic ----
 * Seeded on-device generator with gen_synthetic_keys' distribution
 * (tensor_core.py:226-241): per sub-channel radius ~ lognormal(mean_j, std),
 * angle ~ U[0, 2pi), mean_j += outlier_boost for channels with bit j set in
 * outlier_mask (j < 64).  Writes [n_units][tokens][d] of out_dtype; unit u uses
 * Philox stream (seed, u).  Not bit-identical to numpy's PCG64 stream. */
int pqb_synthetic_keys(uint64_t seed, int64_t n_units, int64_t tokens, int d, int layout,
                       float radius_log_mean, float radius_log_std, uint64_t outlier_mask,
                       float outlier_boost, void* out, int out_dtype, pqb_stream_t stream);
/* Standard-normal fill (values / queries), Philox stream (seed, i/4). */
int pqb_synthetic_normal(uint64_t seed, int64_t count, void* out, int out_dtype,
                         pqb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* PQB200_H_ */
