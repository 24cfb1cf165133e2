// extern "C" entry points of libpqb200.so: argument validation, dispatch to the
// kernel launchers, and status / thread-local error reporting (include/pqb200.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace pqb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int cuda_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return PQB_ECUDA;
  }
  return PQB_OK;
}

#define PQB_CHECK(cond, code, ...)       \
  do {                                   \
    if (!(cond)) {                       \
      ::pqb::set_error(__VA_ARGS__);     \
      return (code);                     \
    }                                    \
  } while (0)

static bool is_vq(int dt) { return dt == PQB_VQ2 || dt == PQB_VQ4 || dt == PQB_VQ8; }
static int vq_bits_host(int dt) { return dt == PQB_VQ2 ? 2 : dt == PQB_VQ4 ? 4 : dt == PQB_VQ8 ? 8 : 0; }
static bool dtype_ok(int dt) { return dt == PQB_F32 || dt == PQB_BF16 || dt == PQB_F16; }
static bool layout_ok(int l) { return l == PQB_ADJACENT || l == PQB_HALF_SPLIT; }
static int elem_bytes(int dt) { return dt == PQB_F32 ? 4 : 2; }

// 8-channel vector loads: tpr = half/8 threads per row must divide 256, rows
// 16-byte aligned.
static bool vec_loads_ok(const void* keys, int dtype, int d, int64_t us, int64_t ts) {
  const int half = d / 2;
  if (half < 8 || half > 256 || (half & (half - 1))) return false;
  if (reinterpret_cast<uintptr_t>(keys) % 16) return false;
  const int eb = elem_bytes(dtype);
  return (us * eb) % 16 == 0 && (ts * eb) % 16 == 0;
}

static int check_store(const pqb_store* st, int d, int m, int n, bool need_values) {
  PQB_CHECK(st != nullptr && st->pool != nullptr, PQB_EINVAL, "store: null descriptor or pool");
  PQB_CHECK(st->page_tokens > 0 && st->page_tokens % 32 == 0, PQB_EINVAL,
            "store: page_tokens=%d must be a positive multiple of 32", st->page_tokens);
  PQB_CHECK(st->max_pages > 0, PQB_EINVAL, "store: max_pages must be > 0");
  PQB_CHECK(st->page_bytes % 16 == 0 && st->angle_off % 4 == 0 && st->radius_off % 4 == 0, PQB_EINVAL,
            "store: page_bytes / region offsets misaligned");
  const int64_t half = d / 2;
  const int64_t ab = st->page_tokens * half * m / 8, rb = st->page_tokens * half * n / 8;
  PQB_CHECK(st->angle_off >= 0 && st->angle_off + ab <= st->page_bytes, PQB_EINVAL,
            "store: angle region exceeds page");
  PQB_CHECK(st->radius_off >= 0 && st->radius_off + rb <= st->page_bytes, PQB_EINVAL,
            "store: radius region exceeds page");
  if (need_values) {
    PQB_CHECK(st->value_off >= 0, PQB_EINVAL, "store: no value region");
    PQB_CHECK(st->value_dtype == PQB_F32 || st->value_dtype == PQB_BF16 || is_vq(st->value_dtype), PQB_EINVAL,
              "store: bad value dtype");
    PQB_CHECK(!is_vq(st->value_dtype) || (d == 128 && st->value_off % 16 == 0), PQB_EUNSUPPORTED,
              "store: quantized values need d = 128 and a 16-byte aligned value region");
    const int64_t vb = static_cast<int64_t>(st->page_tokens) *
                       (is_vq(st->value_dtype) ? 16 * vq_bits_host(st->value_dtype) + 8
                                               : d * (st->value_dtype == PQB_F32 ? 4 : 2));
    PQB_CHECK(st->value_off + vb <= st->page_bytes, PQB_EINVAL, "store: value region exceeds page");
  }
  return PQB_OK;
}

}  // namespace pqb

using namespace pqb;

extern "C" {

int pqb_abi_version(void) { return PQB_ABI_VERSION; }

const char* pqb_last_error(void) { return g_err; }

int pqb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int pqb_radius_scales(const void* keys, int key_dtype, int64_t n_units, int64_t tokens, int d, int64_t unit_stride,
                      int64_t tok_stride, int layout, int radius_bits, unsigned long long* maxsq_ws,
                      uint16_t* scales_out, int32_t* flags, pqb_stream_t stream) {
  PQB_CHECK(d >= 2 && d % 2 == 0, PQB_EINVAL, "vector dimension must be even and >= 2, got %d", d);
  PQB_CHECK(radius_bits >= 1 && radius_bits <= 8, PQB_EINVAL, "radius_bits must be in [1, 8], got %d", radius_bits);
  PQB_CHECK(tokens > 0, PQB_EINVAL, "cannot compute scales from an empty tensor");
  PQB_CHECK(n_units >= 0 && n_units <= 65535, PQB_EINVAL, "n_units=%lld out of range", (long long)n_units);
  PQB_CHECK(dtype_ok(key_dtype) && layout_ok(layout), PQB_EINVAL, "bad dtype or layout");
  PQB_CHECK(keys && maxsq_ws && scales_out && flags, PQB_EINVAL, "null pointer argument");
  if (n_units == 0) return PQB_OK;
  RadiusScalesArgs a{keys, key_dtype, n_units, tokens, d, unit_stride, tok_stride, layout, radius_bits,
                     maxsq_ws, scales_out, flags, vec_loads_ok(keys, key_dtype, d, unit_stride, tok_stride)};
  launch_radius_scales(a, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_radius_scales");
}

int pqb_encode(const void* keys, int key_dtype, int64_t n_units, int64_t tokens, int d, int64_t unit_stride,
               int64_t tok_stride, int layout, int angle_bits, int radius_bits, const uint16_t* scales,
               const pqb_store* store, const int32_t* tok_offset, int64_t tok_offset_const,
               unsigned long long* clamp_counts, int32_t* flags, pqb_stream_t stream) {
  PQB_CHECK(d >= 2 && d % 2 == 0, PQB_EINVAL, "vector dimension must be even and >= 2, got %d", d);
  PQB_CHECK(angle_bits >= 1 && angle_bits <= 8, PQB_EINVAL, "angle_bits must be in [1, 8], got %d", angle_bits);
  PQB_CHECK(radius_bits >= 1 && radius_bits <= 8, PQB_EINVAL, "radius_bits must be in [1, 8], got %d", radius_bits);
  PQB_CHECK(tokens >= 0 && n_units >= 0 && n_units <= 65535, PQB_EINVAL, "bad token / unit count");
  PQB_CHECK(dtype_ok(key_dtype) && layout_ok(layout), PQB_EINVAL, "bad dtype or layout");
  PQB_CHECK(scales && flags && (keys || tokens == 0), PQB_EINVAL, "null pointer argument");
  const int rc = check_store(store, d, angle_bits, radius_bits, false);
  if (rc) return rc;
  if (n_units == 0 || tokens == 0) return PQB_OK;
  const int half = d / 2;
  // vector kernel: whole 32-bit words per token (half % 32 == 0) and one block
  // iteration (256 / (half/8) tokens) crossing at most one page boundary
  const bool vec = vec_loads_ok(keys, key_dtype, d, unit_stride, tok_stride) && half % 32 == 0 &&
                   2048 / half <= store->page_tokens && reinterpret_cast<uintptr_t>(scales) % 16 == 0;
  EncodeArgs a{keys, key_dtype, n_units, tokens, d, unit_stride, tok_stride, layout, angle_bits, radius_bits,
               scales, store, tok_offset, tok_offset_const, clamp_counts, flags, vec};
  launch_encode(a, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_encode");
}

int pqb_store_values(const void* values, int value_dtype, int64_t n_units, int64_t tokens, int d,
                     int64_t unit_stride, int64_t tok_stride, const pqb_store* store, const int32_t* tok_offset,
                     int64_t tok_offset_const, pqb_stream_t stream) {
  return pqb_store_values_ex(values, value_dtype, n_units, tokens, d, unit_stride, tok_stride, store, tok_offset,
                             tok_offset_const, nullptr, stream);
}

int pqb_store_values_ex(const void* values, int value_dtype, int64_t n_units, int64_t tokens, int d,
                        int64_t unit_stride, int64_t tok_stride, const pqb_store* store, const int32_t* tok_offset,
                        int64_t tok_offset_const, int32_t* flags, pqb_stream_t stream) {
  PQB_CHECK(d >= 2 && d % 2 == 0, PQB_EINVAL, "vector dimension must be even and >= 2, got %d", d);
  PQB_CHECK(values == nullptr || dtype_ok(value_dtype), PQB_EINVAL, "bad value dtype");
  PQB_CHECK(store && store->pool && store->value_off >= 0, PQB_EINVAL, "store has no value region");
  PQB_CHECK(store->value_dtype == PQB_F32 || store->value_dtype == PQB_BF16 || is_vq(store->value_dtype),
            PQB_EINVAL, "bad store value dtype");
  PQB_CHECK(!is_vq(store->value_dtype) || (d == 128 && tok_offset == nullptr && tok_offset_const % 32 == 0),
            PQB_EUNSUPPORTED, "quantized value stores take d = 128 and whole 32-token tiles");
  PQB_CHECK(n_units >= 0 && n_units <= 65535 && tokens >= 0, PQB_EINVAL, "bad token / unit count");
  if (n_units == 0 || tokens == 0) return PQB_OK;
  launch_store_values(values, value_dtype, n_units, tokens, d, unit_stride, tok_stride, *store, tok_offset,
                      tok_offset_const, reinterpret_cast<cudaStream_t>(stream), flags);
  return cuda_status("pqb_store_values");
}

int pqb_store_residual(const pqb_cache* cache, const void* keys, int key_dtype, int64_t n_units, int64_t tokens,
                       int64_t unit_stride, int64_t tok_stride, int64_t tok_offset_const, int32_t* flags,
                       pqb_stream_t stream) {
  PQB_CHECK(cache && cache->residual && cache->res_cap > 0, PQB_EINVAL, "cache has no residual ring");
  PQB_CHECK(dtype_ok(key_dtype) && keys && flags, PQB_EINVAL, "bad key arguments");
  PQB_CHECK(tokens >= 0 && tokens <= cache->res_cap, PQB_EINVAL, "residual tokens %lld exceed capacity %d",
            (long long)tokens, cache->res_cap);
  PQB_CHECK(n_units >= 0 && n_units <= 65535, PQB_EINVAL, "bad unit count");
  if (n_units == 0 || tokens == 0) return PQB_OK;
  launch_store_residual(*cache, keys, key_dtype, n_units, tokens, unit_stride, tok_stride, tok_offset_const, flags,
                        reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_store_residual");
}

int pqb_append(const pqb_cache* cache, int64_t n_units, const void* keys, int key_dtype, const void* values,
               int value_dtype, unsigned long long* clamp_counts, int32_t* flags, pqb_stream_t stream) {
  PQB_CHECK(cache != nullptr, PQB_EINVAL, "null cache");
  PQB_CHECK(cache->scales && cache->seq_lens && cache->quant_lens, PQB_ESTATE, "cache is empty; prefill first");
  PQB_CHECK(cache->res_cap == 0 || cache->residual, PQB_EINVAL, "residual ring missing");
  PQB_CHECK(dtype_ok(key_dtype) && keys && flags, PQB_EINVAL, "bad key arguments");
  PQB_CHECK(values == nullptr || dtype_ok(value_dtype), PQB_EINVAL, "bad value dtype");
  PQB_CHECK(n_units >= 0 && n_units <= 2147483647, PQB_EINVAL, "bad unit count");
  const int rc = check_store(&cache->store, cache->d, cache->angle_bits, cache->radius_bits, false);
  if (rc) return rc;
  if (n_units == 0) return PQB_OK;
  launch_append(*cache, n_units, keys, key_dtype, values, value_dtype, clamp_counts, flags,
                reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_append");
}

size_t pqb_decode_workspace_bytes(int64_t n_units, int group, int max_tokens, int d) {
  if (n_units <= 0 || group <= 0 || max_tokens <= 0 || d <= 0) return 0;
  return decode_workspace_bytes(n_units, group, max_tokens, d);
}

int pqb_decode_attn_ex(const pqb_cache* cache, int64_t n_units, int group, const void* q, int q_dtype,
                       float sm_scale, int max_tokens, void* out, int out_dtype, float* scores, int64_t scores_ld,
                       void* workspace, size_t workspace_bytes, int flags, int splits, pqb_stream_t stream) {
  PQB_CHECK(cache != nullptr, PQB_EINVAL, "null cache");
  PQB_CHECK(cache->scales && cache->seq_lens && cache->quant_lens, PQB_ESTATE, "cache is empty; prefill first");
  PQB_CHECK(cache->d >= 2 && cache->d % 2 == 0, PQB_EINVAL, "bad cache dim %d", cache->d);
  PQB_CHECK(group >= 1, PQB_EINVAL, "group must be >= 1");
  PQB_CHECK(q && dtype_ok(q_dtype), PQB_EINVAL, "bad query");
  PQB_CHECK(out || scores, PQB_EINVAL, "nothing to compute: out and scores are both NULL");
  PQB_CHECK(out == nullptr || out_dtype == PQB_F32 || out_dtype == PQB_BF16, PQB_EINVAL, "bad out dtype");
  PQB_CHECK(scores == nullptr || scores_ld >= max_tokens, PQB_EINVAL, "scores_ld < max_tokens");
  PQB_CHECK(max_tokens >= 1, PQB_EINVAL, "max_tokens must be >= 1");
  PQB_CHECK(n_units >= 0 && n_units <= 65535, PQB_EINVAL, "n_units out of range");
  PQB_CHECK(cache->res_cap == 0 || cache->residual, PQB_EINVAL, "residual ring missing");
  const int rc = check_store(&cache->store, cache->d, cache->angle_bits, cache->radius_bits, out != nullptr);
  if (rc) return rc;
  if (n_units == 0) return PQB_OK;
  DecodeArgs a{cache, n_units, group, q, q_dtype, sm_scale, max_tokens, out, out_dtype, scores, scores_ld,
               workspace, workspace_bytes, flags, splits};
  const int lrc = launch_decode(a, reinterpret_cast<cudaStream_t>(stream));
  if (lrc) return lrc;
  return cuda_status("pqb_decode_attn");
}

int pqb_decode_attn(const pqb_cache* cache, int64_t n_units, int group, const void* q, int q_dtype, float sm_scale,
                    int max_tokens, void* out, int out_dtype, float* scores, int64_t scores_ld, void* workspace,
                    size_t workspace_bytes, pqb_stream_t stream) {
  return pqb_decode_attn_ex(cache, n_units, group, q, q_dtype, sm_scale, max_tokens, out, out_dtype, scores,
                            scores_ld, workspace, workspace_bytes, 0, 0, stream);
}

int pqb_decode_attn_peer(const pqb_cache* cache, int64_t n_units, int group, const void* q, int q_dtype,
                         float sm_scale, int max_tokens, const pqb_peer_out* peer, void* workspace,
                         size_t workspace_bytes, pqb_stream_t stream) {
  PQB_CHECK(peer != nullptr, PQB_EINVAL, "null peer descriptor");
  PQB_CHECK(peer->n_peers >= 1 && peer->n_peers <= PQB_MAX_PEERS && peer->rank >= 0 && peer->rank < peer->n_peers,
            PQB_EINVAL, "bad peer count / rank");
  PQB_CHECK(peer->kv_local >= 1 && peer->q_heads >= group && peer->batch0 >= 0 && peer->head0 >= 0, PQB_EINVAL,
            "bad peer layout");
  PQB_CHECK(peer->out_dtype == PQB_F32 || peer->out_dtype == PQB_BF16, PQB_EINVAL, "bad peer out dtype");
  for (int k = 0; k < peer->n_peers; ++k)
    PQB_CHECK(peer->out[k] && peer->flags[k], PQB_EINVAL, "null peer buffer %d", k);
  PQB_CHECK(cache != nullptr, PQB_EINVAL, "null cache");
  PQB_CHECK(cache->scales && cache->seq_lens && cache->quant_lens, PQB_ESTATE, "cache is empty; prefill first");
  PQB_CHECK(q && dtype_ok(q_dtype), PQB_EINVAL, "bad query");
  PQB_CHECK(max_tokens >= 1 && n_units >= 0 && n_units <= 65535, PQB_EINVAL, "bad token / unit count");
  const int rc = check_store(&cache->store, cache->d, cache->angle_bits, cache->radius_bits, true);
  if (rc) return rc;
  if (n_units == 0) return PQB_OK;
  DecodeArgs a{cache, n_units, group, q, q_dtype, sm_scale, max_tokens, peer->out[peer->rank], peer->out_dtype,
               nullptr, 0, workspace, workspace_bytes, 0, 0, peer};
  const int lrc = launch_decode(a, reinterpret_cast<cudaStream_t>(stream));
  if (lrc) return lrc;
  return cuda_status("pqb_decode_attn_peer");
}

int pqb_peer_wait(const uint32_t* flags, int n_peers, int rank, uint32_t* expect, pqb_stream_t stream) {
  PQB_CHECK(flags && expect && n_peers >= 1 && n_peers <= PQB_MAX_PEERS && rank >= 0 && rank < n_peers, PQB_EINVAL,
            "bad peer wait arguments");
  launch_peer_wait(flags, n_peers, rank, expect, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_peer_wait");
}

// ---- peer-visible buffers (pqb_peer_out over CUDA IPC)
static int rt_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PQB_OK;
  (void)cudaGetLastError();
  set_error("%s: %s", what, cudaGetErrorString(e));
  return PQB_ECUDA;
}

static int select_device(int device) {
  int n = 0;
  PQB_CHECK(cudaGetDeviceCount(&n) == cudaSuccess && device >= 0 && device < n, PQB_EINVAL,
            "device %d out of range (%d visible)", device, n);
  return rt_status(cudaSetDevice(device), "cudaSetDevice");
}

int pqb_ipc_alloc(int device, size_t bytes, void** ptr, void* handle) {
  PQB_CHECK(ptr && handle && bytes > 0, PQB_EINVAL, "pqb_ipc_alloc: null output or zero size");
  *ptr = nullptr;
  int rc = select_device(device);
  if (rc != PQB_OK) return rc;
  void* p = nullptr;
  if ((rc = rt_status(cudaMalloc(&p, bytes), "cudaMalloc")) != PQB_OK) return rc;
  cudaIpcMemHandle_t h;
  rc = rt_status(cudaMemset(p, 0, bytes), "cudaMemset");
  if (rc == PQB_OK) rc = rt_status(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
  if (rc != PQB_OK) {
    cudaFree(p);
    return rc;
  }
  static_assert(sizeof(h) == PQB_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return PQB_OK;
}

int pqb_ipc_open(int device, const void* handle, void** ptr) {
  PQB_CHECK(ptr && handle, PQB_EINVAL, "pqb_ipc_open: null handle or output");
  *ptr = nullptr;
  const int rc = select_device(device);
  if (rc != PQB_OK) return rc;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return rt_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int pqb_ipc_close(int device, void* ptr) {
  PQB_CHECK(ptr, PQB_EINVAL, "pqb_ipc_close: null pointer");
  const int rc = select_device(device);
  return rc != PQB_OK ? rc : rt_status(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
}

int pqb_ipc_free(int device, void* ptr) {
  PQB_CHECK(ptr, PQB_EINVAL, "pqb_ipc_free: null pointer");
  const int rc = select_device(device);
  return rc != PQB_OK ? rc : rt_status(cudaFree(ptr), "cudaFree");
}

int pqb_peer_access(int device, int peer_device, int* can_access) {
  PQB_CHECK(can_access, PQB_EINVAL, "pqb_peer_access: null output");
  int n = 0;
  PQB_CHECK(cudaGetDeviceCount(&n) == cudaSuccess && device >= 0 && device < n && peer_device >= 0 &&
                peer_device < n, PQB_EINVAL, "devices %d, %d out of range (%d visible)", device, peer_device, n);
  if (device == peer_device) {
    *can_access = 1;
    return PQB_OK;
  }
  return rt_status(cudaDeviceCanAccessPeer(can_access, device, peer_device), "cudaDeviceCanAccessPeer");
}

int pqb_decode_launches(int64_t n_units, int group, int max_tokens, int flags) {
  if (n_units <= 0 || max_tokens <= 0) return 1;
  return decode_launch_count(n_units, group, max_tokens, flags);
}

int pqb_decode_launches_ex(int64_t n_units, int group, int max_tokens, int flags, int angle_bits, int radius_bits,
                           int value_dtype) {
  if (n_units <= 0 || max_tokens <= 0) return 1;
  return decode_launch_count(n_units, group, max_tokens, flags, angle_bits, radius_bits, value_dtype);
}

int pqb_decode_dq_layout(void) { return decode_dq_layout(); }

int pqb_decode_split_starts(int64_t n_units, int max_tokens, int ctas, int32_t* starts) {
  return starts ? decode_split_starts(n_units, max_tokens, ctas, starts) : -1;
}

int pqb_decode_splits(int64_t n_units, int max_tokens) {
  if (n_units <= 0 || max_tokens <= 0) return 1;
  return decode_splits(n_units, max_tokens);
}

int pqb_angle_table(int angle_bits, float* cos_out, float* sin_out, pqb_stream_t stream) {
  PQB_CHECK(angle_bits >= 1 && angle_bits <= 8, PQB_EINVAL, "angle_bits must be in [1, 8], got %d", angle_bits);
  PQB_CHECK(cos_out && sin_out, PQB_EINVAL, "null output");
  launch_angle_table(angle_bits, cos_out, sin_out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_angle_table");
}

int pqb_query_lut(const void* q, int q_dtype, int64_t n, int d, int layout, int angle_bits, float* out,
                  pqb_stream_t stream) {
  PQB_CHECK(d >= 2 && d % 2 == 0, PQB_EINVAL, "vector dimension must be even and >= 2, got %d", d);
  PQB_CHECK(angle_bits >= 1 && angle_bits <= 8, PQB_EINVAL, "angle_bits must be in [1, 8], got %d", angle_bits);
  PQB_CHECK(dtype_ok(q_dtype) && layout_ok(layout) && q && out && n >= 0, PQB_EINVAL, "bad arguments");
  launch_query_lut(q, q_dtype, n, d, layout, angle_bits, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_query_lut");
}

int pqb_radius_table(const uint16_t* scales, int64_t n_units, int d, int radius_bits, float* out,
                     pqb_stream_t stream) {
  PQB_CHECK(d >= 2 && d % 2 == 0, PQB_EINVAL, "vector dimension must be even and >= 2, got %d", d);
  PQB_CHECK(radius_bits >= 1 && radius_bits <= 8, PQB_EINVAL, "radius_bits must be in [1, 8], got %d", radius_bits);
  PQB_CHECK(scales && out && n_units >= 0, PQB_EINVAL, "bad arguments");
  launch_radius_table(scales, n_units, d, radius_bits, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_radius_table");
}

int pqb_unpack_codes(const pqb_store* store, int64_t unit, int d, int angle_bits, int radius_bits, int64_t tokens,
                     uint8_t* angle_out, uint8_t* radius_out, pqb_stream_t stream) {
  const int rc = check_store(store, d, angle_bits, radius_bits, false);
  if (rc) return rc;
  PQB_CHECK(tokens >= 0 && tokens <= static_cast<int64_t>(store->max_pages) * store->page_tokens, PQB_EINVAL,
            "tokens out of range");
  launch_unpack(*store, unit, d, angle_bits, radius_bits, tokens, angle_out, radius_out,
                reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_unpack_codes");
}

int pqb_export_streams(const pqb_store* store, int64_t unit, int d, int angle_bits, int radius_bits, int64_t tokens,
                       uint8_t* angle_stream, uint8_t* radius_stream, pqb_stream_t stream) {
  const int rc = check_store(store, d, angle_bits, radius_bits, false);
  if (rc) return rc;
  PQB_CHECK(tokens >= 0 && tokens <= static_cast<int64_t>(store->max_pages) * store->page_tokens, PQB_EINVAL,
            "tokens out of range");
  launch_export(*store, unit, d, angle_bits, radius_bits, tokens, angle_stream, radius_stream,
                reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_export_streams");
}

int pqb_read_values(const pqb_store* store, int64_t unit, int d, int64_t tokens, float* out, pqb_stream_t stream) {
  PQB_CHECK(store && store->pool && store->value_off >= 0, PQB_EINVAL, "store has no value region");
  PQB_CHECK(out && tokens >= 0 && d >= 2, PQB_EINVAL, "bad arguments");
  launch_read_values(*store, unit, d, tokens, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_read_values");
}

int pqb_pack_codes(const uint8_t* angle_codes, const uint8_t* radius_codes, int64_t tokens, int d, int angle_bits,
                   int radius_bits, const pqb_store* store, int64_t unit, pqb_stream_t stream) {
  const int rc = check_store(store, d, angle_bits, radius_bits, false);
  if (rc) return rc;
  PQB_CHECK(angle_codes && radius_codes && tokens >= 0 && unit >= 0, PQB_EINVAL, "bad arguments");
  PQB_CHECK(tokens <= static_cast<int64_t>(store->max_pages) * store->page_tokens, PQB_EINVAL, "tokens out of range");
  launch_pack_codes(angle_codes, radius_codes, tokens, d, angle_bits, radius_bits, *store, unit,
                    reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_pack_codes");
}

int pqb_dequantize(const pqb_cache* cache, int64_t unit, int64_t tokens, float* out, pqb_stream_t stream) {
  PQB_CHECK(cache && cache->scales, PQB_ESTATE, "cache is empty; prefill first");
  PQB_CHECK(out && tokens >= 0 && unit >= 0, PQB_EINVAL, "bad arguments");
  const int rc = check_store(&cache->store, cache->d, cache->angle_bits, cache->radius_bits, false);
  if (rc) return rc;
  launch_dequantize(*cache, unit, tokens, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_dequantize");
}

int pqb_quantize_values(const void* values, int dtype, int64_t n, int d, int bits, float* out, pqb_stream_t stream) {
  PQB_CHECK(bits >= 1 && bits <= 8, PQB_EINVAL, "bits must be in [1, 8], got %d", bits);
  PQB_CHECK(values && out && dtype_ok(dtype) && n >= 0 && d >= 1, PQB_EINVAL, "bad arguments");
  launch_quantize_values(values, dtype, n, d, bits, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_quantize_values");
}

int pqb_softmax_f64(const float* scores, int64_t n, double temperature, double* out, pqb_stream_t stream) {
  PQB_CHECK(n > 0, PQB_EINVAL, "cannot take attention weights of an empty score vector");
  PQB_CHECK(scores && out, PQB_EINVAL, "null pointer argument");
  launch_softmax_f64(scores, n, temperature, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_softmax_f64");
}

int pqb_to_polar(const void* x, const void* y, int dtype, int64_t n, void* radius_out, void* theta_out,
                 pqb_stream_t stream) {
  PQB_CHECK(dtype == PQB_F32 || dtype == PQB_F64, PQB_EINVAL, "to_polar: dtype must be PQB_F32 or PQB_F64");
  PQB_CHECK(n >= 0 && (n == 0 || (x && y && radius_out && theta_out)), PQB_EINVAL, "bad arguments");
  launch_to_polar(x, y, dtype, n, radius_out, theta_out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_to_polar");
}

int pqb_quantize_angle(const void* theta, int dtype, int64_t n, int angle_bits, uint8_t* out, pqb_stream_t stream) {
  PQB_CHECK(angle_bits >= 1 && angle_bits <= 8, PQB_EINVAL, "angle_bits must be in [1, 8], got %d", angle_bits);
  PQB_CHECK(dtype == PQB_F32 || dtype == PQB_F64, PQB_EINVAL, "quantize_angle: dtype must be PQB_F32 or PQB_F64");
  PQB_CHECK(n >= 0 && (n == 0 || (theta && out)), PQB_EINVAL, "bad arguments");
  launch_quantize_angle(theta, dtype, n, angle_bits, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_quantize_angle");
}

int pqb_angle_grid(int angle_bits, double* out, pqb_stream_t stream) {
  PQB_CHECK(angle_bits >= 1 && angle_bits <= 8, PQB_EINVAL, "angle_bits must be in [1, 8], got %d", angle_bits);
  PQB_CHECK(out, PQB_EINVAL, "null output");
  launch_angle_grid(angle_bits, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_angle_grid");
}

int pqb_quantize_radius(const void* radius, int dtype, const float* scale, int64_t n, int radius_bits, uint8_t* out,
                        unsigned long long* clamped, pqb_stream_t stream) {
  PQB_CHECK(radius_bits >= 1 && radius_bits <= 8, PQB_EINVAL, "radius_bits must be in [1, 8], got %d", radius_bits);
  PQB_CHECK(dtype == PQB_F32 || dtype == PQB_F64, PQB_EINVAL, "quantize_radius: dtype must be PQB_F32 or PQB_F64");
  PQB_CHECK(n >= 0 && (n == 0 || (radius && scale && out)), PQB_EINVAL, "bad arguments");
  launch_quantize_radius(radius, dtype, scale, n, radius_bits, out, clamped, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_quantize_radius");
}

int pqb_scores_direct(const pqb_cache* cache, int64_t unit, const void* q, int q_dtype, int64_t tokens, float* out,
                      pqb_stream_t stream) {
  PQB_CHECK(cache && cache->scales && cache->seq_lens && cache->quant_lens, PQB_ESTATE,
            "cache is empty; prefill first");
  PQB_CHECK(q && dtype_ok(q_dtype) && unit >= 0 && tokens >= 0 && (tokens == 0 || out), PQB_EINVAL,
            "bad arguments");
  const int rc = check_store(&cache->store, cache->d, cache->angle_bits, cache->radius_bits, false);
  if (rc) return rc;
  launch_scores_direct(*cache, unit, q, q_dtype, tokens, out, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_scores_direct");
}

int pqb_import_streams(const pqb_store* store, int64_t unit, int d, int angle_bits, int radius_bits, int64_t tokens,
                       const uint8_t* angle_stream, const uint8_t* radius_stream, pqb_stream_t stream) {
  const int rc = check_store(store, d, angle_bits, radius_bits, false);
  if (rc) return rc;
  PQB_CHECK(tokens >= 0 && tokens <= static_cast<int64_t>(store->max_pages) * store->page_tokens, PQB_EINVAL,
            "tokens out of range");
  PQB_CHECK(unit >= 0 && (tokens == 0 || (angle_stream && radius_stream)), PQB_EINVAL, "bad arguments");
  launch_import(*store, unit, d, angle_bits, radius_bits, tokens, angle_stream, radius_stream,
                reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_import_streams");
}

int pqb_synthetic_keys(uint64_t seed, int64_t n_units, int64_t tokens, int d, int layout, float radius_log_mean,
                       float radius_log_std, uint64_t outlier_mask, float outlier_boost, void* out, int out_dtype,
                       pqb_stream_t stream) {
  PQB_CHECK(d >= 2 && d % 2 == 0 && layout_ok(layout) && dtype_ok(out_dtype) && out, PQB_EINVAL, "bad arguments");
  PQB_CHECK(n_units >= 0 && n_units <= 65535 && tokens >= 0, PQB_EINVAL, "bad sizes");
  launch_synthetic_keys(seed, n_units, tokens, d, layout, radius_log_mean, radius_log_std, outlier_mask,
                        outlier_boost, out, out_dtype, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_synthetic_keys");
}

int pqb_synthetic_normal(uint64_t seed, int64_t count, void* out, int out_dtype, pqb_stream_t stream) {
  PQB_CHECK(dtype_ok(out_dtype) && out && count >= 0, PQB_EINVAL, "bad arguments");
  launch_synthetic_normal(seed, count, out, out_dtype, reinterpret_cast<cudaStream_t>(stream));
  return cuda_status("pqb_synthetic_normal");
}

}  // extern "C"
