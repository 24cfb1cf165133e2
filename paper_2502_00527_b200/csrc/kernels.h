// Internal launcher interface between the C ABI (abi.cu) and the kernel files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pqb200.h"

namespace pqb {

struct RadiusScalesArgs {
  const void* keys;
  int key_dtype;
  int64_t n_units, tokens;
  int d;
  int64_t unit_stride, tok_stride;
  int layout, radius_bits;
  unsigned long long* maxsq_ws;
  uint16_t* scales_out;
  int32_t* flags;
  bool vector_ok;  // 8-channel vector path legal (alignment / d)
};

struct EncodeArgs {
  const void* keys;
  int key_dtype;
  int64_t n_units, tokens;
  int d;
  int64_t unit_stride, tok_stride;
  int layout, angle_bits, radius_bits;
  const uint16_t* scales;
  const pqb_store* store;
  const int32_t* tok_offset;
  int64_t tok_offset_const;
  unsigned long long* clamp_counts;
  int32_t* flags;
  bool vector_ok;
};

struct DecodeArgs {
  const pqb_cache* cache;
  int64_t n_units;
  int group;
  const void* q;
  int q_dtype;
  float sm_scale;
  int max_tokens;
  void* out;
  int out_dtype;
  float* scores;
  int64_t scores_ld;
  void* workspace;
  size_t workspace_bytes;
  int flags = 0;   // PQB_DECODE_* bits
  int splits = 0;  // 0: automatic
  const pqb_peer_out* peer = nullptr;  // pqb_decode_attn_peer
};

int launch_radius_scales(const RadiusScalesArgs& a, cudaStream_t s);
// decode.cu: kernels a fused DQ decode call enqueues (1, or 2 with the separate split merge)
int decode_launch_count(int64_t n_units, int group, int max_tokens, int flags, int angle_bits = 4, int radius_bits = 4,
                       int value_dtype = PQB_BF16);
int decode_dq_layout();
int decode_split_starts(int64_t n_units, int max_tokens, int ctas, int32_t* starts);
int launch_encode(const EncodeArgs& a, cudaStream_t s);
// encode_fast.cu: persistent TMA-fed encoder for d = 128, m, n in {2,3,4}; false if the call does not qualify.
bool launch_encode_fast(const EncodeArgs& a, cudaStream_t s);
int launch_store_values(const void* vals, int dtype, int64_t n_units, int64_t T, int d, int64_t us, int64_t ts,
                        const pqb_store& st, const int32_t* tok_offset, int64_t tok_offset_const, cudaStream_t s,
                        int32_t* flags = nullptr);
int launch_store_residual(const pqb_cache& c, const void* keys, int dtype, int64_t n_units, int64_t T, int64_t us,
                          int64_t ts, int64_t tok_offset_const, int32_t* flags, cudaStream_t s);
int launch_append(const pqb_cache& c, int64_t n_units, const void* keys, int key_dtype, const void* vals,
                  int val_dtype, unsigned long long* clamp_counts, int32_t* flags, cudaStream_t s);

int decode_splits(int64_t n_units, int max_tokens);
size_t decode_workspace_bytes(int64_t n_units, int group, int max_tokens, int d);
// returns PQB_OK or PQB_EUNSUPPORTED / PQB_EINVAL (message via set_error)
int launch_decode(const DecodeArgs& a, cudaStream_t s);

int launch_angle_table(int m, float* c, float* s, cudaStream_t st);
int launch_query_lut(const void* q, int q_dtype, int64_t n, int d, int layout, int m, float* out, cudaStream_t s);
int launch_radius_table(const uint16_t* scales, int64_t n_units, int d, int n_bits, float* out, cudaStream_t s);
int launch_unpack(const pqb_store& st, int64_t unit, int d, int m, int n, int64_t T, uint8_t* a, uint8_t* r,
                  cudaStream_t s);
int launch_export(const pqb_store& st, int64_t unit, int d, int m, int n, int64_t T, uint8_t* a, uint8_t* r,
                  cudaStream_t s);
int launch_read_values(const pqb_store& st, int64_t unit, int d, int64_t T, float* out, cudaStream_t s);
int launch_pack_codes(const uint8_t* a, const uint8_t* r, int64_t T, int d, int m, int n, const pqb_store& st,
                      int64_t unit, cudaStream_t s);
int launch_dequantize(const pqb_cache& c, int64_t unit, int64_t T, float* out, cudaStream_t s);
int launch_peer_wait(const uint32_t* flags, int n_peers, int rank, uint32_t* expect, cudaStream_t s);
int launch_quantize_values(const void* vals, int dt, int64_t n, int d, int bits, float* out, cudaStream_t s);
int launch_softmax_f64(const float* scores, int64_t n, double temperature, double* out, cudaStream_t s);
int launch_synthetic_keys(uint64_t seed, int64_t n_units, int64_t T, int d, int layout, float mu, float sigma,
                          uint64_t mask, float boost, void* out, int dtype, cudaStream_t s);
int launch_synthetic_normal(uint64_t seed, int64_t count, void* out, int dtype, cudaStream_t s);

// api.cu: element-wise reference API, PQC1 import, qk_scores_direct
int launch_to_polar(const void* x, const void* y, int dtype, int64_t n, void* r, void* t, cudaStream_t s);
int launch_quantize_angle(const void* theta, int dtype, int64_t n, int m, uint8_t* out, cudaStream_t s);
int launch_angle_grid(int m, double* out, cudaStream_t s);
int launch_quantize_radius(const void* radius, int dtype, const float* scale, int64_t n, int bits, uint8_t* out,
                           unsigned long long* clamped, cudaStream_t s);
int launch_import(const pqb_store& st, int64_t unit, int d, int m, int n, int64_t T, const uint8_t* a,
                  const uint8_t* r, cudaStream_t s);
int launch_scores_direct(const pqb_cache& c, int64_t unit, const void* q, int q_dtype, int64_t tokens, float* out,
                         cudaStream_t s);

void set_error(const char* fmt, ...);

}  // namespace pqb
