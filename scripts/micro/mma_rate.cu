// Microbenchmark: legacy mma.sync m16n8k16 bf16->f32 issue rate on one B200
// (148 SMs, 8 warps/SM, 4 independent accumulator chains per warp).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256, 1) mma_loop(float* out, int iters, uint32_t seed) {
  float d[4][4] = {};
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b0 = a0 * 11u, b1 = a0 * 13u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// LDS.64 gather rate (conflict-free, random index within a 128-B row)
__global__ void __launch_bounds__(256, 1) lds_loop(float* out, int iters) {
  __shared__ float2 tab[16 * 64];
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) tab[i] = make_float2(i, -i);
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u;
  float s0 = 0.f, s1 = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float2 t = tab[j * 16 + ((x >> (j & 7) * 4) & 15)];
      s0 += t.x;
      s1 += t.y;
    }
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sms * 256 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    mma_loop<<<sms, 256>>>(out, iters, rep);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = double(sms) * 8 * iters * 4;
    printf("mma.sync m16n8k16 bf16: %.3f ms, %.1f TFLOP/s, %.3f mma/clk/SM @1.9GHz\n", ms,
           mmas * 4096 / (ms * 1e-3) / 1e12, mmas / sms / (ms * 1e-3 * 1.9e9));
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    lds_loop<<<sms, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double lds = double(sms) * 8 * iters * 16;
    printf("LDS.64 warp-instr: %.3f ms, %.3f instr/clk/SM @1.9GHz\n", ms, lds / sms / (ms * 1e-3 * 1.9e9));
  }
  return 0;
}
