// Micro-test of the tcgen05 P.V formulation used by the PQB_DQ_UMMA decode
// build: O^T[128 dims x 8] = V^T[128 x 32 tokens] . P^T[32 x 8] with
//   A = V^T from a 32-token value tile in the grouped page layout (8-token
//       groups of [dims 0-63 | dims 64-127], 128 B rows, 16-B chunks XOR (t & 7)),
//       MN-major, 128-byte swizzle;
//   B = P^T as K-major core matrices (8 rows x 16 B) at a 256-B stride;
//   D = fp32 in tensor memory, read back with tcgen05.ld.32x32b.x8.
// Tries descriptor variants and prints the max error of each against a CPU
// reference:  nvcc -gencode arch=compute_100a,code=sm_100a -I.. -o umma_pv umma_pv.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | ((uint64_t)layout << 61);
}

__global__ void k(const uint8_t* vtile, const uint8_t* pt, float* out, uint32_t a_lbo, uint32_t a_sbo, uint32_t a_lay,
                  uint32_t b_lbo, uint32_t b_sbo, uint32_t idesc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sv = sm;             // 8 KB value tile (1 KB aligned)
  uint8_t* sp = sm + 8192;      // P^T: 4 core matrices, each in the second half of a 256-B slot
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 8192; i += blockDim.x) sv[i] = vtile[i];
  for (int i = tid; i < 1024; i += blockDim.x) sp[i] = pt[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  if (tid == 0) {
    for (int h = 0; h < 2; ++h) {
      const uint64_t ad = desc(smem_u32(sv) + h * 4096, a_lbo, a_sbo, a_lay);
      const uint64_t bd = desc(smem_u32(sp) + 128 + h * 512, b_lbo, b_sbo, 0);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(t), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)h) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncwarp();
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(t + ((32u * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int c = 0; c < 8; ++c) out[(32 * warp + lane) * 8 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
  }
}

static uint16_t bf(float f) { __nv_bfloat16 b = __float2bfloat16(f); return *reinterpret_cast<uint16_t*>(&b); }

int main() {
  // V[t][e], P[t][n] small integers (exact in bf16 and fp32 sums)
  std::vector<float> V(32 * 128), P(32 * 8);
  for (int t = 0; t < 32; ++t) for (int e = 0; e < 128; ++e) V[t * 128 + e] = (float)(((t * 7 + e * 3) % 11) - 5);
  for (int t = 0; t < 32; ++t) for (int n = 0; n < 8; ++n) P[t * 8 + n] = (float)(((t * 5 + n * 3) % 7) - 3);
  std::vector<uint8_t> vt(8192, 0), pt(1024, 0);
  for (int t = 0; t < 32; ++t)
    for (int e = 0; e < 128; ++e) {
      const size_t off = ((t >> 3) << 11) + ((e >> 6) << 10) + ((t & 7) << 7) + (((((e >> 3) & 7) ^ (t & 7))) << 4) + ((e & 7) << 1);
      const uint16_t b = bf(V[t * 128 + e]);
      memcpy(&vt[off], &b, 2);
    }
  // core matrix j (tokens 8j..8j+7) at slot j: second half of 256-B slot, row n = 16 B
  for (int t = 0; t < 32; ++t)
    for (int n = 0; n < 8; ++n) {
      const size_t off = (t >> 3) * 256 + 128 + n * 16 + (t & 7) * 2;
      const uint16_t b = bf(P[t * 8 + n]);
      memcpy(&pt[off], &b, 2);
    }
  std::vector<double> ref(128 * 8, 0.0);
  for (int e = 0; e < 128; ++e) for (int n = 0; n < 8; ++n) for (int t = 0; t < 32; ++t) ref[e * 8 + n] += V[t * 128 + e] * P[t * 8 + n];
  uint8_t *dv, *dp; float* dout;
  cudaMalloc(&dv, 8192); cudaMalloc(&dp, 1024); cudaMalloc(&dout, 128 * 8 * 4);
  cudaMemcpy(dv, vt.data(), 8192, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, pt.data(), 1024, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  const uint32_t idesc_mn = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 17) | (8u << 24);
  struct Var { uint32_t alb, asb, alay, blb, bsb, id; const char* name; } vars[] = {
      {1024, 2048, 2, 256, 256, idesc_mn, "A lbo1K sbo2K sw128 | B lbo256"},
      {2048, 1024, 2, 256, 256, idesc_mn, "A lbo2K sbo1K sw128 | B lbo256"},
      {1024, 2048, 2, 128, 256, idesc_mn, "A lbo1K sbo2K | B lbo128 sbo256"},
      {1024, 2048, 2, 256, 128, idesc_mn, "A lbo1K sbo2K | B lbo256 sbo128"},
      {2048, 1024, 2, 256, 128, idesc_mn, "A lbo2K sbo1K | B lbo256 sbo128"},
  };
  std::vector<float> out(128 * 8);
  for (auto& v : vars) {
    cudaMemset(dout, 0, 128 * 8 * 4);
    k<<<1, 128, 16384>>>(dv, dp, dout, v.alb, v.asb, v.alay, v.blb, v.bsb, v.id);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: CUDA error %s\n", v.name, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(out.data(), dout, 128 * 8 * 4, cudaMemcpyDeviceToHost);
    double err = 0; int bad = 0;
    for (int i = 0; i < 128 * 8; ++i) { const double d = fabs(out[i] - ref[i]); err = d > err ? d : err; bad += d > 1e-3 || std::isnan(out[i]); }
    printf("%-40s max err %.3g  bad %d  out[0..3] %g %g %g %g ref %g %g %g %g\n", v.name, err, bad, out[0], out[1], out[8], out[9],
           ref[0], ref[1], ref[8], ref[9]);
  }
  return 0;
}
