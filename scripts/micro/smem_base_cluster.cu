// Dynamic shared-memory base per CTA rank in a thread-block-cluster launch
// (does the product table's fixed-address layout hold in clusters?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o smem_base_cluster smem_base_cluster.cu
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* out) {
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ uint64_t st[32];
  st[threadIdx.x & 31] = threadIdx.x;
  dyn[threadIdx.x] = 1;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = rank;
    out[blockIdx.x * 4 + 1] = static_cast<unsigned>(__cvta_generic_to_shared(dyn));
    out[blockIdx.x * 4 + 2] = static_cast<unsigned>(__cvta_generic_to_shared(st));
    unsigned remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(dyn))), "r"(0u));
    out[blockIdx.x * 4 + 3] = remote;
  }
}
int main() {
  const int nb = 8;
  unsigned* d; cudaMalloc(&d, nb * 16); unsigned h[nb * 4];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int cl : {1, 2, 4}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 200000;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, d);
    cudaMemcpy(h, d, nb * 16, cudaMemcpyDeviceToHost);
    printf("cluster %d: err=%s\n", cl, cudaGetErrorString(cudaGetLastError()));
    for (int b = 0; b < nb; ++b) printf("  block %d rank %u dyn=0x%x static=0x%x mapa(dyn, rank0)=0x%x\n", b, h[b * 4], h[b * 4 + 1], h[b * 4 + 2], h[b * 4 + 3]);
  }
}
