// Where dynamic shared memory starts in a CTA's shared window (B200 result:
// 1 KB reserved at 0, static from 0x400, dynamic right after static; opt-in
// limit 232448 B for static + dynamic).  Used to size the 64 KB-aligned
// product-table layout discussed in DESIGN.md section 7.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/smem_base smem_base.cu && /tmp/smem_base
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* out) {
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ uint64_t st[64];
  st[threadIdx.x] = threadIdx.x;
  dyn[threadIdx.x] = 1;
  if (threadIdx.x == 0) {
    out[0] = static_cast<unsigned>(__cvta_generic_to_shared(dyn));
    out[1] = static_cast<unsigned>(__cvta_generic_to_shared(st));
  }
}
int main() {
  unsigned* d; cudaMalloc(&d, 8); unsigned h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k<<<1, 64, 200000>>>(d); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  int optin; cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  int reserved; cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, 0);
  printf("dyn=0x%x static=0x%x optin=%d reserved=%d err=%s\n", h[0], h[1], optin, reserved, cudaGetErrorString(cudaGetLastError()));
}
