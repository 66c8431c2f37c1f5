// Where does dynamic shared memory start?  (decides whether the 1 KB
// alignment slack for SW128 tiles is needed)
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* out) {
  extern __shared__ uint8_t smem[];
  out[0] = (unsigned)__cvta_generic_to_shared(smem);
}
__global__ void k2(unsigned* out) {
  __shared__ uint64_t bar[4];
  extern __shared__ uint8_t smem[];
  bar[threadIdx.x & 3] = 0;
  out[1] = (unsigned)__cvta_generic_to_shared(smem);
  out[2] = (unsigned)__cvta_generic_to_shared(bar);
}
int main() {
  unsigned* d; cudaMalloc(&d, 16); unsigned h[3] = {0, 0, 0};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k<<<1, 32, 232448>>>(d); k2<<<1, 32, 200000>>>(d);
  cudaMemcpy(h, d, 12, cudaMemcpyDeviceToHost);
  printf("dynamic smem offset (no static): %u ; with static: dyn %u static %u ; err %s\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
}
