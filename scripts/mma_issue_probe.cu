// Microbenchmark: how long does one thread take to ISSUE tcgen05.mma groups,
// and what is the tensor pipe's execution rate, for the attention shapes
// (M=128, N=128 and N=256, K=16 per instruction, SS operands in smem).
#include <cstdio>
#include "../paper_2511_20426_b200/csrc/sm100.cuh"
using namespace bc;
template <int N, int GROUP>
__global__ void __launch_bounds__(128, 1) k(long long* out, int groups) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_bf16(128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32768);
    long long t_issue = 0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      long long s = clock64();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < GROUP; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_bf16_ss(tmem + (g & 1) * 256, desc_sw128(a0 + off, 16, 1024), desc_sw128(b0 + off, 16, 1024), idesc, kk != 0);
        }
      }
      __syncwarp();
      t_issue += clock64() - s;
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t_issue; out[1] = t1 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}
template <int N, int GROUP> void run(long long* out) {
  const int smem = 96 * 1024;
  cudaFuncSetAttribute(k<N, GROUP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int groups : {1, 2, 4, 64}) {
    k<N, GROUP><<<148, 128, smem>>>(out, groups);
    k<N, GROUP><<<148, 128, smem>>>(out, groups);
    long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    double ideal = (double)groups * GROUP * 128.0 * N / 256.0;  // floor 128*N/256 cycles per MMA
    printf("N=%d group=%d groups=%3d: issue %6.0f cyc/group, total %7lld cyc (ideal %7.0f) -> %.0f%% of tensor peak (err %s)\n",
           N, GROUP, groups, (double)h[0] / groups, h[1], ideal, 100.0 * ideal / h[1], cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  long long* out; cudaMalloc(&out, 64);
  run<128, 8>(out);
  run<256, 8>(out);
  return 0;
}
