// Microbenchmark: MUFU.EX2 throughput per SM vs warps per SM sub-partition,
// and with interleaved FFMA2/F2FP (the softmax mix).
#include <cstdio>
#include <cuda_bf16.h>
template <int MIX>
__global__ void k(float* out, int iters, long long* cyc) {
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float a = v[i], b = v[i + 1];
      if (MIX) { a = fmaf(a, 0.999f, -0.001f); b = fmaf(b, 0.999f, -0.001f); }
      float x, y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(x) : "f"(a));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(b));
      if (MIX) {
        __nv_bfloat162 p = __floats2bfloat162_rn(x, y);
        acc += *reinterpret_cast<unsigned*>(&p);
      }
      v[i] = x * 0.5f; v[i + 1] = y * 0.5f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int mix = 0; mix < 2; ++mix)
  for (int threads : {128, 256, 512, 1024}) {
    int iters = 256;
    if (mix) k<1><<<148, threads>>>(out, iters, cyc); else k<0><<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    if (mix) k<1><<<148, threads>>>(out, iters, cyc); else k<0><<<148, threads>>>(out, iters, cyc);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ex2 = (double)threads * iters * 16;
    printf("mix=%d threads=%4d warps/SMSP=%d: %.2f ex2/clk/SM  (%.2f cyc per warp-MUFU per SMSP)\n", mix, threads,
           threads / 128, ex2 / c, c / (ex2 / 32 / 4));
  }
  return 0;
}
