// Microbenchmark: per-SM throughput of the softmax instruction mix on B200
// (FFMA, FFMA2, FADD2, FMNMX3, F2FP bf16 pack, MUFU.EX2) at 1..4 warps/SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__device__ __forceinline__ uint64_t f2(float lo, float hi) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float v[16]; uint64_t w[8]; uint32_t u[8];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int i = 0; i < 8; ++i) { w[i] = f2(v[i], v[i + 8]); u[i] = i; }
  const uint64_t c2 = f2(0.999f, 0.999f), m2 = f2(-0.001f, -0.001f);
  const float c = 0.999f, m = -0.001f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { v[i] = fmaf(v[i], c, m); v[i + 8] = fmaf(v[i + 8], c, m); }               // 2 FFMA (reg)
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[i]) : "l"(c2), "l"(m2)); // 1 FFMA2
      if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[i]) : "l"(m2));              // 1 FADD2
      if (OP == 3) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[i + 8]), "f"(v[(i + 1) & 15]));  // FMNMX3
      if (OP == 4) { __nv_bfloat162 p = __floats2bfloat162_rn(v[i], v[i + 8]); u[i] += *reinterpret_cast<uint32_t*>(&p); v[i] += 1e-7f; }  // F2FP (+FADD)
      if (OP == 5) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i])); v[i] = y * 0.5f; }  // MUFU (+FMUL)
      if (OP == 7) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(u[i])); u[i] = y ^ 0x00010001u; }  // MUFU f16x2
      if (OP == 8) { uint32_t y; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(v[i]), "f"(v[i + 8])); u[i] += y; v[i] += 1e-7f; }  // F2FP f16
      if (OP == 9) { asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) & 7])); }  // HADD2
      if (OP == 6) { v[i] = fmaf(v[i], 0.999f, -0.001f); v[i + 8] = fmaf(v[i + 8], 0.999f, -0.001f); }  // FFMA imm
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
  for (int i = 0; i < 8; ++i) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(w[i])); s += a + b + u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, int per_iter, float* out, long long* cyc) {
  for (int threads : {128, 256, 512}) {
    int iters = 512;
    k<OP><<<148, threads>>>(out, iters, cyc);
    k<OP><<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double warp_instr_per_smsp = (double)threads / 32 / 4 * iters * per_iter;
    printf("%-12s warps/SMSP=%d: %.2f cycles per warp-instruction per SMSP\n", name, threads / 128, c / warp_instr_per_smsp);
  }
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  run<0>("FFMA reg", 16, out, cyc);
  run<6>("FFMA imm", 16, out, cyc);
  run<1>("FFMA2", 8, out, cyc);
  run<2>("FADD2", 8, out, cyc);
  run<3>("FMNMX3", 8, out, cyc);
  run<4>("F2FP+FADD", 8, out, cyc);
  run<5>("MUFU+FMUL", 8, out, cyc);
  run<7>("MUFU.f16x2", 8, out, cyc);
  run<8>("F2FP.f16+FADD", 8, out, cyc);
  run<9>("HADD2", 8, out, cyc);
  return 0;
}
