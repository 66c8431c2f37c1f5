// Debug timeline of the tcgen05 GEMM: nvcc -DBC_GEMM_TRACE ... (see gemm_trace.sh)
#include "../paper_2511_20426_b200/csrc/gemm.cu"
#include <cstdio>
#include <vector>
int main(int argc, char** argv) {
  int M = 8192, N = 8192, K = 8192, cg = argc > 1 ? atoi(argv[1]) : 1;
  void *A, *B, *C;
  cudaMalloc(&A, (size_t)M * K * 2); cudaMalloc(&B, (size_t)N * K * 2); cudaMalloc(&C, (size_t)M * N * 2);
  cudaMemset(A, 0, (size_t)M * K * 2); cudaMemset(B, 0, (size_t)N * K * 2);
  bc::GemmArgs g{A, B, C, M, N, K, 0, nullptr, nullptr, 0, 1, 256, cg};
  for (int i = 0; i < 3; ++i) bc::gemm_run(g, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); bc::gemm_run(g, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("cg=%d %.1f us %.0f TFLOP/s err=%s\n", cg, ms * 1e3, 2.0 * M * N * K / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  static unsigned long long t[4][3][256];
  cudaMemcpyFromSymbol(t, bc::g_gemm_trace, sizeof(t));
  unsigned long long t0 = t[0][0][0];
  for (int c = 0; c < (cg == 2 ? 2 : 1); ++c) {
    printf("cta %d producer issue (ns):", c);
    for (int k = 0; k < 24; ++k) printf(" %lld", (long long)(t[c][0][k] - t0));
    printf("\ncta %d mma full (ns):", c);
    for (int k = 0; k < 24; ++k) printf(" %lld", (long long)(t[c][1][k] - t0));
    printf("\ncta %d tfull (ns):", c);
    for (int k = 0; k < 2; ++k) printf(" %lld", (long long)(t[c][2][k] - t0));
    printf("\n");
  }
  // steady state per-kb interval of MMA-full on cta 0
  printf("mma interval kb 40..120 avg ns: %.1f\n", (double)(t[0][1][120] - t[0][1][40]) / 80);
  return 0;
}
