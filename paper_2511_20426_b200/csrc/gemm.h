// Host interface of the tcgen05 GEMM (gemm.cu) used by the Wan runtime.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bc {

enum GemmEpilogue {
  kEpiStoreBf16 = 0,    // C bf16 = acc + bias
  kEpiGeluBf16 = 1,     // C bf16 = gelu_tanh(acc + bias)
  kEpiStoreF32 = 2,     // C fp32 = acc + bias
  kEpiResidualF32 = 3,  // C fp32 += gate[row / rows_per_gate] * (acc + bias)
};

struct GemmArgs {
  const void* A;  // bf16 [M][K]
  const void* B;  // bf16 [N][K]
  void* C;
  int M, N, K;
  int mode;
  const float* bias;
  const float* gate;
  int gate_stride;
  int rows_per_gate;
  int bn;  // 0 = auto
  int cg;  // 0 = auto, 1 = single CTA, 2 = CTA pair
  int gate_row0;  // gate row of C row r = (gate_row0 + r) / rows_per_gate
};

int gemm_run(const GemmArgs& g, cudaStream_t st);
int make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
// the same with a 128 / 64 / 32-byte (or 0 = no) swizzle
int make_tmap_2d_swz(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);
// fp32 (the gated-residual GEMM's C tiles)
int make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);
int num_sms();

}  // namespace bc
