// Launch interface of the Wan bandwidth-bound kernels (wan_kernels.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bcb200.h"

namespace bc {

struct EntryPtrs {
  const float* p[BC_MAX_ENTRIES];
  int block[BC_MAX_ENTRIES];
};

struct TimeArgs {
  double t[BC_MAX_ENTRIES];
};

// mode 0: LN(x) * (1 + base_scale + pe_scale[e]) + base_shift + pe_shift[e]
// mode 1: LN(x) * base_scale + base_shift          (affine LayerNorm)
struct LnArgs {
  int mode;
  const float* base_shift;
  const float* base_scale;
  const float* pe_shift;
  const float* pe_scale;
  int entry_stride;
};

struct QkArgs {
  __nv_bfloat16* qout;
  __nv_bfloat16* arena;
  int64_t mat_base;  // matrix index of slot 0's K for this layer
  int slot[BC_MAX_ENTRIES];
  int frame0[BC_MAX_ENTRIES];
  int hp, wp;
  const float* norm_q;
  const float* norm_k;
};

struct UpdArgs {
  float* latents[BC_MAX_ENTRIES];
  const float* eps[BC_MAX_ENTRIES];
  float* out[BC_MAX_ENTRIES];
  double level[BC_MAX_ENTRIES];
  double next_level[BC_MAX_ENTRIES];
  int post[BC_MAX_ENTRIES];
  int block[BC_MAX_ENTRIES];
};

int launch_patchify(const EntryPtrs& lat, int n, int F, int H, int W, __nv_bfloat16* out, cudaStream_t st);
int launch_gemv(const float* in, int n, int K, const __nv_bfloat16* W, const float* b, float* out, int N,
                int act_in, int act_out, cudaStream_t st);
int launch_timestep_sin(const TimeArgs& a, int n, float* out, int freq_dim, cudaStream_t st);
int launch_ln_rows(const float* X, __nv_bfloat16* out, int rows, int d, int rows_per_entry, const LnArgs& a,
                   cudaStream_t st);
int launch_qk_norm_rope(const __nv_bfloat16* qkv, int rows, int d, int T, const QkArgs& a, cudaStream_t st);
int launch_rms_rows(__nv_bfloat16* x, int rows, int d, int ld, const float* w, __nv_bfloat16* out, int ld_out,
                    cudaStream_t st);
int launch_copy_cols(const __nv_bfloat16* src, int ld_src, int c0, __nv_bfloat16* dst, int ld_dst, int rows,
                     int w, cudaStream_t st);
int launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t st);
int launch_head_update(const float* Y, int n, int T, int F, int H, int W, const UpdArgs& u, int32_t* status,
                       cudaStream_t st);
int launch_mod_combine(const float* base, const float* e0, int L, int n, int d, float* out, cudaStream_t st);
int launch_check_finite(const EntryPtrs& lat, int n, int n_el, int32_t* status, cudaStream_t st);

}  // namespace bc
