// Host interface of the tcgen05 flash attention (attention.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bcb200.h"

namespace bc {

// Kernel parameter block (by value).
struct AttnParams {
  int q_tokens;    // query rows per entry
  int kv_tokens;   // keys per slot (per matrix)
  int heads;
  int mat_base;    // matrix index of slot 0's K for this layer
  int mat_stride;  // matrices between consecutive slots
  int v_offset;    // matrices from a slot's K to its V
  float scale;     // softmax scale (1/sqrt(head_dim))
  void* out;       // bf16 [n_entries*q_tokens][heads*128]
  unsigned long long* trace;  // diagnostic timeline (BC_ATTN_TRACE builds)
  int n_vis[BC_MAX_ENTRIES];
  int vis_slot[BC_MAX_ENTRIES][BC_MAX_VIS];
  // multi-GPU: before the first tile of visible slot v, wait until
  // flags[flag_base + slot] >= need[e][v] (0 = no wait; peers publish)
  const uint32_t* flags;
  int flag_base;
  uint32_t need[BC_MAX_ENTRIES][BC_MAX_VIS];
};

struct AttnArgs {
  const void* q;        // bf16 [n_entries*q_tokens][heads*128]
  const void* kv_base;  // bf16 matrices [n_mats][kv_tokens][heads*128]
  int n_mats;
  int n_entries, q_tokens, kv_tokens, heads, head_dim;
  int mat_base, mat_stride, v_offset;
  float scale;
  void* out;
  int n_vis[BC_MAX_ENTRIES];
  int vis_slot[BC_MAX_ENTRIES][BC_MAX_VIS];
  const uint32_t* flags;
  int flag_base;
  uint32_t need[BC_MAX_ENTRIES][BC_MAX_VIS];
};

int attention_run(const AttnArgs& a, cudaStream_t st);

}  // namespace bc
