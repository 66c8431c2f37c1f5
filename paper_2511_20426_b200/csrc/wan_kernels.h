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
  int row0;  // global batch row of local row 0 (entry = (row0 + row) / rows_per_entry)
};

// Multi-GPU temporal parallelism: every rank keeps a full KV-arena replica;
// fresh K/V rows reach every peer's arena over NVLink (P2P stores from the
// q/k kernel; BC_KV_PUSH=copy: side-stream copies) and (layer, slot, producer rank) ready epochs
// are published into each peer's flag array [L][n_slots][n_ranks];
// iteration-done epochs guard slot reuse.
#define BC_MAX_PEERS 8
struct PeerArgs {
  int n_peers;                          // 0 = single GPU
  __nv_bfloat16* arena[BC_MAX_PEERS];   // peers' arenas (same layout as ours)
  uint32_t* flags[BC_MAX_PEERS];        // peers' [L][n_slots][n_ranks] ready epochs
  uint32_t* done[BC_MAX_PEERS];         // peers' [n_ranks] iteration-done epochs
  const uint32_t* my_done;              // ours, written by peers
  int my_rank, n_ranks;
  uint32_t epoch;                       // this iteration's epoch
  uint32_t wait_done;                   // wait until every peer's done >= this (0 = no wait)
  int flag_base;                        // layer * n_slots
  uint32_t* ctr;                        // zeroed launch counter (last-CTA detection)
  int push;                             // 1: q/k kernel stores K/V into peers + publishes
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
  const float2* rope_f;  // [max_frames][22] cos/sin, time pairs
  const float2* rope_h;  // [hp][21]
  const float2* rope_w;  // [wp][21]
  int row0;              // global batch row of local row 0
  PeerArgs peer;
};

struct UpdArgs {
  float* latents[BC_MAX_ENTRIES];
  const float* eps[BC_MAX_ENTRIES];
  float* out[BC_MAX_ENTRIES];
  double level[BC_MAX_ENTRIES];
  double next_level[BC_MAX_ENTRIES];
  int post[BC_MAX_ENTRIES];
  int block[BC_MAX_ENTRIES];
  PeerArgs peer;  // iteration-done signal (flags/arena unused)
};

// tokens of global rows [row0, row0 + rows) of the concatenated batch
// status != nullptr: also the finiteness check of the latents (rows must
// cover every latent of the batch)
int launch_patchify(const EntryPtrs& lat, int F, int H, int W, int row0, int rows, __nv_bfloat16* out,
                    int32_t* status, cudaStream_t st);
// act 0: none, 1: silu, 2: out raw + out2 silu.  in == nullptr: the input
// is the sinusoid (K = freq_dim) of ts->t[e]; mod != nullptr: also
// mod[l][e][o] = base[l][o] + out[e][o] for l < L (the AdaLN tables)
int launch_gemv(const float* in, int n, int K, const __nv_bfloat16* W, const float* b, float* out, int N, int act,
                float* out2, cudaStream_t st, const TimeArgs* ts = nullptr, const float* base = nullptr, int L = 0,
                float* mod = nullptr);
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
int launch_signal_done(const PeerArgs& p, cudaStream_t st);
// release-store `v` to up to kMaxFlagWrites (peer) flag words from one
// thread after a system fence: the fallback of cuStreamWriteValue32
constexpr int kMaxFlagWrites = 64;
struct FlagWrites {
  uint32_t* addr[kMaxFlagWrites];
  int n;
  uint32_t v;
};
int launch_flag_writes(const FlagWrites& f, cudaStream_t st);
int launch_rope_tables(float2* tf, int max_frames, float2* th, int hp, float2* tw, int wp, cudaStream_t st);
constexpr int kRopeMaxFrames = 4096;
int launch_check_finite(const EntryPtrs& lat, int n, int n_el, int32_t* status, cudaStream_t st);

}  // namespace bc
