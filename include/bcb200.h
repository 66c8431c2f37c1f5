/*
 * bcb200.h -- C-ABI of the B200-native Block Cascading hot path.
 *
 * The reference (`blockcascade`, pure Python/numpy) has no FFI; these entry
 * points are what its numeric operator boundary would bind.  Each one names
 * the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/blockcascade/).  Plain pointers and sizes only:
 * device pointers are CUDA global-memory addresses, `stream` is a
 * cudaStream_t passed as void*, host pointers are marked [host].
 *
 * Status codes (mapped onto the reference's exception classes by
 * paper_2511_20426_b200/errors.py):
 *   BC_OK 0, BC_ERR_CONTRACT 1 (ContractViolation), BC_ERR_NUMERIC 2
 *   (NumericError), BC_ERR_CUDA 3 (CUDA/NCCL failure, or no device).
 */
#ifndef BCB200_H_
#define BCB200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BC_OK 0
#define BC_ERR_CONTRACT 1
#define BC_ERR_NUMERIC 2
#define BC_ERR_CUDA 3

#define BC_MAX_ENTRIES 16 /* cascade width cap per launch (ceil(P/o) <= 16) */
#define BC_MAX_VIS 32     /* visible key blocks per query block             */

/* Human-readable text of the last error on this thread. */
const char* bc_last_error(void);
/* Library version / build flags string. */
const char* bc_version(void);
/* Kernels launched by this library so far (process-wide). */
long long bc_launch_count(void);
/* Per-kernel-class CUDA-event timing of bc_wan_step launches (classes:
 * 0 self-attention, 1 cross-attention, 2 GEMM, 3 bandwidth-bound). */
int bc_profile_enable(int on);
int bc_profile_collect(double* ms, double* flops, double* bytes, int64_t* launches, int n_classes);

/* ---------------------------------------------------------------------------
 * Noise: NoiseStream.draw / block_noise (core.py:161-186) and the Philox
 * expansion of embed_prompt (core.py:144-158).  Bit-identical to numpy:
 * Philox4x64-10 bit generator (key, 256-bit counter incremented before each
 * 4-word block) feeding numpy's own ziggurat `random_standard_normal_fill`.
 * Host-side, GIL-free, one thread per stream.
 * ------------------------------------------------------------------------- */
typedef struct {
  uint64_t key[2];     /* Philox key words                           */
  uint64_t counter[4]; /* Philox counter, e.g. {block, pass, frame, 0} */
  int64_t n;           /* normals to draw                            */
  void* out;           /* [host] float64 or float32 destination      */
} bc_noise_task;

/* dtype: 0 = float64, 1 = float32 (rounded from the float64 draw). */
int bc_noise_run(const bc_noise_task* tasks /*[host]*/, int n_tasks, int dtype,
                 int n_threads);

/* Raw Philox4x64-10 output words (for known-answer tests). */
int bc_philox4x64(const uint64_t key[2], const uint64_t counter[4], uint64_t out[4]);

/* ---------------------------------------------------------------------------
 * renoise (denoiser.py:360-368): out = (1 - s) * x0 + s * eps, s = level/1000,
 * evaluated without FMA contraction (bit-identical to numpy for float64).
 * out may alias x0.  `nonfinite` (device int32, may be NULL) is set to 1 if
 * any output is non-finite.
 * ------------------------------------------------------------------------- */
int bc_renoise_f64(const double* x0, const double* eps, double level, double* out,
                   int64_t n, int32_t* nonfinite, void* stream);
int bc_renoise_f32(const float* x0, const float* eps, double level, float* out,
                   int64_t n, int32_t* nonfinite, void* stream);

/* ---------------------------------------------------------------------------
 * Batch description shared by both forwards: one entry per in-flight block
 * (plan order = ascending block).  vis_slot[e][0..n_vis[e]) lists the KV
 * arena slots the entry's queries attend to, in ascending block order --
 * the gather order of denoiser._gather (denoiser.py:284-296) and the column
 * order of build_mask (denoiser.py:172-194).  slot[e] is where the entry
 * writes its fresh per-layer K/V.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t n_entries;
  int32_t block_size; /* latent frames per block (S)              */
  int32_t block_index[BC_MAX_ENTRIES];
  double level[BC_MAX_ENTRIES];
  int32_t slot[BC_MAX_ENTRIES];
  int32_t n_vis[BC_MAX_ENTRIES];
  int32_t vis_slot[BC_MAX_ENTRIES][BC_MAX_VIS];
} bc_batch;

/* ---------------------------------------------------------------------------
 * Toy DiT forward (denoiser.py:299-357, embed_entry 234-250, layer_qkv
 * 253-261, layer_attend 264-277, predict_head 280-281), float64 on device.
 * KV arena layout: [layers][n_slots][2 (K,V)][S][D] float64.
 * ------------------------------------------------------------------------- */
typedef struct {
  const double *w_in, *w_cond, *w_level, *w_q, *w_k, *w_v, *w_o, *w_head;
  int32_t layers, heads, dim, cond_dim;
} bc_toy_weights;

int bc_toy_forward(const bc_toy_weights* w /*[host struct, device ptrs]*/,
                   const bc_batch* batch /*[host]*/,
                   const double* const* latents /*[host] n_entries device ptrs (S,D)*/,
                   const double* const* cond /*[host] n_entries device ptrs (Dc)*/,
                   double* kv_arena, int32_t n_slots,
                   double* const* x0_out /*[host] n_entries device ptrs (S,D)*/,
                   double* workspace /* >= 2*n*S*D doubles */,
                   int32_t* status /* device int32: 1+block of first non-finite input */,
                   void* stream);

/* ---------------------------------------------------------------------------
 * Wan2.1-shaped DiT (configs 2-5).  See wan_runtime.cu / DESIGN.md.
 * ------------------------------------------------------------------------- */
typedef struct bc_wan_ctx bc_wan_ctx;

typedef struct {
  int32_t layers, heads, head_dim, ffn_dim;
  int32_t text_len, text_dim, freq_dim;
  int32_t latent_h, latent_w;  /* latent grid (patch 1x2x2, 16 channels) */
  int32_t block_size;          /* latent frames per block                 */
  int32_t n_slots;             /* KV arena slots                          */
  int32_t max_entries;         /* widest batch the workspace must hold    */
} bc_wan_dims;

/* Parameter block: device pointers into caller-owned (torch) storage.
 * Linear weights are bf16 [out][in] (nn.Linear layout), vectors fp32. */
typedef struct {
  const void* patch_w;  const float* patch_b;    /* [d][64], [d]           */
  const void* text_w1;  const float* text_b1;    /* [d][text_dim]          */
  const void* text_w2;  const float* text_b2;    /* [d][d]                 */
  const void* time_w1;  const float* time_b1;    /* [d][freq_dim]          */
  const void* time_w2;  const float* time_b2;    /* [d][d]                 */
  const void* tproj_w;  const float* tproj_b;    /* [6d][d]                */
  const void* head_w;   const float* head_b;     /* [64][d]                */
  const float* head_mod;                          /* [2][d]                 */
  /* per layer, stacked over layers */
  const void* qkv_w;    const float* qkv_b;      /* [L][3d][d], [L][3d]    */
  const void* o_w;      const float* o_b;        /* [L][d][d]              */
  const void* cq_w;     const float* cq_b;       /* cross q                */
  const void* ckv_w;    const float* ckv_b;      /* [L][2d][d] cross k,v   */
  const void* co_w;     const float* co_b;       /* cross out              */
  const void* ffn1_w;   const float* ffn1_b;     /* [L][ffn][d]            */
  const void* ffn2_w;   const float* ffn2_b;     /* [L][d][ffn]            */
  const float* norm_q;  const float* norm_k;     /* [L][d] RMSNorm weights */
  const float* cnorm_q; const float* cnorm_k;    /* [L][d] cross RMSNorm   */
  const float* norm3_w; const float* norm3_b;    /* [L][d] cross-attn LN   */
  const float* modulation;                        /* [L][6][d]              */
} bc_wan_params;

int bc_wan_create(const bc_wan_dims* dims, const bc_wan_params* params,
                  void* kv_arena /* bf16 [L][n_slots][2][T][d] */,
                  void* workspace, int64_t workspace_bytes, bc_wan_ctx** out);
/* Bytes of workspace bc_wan_create needs for these dims. */
int64_t bc_wan_workspace_bytes(const bc_wan_dims* dims);
int bc_wan_destroy(bc_wan_ctx* ctx);

/* Per prompt: text MLP over the synthetic encoder states (device fp32
 * [text_len][text_dim]) and the per-layer cross-attention K/V. */
int bc_wan_set_text(bc_wan_ctx* ctx, const float* text_states, void* stream);

/* Per-entry fused update applied after the head (the "Euler/renoise step"):
 *   x0 = x_t - sigma_t * v   (flow-matching head, sigma_t = level/1000)
 *   post 0: x_next = (1-s') x0 + s' eps,  s' = next_level/1000
 *   post 1: x_next = x0 and emit_out = x0 (emission)
 *   post 2: nothing (cache pass; KV already written to the slot)
 *   post 3: x0_out = x0 only (operator API: forward without update) */
typedef struct {
  int32_t post[BC_MAX_ENTRIES];
  double next_level[BC_MAX_ENTRIES];
  float* latents[BC_MAX_ENTRIES];     /* (S,16,H,W) fp32, updated in place */
  const float* eps[BC_MAX_ENTRIES];   /* post 0 */
  float* out[BC_MAX_ENTRIES];         /* post 1 / 3 */
} bc_wan_update;

/* One cascade iteration: batched forward of every entry + fused update.
 * Launched as a CUDA graph (re-captured per step, one executable per batch
 * width) unless disabled; results are identical either way. */
int bc_wan_step(bc_wan_ctx* ctx, const bc_batch* batch, const bc_wan_update* upd,
                int32_t* status, void* stream);
/* Work list the balanced kernel would run for bc_attention_paged's arguments
   (host logic, no device work): item words into items[0..ret), per-CTA
   offsets into start[0..*n_ctas]; item = e | head << 8 | tile << 16, plus bit
   31 = pair of tiles (tile, tile + 1), or bit 30 = cross-entry pair (the last
   tiles of entries e and bits 16-23).  Returns -1 if the grid kernel would
   run instead. */
int bc_attention_plan(const bc_batch* batch, int32_t q_per_entry, int32_t kv_tokens, int32_t heads,
                      uint32_t* items, int32_t items_cap, uint16_t* start, int32_t* n_ctas);
int bc_attention_set_balance(int on); /* 1: balanced persistent self-attention (default, or BC_ATTN_BALANCE env), 0: one CTA per query-tile pair; identical results */
int bc_wan_set_graphs(int on); /* 1: CUDA graphs (default, or BC_GRAPHS env), 0: eager launches */

/* ---- multi-GPU temporal parallelism (one process per GPU, NVLink P2P) ----
 * Every rank holds a full KV-arena replica.  Fresh K/V rows computed by a
 * rank are stored into every peer's replica (P2P stores from the q/k
 * kernel; BC_KV_PUSH=copy: side-stream cudaMemcpyAsync) and the rank publishes
 * epoch into peers' flags[layer][slot][my_rank]; attention waits (per
 * visible slot) until the flag of every producer rank in pmask is >= need
 * before its first tile of that slot; the head kernel publishes
 * iteration-done epochs, which the next iteration's first K/V write waits
 * for (no reader of a slot is overtaken).
 * Two partitions of an iteration (the caller chooses per step):
 *  - blocks: a rank runs whole entries (row1 = 0; batch = its own entries);
 *  - rows:   every rank gets the whole batch and runs the global rows
 *            [row0, row1) of the n*T concatenated rows; Y rows are exchanged
 *            (my_y / peer_y, yready flags) and every rank updates every
 *            entry's latents (replicated, so latents never move).
 * Pointers are device (IPC-mapped) addresses. */
#define BC_MAX_PEERS 8
typedef struct {
  int32_t n_peers, my_rank, n_ranks;             /* n_ranks = n_peers + 1      */
  void* peer_arena[BC_MAX_PEERS];
  uint32_t* peer_flags[BC_MAX_PEERS];            /* peers' [L][n_slots][n_ranks] */
  uint32_t* peer_done[BC_MAX_PEERS];             /* peers' [n_ranks]           */
  uint32_t* my_flags;                            /* ours, written by peers     */
  uint32_t* my_done;
  uint32_t* counters;                            /* >= 1 zeroed u32 (scratch)  */
  /* row-sharded steps only (else NULL): Y [max_entries*T][64] fp32 */
  float* my_y;
  void* peer_y[BC_MAX_PEERS];
  uint32_t* my_yready;                           /* ours [n_ranks], written by peers */
  uint32_t* peer_yready[BC_MAX_PEERS];
} bc_wan_peers;
int bc_wan_set_peers(bc_wan_ctx* ctx, const bc_wan_peers* peers);

typedef struct {
  uint32_t epoch;                                 /* iteration epoch, 1 .. 2^24-1 */
  uint32_t need[BC_MAX_ENTRIES][BC_MAX_VIS];      /* wait epoch per visible slot (0 = none) */
  uint8_t pmask[BC_MAX_ENTRIES][BC_MAX_VIS];      /* producer ranks to wait for (bit r) */
  int32_t stage;  /* -1 whole step; 0 begin; 1 layer part A; 2 part B; 3 head (+Y push); 4 update */
  int32_t layer;
  int32_t row0, row1;                             /* rows partition: global row slice; row1 = 0: blocks */
} bc_wan_dist;
int bc_wan_step_dist(bc_wan_ctx* ctx, const bc_batch* batch, const bc_wan_update* upd,
                     const bc_wan_dist* dist, int32_t* status, void* stream);
int bc_wan_signal_done(bc_wan_ctx* ctx, uint32_t epoch, void* stream);

/* Device memory that can be shared with the other ranks' processes. */
int bc_ipc_malloc(int64_t bytes, void** ptr, char handle[64]);
int bc_ipc_open(const char handle[64], void** ptr);
int bc_ipc_close(void* ptr);
int bc_free(void* ptr);
int bc_memset_async(void* ptr, int value, int64_t bytes, void* stream);
/* Stream-ordered handoff between ranks (decode GPU inbox): a device copy
 * (peer / IPC-mapped buffers allowed), and a 32-bit flag write / wait
 * (value >= `value`) executed by the stream (cuStreamWriteValue32 with a
 * memory fence / cuStreamWaitValue32). */
int bc_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
int bc_stream_write_u32(void* addr, uint32_t value, void* stream);
int bc_stream_wait_geq_u32(void* addr, uint32_t value, void* stream);

/* ---------------------------------------------------------------------------
 * Building blocks, exported for the parity tests and the multi-GPU executor.
 * ------------------------------------------------------------------------- */
/* C[M,N] (+)= epilogue(A[M,K] . B[N,K]^T + bias); bf16 in, fp32 accumulate.
 * mode 0: C bf16 = acc+bias;  1: C bf16 = gelu_tanh(acc+bias);
 * 2: C fp32 = acc+bias;       3: C fp32 += gate[row/rows_per_gate] * (acc+bias)
 * K % 64 == 0, N % 64 == 0; lda = ldb = K, ldc = N.
 * Tuning bits above the epilogue (0 = automatic): bits 8-15 force the tile
 * width in units of 64 columns (of 32 columns when bit 18 is set: 224 =
 * 7 << 8 | 1 << 18); bits 16-17 = 1 single-CTA tiles, 2 CTA-pair tiles
 * (tcgen05 cta_group::2, 256 rows; widths 256 / 224 / 192, 224 may end in a
 * ragged, masked column tile).  Results are identical for every choice
 * (fixed K order, no split-K). */
int bc_gemm_bf16(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                 int32_t mode, const float* bias, const float* gate, int32_t gate_stride,
                 int32_t rows_per_gate, void* stream);

/* The tiling bc_gemm_bf16 chooses automatically for this shape / epilogue:
 * tile width (*bn columns) and CTAs per tile (*cg: 1, or 2 = CTA pair). */
int bc_gemm_plan(int32_t M, int32_t N, int32_t K, int32_t mode, int32_t* bn, int32_t* cg);

/* Paged flash attention over KV-arena slots (self-attention) or a dense
 * K/V (cross-attention).  q: bf16 [rows][heads][128]; out: bf16 same.
 * For entry e, query rows [e*q_per_entry, (e+1)*q_per_entry) attend to the
 * concatenation of vis_slot[e][*] (each `kv_tokens` rows) in order. */
int bc_attention_paged(const void* q, const void* k_arena, const void* v_arena,
                       int64_t slot_stride_elems, int32_t kv_tokens,
                       const bc_batch* batch, int32_t q_per_entry, int32_t heads,
                       void* out, void* stream);


/* ---------------------------------------------------------------------------
 * VAE decode.  Replaces the reference's decode lane
 * (engine.py:151-158, a cost-model charge) and its linear stand-in
 * decode_block / make_decode_map (executor.py:189-212) with the public
 * Wan2.1 causal 3-D VAE decoder.  Activations are "padded frames":
 * channels-last [n_frames][H+2][W+2][C] with a zero border; frames 0-1 of a
 * causal conv input hold its history (the previous block's last two input
 * frames, zeros before the first block).  Host orchestration:
 * paper_2511_20426_b200/vae.py.
 * ------------------------------------------------------------------------- */
#define BC_VAE_MAX_FRAMES 16

typedef struct {
  const void* in;      /* bf16 padded frames [n_frames][H+2][W+2][cin]          */
  const void* w;       /* bf16 [cout][kt*kh*kw][cin] (tap-major, K-contiguous)  */
  const float* bias;   /* fp32 [cout]                                           */
  int32_t H, W;        /* valid extent                                          */
  int32_t n_frames;    /* frames in the input / output buffers                  */
  int32_t frame0;      /* first output frame (>= kt-1: causal taps read frame0-2..frame0) */
  int32_t n_out_frames;
  int32_t cin, cout;   /* cin % 32 == 0, cout % 16 == 0                         */
  int32_t kt, kh, kw;  /* 3x3x3, 1x3x3, 3x1x1 or 1x1x1                           */
  const float* res;    /* optional fp32 residual, same layout as out32          */
  float* out32;        /* optional fp32 y = conv + bias (+ res), padded frames  */
  void* out16;         /* optional bf16 y                                       */
  void* act;           /* optional bf16 silu?(RMS_norm(y) * gamma): the next conv's input */
  const float* gamma;  /* fp32 [cout] for act                                   */
  int32_t act_silu;    /* 1: silu(norm), 0: norm only (attention block input)   */
  float* video;        /* optional fp32 [frames][video_channels][H][W], clamped to [-1,1] */
  int32_t video_channels, video_frame0;
} bc_vae_conv_args;

/* Output frame j of an upsample reads source (src[j] ? b : a) frame frame[j]
 * at channel offset chan[j] (b has 2C channels: the time conv's two halves). */
typedef struct {
  int32_t src[BC_VAE_MAX_FRAMES];
  int32_t frame[BC_VAE_MAX_FRAMES];
  int32_t chan[BC_VAE_MAX_FRAMES];
} bc_vae_frame_map;

/* Causal conv as a tcgen05 implicit GEMM with fused bias / residual / RMS
 * norm + SiLU / clamp epilogues (CausalConv3d, Conv2d of Resample, the 1x1
 * shortcut and to_qkv of the Wan2.1 decoder). */
int bc_vae_conv(const bc_vae_conv_args* args /*[host]*/, void* stream);
/* z [T][zc][H][W] fp32 -> z*std+mean -> 1x1x1 conv (WanVAE_.conv2) -> bf16
 * padded frames [frame0+t] with cpad channels (zc..cpad-1 left as they are). */
int bc_vae_prep(const float* z, const float* w2, const float* b2, const float* mean, const float* stdv,
                void* out, int32_t T, int32_t zc, int32_t H, int32_t W, int32_t frame0, int32_t cpad,
                void* stream);
/* nearest-exact x2 (Resample) of fp32 padded frames into bf16 padded frames
 * [out_frame0 + j] of the next level (2H x 2W). */
int bc_vae_upsample(const float* a, const float* b, const bc_vae_frame_map* map /*[host]*/, int32_t C,
                    int32_t H, int32_t W, void* out, int32_t out_frame0, int32_t n_out, void* stream);
/* AttentionBlock helpers (one frame): q, k [np][C], v^T [C][np] from the
 * padded qkv rows; row softmax of S [rows][np] over n_valid columns; and the
 * residual x += proj followed by the next conv's silu(RMS_norm(x) * gamma). */
int bc_vae_attn_gather(const void* qkv, int32_t frame, int32_t H, int32_t W, int32_t C, int32_t np,
                       void* q, void* k, void* vt, void* stream);
int bc_vae_softmax(const float* S, void* P, int32_t rows, int32_t np, int32_t n_valid, float scale,
                   void* stream);
/* silu?(RMS_norm(x) * gamma) of fp32 padded frames [frame0, frame0+n) into
 * bf16 -- the next conv's input when a conv's rows do not fit one unit. */
int bc_vae_norm_act(const float* x, const float* gamma, void* act, int32_t frame0, int32_t n_frames,
                    int32_t H, int32_t W, int32_t C, int32_t use_silu, void* stream);
int bc_vae_attn_out(float* x, const float* proj, const float* gamma, void* act, int32_t frame, int32_t H,
                    int32_t W, int32_t C, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BCB200_H_ */
