// Wan2.1-shaped DiT runtime: one cascade iteration = one bc_wan_step call.
//
// The host scheduler hands over the batch (one entry per in-flight block,
// ascending) with each entry's KV-arena slot and visible-slot list; this
// file launches the whole batched forward on one stream:
//
//   patchify -> patch GEMM -> time MLP -> per layer {
//     LN+AdaLN -> QKV GEMM -> q/k RMSNorm+RoPE (K/V -> own slot) ->
//     paged self-attention over visible slots -> O GEMM (+gate*res) ->
//     affine LN -> cross-q GEMM -> RMSNorm -> cross-attention (text K/V) ->
//     cross-O GEMM (+res) -> LN+AdaLN -> FFN1 GEMM (+GELU) -> FFN2 GEMM (+gate*res) }
//   -> head LN+mod -> head GEMM -> unpatchify + flow->x0 + renoise/emit.
//
// Entries of all cascade levels run through the same GEMMs (rows are
// concatenated); only the per-entry modulation vectors and the attention
// slot tables differ.  Memory: caller-owned (torch) weights, KV arena
// [L][n_slots][2][T][d] bf16 and workspace; nothing is allocated here.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "attention.h"
#include "bc_common.h"
#include "gemm.h"
#include "wan_kernels.h"

struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

struct bc_wan_ctx {
  bc_wan_dims dims;
  bc_wan_params prm;
  __nv_bfloat16* arena;
  int d, T, R, E;
  // workspace carve-outs
  float* X;
  __nv_bfloat16 *xn, *qkv, *Q, *attn, *H1, *patches;
  float* Y;
  float *t_h, *t_e, *t_es, *t_e0, *mod_all;
  __nv_bfloat16 *text_in, *text_h, *ctx, *text_tmp, *textkv;
  float2 *rope_f, *rope_h, *rope_w;
  bool text_ready, rope_ready;
  std::vector<std::string> layer_names;  // NVTX range names "layer N"
  // CUDA graphs of the single-GPU step, one executable per batch width
  // (the kernel sequence -- incl. the GEMM tile variants -- depends on it);
  // each step is re-captured and its parameters pushed with
  // cudaGraphExecUpdate, so the ~400 launches reach the GPU as one graph
  cudaGraphExec_t graph_exec[BC_MAX_ENTRIES + 1] = {};
  bool width_seen[BC_MAX_ENTRIES + 1] = {};
  cudaStream_t gstream = nullptr;  // capture / launch stream (the caller's may be the legacy stream)
  bool graphs_broken = false;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  bc_wan_peers peers;
  // BC_KV_PUSH=copy: side-stream push of fresh K/V to the peers' replicas
  bool push_by_copy;
  cudaStream_t side;
  cudaEvent_t ev_qk, ev_side;
  struct StepState {
    bc_batch batch;
    bc_wan_update upd;
    int32_t* status;
    uint32_t epoch;
    int n, R;       // entries; rows of this launch (local slice of the batch's n*T rows)
    int row0;       // global batch row of local row 0
    bool rows_mode; // row-sharded multi-GPU step: Y rows are exchanged, every rank updates all latents
    double self_flops;
    bc::AttnArgs sa, ca;
    bc::QkArgs qa;
  } step;
};
using StepState = bc_wan_ctx::StepState;

namespace {

struct Carver {
  char* base;
  int64_t off = 0;
  template <typename T>
  T* take(int64_t count) {
    off = (off + 255) & ~int64_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * (int64_t)sizeof(T);
    return p;
  }
};

int64_t carve(bc_wan_ctx* c, const bc_wan_dims& dm, char* base) {
  Carver cv{base};
  const int64_t d = (int64_t)dm.heads * dm.head_dim;
  const int64_t T = (int64_t)dm.block_size * (dm.latent_h / 2) * (dm.latent_w / 2);
  const int64_t E = dm.max_entries;
  const int64_t R = E * T;
  bc_wan_ctx tmp;
  bc_wan_ctx* t = c ? c : &tmp;
  t->X = cv.take<float>(R * d);
  t->xn = cv.take<__nv_bfloat16>(R * d);
  t->qkv = cv.take<__nv_bfloat16>(R * 3 * d);
  t->Q = cv.take<__nv_bfloat16>(R * d);
  t->attn = cv.take<__nv_bfloat16>(R * d);
  t->H1 = cv.take<__nv_bfloat16>(R * dm.ffn_dim);
  t->patches = cv.take<__nv_bfloat16>(R * 64);
  t->Y = cv.take<float>(R * 64);
  t->t_h = cv.take<float>(E * d);
  t->t_e = cv.take<float>(E * d);
  t->t_es = cv.take<float>(E * d);
  t->t_e0 = cv.take<float>(E * 6 * d);
  t->mod_all = cv.take<float>((int64_t)dm.layers * E * 6 * d);
  t->text_in = cv.take<__nv_bfloat16>((int64_t)dm.text_len * dm.text_dim);
  t->text_h = cv.take<__nv_bfloat16>((int64_t)dm.text_len * d);
  t->ctx = cv.take<__nv_bfloat16>((int64_t)dm.text_len * d);
  t->text_tmp = cv.take<__nv_bfloat16>((int64_t)dm.text_len * 2 * d);
  t->textkv = cv.take<__nv_bfloat16>((int64_t)dm.layers * 2 * dm.text_len * d);
  t->rope_f = cv.take<float2>((int64_t)bc::kRopeMaxFrames * 22);
  t->rope_h = cv.take<float2>((int64_t)(dm.latent_h / 2) * 21);
  t->rope_w = cv.take<float2>((int64_t)(dm.latent_w / 2) * 21);
  return cv.off + 256;
}

int check_dims(const bc_wan_dims& dm) {
  if (dm.head_dim != 128) return bc_fail(BC_ERR_CONTRACT, "wan: head_dim must be 128");
  const int d = dm.heads * dm.head_dim;
  if (d % 256 || dm.ffn_dim % 256 || dm.text_dim % 64 || dm.freq_dim % 2)
    return bc_fail(BC_ERR_CONTRACT, "wan: dims must be multiples of 256 (d, ffn) / 64 (text_dim)");
  if (dm.latent_h % 2 || dm.latent_w % 2 || dm.block_size < 1 || dm.layers < 1)
    return bc_fail(BC_ERR_CONTRACT, "wan: bad latent geometry");
  if (dm.max_entries < 1 || dm.max_entries > BC_MAX_ENTRIES || dm.n_slots < 1)
    return bc_fail(BC_ERR_CONTRACT, "wan: bad max_entries / n_slots");
  return BC_OK;
}

#define RC(x)              \
  do {                     \
    int _rc = (x);         \
    if (_rc) return _rc;   \
  } while (0)

int gemm(const void* A, const void* B, void* C, int M, int N, int K, int mode, const float* bias,
         const float* gate, int gate_stride, int rows_per_gate, cudaStream_t st, int gate_row0 = 0) {
  if (M == 0) return BC_OK;  // empty row slice (row-sharded multi-GPU step)
  bc::GemmArgs g{A, B, C, M, N, K, mode, bias, gate, gate_stride, rows_per_gate, 0, 0, gate_row0};
  return bc::gemm_run(g, st);
}

// ---- optional per-kernel-class timing with CUDA events on the launch stream
enum ProfClass { kSelfAttn = 0, kCrossAttn = 1, kGemm = 2, kBandwidth = 3, kNumProf = 4 };
struct ProfRec {
  cudaEvent_t a, b;
  int cls;
  double flops, bytes;
};
bool g_prof = false;
int g_graphs = -1;  // -1: BC_GRAPHS env (default on)
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_free_events;

cudaEvent_t ev_get() {
  if (!g_free_events.empty()) {
    cudaEvent_t e = g_free_events.back();
    g_free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

template <class F>
int timed(int cls, double flops, double bytes, cudaStream_t st, F&& f) {
  if (!g_prof) return f();
  cudaEvent_t a = ev_get(), b = ev_get();
  cudaEventRecord(a, st);
  const int rc = f();
  cudaEventRecord(b, st);
  g_recs.push_back({a, b, cls, flops, bytes});
  return rc;
}

PFN_cuStreamWaitValue32_v11070 wait_value32() {
  static const PFN_cuStreamWaitValue32_v11070 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    return (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p)
               : nullptr;
  }();
  return fn;
}

PFN_cuStreamWriteValue32_v11070 write_value32() {
  static const PFN_cuStreamWriteValue32_v11070 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    return (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p)
               : nullptr;
  }();
  return fn;
}

// Publish `v` into (peer) flag words in stream order.  cuStreamWriteValue32
// (a memory barrier, then the write, executed by the stream itself) is the
// default; if the driver rejects a peer address the writes go through a
// 1-thread kernel (system fence + release stores) from then on -- never
// lost, only a launch more per publication.
std::atomic<int> g_memops_ok{getenv("BC_NO_MEMOP_WRITES") ? 0 : 1};  // env: force the kernel path (tests)
int write_flags(cudaStream_t st, const bc::FlagWrites& f) {
  if (f.n <= 0) return BC_OK;
  if (g_memops_ok.load(std::memory_order_relaxed)) {
    auto wv = write_value32();
    int done = 0;
    if (wv) {
      for (; done < f.n; ++done)
        if (wv((CUstream)st, (CUdeviceptr)f.addr[done], f.v, 0) != CUDA_SUCCESS) break;
    }
    if (done == f.n) return BC_OK;
    (void)cudaGetLastError();
    g_memops_ok.store(0);
  }
  return bc::launch_flag_writes(f, st);
}

template <typename T>
const T* at(const void* base, int64_t elems) {
  return static_cast<const T*>(base) + elems;
}

}  // namespace

// Launch single-GPU steps as CUDA graphs (1, default) or eagerly (0).
extern "C" int bc_wan_set_graphs(int on) {
  g_graphs = on ? 1 : 0;
  return BC_OK;
}

extern "C" int bc_profile_enable(int on) {
  g_prof = on != 0;
  return BC_OK;
}

// Sums (ms, algorithmic flops, algorithmic bytes, launches) per class since
// the last collect: 0 self-attention, 1 cross-attention, 2 GEMM, 3 others.
extern "C" int bc_profile_collect(double* ms, double* flops, double* bytes, int64_t* count, int n_cls) {
  for (int i = 0; i < n_cls; ++i) ms[i] = flops[i] = bytes[i] = 0.0, count[i] = 0;
  for (auto& r : g_recs) {
    BC_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    BC_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    if (r.cls < n_cls) {
      ms[r.cls] += t;
      flops[r.cls] += r.flops;
      bytes[r.cls] += r.bytes;
      count[r.cls] += 1;
    }
    g_free_events.push_back(r.a);
    g_free_events.push_back(r.b);
  }
  g_recs.clear();
  return BC_OK;
}

extern "C" int64_t bc_wan_workspace_bytes(const bc_wan_dims* dims) {
  if (!dims || check_dims(*dims)) return -1;
  return carve(nullptr, *dims, nullptr);
}

extern "C" int bc_wan_create(const bc_wan_dims* dims, const bc_wan_params* params, void* kv_arena,
                             void* workspace, int64_t workspace_bytes, bc_wan_ctx** out) {
  if (!dims || !params || !kv_arena || !workspace || !out)
    return bc_fail(BC_ERR_CONTRACT, "bc_wan_create: null argument");
  RC(check_dims(*dims));
  const int64_t need = carve(nullptr, *dims, nullptr);
  if (workspace_bytes < need)
    return bc_fail(BC_ERR_CONTRACT, "bc_wan_create: workspace %lld < %lld bytes", (long long)workspace_bytes,
                   (long long)need);
  bc_wan_ctx* c = new (std::nothrow) bc_wan_ctx();
  if (!c) return bc_fail(BC_ERR_CUDA, "bc_wan_create: out of host memory");
  c->dims = *dims;
  c->prm = *params;
  c->arena = static_cast<__nv_bfloat16*>(kv_arena);
  c->d = dims->heads * dims->head_dim;
  c->T = dims->block_size * (dims->latent_h / 2) * (dims->latent_w / 2);
  c->E = dims->max_entries;
  c->R = c->E * c->T;
  carve(c, *dims, static_cast<char*>(workspace));
  c->text_ready = false;
  for (int l = 0; l < dims->layers; ++l) c->layer_names.push_back("layer " + std::to_string(l));
  *out = c;
  return BC_OK;
}

extern "C" int bc_wan_destroy(bc_wan_ctx* ctx) {
  if (ctx) {
    for (auto& ex : ctx->graph_exec)
      if (ex) {
        cudaGraphExecDestroy(ex);
        ex = nullptr;
      }
    if (ctx->gstream) {
      cudaStreamSynchronize(ctx->gstream);
      cudaStreamDestroy(ctx->gstream);
      cudaEventDestroy(ctx->gev_in);
      cudaEventDestroy(ctx->gev_out);
    }
  }
  if (ctx && ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->ev_qk);
    cudaEventDestroy(ctx->ev_side);
  }
  delete ctx;
  return BC_OK;
}

// Text encoder MLP (Linear(text_dim,d) -> GELU(tanh) -> Linear(d,d)) and the
// per-layer cross-attention K = RMSNorm(ctx Wk + bk) * w, V = ctx Wv + bv.
extern "C" int bc_wan_set_text(bc_wan_ctx* c, const float* states, void* stream) {
  if (!c || !states) return bc_fail(BC_ERR_CONTRACT, "bc_wan_set_text: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const bc_wan_dims& dm = c->dims;
  const bc_wan_params& p = c->prm;
  const int d = c->d, Lt = dm.text_len;
  if (!c->rope_ready) {
    RC(bc::launch_rope_tables(c->rope_f, bc::kRopeMaxFrames, c->rope_h, dm.latent_h / 2, c->rope_w, dm.latent_w / 2, st));
    c->rope_ready = true;
  }
  RC(bc::launch_f32_to_bf16(states, c->text_in, (int64_t)Lt * dm.text_dim, st));
  RC(gemm(c->text_in, p.text_w1, c->text_h, Lt, d, dm.text_dim, bc::kEpiGeluBf16, p.text_b1, nullptr, 0, 1, st));
  RC(gemm(c->text_h, p.text_w2, c->ctx, Lt, d, d, bc::kEpiStoreBf16, p.text_b2, nullptr, 0, 1, st));
  for (int l = 0; l < dm.layers; ++l) {
    RC(gemm(c->ctx, at<__nv_bfloat16>(p.ckv_w, (int64_t)l * 2 * d * d), c->text_tmp, Lt, 2 * d, d,
            bc::kEpiStoreBf16, p.ckv_b + (size_t)l * 2 * d, nullptr, 0, 1, st));
    __nv_bfloat16* kdst = c->textkv + (size_t)l * 2 * Lt * d;
    RC(bc::launch_rms_rows(c->text_tmp, Lt, d, 2 * d, p.cnorm_k + (size_t)l * d, kdst, d, st));
    RC(bc::launch_copy_cols(c->text_tmp, 2 * d, d, kdst + (size_t)Lt * d, d, Lt, d, st));
  }
  c->text_ready = true;
  return BC_OK;
}

// ---------------------------------------------------------------- stepping
namespace {

int validate_step(const bc_wan_ctx* c, const bc_batch* batch, const bc_wan_update* upd) {
  const bc_wan_dims& dm = c->dims;
  const int n = batch->n_entries;
  if (n < 1 || n > c->E) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: %d entries (max %d)", n, c->E);
  if (batch->block_size != dm.block_size) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: block size mismatch");
  for (int e = 0; e < n; ++e) {
    if (batch->slot[e] < 0 || batch->slot[e] >= dm.n_slots || batch->n_vis[e] < 1 || batch->n_vis[e] > BC_MAX_VIS)
      return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: bad slot table (entry %d)", e);
    for (int v = 0; v < batch->n_vis[e]; ++v)
      if (batch->vis_slot[e][v] < 0 || batch->vis_slot[e][v] >= dm.n_slots)
        return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: visible slot out of range");
    if (!(batch->level[e] >= 0.0 && batch->level[e] <= 1000.0) || !upd->latents[e])
      return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: bad level / latents (entry %d)", e);
    if (upd->post[e] == 0 && (!upd->eps[e] || !(upd->next_level[e] >= 0.0 && upd->next_level[e] <= 1000.0)))
      return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: renoise entry %d needs eps and a level", e);
    if ((upd->post[e] == 1 || upd->post[e] == 3) && !upd->out[e])
      return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: entry %d needs an output buffer", e);
  }
  return BC_OK;
}

bc::PeerArgs peer_args(const bc_wan_ctx* c, uint32_t epoch) {
  bc::PeerArgs pa{};
  pa.n_peers = c->peers.n_peers;
  for (int p = 0; p < pa.n_peers; ++p) {
    pa.arena[p] = static_cast<__nv_bfloat16*>(c->peers.peer_arena[p]);
    pa.flags[p] = c->peers.peer_flags[p];
    pa.done[p] = c->peers.peer_done[p];
  }
  pa.my_done = c->peers.my_done;
  pa.my_rank = c->peers.my_rank;
  pa.n_ranks = c->peers.n_ranks;
  pa.epoch = epoch;
  pa.ctr = c->peers.counters;
  return pa;
}

// stage 0: validation, patch embedding, time MLP, per-step argument blocks
int stage_begin(bc_wan_ctx* c, const bc_batch* batch, const bc_wan_update* upd, const bc_wan_dist* dist,
                int32_t* status, cudaStream_t st) {
  RC(validate_step(c, batch, upd));
  StepState& S = c->step;
  S.batch = *batch;
  S.upd = *upd;
  S.status = status;
  S.epoch = dist ? dist->epoch : 0u;
  const bc_wan_dims& dm = c->dims;
  const bc_wan_params& p = c->prm;
  const int n = batch->n_entries;
  const int d = c->d, T = c->T, L = dm.layers, F = dm.block_size;
  const int H = dm.latent_h, W = dm.latent_w;
  const bool multi = c->peers.n_peers > 0 && dist;
  // row-sharded step: this rank runs global rows [row0, row1) of the n*T
  // concatenated rows (every entry of the iteration, a slice of its tokens)
  S.rows_mode = multi && dist->row1 > 0;
  S.row0 = S.rows_mode ? dist->row0 : 0;
  const int row1 = S.rows_mode ? dist->row1 : n * T;
  if (S.row0 < 0 || row1 > n * T || row1 < S.row0)
    return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: bad row slice [%d, %d) of %d rows", S.row0, row1, n * T);
  if (S.rows_mode && (!c->peers.my_y || !c->peers.my_yready))
    return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: row-sharded steps need shared Y buffers (bc_wan_peers.my_y)");
  const int R = row1 - S.row0;
  S.n = n;
  S.R = R;

  bc::EntryPtrs lat{};
  for (int e = 0; e < n; ++e) {
    lat.p[e] = upd->latents[e];
    lat.block[e] = batch->block_index[e];
  }
  // the finiteness check of the inputs rides on patchify when this rank's
  // rows cover the whole batch; a row slice checks every latent separately
  const bool whole = S.row0 == 0 && R == n * T;
  if (!whole)
    RC(timed(kBandwidth, 0.0, 4.0 * n * F * 16 * H * W, st, [&] { return bc::launch_check_finite(lat, n, F * 16 * H * W, status, st); }));
  if (R > 0)
    RC(timed(kBandwidth, 0.0, 6.0 * R * 64, st, [&] { return bc::launch_patchify(lat, F, H, W, S.row0, R, c->patches, whole ? status : nullptr, st); }));
  RC(timed(kGemm, 2.0 * R * d * 64, 0.0, st, [&] { return gemm(c->patches, p.patch_w, c->X, R, d, 64, bc::kEpiStoreF32, p.patch_b, nullptr, 0, 1, st); }));

  // time embedding: e = W2 silu(W1 sin(t) + b1) + b2 ; e0 = Wp silu(e) + bp
  bc::TimeArgs ta{};
  for (int e = 0; e < n; ++e) ta.t[e] = batch->level[e];
  // (three launches: the sinusoid is computed inside the first GEMV, the
  // per-layer AdaLN tables are written by the last)
  RC(bc::launch_gemv(nullptr, n, dm.freq_dim, static_cast<const __nv_bfloat16*>(p.time_w1), p.time_b1, c->t_h, d,
                     1, nullptr, st, &ta));
  RC(bc::launch_gemv(c->t_h, n, d, static_cast<const __nv_bfloat16*>(p.time_w2), p.time_b2, c->t_e, d, 2, c->t_es,
                     st));
  RC(bc::launch_gemv(c->t_es, n, d, static_cast<const __nv_bfloat16*>(p.tproj_w), p.tproj_b, c->t_e0, 6 * d, 0,
                     nullptr, st, nullptr, p.modulation, L, c->mod_all));

  bc::AttnArgs& sa = S.sa;
  sa = bc::AttnArgs{};
  sa.kv_base = c->arena;
  sa.n_mats = L * dm.n_slots * 2;
  sa.n_entries = n;
  sa.q_tokens = T;
  sa.kv_tokens = T;
  sa.heads = dm.heads;
  sa.head_dim = 128;
  sa.mat_stride = 2;
  sa.v_offset = 1;
  sa.scale = 0.08838834764831845f;  // 1/sqrt(128)
  sa.q = c->Q;
  sa.out = c->attn;
  sa.flags = multi ? c->peers.my_flags : nullptr;
  sa.n_ranks = multi ? c->peers.n_ranks : 1;
  sa.ranged = 1;
  sa.q_rows = R;
  sa.balance = 1;  // persistent balanced kernel (peer-flag waits per item)
  for (int e = 0; e < n; ++e) {
    sa.n_vis[e] = batch->n_vis[e];
    for (int v = 0; v < batch->n_vis[e]; ++v) {
      sa.vis_slot[e][v] = batch->vis_slot[e][v];
      // packed wait word: epoch << 8 | producer-rank mask (0 = no wait)
      const uint32_t ep = multi ? dist->need[e][v] : 0u, pm = multi ? dist->pmask[e][v] : 0u;
      if (ep >= (1u << 24)) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: epoch overflow");
      sa.need[e][v] = (ep && pm) ? (ep << 8) | pm : 0u;
    }
    const int lo = S.row0 - e * T > 0 ? S.row0 - e * T : 0;
    const int hi = row1 - e * T < T ? row1 - e * T : T;
    sa.q_lo[e] = hi > lo ? lo : 0;
    sa.q_hi[e] = hi > lo ? hi : 0;
    sa.q_row[e] = hi > lo ? e * T + lo - S.row0 : 0;
  }
  bc::AttnArgs& ca = S.ca;
  ca = sa;
  ca.kv_base = c->textkv;
  ca.n_mats = L * 2;
  ca.kv_tokens = dm.text_len;
  ca.flags = nullptr;
  for (int e = 0; e < n; ++e) {
    ca.n_vis[e] = 1;
    ca.vis_slot[e][0] = 0;
  }
  bc::QkArgs& qa = S.qa;
  qa = bc::QkArgs{};
  qa.qout = c->Q;
  qa.arena = c->arena;
  qa.hp = H / 2;
  qa.wp = W / 2;
  qa.rope_f = c->rope_f;
  qa.rope_h = c->rope_h;
  qa.rope_w = c->rope_w;
  qa.row0 = S.row0;
  for (int e = 0; e < n; ++e) {
    qa.slot[e] = batch->slot[e];
    qa.frame0[e] = batch->block_index[e] * F;
    if ((batch->block_index[e] + 1) * F > bc::kRopeMaxFrames)
      return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: frame index beyond the RoPE table (%d)", bc::kRopeMaxFrames);
  }
  if (multi) qa.peer = peer_args(c, S.epoch);
  S.self_flops = 0.0;
  for (int e = 0; e < n; ++e)
    S.self_flops += 4.0 * (sa.q_hi[e] - sa.q_lo[e]) * ((double)batch->n_vis[e] * T) * d;
  return BC_OK;
}

// stage 1: LN+AdaLN -> QKV GEMM -> q/k RMSNorm + RoPE, K/V into the own slot
// (and pushed to every peer replica in multi-GPU mode)
int stage_layer_a(bc_wan_ctx* c, int l, cudaStream_t st) {
  StepState& S = c->step;
  const bc_wan_dims& dm = c->dims;
  const bc_wan_params& p = c->prm;
  const int d = c->d, T = c->T, R = S.R, n = S.n;
  const float* mod = c->mod_all + (size_t)l * n * 6 * d;  // [e][6][d]
  bc::QkArgs& qa = S.qa;
  qa.mat_base = (int64_t)l * dm.n_slots * 2;
  qa.norm_q = p.norm_q + (size_t)l * d;
  qa.norm_k = p.norm_k + (size_t)l * d;
  qa.peer.flag_base = l * dm.n_slots;
  // the first K/V write of an iteration waits until every peer finished
  // reading the previous iteration's KV (slot reuse / in-place rewrite)
  qa.peer.wait_done = (l == 0 && S.epoch > 1) ? S.epoch - 1 : 0u;
  qa.peer.push = (c->peers.n_peers > 0 && !c->push_by_copy) ? 1 : 0;
  if (R > 0) {
    bc::LnArgs ln{0, nullptr, nullptr, mod + 0 * d, mod + 1 * d, 6 * d, S.row0};
    RC(timed(kBandwidth, 0.0, 6.0 * R * d, st, [&] { return bc::launch_ln_rows(c->X, c->xn, R, d, T, ln, st); }));
    RC(timed(kGemm, 2.0 * R * 3.0 * d * d, 0.0, st, [&] { return gemm(c->xn, at<__nv_bfloat16>(p.qkv_w, (int64_t)l * 3 * d * d), c->qkv, R, 3 * d, d, bc::kEpiStoreBf16,
            p.qkv_b + (size_t)l * 3 * d, nullptr, 0, 1, st); }));
    RC(timed(kBandwidth, 0.0, 12.0 * R * d, st, [&] { return bc::launch_qk_norm_rope(c->qkv, R, d, T, qa, st); }));
  }
  if (c->peers.n_peers > 0 && c->push_by_copy && S.epoch > 0) {
    // (BC_KV_PUSH=copy) cudaMemcpyAsync moves this rank's fresh K/V rows of
    // layer l (per entry: the token range it computed, K and V halves of the
    // slot's [2][T][d] matrix) into every peer replica, then a stream memory
    // op publishes flags[layer][slot][my_rank] = epoch.  Safe only when the
    // copy runs on a copy engine (see bc_wan_set_peers).
    BC_CUDA(cudaEventRecord(c->ev_qk, st));
    BC_CUDA(cudaStreamWaitEvent(c->side, c->ev_qk, 0));
    const size_t row_bytes = (size_t)d * sizeof(__nv_bfloat16);
    const size_t mat_bytes = (size_t)T * row_bytes;
    int e_used[BC_MAX_ENTRIES];
    int n_used = 0;
    for (int e = 0; e < n; ++e) {
      const int lo = S.sa.q_lo[e], hi = S.sa.q_hi[e];
      if (hi <= lo) continue;
      e_used[n_used++] = e;
      const size_t off = ((size_t)qa.mat_base + (size_t)S.batch.slot[e] * 2) * mat_bytes;
      for (int pp = 0; pp < c->peers.n_peers; ++pp) {
        char* dst = static_cast<char*>(c->peers.peer_arena[pp]) + off;
        const char* src = reinterpret_cast<const char*>(c->arena) + off;
        if (lo == 0 && hi == T) {  // the whole block: one [2][T][d] copy
          BC_CUDA(cudaMemcpyAsync(dst, src, 2 * mat_bytes, cudaMemcpyDeviceToDevice, c->side));
        } else {                   // a token range: K rows and V rows
          const size_t r0 = (size_t)lo * row_bytes, nb = (size_t)(hi - lo) * row_bytes;
          BC_CUDA(cudaMemcpyAsync(dst + r0, src + r0, nb, cudaMemcpyDeviceToDevice, c->side));
          BC_CUDA(cudaMemcpyAsync(dst + mat_bytes + r0, src + mat_bytes + r0, nb, cudaMemcpyDeviceToDevice,
                                  c->side));
        }
      }
    }
    bc::FlagWrites fw{};
    fw.v = S.epoch;
    for (int pp = 0; pp < c->peers.n_peers; ++pp)
      for (int k = 0; k < n_used && fw.n < bc::kMaxFlagWrites; ++k) {
        const size_t fi = ((size_t)l * dm.n_slots + S.batch.slot[e_used[k]]) * c->peers.n_ranks + c->peers.my_rank;
        fw.addr[fw.n++] = c->peers.peer_flags[pp] + fi;
      }
    RC(write_flags(c->side, fw));
  }
  return BC_OK;
}

// stage 2: self-attention -> O GEMM (+gate) -> cross-attention -> FFN
int stage_layer_b(bc_wan_ctx* c, int l, cudaStream_t st) {
  StepState& S = c->step;
  const bc_wan_dims& dm = c->dims;
  const bc_wan_params& p = c->prm;
  const int d = c->d, T = c->T, R = S.R, n = S.n, r0 = S.row0;
  if (R == 0) return BC_OK;
  const float* mod = c->mod_all + (size_t)l * n * 6 * d;
  S.sa.mat_base = l * dm.n_slots * 2;
  S.sa.flag_base = l * dm.n_slots;
  RC(timed(kSelfAttn, S.self_flops, 0.0, st, [&] { return bc::attention_run(S.sa, st); }));
  RC(timed(kGemm, 2.0 * R * d * d, 0.0, st, [&] { return gemm(c->attn, at<__nv_bfloat16>(p.o_w, (int64_t)l * d * d), c->X, R, d, d, bc::kEpiResidualF32,
          p.o_b + (size_t)l * d, mod + 2 * d, 6 * d, T, st, r0); }));
  bc::LnArgs ln3{1, p.norm3_b + (size_t)l * d, p.norm3_w + (size_t)l * d, nullptr, nullptr, 0, r0};
  RC(timed(kBandwidth, 0.0, 6.0 * R * d, st, [&] { return bc::launch_ln_rows(c->X, c->xn, R, d, T, ln3, st); }));
  RC(timed(kGemm, 2.0 * R * d * d, 0.0, st, [&] { return gemm(c->xn, at<__nv_bfloat16>(p.cq_w, (int64_t)l * d * d), c->Q, R, d, d, bc::kEpiStoreBf16,
          p.cq_b + (size_t)l * d, nullptr, 0, 1, st); }));
  RC(timed(kBandwidth, 0.0, 4.0 * R * d, st, [&] { return bc::launch_rms_rows(c->Q, R, d, d, p.cnorm_q + (size_t)l * d, c->Q, d, st); }));
  S.ca.mat_base = l * 2;
  RC(timed(kCrossAttn, 4.0 * R * (double)dm.text_len * d, 0.0, st, [&] { return bc::attention_run(S.ca, st); }));
  RC(timed(kGemm, 2.0 * R * d * d, 0.0, st, [&] { return gemm(c->attn, at<__nv_bfloat16>(p.co_w, (int64_t)l * d * d), c->X, R, d, d, bc::kEpiResidualF32,
          p.co_b + (size_t)l * d, nullptr, 0, 1, st); }));
  bc::LnArgs ln2{0, nullptr, nullptr, mod + 3 * d, mod + 4 * d, 6 * d, r0};
  RC(timed(kBandwidth, 0.0, 6.0 * R * d, st, [&] { return bc::launch_ln_rows(c->X, c->xn, R, d, T, ln2, st); }));
  RC(timed(kGemm, 2.0 * R * (double)dm.ffn_dim * d, 0.0, st, [&] { return gemm(c->xn, at<__nv_bfloat16>(p.ffn1_w, (int64_t)l * dm.ffn_dim * d), c->H1, R, dm.ffn_dim, d,
          bc::kEpiGeluBf16, p.ffn1_b + (size_t)l * dm.ffn_dim, nullptr, 0, 1, st); }));
  RC(timed(kGemm, 2.0 * R * (double)dm.ffn_dim * d, 0.0, st, [&] { return gemm(c->H1, at<__nv_bfloat16>(p.ffn2_w, (int64_t)l * d * dm.ffn_dim), c->X, R, d, dm.ffn_dim,
          bc::kEpiResidualF32, p.ffn2_b + (size_t)l * d, mod + 5 * d, 6 * d, T, st, r0); }));
  return BC_OK;
}

// stage 3: head LN + modulation -> head GEMM (this rank's rows of Y); a
// row-sharded step pushes its Y rows into every peer's Y and publishes
// yready[my_rank] = epoch there
int stage_head(bc_wan_ctx* c, cudaStream_t st) {
  StepState& S = c->step;
  const bc_wan_params& p = c->prm;
  const int d = c->d, T = c->T, R = S.R;
  float* y = c->Y + (size_t)S.row0 * 64;
  if (R > 0) {
    bc::LnArgs lh{0, p.head_mod, p.head_mod + d, c->t_e, c->t_e, d, S.row0};
    RC(timed(kBandwidth, 0.0, 6.0 * R * d, st, [&] { return bc::launch_ln_rows(c->X, c->xn, R, d, T, lh, st); }));
    RC(timed(kGemm, 2.0 * R * 64.0 * d, 0.0, st, [&] { return gemm(c->xn, p.head_w, y, R, 64, d, bc::kEpiStoreF32, p.head_b, nullptr, 0, 1, st); }));
  }
  if (S.rows_mode) {
    BC_CUDA(cudaEventRecord(c->ev_qk, st));
    BC_CUDA(cudaStreamWaitEvent(c->side, c->ev_qk, 0));
    bc::FlagWrites fw{};
    fw.v = S.epoch;
    for (int pp = 0; pp < c->peers.n_peers; ++pp) {
      if (R > 0)
        BC_CUDA(cudaMemcpyAsync(static_cast<float*>(c->peers.peer_y[pp]) + (size_t)S.row0 * 64, y,
                                (size_t)R * 64 * sizeof(float), cudaMemcpyDeviceToDevice, c->side));
      if (fw.n < bc::kMaxFlagWrites) fw.addr[fw.n++] = c->peers.peer_yready[pp] + c->peers.my_rank;
    }
    RC(write_flags(c->side, fw));
  }
  return BC_OK;
}

// stage 4: unpatchify + x0 + renoise/emit of every entry of this launch (a
// row-sharded step first waits for every peer's Y rows: each rank then
// updates ALL latents identically, so latents never move between GPUs)
int stage_update(bc_wan_ctx* c, cudaStream_t st) {
  StepState& S = c->step;
  const bc_wan_dims& dm = c->dims;
  const int T = c->T, n = S.n, F = dm.block_size;
  if (S.rows_mode) {
    auto wt = wait_value32();
    if (!wt) return bc_fail(BC_ERR_CUDA, "cuStreamWaitValue32 unavailable");
    for (int r = 0; r < c->peers.n_ranks; ++r) {
      if (r == c->peers.my_rank) continue;
      CUresult rr = wt((CUstream)st, (CUdeviceptr)(c->peers.my_yready + r), S.epoch, CU_STREAM_WAIT_VALUE_GEQ);
      if (rr != CUDA_SUCCESS) return bc_fail(BC_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)rr);
    }
  }
  bc::UpdArgs u{};
  for (int e = 0; e < n; ++e) {
    u.latents[e] = S.upd.latents[e];
    u.eps[e] = S.upd.eps[e];
    u.out[e] = S.upd.out[e];
    u.level[e] = S.batch.level[e];
    u.next_level[e] = S.upd.next_level[e];
    u.post[e] = S.upd.post[e];
    u.block[e] = S.batch.block_index[e];
  }
  if (c->peers.n_peers > 0 && S.epoch > 0) {
    u.peer = peer_args(c, S.epoch);
    if (c->push_by_copy || S.rows_mode) {  // this iteration's pushes are ordered before our done signal
      BC_CUDA(cudaEventRecord(c->ev_side, c->side));
      BC_CUDA(cudaStreamWaitEvent(st, c->ev_side, 0));
    }
  }
  const int R = n * T;  // Y holds every entry's rows here
  RC(timed(kBandwidth, 0.0, (4.0 * 64 + 16.0 * 16) * R, st, [&] { return bc::launch_head_update(c->Y, n, T, F, dm.latent_h, dm.latent_w, u, S.status, st); }));
  return BC_OK;
}

int stage_end(bc_wan_ctx* c, cudaStream_t st) {
  RC(stage_head(c, st));
  return stage_update(c, st);
}

// Record one step's launches into a CUDA graph on the context's own stream
// and replay it through the width's executable graph (cudaGraphExecUpdate;
// re-instantiated when the kernel sequence changed).  The first step of each
// batch width runs eagerly (per-kernel static setup must not happen inside a
// capture), as do profiled steps; a failed capture disables graphs for the
// context and the step runs eagerly.
template <class F>
int run_graphed(bc_wan_ctx* c, cudaStream_t& st, int n, F&& run_all) {
  if (g_graphs < 0) {
    const char* e = getenv("BC_GRAPHS");
    g_graphs = e ? atoi(e) != 0 : 1;
  }
  // (per-kernel profiling records events between the launches: eager)
  if (!g_graphs || g_prof || c->graphs_broken || n < 1 || n > BC_MAX_ENTRIES || !c->width_seen[n]) {
    if (n >= 1 && n <= BC_MAX_ENTRIES) c->width_seen[n] = true;
    return run_all();
  }
  if (!c->gstream) {
    BC_CUDA(cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
    BC_CUDA(cudaEventCreateWithFlags(&c->gev_in, cudaEventDisableTiming));
    BC_CUDA(cudaEventCreateWithFlags(&c->gev_out, cudaEventDisableTiming));
  }
  // capture on the context's own stream (the caller's may be the legacy
  // stream, which cannot be captured); ordered after the caller's earlier
  // work and before its later work by two events
  const cudaStream_t caller = st;
  st = c->gstream;
  cudaGraph_t graph = nullptr;
  BC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const int rc = run_all();
  const cudaError_t ec = cudaStreamEndCapture(st, &graph);
  st = caller;
  if (rc || ec != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    if (rc) return rc;
    c->graphs_broken = true;  // something in the step cannot be captured: stay eager
    return run_all();
  }
  cudaGraphExec_t& ex = c->graph_exec[n];
  if (ex) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(ex, graph, &info) != cudaSuccess) {
      (void)cudaGetLastError();
      cudaGraphExecDestroy(ex);
      ex = nullptr;
    }
  }
  if (!ex) {
    const cudaError_t ei = cudaGraphInstantiate(&ex, graph, 0);
    if (ei != cudaSuccess) {
      cudaGraphDestroy(graph);
      ex = nullptr;
      (void)cudaGetLastError();
      c->graphs_broken = true;
      return run_all();
    }
  }
  cudaGraphDestroy(graph);
  BC_CUDA(cudaEventRecord(c->gev_in, caller));
  BC_CUDA(cudaStreamWaitEvent(c->gstream, c->gev_in, 0));
  BC_CUDA(cudaGraphLaunch(ex, c->gstream));
  BC_CUDA(cudaEventRecord(c->gev_out, c->gstream));
  BC_CUDA(cudaStreamWaitEvent(caller, c->gev_out, 0));
  return BC_OK;
}

}  // namespace

extern "C" int bc_wan_step(bc_wan_ctx* c, const bc_batch* batch, const bc_wan_update* upd, int32_t* status,
                           void* stream) {
  if (!c || !batch || !upd || !status) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: null argument");
  if (!c->text_ready) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: bc_wan_set_text not called");
  if (c->peers.n_peers > 0) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step: peers attached, use bc_wan_step_dist");
  cudaStream_t st = (cudaStream_t)stream;
  // NVTX ranges (free without a tool attached): one per step and per layer,
  // so ncu --nvtx / nsys timelines map launches to (iteration, layer)
  NvtxScope step_range("bc_wan_step");
  auto run_all = [&]() -> int {
    RC(stage_begin(c, batch, upd, nullptr, status, st));
    for (int l = 0; l < c->dims.layers; ++l) {
      NvtxScope layer_range(c->layer_names[l].c_str());
      RC(stage_layer_a(c, l, st));
      RC(stage_layer_b(c, l, st));
    }
    return stage_end(c, st);
  };
  return run_graphed(c, st, batch->n_entries, run_all);
}

extern "C" int bc_wan_set_peers(bc_wan_ctx* c, const bc_wan_peers* peers) {
  if (!c || !peers) return bc_fail(BC_ERR_CONTRACT, "bc_wan_set_peers: null argument");
  if (peers->n_peers < 0 || peers->n_peers > BC_MAX_PEERS || peers->n_ranks != peers->n_peers + 1 ||
      peers->my_rank < 0 || peers->my_rank >= peers->n_ranks)
    return bc_fail(BC_ERR_CONTRACT, "bc_wan_set_peers: bad rank geometry");
  if (peers->n_peers > 0 && (!peers->my_flags || !peers->my_done || !peers->counters))
    return bc_fail(BC_ERR_CONTRACT, "bc_wan_set_peers: flags / done / counters required");
  for (int p = 0; p < peers->n_peers; ++p)
    if (!peers->peer_arena[p] || !peers->peer_flags[p] || !peers->peer_done[p])
      return bc_fail(BC_ERR_CONTRACT, "bc_wan_set_peers: null peer pointer");
  if (peers->my_y) {  // row-sharded steps: Y lives in memory the peers can write
    if (!peers->my_yready) return bc_fail(BC_ERR_CONTRACT, "bc_wan_set_peers: my_y needs my_yready");
    for (int p = 0; p < peers->n_peers; ++p)
      if (!peers->peer_y[p] || !peers->peer_yready[p])
        return bc_fail(BC_ERR_CONTRACT, "bc_wan_set_peers: null peer Y pointer");
    c->Y = peers->my_y;
  }
  c->peers = *peers;
  // Default: the q/k kernel itself stores each fresh K/V row into every
  // peer's replica (NVLink P2P) and its last CTA publishes the flags, so a
  // consumer's spinning attention only ever waits on work that precedes it
  // on some stream -- deadlock-free whatever else occupies the SMs.
  // BC_KV_PUSH=copy: cudaMemcpyAsync on a side stream + stream-memop flags;
  // overlaps the transfer with compute but needs the copy to run on a copy
  // engine -- a same-device copy (one-GPU emulation of the ranks) is an SM
  // kernel that a spinning attention can starve (measured: hangs at full
  // Wan-1.3B geometry, scripts/emulated_full.py).
  // Default by device identity: when every peer replica lives on ANOTHER
  // GPU the copies run on copy engines (DMA over NVLink, no SMs), so the
  // transfer overlaps the producer's own attention instead of lengthening
  // its q/k kernel by the NVLink store time; peers on this device (the
  // one-GPU emulation, two processes on one GPU) keep the kernel stores.
  // BC_KV_PUSH=copy / kernel overrides.
  const char* how = getenv("BC_KV_PUSH");
  if (how && std::strcmp(how, "copy") == 0) {
    c->push_by_copy = true;
  } else if (how && std::strcmp(how, "kernel") == 0) {
    c->push_by_copy = false;
  } else {
    int me = -1;
    cudaGetDevice(&me);
    bool all_remote = peers->n_peers > 0;
    for (int p = 0; p < peers->n_peers && all_remote; ++p) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, peers->peer_arena[p]) != cudaSuccess || at.device == me) all_remote = false;
    }
    (void)cudaGetLastError();
    c->push_by_copy = all_remote;
  }
  if (peers->n_peers > 0 && !c->side) {
    BC_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    BC_CUDA(cudaEventCreateWithFlags(&c->ev_qk, cudaEventDisableTiming));
    BC_CUDA(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
  }
  return BC_OK;
}

// Multi-GPU step of this rank's entries (or one stage of it, for drivers
// that interleave several ranks on one device).
extern "C" int bc_wan_step_dist(bc_wan_ctx* c, const bc_batch* batch, const bc_wan_update* upd,
                                const bc_wan_dist* dist, int32_t* status, void* stream) {
  if (!c || !dist || !status) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: null argument");
  if (!c->text_ready) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: bc_wan_set_text not called");
  if (dist->epoch < 1) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: epoch must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  static const char* kStageNames[] = {"bc_wan_step_dist", "begin", "layer part A", "layer part B", "head",
                                      "update"};
  NvtxScope range(kStageNames[(dist->stage >= -1 && dist->stage <= 4) ? dist->stage + 1 : 0]);
  switch (dist->stage) {
    case -1:
      // eager: multi-GPU sessions are re-created per run, so per-width graph
      // instantiation would not amortise (measured slower in the two-process
      // one-GPU test)
      if (!batch || !upd) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: null batch");
      RC(stage_begin(c, batch, upd, dist, status, st));
      for (int l = 0; l < c->dims.layers; ++l) {
        RC(stage_layer_a(c, l, st));
        RC(stage_layer_b(c, l, st));
      }
      return stage_end(c, st);
    case 0:
      if (!batch || !upd) return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: null batch");
      return stage_begin(c, batch, upd, dist, status, st);
    case 1:
      return stage_layer_a(c, dist->layer, st);
    case 2:
      return stage_layer_b(c, dist->layer, st);
    case 3:
      return stage_head(c, st);
    case 4:
      return stage_update(c, st);
  }
  return bc_fail(BC_ERR_CONTRACT, "bc_wan_step_dist: bad stage %d", dist->stage);
}

// A rank with no entries this iteration still publishes iteration-done.
extern "C" int bc_wan_signal_done(bc_wan_ctx* c, uint32_t epoch, void* stream) {
  if (!c) return bc_fail(BC_ERR_CONTRACT, "bc_wan_signal_done: null ctx");
  if (c->peers.n_peers == 0) return BC_OK;
  return bc::launch_signal_done(peer_args(c, epoch), (cudaStream_t)stream);
}

// ---------------------------------------------------------------- IPC memory
extern "C" int bc_ipc_malloc(int64_t bytes, void** ptr, char handle[64]) {
  if (!ptr || bytes <= 0) return bc_fail(BC_ERR_CONTRACT, "bc_ipc_malloc: bad arguments");
  BC_CUDA(cudaMalloc(ptr, (size_t)bytes));
  BC_CUDA(cudaMemset(*ptr, 0, (size_t)bytes));
  if (handle) {
    cudaIpcMemHandle_t h;
    BC_CUDA(cudaIpcGetMemHandle(&h, *ptr));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle, &h, 64);
  }
  return BC_OK;
}

extern "C" int bc_ipc_open(const char handle[64], void** ptr) {
  if (!handle || !ptr) return bc_fail(BC_ERR_CONTRACT, "bc_ipc_open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  BC_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BC_OK;
}

extern "C" int bc_ipc_close(void* ptr) {
  BC_CUDA(cudaIpcCloseMemHandle(ptr));
  return BC_OK;
}

extern "C" int bc_free(void* ptr) {
  BC_CUDA(cudaFree(ptr));
  return BC_OK;
}

extern "C" int bc_memset_async(void* ptr, int value, int64_t bytes, void* stream) {
  BC_CUDA(cudaMemsetAsync(ptr, value, (size_t)bytes, (cudaStream_t)stream));
  return BC_OK;
}

// ---------------------------------------------------------------- stream-ordered handoff primitives
// (the decode-GPU inbox, decode_rank.py): a copy between (possibly peer /
// IPC-mapped) device buffers, and 32-bit flag writes / waits executed by the
// stream itself -- the waiting stream's GPU spins in the front end, not on
// an SM, so a peer that shares the GPU is never starved.
extern "C" int bc_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (!dst || !src || bytes < 0) return bc_fail(BC_ERR_CONTRACT, "bc_copy_async: bad arguments");
  BC_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return BC_OK;
}

extern "C" int bc_stream_write_u32(void* addr, uint32_t value, void* stream) {
  if (!addr) return bc_fail(BC_ERR_CONTRACT, "bc_stream_write_u32: null address");
  // default flags: a memory fence orders the stream's earlier writes (the
  // copy) before the flag for every observer (kernel fallback: write_flags)
  bc::FlagWrites fw{};
  fw.addr[0] = static_cast<uint32_t*>(addr);
  fw.n = 1;
  fw.v = value;
  return write_flags((cudaStream_t)stream, fw);
}

extern "C" int bc_stream_wait_geq_u32(void* addr, uint32_t value, void* stream) {
  auto wt = wait_value32();
  if (!wt) return bc_fail(BC_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  const CUresult r = wt((CUstream)stream, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return bc_fail(BC_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return BC_OK;
}
