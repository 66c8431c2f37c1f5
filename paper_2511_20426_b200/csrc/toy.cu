// Toy DiT forward (the reference's own model, blockcascade/denoiser.py),
// float64 on the device, plus the renoise kernel shared by both model
// families.
//
// The toy has one token per latent frame and D <= a few hundred; every
// phase is a grid of (entry, 32-column chunk) CTAs with warp-level dot
// products, 2 + 3L launches per forward.  This path exists for numeric
// parity with the reference's float64 forward (its only reference-pinned
// numeric oracle); it is launch-bound by construction.
//
// Phase order per layer mirrors forward() (denoiser.py:333-353): QKV for
// every entry (fresh K/V written to the entry's arena slot), then attention
// for every entry -- the kernel boundary is the per-layer barrier of
// executor.py:3-7.  Key order inside attention is the slot order supplied
// by the host (ascending block), i.e. _gather's order (denoiser.py:284-296).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "bc_common.h"

namespace {

constexpr int kThreads = 256;
constexpr int kLevelFeats = 8;
constexpr double kRmsEps = 1e-6;

struct ToyPtrs {
  const double* x[BC_MAX_ENTRIES];
  const double* cond[BC_MAX_ENTRIES];
  double* x0[BC_MAX_ENTRIES];
};


// Every kernel below spreads one entry's work over many CTAs: grid
// (entry, 32-column chunk of the output), one warp per output element with
// the dot product split over the lanes (fixed xor-tree reduction order, so
// results are deterministic and independent of the batch).  The first
// version ran each phase as ONE CTA per entry with thread-serial 256-long
// dot products and a single-thread softmax: ~1 ms per iteration, no faster
// than the numpy oracle on the host.

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// sum_k a[k] * b[k] over k < n, lanes interleaved, then the xor tree
__device__ __forceinline__ double warp_dot(const double* a, const double* b, int n) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int k = lane; k < n; k += 32) acc += a[k] * b[k];
  return warp_sum_d(acc);
}

constexpr int kCols = 32;  // output columns per CTA

// RMS-normalise the S rows of h into smem hn (every CTA of the entry redoes
// this: S*D reads, negligible)
__device__ __forceinline__ void rms_rows_smem(const double* h, double* hn, int S, int D) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < S; i += nw) {
    const double ss = warp_dot(h + (size_t)i * D, h + (size_t)i * D, D);
    const double inv = 1.0 / sqrt(ss / (double)D + kRmsEps);
    for (int k = threadIdx.x & 31; k < D; k += 32) hn[i * D + k] = h[(size_t)i * D + k] * inv;
  }
  __syncthreads();
}

// h[e] = x W_in^T + pos(b*S+i) + W_level feats(level) + W_cond cond
// (embed_entry, denoiser.py:234-250; _position_encoding 214-221;
//  _level_features 224-227).  grid (n, D / 32)
__global__ void toy_embed(bc_toy_weights w, bc_batch bt, ToyPtrs p, double* hidden,
                          int32_t* status) {
  const int e = blockIdx.x, j0 = blockIdx.y * kCols;
  const int S = bt.block_size, D = w.dim, Dc = w.cond_dim;
  const double* x = p.x[e];
  const double* c = p.cond[e];
  double* h = hidden + (size_t)e * S * D;
  const double s = bt.level[e] / 1000.0;
  double feat[kLevelFeats];
#pragma unroll
  for (int k = 0; k < kLevelFeats / 2; ++k) {
    feat[k] = sin(2.0 * M_PI * s * (double)(k + 1));
    feat[k + kLevelFeats / 2] = cos(2.0 * M_PI * s * (double)(k + 1));
  }
  if (blockIdx.y == 0)
    for (int idx = threadIdx.x; idx < S * D; idx += blockDim.x)
      if (!isfinite(x[idx])) atomicCAS(status, 0, 1 + bt.block_index[e]);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = warp; o < S * kCols; o += nw) {
    const int i = o / kCols, j = j0 + o % kCols;
    if (j >= D) continue;
    double acc = warp_dot(x + (size_t)i * D, w.w_in + (size_t)j * D, D);
    const double cv = warp_dot(w.w_cond + (size_t)j * Dc, c, Dc);
    if ((threadIdx.x & 31) == 0) {
      const double pos = (double)(bt.block_index[e] * S + i);
      const double expo = 2.0 * (double)(j >> 1) / (double)D;
      const double ang = pos / pow(10000.0, expo);
      acc += (j & 1) ? cos(ang) : sin(ang);
      double lv = 0.0;
      for (int f = 0; f < kLevelFeats; ++f) lv += w.w_level[(size_t)j * kLevelFeats + f] * feat[f];
      h[(size_t)i * D + j] = acc + lv + cv;
    }
  }
}

// hn = rmsnorm(h); out = hn W^T for W in {q,k,v} (layer_qkv, 253-261).
// grid (n, 3, D / 32): y = 0 -> q workspace, 1 -> K slot, 2 -> V slot.
__global__ void toy_qkv(bc_toy_weights w, bc_batch bt, int layer, const double* hidden,
                        double* qbuf, double* arena, int n_slots) {
  extern __shared__ double sm[];
  const int e = blockIdx.x, which = blockIdx.y, j0 = blockIdx.z * kCols;
  const int S = bt.block_size, D = w.dim;
  double* hn = sm;  // S*D
  rms_rows_smem(hidden + (size_t)e * S * D, hn, S, D);
  const double* W = (which == 0 ? w.w_q : which == 1 ? w.w_k : w.w_v) + (size_t)layer * D * D;
  double* dst = which == 0 ? qbuf + (size_t)e * S * D
                           : arena + ((((size_t)layer * n_slots + bt.slot[e]) * 2 + (which - 1)) * S) * D;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = warp; o < S * kCols; o += nw) {
    const int i = o / kCols, j = j0 + o % kCols;
    if (j >= D) continue;
    const double acc = warp_dot(hn + i * D, W + (size_t)j * D, D);
    if ((threadIdx.x & 31) == 0) dst[(size_t)i * D + j] = acc;
  }
}

// One head of one entry: softmax(q K^T / sqrt(hd)) V over the visible slots
// in order (layer_attend 264-277, _gather 284-296); the head's output
// overwrites its own q columns in qbuf (q was copied to smem first).
// grid (n, H)
__global__ void toy_attend(bc_toy_weights w, bc_batch bt, int layer, double* qbuf, const double* arena,
                           int n_slots) {
  extern __shared__ double sm[];
  const int e = blockIdx.x, hh = blockIdx.y;
  const int S = bt.block_size, D = w.dim, H = w.heads, hd = D / H;
  const int nk = bt.n_vis[e] * S;
  double* q = sm;            // S*hd
  double* sc = sm + S * hd;  // S*nk
  const double scale = 1.0 / sqrt((double)hd);
  double* qg = qbuf + (size_t)e * S * D + hh * hd;
  for (int idx = threadIdx.x; idx < S * hd; idx += blockDim.x) q[idx] = qg[(size_t)(idx / hd) * D + idx % hd];
  __syncthreads();
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int o = warp; o < S * nk; o += nw) {
    const int i = o / nk, t = o % nk;
    const int slot = bt.vis_slot[e][t / S], r = t % S;
    const double* k = arena + ((((size_t)layer * n_slots + slot) * 2 + 0) * S + r) * D + hh * hd;
    const double acc = warp_dot(q + i * hd, k, hd);
    if (lane == 0) sc[i * nk + t] = acc * scale;
  }
  __syncthreads();
  for (int i = warp; i < S; i += nw) {  // max-subtracted softmax of row i
    double* row = sc + i * nk;
    double m = -INFINITY;
    for (int t = lane; t < nk; t += 32) m = fmax(m, row[t]);
    m = warp_max_d(m);
    double z = 0.0;
    for (int t = lane; t < nk; t += 32) {
      const double v = exp(row[t] - m);
      row[t] = v;
      z += v;
    }
    z = warp_sum_d(z);
    for (int t = lane; t < nk; t += 32) row[t] /= z;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < S * hd; idx += blockDim.x) {
    const int i = idx / hd, d = idx % hd;
    double acc = 0.0;
    for (int t = 0; t < nk; ++t) {
      const int slot = bt.vis_slot[e][t / S], r = t % S;
      acc += sc[i * nk + t] * arena[((((size_t)layer * n_slots + slot) * 2 + 1) * S + r) * D + hh * hd + d];
    }
    qg[(size_t)i * D + d] = acc;
  }
}

// h += att W_o^T (the tail of layer_attend).  grid (n, D / 32)
__global__ void toy_oproj(bc_toy_weights w, bc_batch bt, int layer, double* hidden, const double* att) {
  const int e = blockIdx.x, j0 = blockIdx.y * kCols;
  const int S = bt.block_size, D = w.dim;
  const double* a = att + (size_t)e * S * D;
  double* h = hidden + (size_t)e * S * D;
  const double* Wo = w.w_o + (size_t)layer * D * D;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = warp; o < S * kCols; o += nw) {
    const int i = o / kCols, j = j0 + o % kCols;
    if (j >= D) continue;
    const double acc = warp_dot(a + (size_t)i * D, Wo + (size_t)j * D, D);
    if ((threadIdx.x & 31) == 0) h[(size_t)i * D + j] += acc;
  }
}

// x0 = rmsnorm(h) W_head^T (predict_head, 280-281).  grid (n, D / 32)
__global__ void toy_head(bc_toy_weights w, bc_batch bt, const double* hidden, ToyPtrs p) {
  extern __shared__ double sm[];
  const int e = blockIdx.x, j0 = blockIdx.y * kCols;
  const int S = bt.block_size, D = w.dim;
  double* hn = sm;
  rms_rows_smem(hidden + (size_t)e * S * D, hn, S, D);
  double* out = p.x0[e];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = warp; o < S * kCols; o += nw) {
    const int i = o / kCols, j = j0 + o % kCols;
    if (j >= D) continue;
    const double acc = warp_dot(hn + i * D, w.w_head + (size_t)j * D, D);
    if ((threadIdx.x & 31) == 0) out[(size_t)i * D + j] = acc;
  }
}

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <>
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// (1 - s) x0 + s eps, two rounded products and a rounded add (no FMA):
// the exact numpy evaluation order of renoise (denoiser.py:367-368).
template <typename T>
__global__ void renoise_kernel(const T* __restrict__ x0, const T* __restrict__ eps, T keep,
                               T sigma, T* out, int64_t n, int32_t* nonfinite) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = add_rn(mul_rn(keep, x0[i]), mul_rn(sigma, eps[i]));
    out[i] = v;
    bad |= !isfinite(v);
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(nonfinite, 1);
}

template <typename T>
int launch_renoise(const T* x0, const T* eps, double level, T* out, int64_t n, int32_t* nf,
                   void* stream) {
  if (n < 0 || !(level >= 0.0 && level <= 1000.0))
    return bc_fail(BC_ERR_CONTRACT, "renoise: level %g out of [0,1000] or n < 0", level);
  if (n == 0) return BC_OK;
  const double sig = level / 1000.0;
  const double keep = 1.0 - sig;
  int grid = (int)((n + kThreads - 1) / kThreads);
  if (grid > 148 * 16) grid = 148 * 16;
  renoise_kernel<T><<<grid, kThreads, 0, (cudaStream_t)stream>>>(x0, eps, (T)keep, (T)sig, out, n, nf);
  BC_LAUNCHED();
  return BC_OK;
}

}  // namespace

extern "C" int bc_renoise_f64(const double* x0, const double* eps, double level, double* out,
                              int64_t n, int32_t* nonfinite, void* stream) {
  return launch_renoise<double>(x0, eps, level, out, n, nonfinite, stream);
}

extern "C" int bc_renoise_f32(const float* x0, const float* eps, double level, float* out,
                              int64_t n, int32_t* nonfinite, void* stream) {
  return launch_renoise<float>(x0, eps, level, out, n, nonfinite, stream);
}

extern "C" int bc_toy_forward(const bc_toy_weights* w, const bc_batch* batch,
                              const double* const* latents, const double* const* cond,
                              double* kv_arena, int32_t n_slots, double* const* x0_out,
                              double* workspace, int32_t* status, void* stream) {
  if (!w || !batch || !latents || !cond || !x0_out || !kv_arena || !workspace)
    return bc_fail(BC_ERR_CONTRACT, "bc_toy_forward: null argument");
  const bc_batch& b = *batch;
  if (b.n_entries < 1 || b.n_entries > BC_MAX_ENTRIES || b.block_size < 1)
    return bc_fail(BC_ERR_CONTRACT, "bc_toy_forward: bad batch (n=%d)", b.n_entries);
  if (w->dim % w->heads) return bc_fail(BC_ERR_CONTRACT, "bc_toy_forward: heads must divide dim");
  for (int e = 0; e < b.n_entries; ++e) {
    if (b.n_vis[e] < 1 || b.n_vis[e] > BC_MAX_VIS || b.slot[e] < 0 || b.slot[e] >= n_slots)
      return bc_fail(BC_ERR_CONTRACT, "bc_toy_forward: bad slot table for entry %d", e);
    for (int v = 0; v < b.n_vis[e]; ++v)
      if (b.vis_slot[e][v] < 0 || b.vis_slot[e][v] >= n_slots)
        return bc_fail(BC_ERR_CONTRACT, "bc_toy_forward: visible slot out of range");
  }
  ToyPtrs p{};
  for (int e = 0; e < b.n_entries; ++e) {
    p.x[e] = latents[e];
    p.cond[e] = cond[e];
    p.x0[e] = x0_out[e];
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int S = b.block_size, D = w->dim, n = b.n_entries;
  double* hidden = workspace;
  double* qbuf = workspace + (size_t)n * S * D;   // q, then each head's attention output in place
  const size_t sm_norm = (size_t)S * D * sizeof(double);
  int max_k = 0;
  for (int e = 0; e < n; ++e) max_k = b.n_vis[e] * S > max_k ? b.n_vis[e] * S : max_k;
  const int hd = D / w->heads;
  const size_t sm_att = ((size_t)S * hd + (size_t)S * max_k) * sizeof(double);
  if (sm_norm > 200 * 1024 || sm_att > 200 * 1024)
    return bc_fail(BC_ERR_CONTRACT, "bc_toy_forward: toy dims too large for one CTA");
  static bool attr_done = false;
  if (!attr_done) {
    BC_CUDA(cudaFuncSetAttribute(toy_qkv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    BC_CUDA(cudaFuncSetAttribute(toy_attend, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    BC_CUDA(cudaFuncSetAttribute(toy_head, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done = true;
  }
  const int chunks = (D + kCols - 1) / kCols;
  toy_embed<<<dim3(n, chunks), kThreads, 0, st>>>(*w, b, p, hidden, status);
  BC_LAUNCHED();
  for (int l = 0; l < w->layers; ++l) {
    toy_qkv<<<dim3(n, 3, chunks), kThreads, sm_norm, st>>>(*w, b, l, hidden, qbuf, kv_arena, n_slots);
    BC_LAUNCHED();
    toy_attend<<<dim3(n, w->heads), kThreads, sm_att, st>>>(*w, b, l, qbuf, kv_arena, n_slots);
    BC_LAUNCHED();
    toy_oproj<<<dim3(n, chunks), kThreads, 0, st>>>(*w, b, l, hidden, qbuf);
    BC_LAUNCHED();
  }
  toy_head<<<dim3(n, chunks), kThreads, sm_norm, st>>>(*w, b, hidden, p);
  BC_LAUNCHED();
  return BC_OK;
}
