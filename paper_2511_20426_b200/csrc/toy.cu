// Toy DiT forward (the reference's own model, blockcascade/denoiser.py),
// float64 on the device, plus the renoise kernel shared by both model
// families.
//
// The toy has one token per latent frame and D <= a few hundred, so each
// phase is one CTA per batch entry; the whole forward is 2 + 2L launches.
// The work is launch-bound by construction -- this path exists for
// numeric parity with the reference's float64 forward (its only
// reference-pinned numeric oracle), not for throughput.
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

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  // fixed order over warps -> deterministic
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

// h[e] = x W_in^T + pos(b*S+i) + W_level feats(level) + W_cond cond
// (embed_entry, denoiser.py:234-250; _position_encoding 214-221;
//  _level_features 224-227)
__global__ void toy_embed(bc_toy_weights w, bc_batch bt, ToyPtrs p, double* hidden,
                          int32_t* status) {
  const int e = blockIdx.x;
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
  for (int idx = threadIdx.x; idx < S * D; idx += blockDim.x) {
    const int i = idx / D, j = idx % D;
    const double* xi = x + (size_t)i * D;
    if (!isfinite(xi[j])) atomicCAS(status, 0, 1 + bt.block_index[e]);
    double acc = 0.0;
    const double* wr = w.w_in + (size_t)j * D;
    for (int k = 0; k < D; ++k) acc += xi[k] * wr[k];
    const double pos = (double)(bt.block_index[e] * S + i);
    const double expo = 2.0 * (double)(j >> 1) / (double)D;
    const double ang = pos / pow(10000.0, expo);
    acc += (j & 1) ? cos(ang) : sin(ang);
    double lv = 0.0;
    for (int f = 0; f < kLevelFeats; ++f) lv += w.w_level[(size_t)j * kLevelFeats + f] * feat[f];
    double cv = 0.0;
    for (int f = 0; f < Dc; ++f) cv += w.w_cond[(size_t)j * Dc + f] * c[f];
    h[idx] = acc + lv + cv;
  }
}

// hn = rmsnorm(h); out = hn W^T for W in {q,k,v} (layer_qkv, 253-261).
// grid (n_entries, 3): y = 0 -> q workspace, 1 -> K slot, 2 -> V slot.
__global__ void toy_qkv(bc_toy_weights w, bc_batch bt, int layer, const double* hidden,
                        double* qbuf, double* arena, int n_slots) {
  extern __shared__ double sm[];
  const int e = blockIdx.x, which = blockIdx.y;
  const int S = bt.block_size, D = w.dim;
  double* hn = sm;              // S*D
  double* red = sm + S * D;     // 32
  const double* h = hidden + (size_t)e * S * D;
  for (int i = 0; i < S; ++i) {
    double ss = 0.0;
    for (int k = threadIdx.x; k < D; k += blockDim.x) ss += h[(size_t)i * D + k] * h[(size_t)i * D + k];
    const double tot = block_sum(ss, red);
    const double inv = 1.0 / sqrt(tot / (double)D + kRmsEps);
    for (int k = threadIdx.x; k < D; k += blockDim.x) hn[i * D + k] = h[(size_t)i * D + k] * inv;
  }
  __syncthreads();
  const double* W = (which == 0 ? w.w_q : which == 1 ? w.w_k : w.w_v) + (size_t)layer * D * D;
  double* dst;
  if (which == 0) {
    dst = qbuf + (size_t)e * S * D;
  } else {
    dst = arena + ((((size_t)layer * n_slots + bt.slot[e]) * 2 + (which - 1)) * S) * D;
  }
  for (int idx = threadIdx.x; idx < S * D; idx += blockDim.x) {
    const int i = idx / D, j = idx % D;
    const double* wr = W + (size_t)j * D;
    double acc = 0.0;
    for (int k = 0; k < D; ++k) acc += hn[i * D + k] * wr[k];
    dst[idx] = acc;
  }
}

// Per head: softmax(q K^T / sqrt(hd)) V over the visible slots in order,
// then h += out W_o^T (layer_attend, 264-277).
__global__ void toy_attend(bc_toy_weights w, bc_batch bt, int layer, double* hidden,
                           const double* qbuf, const double* arena, int n_slots) {
  extern __shared__ double sm[];
  const int e = blockIdx.x;
  const int S = bt.block_size, D = w.dim, H = w.heads, hd = D / H;
  const int nk = bt.n_vis[e] * S;
  double* att = sm;              // S*D
  double* sc = sm + S * D;       // nk
  const double scale = 1.0 / sqrt((double)hd);
  const double* q = qbuf + (size_t)e * S * D;
  for (int i = 0; i < S; ++i) {
    for (int hh = 0; hh < H; ++hh) {
      for (int t = threadIdx.x; t < nk; t += blockDim.x) {
        const int slot = bt.vis_slot[e][t / S], r = t % S;
        const double* k = arena + ((((size_t)layer * n_slots + slot) * 2 + 0) * S + r) * D + hh * hd;
        double acc = 0.0;
        for (int d = 0; d < hd; ++d) acc += q[(size_t)i * D + hh * hd + d] * k[d];
        sc[t] = acc * scale;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double m = sc[0];
        for (int t = 1; t < nk; ++t) m = fmax(m, sc[t]);
        double z = 0.0;
        for (int t = 0; t < nk; ++t) {
          sc[t] = exp(sc[t] - m);
          z += sc[t];
        }
        for (int t = 0; t < nk; ++t) sc[t] /= z;
      }
      __syncthreads();
      for (int d = threadIdx.x; d < hd; d += blockDim.x) {
        double acc = 0.0;
        for (int t = 0; t < nk; ++t) {
          const int slot = bt.vis_slot[e][t / S], r = t % S;
          acc += sc[t] * arena[((((size_t)layer * n_slots + slot) * 2 + 1) * S + r) * D + hh * hd + d];
        }
        att[i * D + hh * hd + d] = acc;
      }
      __syncthreads();
    }
  }
  double* h = hidden + (size_t)e * S * D;
  const double* Wo = w.w_o + (size_t)layer * D * D;
  for (int idx = threadIdx.x; idx < S * D; idx += blockDim.x) {
    const int i = idx / D, j = idx % D;
    double acc = 0.0;
    for (int k = 0; k < D; ++k) acc += att[i * D + k] * Wo[(size_t)j * D + k];
    h[idx] += acc;
  }
}

// x0 = rmsnorm(h) W_head^T (predict_head, 280-281)
__global__ void toy_head(bc_toy_weights w, bc_batch bt, const double* hidden, ToyPtrs p) {
  extern __shared__ double sm[];
  const int e = blockIdx.x;
  const int S = bt.block_size, D = w.dim;
  double* hn = sm;
  double* red = sm + S * D;
  const double* h = hidden + (size_t)e * S * D;
  for (int i = 0; i < S; ++i) {
    double ss = 0.0;
    for (int k = threadIdx.x; k < D; k += blockDim.x) ss += h[(size_t)i * D + k] * h[(size_t)i * D + k];
    const double tot = block_sum(ss, red);
    const double inv = 1.0 / sqrt(tot / (double)D + kRmsEps);
    for (int k = threadIdx.x; k < D; k += blockDim.x) hn[i * D + k] = h[(size_t)i * D + k] * inv;
  }
  __syncthreads();
  double* out = p.x0[e];
  for (int idx = threadIdx.x; idx < S * D; idx += blockDim.x) {
    const int i = idx / D, j = idx % D;
    double acc = 0.0;
    for (int k = 0; k < D; ++k) acc += hn[i * D + k] * w.w_head[(size_t)j * D + k];
    out[idx] = acc;
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
  double* qbuf = workspace + (size_t)n * S * D;
  size_t sm_norm = ((size_t)S * D + 32) * sizeof(double);
  int max_k = 0;
  for (int e = 0; e < n; ++e) max_k = b.n_vis[e] * S > max_k ? b.n_vis[e] * S : max_k;
  size_t sm_att = ((size_t)S * D + max_k) * sizeof(double);
  if (sm_norm > 200 * 1024 || sm_att > 200 * 1024)
    return bc_fail(BC_ERR_CONTRACT, "bc_toy_forward: toy dims too large for one CTA");
  static bool attr_done = false;
  if (!attr_done) {
    BC_CUDA(cudaFuncSetAttribute(toy_qkv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    BC_CUDA(cudaFuncSetAttribute(toy_attend, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    BC_CUDA(cudaFuncSetAttribute(toy_head, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done = true;
  }
  toy_embed<<<n, kThreads, 0, st>>>(*w, b, p, hidden, status);
  BC_LAUNCHED();
  for (int l = 0; l < w->layers; ++l) {
    toy_qkv<<<dim3(n, 3), kThreads, sm_norm, st>>>(*w, b, l, hidden, qbuf, kv_arena, n_slots);
    BC_LAUNCHED();
    toy_attend<<<n, kThreads, sm_att, st>>>(*w, b, l, hidden, qbuf, kv_arena, n_slots);
    BC_LAUNCHED();
  }
  toy_head<<<n, kThreads, sm_norm, st>>>(*w, b, hidden, p);
  BC_LAUNCHED();
  return BC_OK;
}
