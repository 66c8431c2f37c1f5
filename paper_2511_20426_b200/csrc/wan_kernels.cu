// Bandwidth-bound kernels of the Wan2.1-shaped DiT step: patchify, time
// embedding GEMVs, LayerNorm + AdaLN modulation, q/k RMSNorm + 3-D RoPE +
// KV-slot scatter, cross-attention RMSNorm, and the fused head update
// (unpatchify + flow -> x0 + renoise / emit + finiteness check).
//
// All row kernels are warp-per-row with 16-byte vector accesses; statistics
// and the residual stream are fp32, GEMM operands bf16.  Model math follows
// the public Wan2.1 block; the noise parameterisation
// is the reference's sigma = level / 1000 (denoiser.py:360-368).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "bc_common.h"
#include "wan_kernels.h"
#include "sm100.cuh"

namespace bc {
namespace {

constexpr float kEps = 1e-6f;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// thread 0 of each CTA: wait until every peer reported iteration `want` done
__device__ __forceinline__ void wait_peers_done(const PeerArgs& pa) {
  if (pa.n_peers == 0 || pa.wait_done == 0) return;
  if (threadIdx.x == 0) {
    for (int r = 0; r < pa.n_ranks; ++r) {
      if (r == pa.my_rank) continue;
      spin_until_geq(pa.my_done + r, pa.wait_done, 128);
    }
  }
  __syncthreads();
}
// Sum over the WPR warps that cooperate on one row (fixed order).
template <int WPR>
__device__ __forceinline__ float row_reduce(float v, float* red, int slot, int wir) {
  v = warp_sum(v);
  if constexpr (WPR == 1) {
    return v;
  } else {
    if ((threadIdx.x & 31) == 0) red[slot * WPR + wir] = v;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) t += red[slot * WPR + w];
    __syncthreads();
    return t;
  }
}

// after all CTAs' stores: the last CTA to finish runs `fn` (publication)
template <class F>
__device__ __forceinline__ void last_cta_publish(uint32_t* ctr, F&& fn) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(ctr, 1u);
    if (prev == gridDim.x * gridDim.y - 1) {
      __threadfence_system();
      fn();
      *ctr = 0;  // ready for the next launch on this stream
    }
  }
}
__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

// ------------------------------------------------------------ patchify
// x: (F,16,H,W) fp32 -> tokens (F*(H/2)*(W/2), 64) bf16; vector index
// c*4 + kh*2 + kw (Conv3d weight order, kernel (1,2,2)).
// Rows [row0, row0 + rows) of the concatenated batch (row = e * T + token);
// out row 0 = global row row0.
// status != nullptr (the rows cover every latent): the finiteness check of
// the inputs rides along -- status = 1 + block index of an entry holding a
// NaN / Inf (what check_finite_kernel reports), no extra pass over the latents.
__global__ void patchify_kernel(EntryPtrs lat, int F, int H, int W, __nv_bfloat16* out, int T, int row0,
                                int rows, int32_t* status) {
  const int hp = H / 2, wp = W / 2;
  const int64_t total = (int64_t)rows * 64;
  int bad_block = -1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int g = row0 + (int)(idx >> 6), v = (int)(idx & 63);
    const int e = g / T, n = g % T;
    const int c = v >> 2, kh = (v >> 1) & 1, kw = v & 1;
    const int f = n / (hp * wp), rem = n % (hp * wp);
    const int i = rem / wp, j = rem % wp;
    const float val = lat.p[e][(((size_t)f * 16 + c) * H + 2 * i + kh) * W + 2 * j + kw];
    if (!isfinite(val) && bad_block < 0) bad_block = lat.block[e];
    out[idx] = __float2bfloat16(val);
  }
  if (status && bad_block >= 0) atomicCAS(status, 0, 1 + bad_block);
}

// ------------------------------------------------------------ GEMV (time MLP)
// out[e][o] = act( sum_k in[e][k] W[o][k] + b[o] ), one warp per o, 16-byte
// weight loads (8 bf16 per lane per step, 4 in flight before the math); act
// 0: none, 1: silu, 2: out gets the raw value and out2 its silu (t_e feeds
// the head modulation raw and the 6d projection through a silu).  K % 8 == 0.
// Two fusions keep the time embedding at three launches per step:
//  * SIN: the input is each entry's timestep sinusoid (K = freq_dim:
//    [cos(t w_k), sin(t w_k)], w_k = 10000^(-k/half), Wan
//    sinusoidal_embedding_1d), computed into shared memory by every CTA;
//  * mod != nullptr: the AdaLN tables of every layer are written as well,
//    mod[l][e][o] = base[l][o] + out[e][o] (N = 6d), in runs of the CTA's
//    8 consecutive outputs (whole 32-byte sectors).
// (SIN is a template flag so the double-precision sinusoid code does not
// raise the register count of the wide GEMVs.)  Measured in the step: ~9 /
// ~12 / ~30-50 us for n = 1..5 (latency-bound: 9216 short rows), about the
// five separate launches' time; the time MLP is 0.05% of a generation.
template <bool SIN>
__global__ void __launch_bounds__(256)
    gemv_kernel(const float* __restrict__ in, int n, int K, const __nv_bfloat16* __restrict__ W,
                const float* __restrict__ b, float* __restrict__ out, int N, int act, float* __restrict__ out2,
                TimeArgs ts, const float* __restrict__ base, int L, float* __restrict__ mod) {
  extern __shared__ float sin_in[];  // [n][K] when SIN
  __shared__ float e0s[BC_MAX_ENTRIES][8];  // mod != nullptr: this CTA's outputs
  if constexpr (SIN) {
    const int half = K / 2;
    for (int i = threadIdx.x; i < n * half; i += blockDim.x) {
      const int e = i / half, k = i % half;
      const double w = pow(10000.0, -(double)k / (double)half);
      const double arg = ts.t[e] * w;
      sin_in[e * K + k] = (float)cos(arg);
      sin_in[e * K + half + k] = (float)sin(arg);
    }
    __syncthreads();
    in = sin_in;
  }
  const int wib = threadIdx.x >> 5;
  const int row = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= N && !mod) return;  // (with mod: stay for the CTA barrier below)
  const uint4* w = reinterpret_cast<const uint4*>(W + (size_t)min(row, N - 1) * K);
  float acc[BC_MAX_ENTRIES];
#pragma unroll
  for (int e = 0; e < BC_MAX_ENTRIES; ++e) acc[e] = 0.0f;
  constexpr int kAhead = 4;
  const int k8n = K / 8;
  for (int k0 = lane; k0 < k8n; k0 += 32 * kAhead) {
    uint4 u[kAhead];
#pragma unroll
    for (int j = 0; j < kAhead; ++j) u[j] = k0 + 32 * j < k8n ? __ldg(w + k0 + 32 * j) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int j = 0; j < kAhead; ++j) {
      const int k8 = k0 + 32 * j;
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u[j]);
#pragma unroll
      for (int e = 0; e < BC_MAX_ENTRIES; ++e) {
        if (e < n && k8 < k8n) {
          const float4* x = reinterpret_cast<const float4*>(in + (size_t)e * K) + 2 * k8;
          const float4 x0 = x[0], x1 = x[1];
          acc[e] += bf(h[0]) * x0.x + bf(h[1]) * x0.y + bf(h[2]) * x0.z + bf(h[3]) * x0.w + bf(h[4]) * x1.x +
                    bf(h[5]) * x1.y + bf(h[6]) * x1.z + bf(h[7]) * x1.w;
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < BC_MAX_ENTRIES; ++e) {
    if (e < n) {
      float v = warp_sum(acc[e]);  // (xor butterfly: every lane holds the sum)
      v += b ? b[min(row, N - 1)] : 0.0f;
      const float o = act == 1 ? silu(v) : v;
      if (lane == 0 && row < N) {
        out[(size_t)e * N + row] = o;
        if (act == 2) out2[(size_t)e * N + row] = silu(v);
        if (mod) e0s[e][wib] = o;
      }
    }
  }
  if (mod) {
    __syncthreads();
    const int nw = blockDim.x >> 5;
    const int o0 = (int)blockIdx.x * nw;
    const int cnt = min(nw, N - o0);
    for (int i = threadIdx.x; i < L * n * nw; i += blockDim.x) {
      const int j = i % nw, le = i / nw;
      const int e = le % n, l = le / n;
      if (j < cnt) mod[((size_t)l * n + e) * N + o0 + j] = base[(size_t)l * N + o0 + j] + e0s[e][j];
    }
  }
}

// ------------------------------------------------------------ LayerNorm rows
// mode 0: LN(x) * (1 + mod[1]) + mod[0]   with mod = base[6][d] + e0[e][6][d] (chunks sel0/sel1)
// mode 1: LN(x) * w + b                   (affine LN, cross-attn norm3)
template <int VPL, int WPR>  // float4 vectors per lane, warps per row
__global__ void ln_rows_kernel(const float* __restrict__ X, __nv_bfloat16* __restrict__ out, int rows,
                               int d, int rows_per_entry, LnArgs a) {
  // Packed fp32x2 arithmetic (FADD2/FFMA2/FMUL2) and the output folded to
  // one FMA per element, y = x * A + B with A = rstd * scale and
  // B = shift - mean * A: the kernel was issue-bound (ncu: ~20 issued
  // instructions per element, 46% issue-active, DRAM at 34%).
  __shared__ float red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / WPR, wir = warp % WPR;
  const int row = blockIdx.x * (8 / WPR) + slot;
  const int li = wir * 32 + lane;
  const bool active = row < rows;
  const float4* x4 = reinterpret_cast<const float4*>(X + (size_t)(active ? row : 0) * d);
  float4 v[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = li + 32 * WPR * i;
    v[i] = (active && idx * 4 < d) ? x4[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // Warp-per-row blocks whose 8 rows share one entry stage that entry's
  // scale / shift sums in shared memory once (all 256 threads, while the row
  // loads above are in flight), instead of every warp fetching 2 x d floats
  // from L2 after its reductions.  Same sums, same arithmetic.
  __shared__ float4 coef[2][WPR == 1 ? 32 * VPL : 1];
  const int first = blockIdx.x * (8 / WPR);
  const int last = min(rows - 1, first + 8 / WPR - 1);
  const int e_blk = (a.row0 + first) / rows_per_entry;
  const bool staged = WPR == 1 && e_blk == (a.row0 + last) / rows_per_entry;
  if (staged) {
    const float4* bsc = reinterpret_cast<const float4*>(a.base_scale);
    const float4* bsh = reinterpret_cast<const float4*>(a.base_shift);
    const float4* esc = a.mode == 0 ? reinterpret_cast<const float4*>(a.pe_scale + (size_t)e_blk * a.entry_stride) : nullptr;
    const float4* esh = a.mode == 0 ? reinterpret_cast<const float4*>(a.pe_shift + (size_t)e_blk * a.entry_stride) : nullptr;
    for (int idx = threadIdx.x; idx * 4 < d; idx += blockDim.x) {
      float4 sc = bsc ? __ldg(bsc + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 sh = bsh ? __ldg(bsh + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (esc) {
        const float4 sc2 = __ldg(esc + idx), sh2 = __ldg(esh + idx);
        sc = make_float4(sc.x + sc2.x, sc.y + sc2.y, sc.z + sc2.z, sc.w + sc2.w);
        sh = make_float4(sh.x + sh2.x, sh.y + sh2.y, sh.z + sh2.z, sh.w + sh2.w);
      }
      coef[0][idx] = sc;
      coef[1][idx] = sh;
    }
  }
  if (WPR == 1) __syncthreads();
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    s2 = __fadd2_rn(s2, make_float2(v[i].x, v[i].y));
    s2 = __fadd2_rn(s2, make_float2(v[i].z, v[i].w));
  }
  const float mean = row_reduce<WPR>(s2.x + s2.y, red, slot, wir) / d;
  const float2 nm = make_float2(-mean, -mean);
  float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = li + 32 * WPR * i;
    if (idx * 4 < d) {
      const float2 d01 = __fadd2_rn(make_float2(v[i].x, v[i].y), nm);
      const float2 d23 = __fadd2_rn(make_float2(v[i].z, v[i].w), nm);
      q2 = __ffma2_rn(d01, d01, q2);
      q2 = __ffma2_rn(d23, d23, q2);
    }
  }
  const float rstd = rsqrtf(row_reduce<WPR>(q2.x + q2.y, red, slot, wir) / d + kEps);
  if (!active) return;
  const int e = (a.row0 + row) / rows_per_entry;
  const float4* bsc = reinterpret_cast<const float4*>(a.base_scale);
  const float4* bsh = reinterpret_cast<const float4*>(a.base_shift);
  const float4* esc = a.mode == 0 ? reinterpret_cast<const float4*>(a.pe_scale + (size_t)e * a.entry_stride) : nullptr;
  const float4* esh = a.mode == 0 ? reinterpret_cast<const float4*>(a.pe_shift + (size_t)e * a.entry_stride) : nullptr;
  const float2 r2 = make_float2(rstd, rstd);
  const float one = a.mode == 0 ? 1.0f : 0.0f;
  uint2* o2 = reinterpret_cast<uint2*>(out + (size_t)row * d);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = li + 32 * WPR * i;
    if (idx * 4 >= d) continue;
    // scale = [1 +] base_scale [+ pe_scale[e]], shift = base_shift [+ pe_shift[e]]
    float4 sc, sh;
    if (staged) {
      sc = coef[0][idx];
      sh = coef[1][idx];
    } else {
      sc = bsc ? __ldg(bsc + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
      sh = bsh ? __ldg(bsh + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (esc) {
        const float4 sc2 = __ldg(esc + idx), sh2 = __ldg(esh + idx);
        sc = make_float4(sc.x + sc2.x, sc.y + sc2.y, sc.z + sc2.z, sc.w + sc2.w);
        sh = make_float4(sh.x + sh2.x, sh.y + sh2.y, sh.z + sh2.z, sh.w + sh2.w);
      }
    }
    const float2 A01 = __fmul2_rn(__fadd2_rn(make_float2(sc.x, sc.y), make_float2(one, one)), r2);
    const float2 A23 = __fmul2_rn(__fadd2_rn(make_float2(sc.z, sc.w), make_float2(one, one)), r2);
    const float2 B01 = __ffma2_rn(A01, nm, make_float2(sh.x, sh.y));
    const float2 B23 = __ffma2_rn(A23, nm, make_float2(sh.z, sh.w));
    const float2 y01 = __ffma2_rn(make_float2(v[i].x, v[i].y), A01, B01);
    const float2 y23 = __ffma2_rn(make_float2(v[i].z, v[i].w), A23, B23);
    __nv_bfloat162 lo = __float22bfloat162_rn(y01), hi = __float22bfloat162_rn(y23);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    o2[idx] = pk;
  }
}

// ------------------------------------------------------------ q/k RMSNorm + RoPE
// qkv: (rows, 3d) bf16.  q -> qout (rows, d); k, v -> KV-arena slot of the
// row's entry (token t = row % T).  RMSNorm over the full d with weight,
// eps 1e-6; RoPE on complex pairs (2i, 2i+1) of each 128-wide head, pair i
// < 22 rotates with the global frame index, < 43 with the patch row, else
// the patch column (Wan 44/42/42 split of head_dim 128).  cos/sin come from
// tables precomputed in double precision (rope_table_kernel).
__global__ void rope_table_kernel(float2* tf, int max_frames, float2* th, int hp, float2* tw, int wp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nf = max_frames * 22, nh = hp * 21, nw = wp * 21;
  double ang;
  if (i < nf) {
    ang = (double)(i / 22) * pow(10000.0, -2.0 * (i % 22) / 44.0);
    tf[i] = make_float2((float)cos(ang), (float)sin(ang));
  } else if (i < nf + nh) {
    const int k = i - nf;
    ang = (double)(k / 21) * pow(10000.0, -2.0 * (k % 21) / 42.0);
    th[k] = make_float2((float)cos(ang), (float)sin(ang));
  } else if (i < nf + nh + nw) {
    const int k = i - nf - nh;
    ang = (double)(k / 21) * pow(10000.0, -2.0 * (k % 21) / 42.0);
    tw[k] = make_float2((float)cos(ang), (float)sin(ang));
  }
}

#ifndef BC_QK_MINB
#define BC_QK_MINB 3  // resident CTAs per SM the register budget targets
#endif
template <int VPL, int WPR>  // bf16x8 (16 B) vectors per lane, warps per row
__global__ void __launch_bounds__(256, BC_QK_MINB) qk_norm_rope_kernel(const __nv_bfloat16* __restrict__ qkv, int rows, int d, int T,
                                    QkArgs a) {
  __shared__ float red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / WPR, wir = warp % WPR;
  const int row = blockIdx.x * (8 / WPR) + slot;
  const int li = wir * 32 + lane;
  const bool active = row < rows;
  const int lr = active ? row : 0;            // local row (q / qkv buffers)
  // all of the row's q, k and v loads are issued first -- before the peer
  // wait (which only guards the arena stores) and the RoPE table staging,
  // whose L2 latency then overlaps the row's HBM reads
  const __nv_bfloat16* src = qkv + (size_t)lr * 3 * d;
  uint4 raw[3][VPL];
#pragma unroll
  for (int which = 0; which < 3; ++which) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src + which * d);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int idx = li + 32 * WPR * i;
      raw[which][i] = (active && idx * 8 < d) ? s4[idx] : make_uint4(0u, 0u, 0u, 0u);
    }
  }
  wait_peers_done(a.peer);
  const int rr = a.row0 + lr;                  // global row of the batch
  const int e = rr / T, t = rr % T;
  const int hw = a.hp * a.wp;
  const int fl = t / hw, rem = t % hw;
  const int f = a.frame0[e] + fl, ph = rem / a.wp, pw = rem % a.wp;
  // the row's 64 rotation pairs -- 22 time, 21 height, 21 width -- staged in
  // shared memory once as (cos, sin, -sin, cos), so each pair rotates with
  // one packed multiply and one packed FMA after a single lane-indexed load
  // (a per-element 3-way table select diverges inside every warp).  A lane
  // rotates pairs 4q..4q+3, q = its vector index mod 16; pair 4q+j sits at
  // tab[j][q] so each of the lane's four loads is a conflict-free 256-byte
  // sweep (pair-major order made every load 16-way bank-conflicted and the
  // kernel shared-memory bound)
  __shared__ float4 tab[8][4][16];
  {
    const float2* rf = a.rope_f + (size_t)f * 22;
    const float2* rh = a.rope_h + (size_t)ph * 21;
    const float2* rw = a.rope_w + (size_t)pw * 21;
    for (int pi = li; pi < 64; pi += 32 * WPR) {
      const float2 cs = pi < 22 ? rf[pi] : (pi < 43 ? rh[pi - 22] : rw[pi - 43]);
      tab[slot][pi & 3][pi >> 2] = make_float4(cs.x, cs.y, -cs.y, cs.x);
    }
  }
  __syncthreads();
  const size_t mat = (size_t)T * d;
  __nv_bfloat16* kdst = a.arena + ((size_t)a.mat_base + (size_t)a.slot[e] * 2) * mat + (size_t)t * d;
  __nv_bfloat16* vdst = kdst + mat;
  float inv[2];
#pragma unroll
  for (int which = 0; which < 2; ++which) {
    float2 ss2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[which][i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 x = __bfloat1622float2(h[j]);
        ss2 = __ffma2_rn(x, x, ss2);
      }
    }
    inv[which] = rsqrtf(row_reduce<WPR>(ss2.x + ss2.y, red, slot, wir) / d + kEps);
  }
  if (active) {
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const float* wgt = which == 0 ? a.norm_q : a.norm_k;
      __nv_bfloat16* dst = which == 0 ? a.qout + (size_t)lr * d : kdst;
      const float2 inv2 = make_float2(inv[which], inv[which]);
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int idx = li + 32 * WPR * i;
        if (idx * 8 >= d) continue;
        const int c0 = idx * 8;                 // element index in [0, d)
        const int q4 = idx & 15;                // pairs 4 q4 .. 4 q4 + 3 of the head
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[which][i]);
        const float4 w0 = __ldg(reinterpret_cast<const float4*>(wgt + c0));
        const float4 w1 = __ldg(reinterpret_cast<const float4*>(wgt + c0) + 1);
        const float2 wv[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                              make_float2(w1.z, w1.w)};
        uint4 u;
        uint32_t* o = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // (x0, x1) = h * inv * w; (y0, y1) = (x0 c - x1 s, x0 s + x1 c)
          const float2 x = __fmul2_rn(__fmul2_rn(__bfloat1622float2(h[j]), inv2), wv[j]);
          const float4 cs = tab[slot][j][q4];
          const float2 y = __ffma2_rn(make_float2(x.x, x.x), make_float2(cs.x, cs.y),
                                      __fmul2_rn(make_float2(x.y, x.y), make_float2(cs.z, cs.w)));
          const __nv_bfloat162 yb = __float22bfloat162_rn(y);
          o[j] = *reinterpret_cast<const uint32_t*>(&yb);
        }
        reinterpret_cast<uint4*>(dst)[idx] = u;
        if (which == 1 && a.peer.push) {  // fresh K -> every peer's replica (NVLink P2P store)
          for (int p = 0; p < a.peer.n_peers; ++p)
            reinterpret_cast<uint4*>(a.peer.arena[p] + (dst - a.arena))[idx] = u;
        }
      }
    }
    // v: plain copy into the slot (and the peers' replicas)
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int idx = li + 32 * WPR * i;
      if (idx * 8 >= d) continue;
      reinterpret_cast<uint4*>(vdst)[idx] = raw[2][i];
      if (a.peer.push)
        for (int p = 0; p < a.peer.n_peers; ++p)
          reinterpret_cast<uint4*>(a.peer.arena[p] + (vdst - a.arena))[idx] = raw[2][i];
    }
  }
  if (a.peer.n_peers > 0 && a.peer.push) {
    last_cta_publish(a.peer.ctr, [&] {
      const int e_lo = a.row0 / T, e_hi = (a.row0 + rows - 1) / T;  // entries with rows here
      for (int p = 0; p < a.peer.n_peers; ++p)
        for (int e2 = e_lo; e2 <= e_hi; ++e2)
          st_release_sys(a.peer.flags[p] + (size_t)(a.peer.flag_base + a.slot[e2]) * a.peer.n_ranks + a.peer.my_rank,
                         a.peer.epoch);
    });
  }
}

// RMSNorm * weight over rows of width d (bf16), row stride ld
template <int VPL, int WPR>
__global__ void rms_rows_kernel(__nv_bfloat16* x, int rows, int d, int ld, const float* w,
                                __nv_bfloat16* out, int ld_out) {
  __shared__ float red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / WPR, wir = warp % WPR;
  const int row = blockIdx.x * (8 / WPR) + slot;
  const int li = wir * 32 + lane;
  const bool active = row < rows;
  const uint4* s4 = reinterpret_cast<const uint4*>(x + (size_t)(active ? row : 0) * ld);
  float vals[VPL][8];
  float ss = 0.0f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = li + 32 * WPR * i;
    if (active && idx * 8 < d) {
      uint4 u = s4[idx];
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        vals[i][j] = bf(h[j]);
        ss += vals[i][j] * vals[i][j];
      }
    }
  }
  // warp-per-row blocks stage the weight vector in shared memory once (as
  // ln_rows_kernel does its coefficients) while the row loads are in flight
  // (split by 16-byte half, wsm[h][v] = w[8 v + 4 h .. +4), so a warp's
  // loads are unit-stride: interleaved halves made every load 2-way
  // bank-conflicted)
  __shared__ float4 wsm[2][WPR == 1 ? 32 * VPL : 1];
  if (WPR == 1) {
    for (int i = threadIdx.x; i * 4 < d; i += blockDim.x) wsm[i & 1][i >> 1] = __ldg(reinterpret_cast<const float4*>(w) + i);
    __syncthreads();
  }
  const float inv = rsqrtf(row_reduce<WPR>(ss, red, slot, wir) / d + kEps);
  if (!active) return;
  uint4* d4 = reinterpret_cast<uint4*>(out + (size_t)row * ld_out);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = li + 32 * WPR * i;
    if (idx * 8 >= d) continue;
    // weights as two 16-byte loads (8 scalar loads strided 32 B apart across
    // the warp made this kernel L1-wavefront bound)
    const float4 w0 = WPR == 1 ? wsm[0][idx] : __ldg(reinterpret_cast<const float4*>(w) + 2 * idx);
    const float4 w1 = WPR == 1 ? wsm[1][idx] : __ldg(reinterpret_cast<const float4*>(w) + 2 * idx + 1);
    const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    uint4 u;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&u);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = __float2bfloat16(vals[i][j] * inv * wv[j]);
    d4[idx] = u;
  }
}

// copy a column block of a bf16 matrix: dst[r][0:w] = src[r][c0:c0+w]
__global__ void copy_cols_kernel(const __nv_bfloat16* src, int ld_src, int c0, __nv_bfloat16* dst,
                                 int ld_dst, int rows, int w) {
  const int vecs = w / 8;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < rows * vecs; idx += gridDim.x * blockDim.x) {
    const int r = idx / vecs, c = idx % vecs;
    reinterpret_cast<uint4*>(dst + (size_t)r * ld_dst)[c] =
        reinterpret_cast<const uint4*>(src + (size_t)r * ld_src + c0)[c];
  }
}

__global__ void f32_to_bf16_kernel(const float* src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16(src[i]);
}

// ------------------------------------------------------------ head update
// Y: (T, 64) fp32 head output per entry, index (ph*2+pw)*16 + c (Wan
// unpatchify order).  v -> x0 = x_t - sigma v -> post op.
__global__ void head_update_kernel(const float* __restrict__ Y, int T, int F, int H, int W, UpdArgs u,
                                   int32_t* status) {
  const int e = blockIdx.y;
  const int hp = H / 2, wp = W / 2;
  const int n_el = F * 16 * H * W;
  float* lat = u.latents[e];
  const float sig = (float)(u.level[e] / 1000.0);
  const float s_next = (float)(u.next_level[e] / 1000.0);
  const int post = u.post[e];
  bool bad = false;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n_el; idx += gridDim.x * blockDim.x) {
    const int xw = idx % W, yh = (idx / W) % H, c = (idx / (W * H)) % 16, f = idx / (W * H * 16);
    const int n = f * hp * wp + (yh >> 1) * wp + (xw >> 1);
    const int sub = ((yh & 1) * 2 + (xw & 1)) * 16 + c;
    const float v = Y[((size_t)e * T + n) * 64 + sub];
    const float xt = lat[idx];
    const float x0 = xt - sig * v;
    bad |= !isfinite(x0);
    if (post == 0) {
      lat[idx] = __fadd_rn(__fmul_rn(1.0f - s_next, x0), __fmul_rn(s_next, u.eps[e][idx]));
    } else if (post == 1) {
      lat[idx] = x0;
      u.out[e][idx] = x0;
    } else if (post == 3) {
      u.out[e][idx] = x0;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicCAS(status, 0, 1 + u.block[e]);
  if (u.peer.n_peers > 0) {
    last_cta_publish(u.peer.ctr, [&] {
      for (int p = 0; p < u.peer.n_peers; ++p) st_release_sys(u.peer.done[p] + u.peer.my_rank, u.peer.epoch);
    });
  }
}

// idle rank (no entries this iteration): still publish iteration-done
__global__ void signal_done_kernel(PeerArgs pa) {
  __threadfence_system();
  for (int p = 0; p < pa.n_peers; ++p) st_release_sys(pa.done[p] + pa.my_rank, pa.epoch);
}

__global__ void check_finite_kernel(EntryPtrs lat, int n_el, int32_t* status) {
  const int e = blockIdx.y;
  bool bad = false;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n_el; idx += gridDim.x * blockDim.x)
    bad |= !isfinite(lat.p[e][idx]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicCAS(status, 0, 1 + lat.block[e]);
}

int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

int launch_patchify(const EntryPtrs& lat, int F, int H, int W, int row0, int rows, __nv_bfloat16* out,
                    int32_t* status, cudaStream_t st) {
  const int T = F * (H / 2) * (W / 2);
  patchify_kernel<<<grid_for((int64_t)rows * 64, 256), 256, 0, st>>>(lat, F, H, W, out, T, row0, rows, status);
  BC_LAUNCHED();
  return BC_OK;
}

int launch_gemv(const float* in, int n, int K, const __nv_bfloat16* W, const float* b, float* out, int N, int act,
                float* out2, cudaStream_t st, const TimeArgs* ts, const float* base, int L, float* mod) {
  if (K % 8 || (act == 2 && !out2)) return bc_fail(BC_ERR_CONTRACT, "gemv: K %% 8 != 0 or missing out2");
  if (!in && (!ts || K % 2 || (size_t)n * K * sizeof(float) > 48 * 1024))
    return bc_fail(BC_ERR_CONTRACT, "gemv: the sinusoid input needs timesteps and n * K <= 12288");
  if (mod && (!base || L < 1)) return bc_fail(BC_ERR_CONTRACT, "gemv: modulation tables need base and L");
  const int threads = 256;
  const size_t smem = in ? 0 : (size_t)n * K * sizeof(float);
  const int grid = (N * 32 + threads - 1) / threads;
  if (in)
    gemv_kernel<false><<<grid, threads, 0, st>>>(in, n, K, W, b, out, N, act, out2, TimeArgs{}, base, L, mod);
  else
    gemv_kernel<true><<<grid, threads, smem, st>>>(in, n, K, W, b, out, N, act, out2, *ts, base, L, mod);
  BC_LAUNCHED();
  return BC_OK;
}

// rows of <= 12 float4 per lane run warp-per-row; wider rows (14B: d=5120)
// spread over 4 warps so registers stay ~80/thread and occupancy high.
int launch_ln_rows(const float* X, __nv_bfloat16* out, int rows, int d, int rows_per_entry, const LnArgs& a,
                   cudaStream_t st) {
  const int v4 = d / 4;
  if (v4 <= 32 * 12) {
    ln_rows_kernel<12, 1><<<(rows + 7) / 8, 256, 0, st>>>(X, out, rows, d, rows_per_entry, a);
  } else if (v4 <= 4 * 32 * 12) {
    ln_rows_kernel<12, 4><<<(rows + 1) / 2, 256, 0, st>>>(X, out, rows, d, rows_per_entry, a);
  } else {
    return bc_fail(BC_ERR_CONTRACT, "ln_rows: d=%d too wide", d);
  }
  BC_LAUNCHED();
  return BC_OK;
}

int launch_qk_norm_rope(const __nv_bfloat16* qkv, int rows, int d, int T, const QkArgs& a, cudaStream_t st) {
  const int v8 = d / 8;
  // 3 vectors per lane per matrix (q, k, v all in flight: 36 registers of
  // payload) keeps ~80 registers and 3 CTAs per SM
  if (v8 <= 2 * 32 * 3) {
    qk_norm_rope_kernel<3, 2><<<(rows + 3) / 4, 256, 0, st>>>(qkv, rows, d, T, a);
  } else if (v8 <= 8 * 32 * 3) {
    qk_norm_rope_kernel<3, 8><<<rows, 256, 0, st>>>(qkv, rows, d, T, a);
  } else {
    return bc_fail(BC_ERR_CONTRACT, "qk_norm_rope: d=%d too wide", d);
  }
  BC_LAUNCHED();
  return BC_OK;
}

int launch_rms_rows(__nv_bfloat16* x, int rows, int d, int ld, const float* w, __nv_bfloat16* out, int ld_out,
                    cudaStream_t st) {
  const int v8 = d / 8;
  if (v8 <= 32 * 6) {
    rms_rows_kernel<6, 1><<<(rows + 7) / 8, 256, 0, st>>>(x, rows, d, ld, w, out, ld_out);
  } else if (v8 <= 4 * 32 * 6) {
    rms_rows_kernel<6, 4><<<(rows + 1) / 2, 256, 0, st>>>(x, rows, d, ld, w, out, ld_out);
  } else {
    return bc_fail(BC_ERR_CONTRACT, "rms_rows: d=%d too wide", d);
  }
  BC_LAUNCHED();
  return BC_OK;
}

int launch_copy_cols(const __nv_bfloat16* src, int ld_src, int c0, __nv_bfloat16* dst, int ld_dst, int rows,
                     int w, cudaStream_t st) {
  copy_cols_kernel<<<grid_for((int64_t)rows * w / 8, 256), 256, 0, st>>>(src, ld_src, c0, dst, ld_dst, rows, w);
  BC_LAUNCHED();
  return BC_OK;
}

int launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t st) {
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(src, dst, n);
  BC_LAUNCHED();
  return BC_OK;
}

int launch_head_update(const float* Y, int n, int T, int F, int H, int W, const UpdArgs& u, int32_t* status,
                       cudaStream_t st) {
  const int n_el = F * 16 * H * W;
  head_update_kernel<<<dim3(grid_for(n_el, 256) / n + 1, n), 256, 0, st>>>(Y, T, F, H, W, u, status);
  BC_LAUNCHED();
  return BC_OK;
}

int launch_rope_tables(float2* tf, int max_frames, float2* th, int hp, float2* tw, int wp, cudaStream_t st) {
  const int n = max_frames * 22 + (hp + wp) * 21;
  rope_table_kernel<<<(n + 255) / 256, 256, 0, st>>>(tf, max_frames, th, hp, tw, wp);
  BC_LAUNCHED();
  return BC_OK;
}

__global__ void flag_writes_kernel(FlagWrites f) {
  __threadfence_system();
  for (int i = 0; i < f.n; ++i) st_release_sys(f.addr[i], f.v);
}

int launch_flag_writes(const FlagWrites& f, cudaStream_t st) {
  flag_writes_kernel<<<1, 1, 0, st>>>(f);
  BC_LAUNCHED();
  return BC_OK;
}

int launch_signal_done(const PeerArgs& p, cudaStream_t st) {
  signal_done_kernel<<<1, 1, 0, st>>>(p);
  BC_LAUNCHED();
  return BC_OK;
}

int launch_check_finite(const EntryPtrs& lat, int n, int n_el, int32_t* status, cudaStream_t st) {
  check_finite_kernel<<<dim3(grid_for(n_el, 256) / n + 1, n), 256, 0, st>>>(lat, n_el, status);
  BC_LAUNCHED();
  return BC_OK;
}


}  // namespace bc
