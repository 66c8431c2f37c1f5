// tcgen05 flash attention over the paged KV arena (self-attention of the
// cascade) or a dense K/V (text cross-attention).
//
// Semantics = reference layer_attend + _gather (denoiser.py:264-296):
// for the queries of batch entry e, keys/values are the concatenation of the
// visible blocks' K/V in ascending block order -- here the arena slots
// vis_slot[e][0..n_vis) in that order -- and softmax runs over exactly those
// keys.  Key tiles are consumed strictly in that order (no split-K, no
// atomics), so an entry's result does not depend on which other entries
// share the launch.
//
// One CTA = two 128-row query tiles (A, B) x one head x one entry, so the
// tensor core always has the other tile's work while one tile's softmax runs
// on the MUFU/FMA pipes (ping-pong).
//   warp 0     TMA: Q_A, Q_B once; then K_j, V_j through a 3-slot ring
//   warp 1     MMA: S_X = Q_X K_j^T -> TMEM, O_X += P_X V_j (P from smem,
//              V MN-major), X in {A, B}
//   warps 4-7  softmax/correction/epilogue of tile A (thread = query row)
//   warps 8-11 same for tile B
// Online softmax with lazy rescale: the reference max only moves when the
// running max grows by more than 2^8, so O (in TMEM) is rarely rescaled.
// TMEM columns: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <queue>
#include <utility>
#include <vector>

#include "attention.h"
#include "bc_common.h"
#include "sm100.cuh"

#ifdef BC_ATTN_TRACE
unsigned long long* bc_attn_trace_ptr = nullptr;
extern "C" int bc_attn_trace_read(unsigned long long* host) {
  if (!bc_attn_trace_ptr) return 1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, bc_attn_trace_ptr, (32 * 64 + 256 * 8) * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 0;
}
#endif

namespace bc {
namespace {

constexpr int kRows = 128;            // query rows per tile
constexpr int kKeys = 128;            // keys per K/V tile
constexpr int kHd = 128;              // head dim
constexpr int kHalf = 128 * 64 * 2;   // 64-column half of a 128x128 bf16 tile (16 KB)
constexpr int kTile = 2 * kHalf;      // 32 KB
constexpr int kRing = 3;              // K/V ring slots
constexpr int kThreads = 384;
constexpr float kRescaleThresh = 8.0f;  // log2 domain
// setmaxnreg only moves registers inside the CTA's launch allocation
// (384 x 168): the softmax warps' increase must be covered by what the
// control warpgroup releases (128 x (168 - 56) = 256 x (224 - 168)), or the
// increasing warps block forever
constexpr int kRegsLaunch = 168;
constexpr int kRegsCtl = 56;
constexpr int kRegsSoftmax = 224;
static_assert(128 * (kRegsLaunch - kRegsCtl) >= 256 * (kRegsSoftmax - kRegsLaunch), "register split");
#ifndef BC_ATTN_SCHED_POLY
#define BC_ATTN_SCHED_POLY 0
#endif
constexpr int kDefaultPoly = 0;
constexpr int kSchedPoly = BC_ATTN_SCHED_POLY;  // FMA-pipe exp pairs (of 8) in the balanced kernel

struct Smem {
  static constexpr int qa = 0;
  static constexpr int qb = qa + kTile;
  static constexpr int ring = qb + kTile;
  static constexpr int pa = ring + kRing * kTile;
  static constexpr int pb = pa + kTile;
  static constexpr int bars = pb + kTile;
  static constexpr int total = bars + 256;
};

__device__ __forceinline__ float ex2(float x) {
#ifdef BC_ATTN_FAKE_EXP  // timing experiment only (wrong numerics): no MUFU
  return fmaf(x, 0.0009765625f, 1.0f);
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}

// 3-input max (FMNMX3, sm_100+): halves the ALU ops of the row max
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// packed fp32x2 (FFMA2 / FADD2, sm_100+): half the FMA-pipe instructions
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_split(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// 2^x for a pair on the FMA pipe (Cody-Waite split + degree-3 minimax on
// [-0.5, 0.5], max rel. error 7.7e-5 << bf16's 3.9e-3; packed FFMA2/FADD2,
// ~6 FMA-pipe instructions per pair) to offload part of the MUFU work, which
// is 16 ex2/clk/SM (measured, scripts/mufu_probe.cu).  Off by default
// (BC_ATTN_POLY): measured no faster, see profiles/README.md.
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  const uint64_t x = f2(fmaxf(x0, -126.0f), fmaxf(x1, -126.0f));
  const uint64_t t = fadd2(x, f2(kMagic, kMagic));
  const uint64_t n = fadd2(t, f2(-kMagic, -kMagic));
  const uint64_t fr = ffma2(n, f2(-1.0f, -1.0f), x);
  uint64_t p = ffma2(f2(0.05508868380751114f, 0.05508868380751114f), fr,
                     f2(0.24260405145947936f, 0.24260405145947936f));
  p = ffma2(p, fr, f2(0.6932762416819607f, 0.6932762416819607f));
  p = ffma2(p, fr, f2(0.9999289403695112f, 0.9999289403695112f));
  float p0, p1, t0, t1;
  f2_split(p, p0, p1);
  f2_split(t, t0, t1);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// Diagnostic timeline (BC_ATTN_TRACE builds only): CTA (0,0,0) records
// clock64() at protocol points into prm.trace[slot*64 + j].
#ifdef BC_ATTN_TRACE
#define ATRACE(slot, j)                                                                       \
  do {                                                                                        \
    if (prm.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane_id() == 0 && \
        (j) < 64)                                                                             \
      prm.trace[(slot) * 64 + (j)] = clock64();                                               \
  } while (0)
#else
#define ATRACE(slot, j) \
  do {                  \
  } while (0)
#endif

// Ring positions: K_0 -> 0, K_m -> 2m-1 (m >= 1); V_m -> 2m+2, except the
// last V_{n-1} -> 2n-1.  (Emission order K0 K1 V0 K2 V1 ... K_{n-1} V_{n-2} V_{n-1}.)
__device__ __forceinline__ int kpos(int m) { return m == 0 ? 0 : 2 * m - 1; }
__device__ __forceinline__ int vpos(int m, int n) { return m == n - 1 ? 2 * n - 1 : 2 * m + 2; }
__device__ __forceinline__ void ring_item(int i, int n, int& j, int& is_v) {
  if (i == 0) {
    j = 0;
    is_v = 0;
  } else if (i == 2 * n - 1) {
    j = n - 1;
    is_v = 1;
  } else if (i & 1) {  // odd positions are K_{(i+1)/2}
    j = (i + 1) >> 1;
    is_v = 0;
  } else {             // even positions >= 2 are V_{(i-2)/2}
    j = (i - 2) >> 1;
    is_v = 1;
  }
}

struct SoftmaxBars {
  uint64_t* s_full;
  uint64_t* s_empty;
  uint64_t* p_full;
  uint64_t* o_ready;
  // CTA-pair kernel: s_empty / p_full / o_free live in the LEADER CTA and
  // count one elected arrival per warp of both CTAs (cluster addresses)
  uint32_t s_empty_cl = 0, p_full_cl = 0, o_free_cl = 0;
};

// arrive on a softmax-side barrier: every thread locally (count 128), or one
// elected lane per warp on the leader's barrier (CTA pairs, count 8)
__device__ __forceinline__ void sm_arrive(uint64_t* local, uint32_t cluster_addr) {
  if (cluster_addr) {
    __syncwarp();
    if (lane_id() == 0) cl_arrive(cluster_addr);
  } else {
    mbar_arrive(local);
  }
}


// One softmax warpgroup: 128 threads, thread <-> query row of its tile.
template <int kPoly>
__device__ __forceinline__ void softmax_tile(const AttnParams& prm, uint32_t tmem_s, uint32_t tmem_o,
                                             uint8_t* sp, SoftmaxBars b, int n_tiles, int tiles_per_slot,
                                             uint32_t quad, int q_tok0, int e, int head, int tile_x,
                                             uint32_t jb = 0, uint64_t* o_free = nullptr,
                                             const CUtensorMap* map_o = nullptr) {
  const uint32_t row = quad * 32 + lane_id();
  const uint32_t lane_base = (quad * 32) << 16;
  const float c = prm.scale * 1.4426950408889634f;
  const uint32_t sp_u32 = smem_u32(sp);
  float m_used = -INFINITY, l_sum = 0.0f;
  int t0 = 0;  // first key of tile j within its visible block
  for (int j = 0; j < n_tiles; ++j, t0 = (t0 + kKeys < prm.kv_tokens) ? t0 + kKeys : 0) {
    const int valid = min(kKeys, prm.kv_tokens - t0);
    mbar_wait(b.s_full, (jb + j) & 1);
    if ((quad) == 0) ATRACE(0 + tile_x * 8, j);
    tc_fence_after();
    float s[128];
    {  // all four 32-column loads in flight, one wait
      uint32_t r[4][32];
#pragma unroll
      for (int k = 0; k < 4; ++k) tmem_ld32(tmem_s + lane_base + k * 32, r[k]);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 32; ++i) s[k * 32 + i] = __uint_as_float(r[k][i]);
    }
    tc_fence_before();
    sm_arrive(b.s_empty, b.s_empty_cl);  // S buffer may now be overwritten by the next QK^T
    if (quad == 0) ATRACE(4 + tile_x * 8, j);
#ifdef BC_ATTN_NOSOFTMAX  // timing experiment only: MMA/TMA skeleton
    if (j > 0) mbar_wait(b.o_ready, (j - 1) & 1);
    if (s[5] == 1234.5f) l_sum += 1.0f;
#ifdef BC_ATTN_SKEL_STS  // + the P stores: does the smem write traffic cost tensor time?
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int half = q >> 3, ch = q & 7;
      sts128(sp_u32 + half * kHalf + row * 128 + ((ch ^ (row & 7)) << 4), __float_as_uint(s[8 * q]),
             __float_as_uint(s[8 * q + 1]), __float_as_uint(s[8 * q + 2]), __float_as_uint(s[8 * q + 3]));
    }
#endif
    fence_async_shared();
    tc_fence_before();
    sm_arrive(b.p_full, b.p_full_cl);
    continue;
#endif
    if (valid < kKeys) {     // ragged last tile of a slot (warp-uniform)
#pragma unroll
      for (int i = 0; i < 128; ++i)
        if (i >= valid) s[i] = -INFINITY;
    }
    // row max as 8 independent FMNMX3 chains (a single fmaxf chain is a
    // 128-deep dependency: ~500 cycles of latency on the softmax critical path)
    auto row_max = [&]() {
      float m8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = fmax3(s[k], s[8 + k], s[16 + k]);
#pragma unroll
      for (int i = 24; i < 120; i += 16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], s[i + k], s[i + 8 + k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[120 + k]);
      return fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
    };
    float alpha = 1.0f;
    bool bump;
    {
#ifdef BC_ABL_MAX  // timing ablation only: no row max
      const float mt = s[0] * c;
#else
      const float mt = row_max() * c;
#endif
      bump = (j == 0) || (mt > m_used + kRescaleThresh);
      if (bump) {
        const float m_new = fmaxf(m_used, mt);
        alpha = (j == 0) ? 0.0f : ex2(m_used - m_new);
        m_used = m_new;
      }
    }
    // P = 2^(s*c - m) -> packed bf16 in registers (s dies as P is formed)
    uint64_t sum2[2] = {0ull, 0ull};  // (+0.0f, +0.0f) pairs
    const uint64_t c2 = f2(c, c), nm2 = f2(-m_used, -m_used);
    uint32_t pk[64];
    if (quad == 0) ATRACE(1 + tile_x * 8, j);
    if (valid == kKeys) {
#pragma unroll
      for (int t = 0; t < 64; ++t) {
        float x0, x1, p0, p1;
        f2_split(ffma2(f2(s[2 * t], s[2 * t + 1]), c2, nm2), x0, x1);
        if (((t * kPoly) & 7) < kPoly) {  // kPoly of every 8 pairs, spread out
          ex2_poly2(x0, x1, p0, p1);
        } else {
          p0 = ex2(x0);
          p1 = ex2(x1);
        }
        const uint64_t pp = f2(p0, p1);
#ifndef BC_ABL_SUM  // timing ablation only: no row sum
        sum2[t & 1] = fadd2(sum2[t & 1], pp);
#endif
#ifdef BC_ABL_PACK  // timing ablation only: no bf16 conversion
        pk[t] = __float_as_uint(p0) ^ __float_as_uint(p1);
#else
        pk[t] = pack_bf16(p0, p1);
#endif
      }
    } else {
#pragma unroll
      for (int t = 0; t < 64; ++t) {
        float x0, x1;
        f2_split(ffma2(f2(s[2 * t], s[2 * t + 1]), c2, nm2), x0, x1);
        const float p0 = ex2(x0);
        const float p1 = ex2(x1);
        sum2[t & 1] = fadd2(sum2[t & 1], f2(p0, p1));
        pk[t] = pack_bf16(p0, p1);
      }
    }
    if (quad == 0) ATRACE(2 + tile_x * 8, j);
    // PV(j-1) must be complete before O is rescaled or P is overwritten
#ifdef BC_ABL_OWAIT  // timing ablation only (races): no wait for PV(j-1)
    if (false) {
#else
    if (j > 0) {
#endif
      mbar_wait(b.o_ready, (jb + j - 1) & 1);
      tc_fence_after();
      if (quad == 0) ATRACE(5 + tile_x * 8, j);
      if (__any_sync(0xffffffffu, bump)) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t r[32];
          tmem_ld32(tmem_o + lane_base + k * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st32(tmem_o + lane_base + k * 32, r);
        }
        tmem_st_wait();
      }
    }
    // map_o: the previous item's O tile left this P buffer by TMA; it must
    // have been read out before the first P of this item overwrites it
    if (map_o && j == 0) {
      if (row == 0) bulk_wait_read<0>();
      named_bar_sync(1 + tile_x, 128);
    }
    // P -> smem in the UMMA K-major SW128 layout: half h holds keys
    // [64h, 64h+64); 16-byte chunk q of row r sits at chunk (q ^ (r & 7)).
#ifndef BC_ABL_STS  // timing ablation only: no P stores
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int half = q >> 3, ch = q & 7;
      sts128(sp_u32 + half * kHalf + row * 128 + ((ch ^ (row & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2],
             pk[4 * q + 3]);
    }
#else
    if (pk[5] == 0x12345u) sts128(sp_u32 + row * 16, pk[0], pk[1], pk[2], pk[3]);
#endif
    float sa, sb, sc, sd;
    f2_split(sum2[0], sa, sb);
    f2_split(sum2[1], sc, sd);
    l_sum = l_sum * alpha + ((sa + sc) + (sb + sd));
    fence_async_shared();
    tc_fence_before();
    sm_arrive(b.p_full, b.p_full_cl);
    if (quad == 0) ATRACE(3 + tile_x * 8, j);
  }
  // epilogue: O / l -> bf16
  if (n_tiles > 0) {
    mbar_wait(b.o_ready, (jb + n_tiles - 1) & 1);
    tc_fence_after();
  }
  const int qtok = q_tok0 + (int)row;
  const bool live = qtok < prm.q_hi[e];
  const float inv = (l_sum > 0.0f) ? 1.0f / l_sum : 0.0f;
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(prm.out) +
                       ((size_t)(prm.q_row[e] + qtok - prm.q_lo[e]) * prm.heads + head) * kHd;
  // all four 32-column loads of O in flight, one wait (the epilogue sits
  // between a work item's last PV and the next item's first P)
  uint32_t r[4][32];
#pragma unroll
  for (int k = 0; k < 4; ++k) tmem_ld32(tmem_o + lane_base + k * 32, r[k]);
  tmem_ld_wait();
  if (map_o && n_tiles > 0 && q_tok0 + kRows <= prm.q_hi[e]) {
    // whole tile: stage the bf16 rows in this tile's P buffer (free: the
    // last PV is complete) in the SW128 layout and store them with two TMA
    // boxes -- 16 shared stores per thread instead of 16 global stores that
    // each touch 32 rows; one thread waits for the read before the next
    // item's first P store (above)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int k = q >> 2, o = 8 * (q & 3);
      const int half = q >> 3, ch = q & 7;
      sts128(sp_u32 + half * kHalf + row * 128 + ((ch ^ (row & 7)) << 4),
             pack_bf16(__uint_as_float(r[k][o + 0]) * inv, __uint_as_float(r[k][o + 1]) * inv),
             pack_bf16(__uint_as_float(r[k][o + 2]) * inv, __uint_as_float(r[k][o + 3]) * inv),
             pack_bf16(__uint_as_float(r[k][o + 4]) * inv, __uint_as_float(r[k][o + 5]) * inv),
             pack_bf16(__uint_as_float(r[k][o + 6]) * inv, __uint_as_float(r[k][o + 7]) * inv));
    }
    fence_async_shared();
    named_bar_sync(1 + tile_x, 128);
    if (row == 0) {
      const int orow = prm.q_row[e] + q_tok0 - prm.q_lo[e];
      tma_store_3d(map_o, sp, 0, head, orow);
      tma_store_3d(map_o, sp + kHalf, 64, head, orow);
      bulk_commit();
    }
  } else if (live) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint4* dst = reinterpret_cast<uint4*>(out + k * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v;
        v.x = pack_bf16(__uint_as_float(r[k][8 * q + 0]) * inv, __uint_as_float(r[k][8 * q + 1]) * inv);
        v.y = pack_bf16(__uint_as_float(r[k][8 * q + 2]) * inv, __uint_as_float(r[k][8 * q + 3]) * inv);
        v.z = pack_bf16(__uint_as_float(r[k][8 * q + 4]) * inv, __uint_as_float(r[k][8 * q + 5]) * inv);
        v.w = pack_bf16(__uint_as_float(r[k][8 * q + 6]) * inv, __uint_as_float(r[k][8 * q + 7]) * inv);
        dst[q] = v;
      }
    }
  }
  if (o_free) {  // O is read out: the next work item's first PV may overwrite it
    tc_fence_before();
    sm_arrive(o_free, b.o_free_cl);
  }
}

template <int kPoly>
__global__ void __launch_bounds__(kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                AttnParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* q_full = bars + 0;
  uint64_t* ring_full = bars + 1;   // [3]
  uint64_t* ring_empty = bars + 4;  // [3]
  uint64_t* s_full = bars + 7;      // [2] (A, B)
  uint64_t* s_empty = bars + 9;     // [2]
  uint64_t* p_full = bars + 11;     // [2]
  uint64_t* o_ready = bars + 13;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  // grid: x = query-tile pair, y = entry, z = head (concurrent CTAs share a
  // head's K/V in L2)
  const int pair = blockIdx.x, e = blockIdx.y, head = blockIdx.z;
  const int q0 = prm.q_lo[e] + pair * 2 * kRows;  // first query token of tile A
  if (q0 >= prm.q_hi[e]) return;                  // this entry has fewer tiles here
  const bool has_b = q0 + kRows < prm.q_hi[e];
  const int n_vis = prm.n_vis[e];
  const int tiles_per_slot = (prm.kv_tokens + kKeys - 1) / kKeys;
  const int n_tiles = n_vis * tiles_per_slot;
  const uint32_t warp = warp_id();

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_kv);
    mbar_init(q_full, 1);
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&ring_full[i], 1);
      mbar_init(&ring_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_ready[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // register split (setmaxnreg, per warpgroup, inside each role's branch so
  // the allocator sees disjoint regions): the TMA/MMA warpgroup needs few
  // registers, the softmax warpgroups hold a 128-float score row + 64 packed
  // P words per thread
  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
  if (warp == 0) {
    if (lane_id() == 0) {
      const int qrow = prm.q_row[e] + (q0 - prm.q_lo[e]);
      mbar_arrive_expect_tx(q_full, has_b ? 2 * kTile : kTile);
      tma_load_3d(smem + Smem::qa, &map_q, q_full, 0, head, qrow);
      tma_load_3d(smem + Smem::qa + kHalf, &map_q, q_full, 64, head, qrow);
      if (has_b) {
        tma_load_3d(smem + Smem::qb, &map_q, q_full, 0, head, qrow + kRows);
        tma_load_3d(smem + Smem::qb + kHalf, &map_q, q_full, 64, head, qrow + kRows);
      }
      // ring order K0 K1 V0 K2 V1 K3 V2 ... (K runs one tile ahead of V, see
      // ring_pos): K_{j+1} is consumed in the same period as V_j, so with
      // this order every load has about one period of prefetch slack in a
      // 3-slot ring.
      for (int i = 0; i < 2 * n_tiles; ++i) {
        int j, is_v;
        ring_item(i, n_tiles, j, is_v);
        const int slot = i % kRing;
        const uint32_t ph = (i / kRing) & 1;
        const int kv_slot = prm.vis_slot[e][j / tiles_per_slot];
        const int t0 = (j % tiles_per_slot) * kKeys;
        const int mat = prm.mat_base + kv_slot * prm.mat_stride + (is_v ? prm.v_offset : 0);
        if (!is_v && prm.flags && (j % tiles_per_slot) == 0) {
          const uint32_t need = prm.need[e][j / tiles_per_slot];
          if (need) {  // K/V rows of this block come from peer GPUs: wait for each producer
            const uint32_t ep = need >> 8;
            const uint32_t* f = prm.flags + (size_t)(prm.flag_base + kv_slot) * prm.n_ranks;
            for (uint32_t m = need & 0xffu; m; m &= m - 1) {
              spin_until_geq(f + (__ffs(m) - 1), ep, 256);
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        }
        mbar_wait(&ring_empty[slot], ph ^ 1);
        mbar_arrive_expect_tx(&ring_full[slot], kTile);
        uint8_t* dst = smem + Smem::ring + slot * kTile;
        tma_load_4d(dst, &map_kv, &ring_full[slot], 0, head, t0, mat);
        tma_load_4d(dst + kHalf, &map_kv, &ring_full[slot], 64, head, t0, mat);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_qk = idesc_bf16(kRows, kKeys);
    constexpr uint32_t idesc_pv = idesc_bf16(kRows, kHd, 0, 1);  // B (= V) MN-major
    const uint32_t sq[2] = {smem_u32(smem + Smem::qa), smem_u32(smem + Smem::qb)};
    const uint32_t sp[2] = {smem_u32(smem + Smem::pa), smem_u32(smem + Smem::pb)};
    const int n_q = has_b ? 2 : 1;
    auto ring_slot = [&](int i) { return smem_u32(smem + Smem::ring + (i % kRing) * kTile); };
    auto issue_qk = [&](int x, int j) {  // S_x = Q_x K_j^T ; K_j is ring item 2j
      if (elect_one()) {
        const uint32_t sk = ring_slot(kpos(j));
#pragma unroll
        for (int k = 0; k < kHd / 16; ++k) {
          const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
          mma_bf16_ss(tmem + x * 128, desc_sw128(sq[x] + off, 16, 1024), desc_sw128(sk + off, 16, 1024),
                      idesc_qk, k != 0);
        }
        mma_commit(&s_full[x]);
      }
      __syncwarp();
    };
    // O_x += P_x V_j over keys [16 k0, 16 k1) ; V_j is ring item vpos(j)
    auto issue_pv = [&](int x, int j, int k0, int k1) {
      if (elect_one()) {
        const uint32_t sv = ring_slot(vpos(j, n_tiles));
#pragma unroll
        for (int k = k0; k < k1; ++k) {
          const uint32_t aoff = (k >> 2) * kHalf + (k & 3) * 32;
          mma_bf16_ss(tmem + 256 + x * 128, desc_sw128(sp[x] + aoff, 16, 1024),
                      desc_sw128(sv + k * 2048, kHalf, 1024), idesc_pv, (j | k) != 0);
        }
        if (k1 == kKeys / 16) mma_commit(&o_ready[x]);
      }
      __syncwarp();
    };
    auto release = [&](int i) {
      if (elect_one()) mma_commit(&ring_empty[i % kRing]);
      __syncwarp();
    };
    // Issue order per key tile j: S_A(j+1), O_A += P_A(j) V_j, S_B(j+1),
    // O_B += P_B(j) V_j.  Issuing PV_A before QK_B lets softmax A (which waits
    // for PV_A(j) before overwriting P_A) start tile j+1 earlier; measured
    // faster than issuing both QKs first or an event-driven polling issuer.
    auto ring_wait = [&](int i) { mbar_wait(&ring_full[i % kRing], (i / kRing) & 1); };
    mbar_wait(q_full, 0);
    if (n_tiles > 0) {
      ring_wait(0);
      tc_fence_after();
      for (int x = 0; x < n_q; ++x) issue_qk(x, 0);
      release(0);
    }
    for (int j = 0; j < n_tiles; ++j) {
      const bool next = j + 1 < n_tiles;
      for (int x = 0; x < n_q; ++x) {
        if (next) {
          mbar_wait(&s_empty[x], j & 1);  // softmax x has read S_x(j)
          ATRACE(16 + x * 4, j);
          if (x == 0) ring_wait(kpos(j + 1));
          if (x == 0) ATRACE(24, j);
          tc_fence_after();
          issue_qk(x, j + 1);
          ATRACE(17 + x * 4, j);
          // K_{j+1} is free once the last tile's QK^T on it completes:
          // release it now (not after PV_B(j)) so the TMA refills its ring
          // slot (with V_{j+1}) one MMA group earlier
          if (x == n_q - 1) release(kpos(j + 1));
        }
        mbar_wait(&p_full[x], j & 1);
        ATRACE(18 + x * 4, j);
        if (x == 0) ring_wait(vpos(j, n_tiles));
        if (x == 0) ATRACE(25, j);
        tc_fence_after();
        issue_pv(x, j, 0, kKeys / 16);
        ATRACE(19 + x * 4, j);
      }
      release(vpos(j, n_tiles));
    }
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    const int x = (warp >= 8) ? 1 : 0;
    if (x == 0 || has_b) {
      SoftmaxBars b{&s_full[x], &s_empty[x], &p_full[x], &o_ready[x]};
      softmax_tile<kPoly>(prm, tmem + x * 128, tmem + 256 + x * 128, smem + (x ? Smem::pb : Smem::pa), b, n_tiles,
                   tiles_per_slot, warp & 3, q0 + x * kRows, e, head, x);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// CTA-pair variant (cluster of 2 on one TPC, tcgen05 cta_group::2): the two
// CTAs hold two 128-row query tiles each (4 tiles = 512 query rows of one
// entry and head per cluster) and share every K/V tile: QK^T runs as M=256
// MMAs with the key tile's 128 rows split 64 / 64 across the pair, PV as
// M=256 MMAs with V's 128 head-dim columns split 64 / 64.  Each CTA loads
// only ITS half of every K/V tile (16 KB instead of 32 KB per tile), so the
// L2 -> SM traffic, the TMA shared-memory writes and the tensor core's
// B-operand reads per SM halve -- measured, halving the K/V bytes (numerics
// aside, BC_ABL_HALFKV) lets the power-capped GPU clock 8% higher.  The
// leader CTA issues all MMAs; TMA loads of both CTAs complete on the
// leader's barriers; MMA completions are multicast to both CTAs; each CTA's
// softmax warps signal the leader with one elected arrival per warp.
// Per-row arithmetic and key order are those of attn_kernel (the pair MMA
// computes each output element as the single-CTA one does): bit-identical.
constexpr int kRingP = 6;                 // half-tile ring slots (16 KB each)
constexpr int kItemP = 16 * 1024;         // a CTA's half of a K or V tile
constexpr int kHalfK = 64 * 128;          // one 64-column d-half of a 64-key K half-tile (8 KB)
static_assert(Smem::pa - Smem::ring == kRingP * kItemP, "pair ring fits the single-CTA ring");

template <int kPoly>
__global__ void __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kh,
                     const __grid_constant__ CUtensorMap map_kv, AttnParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* q_full = bars + 0;
  uint64_t* ring_full = bars + 1;    // [6] (leader's are the ones waited on)
  uint64_t* ring_empty = bars + 7;   // [6] (both CTAs: multicast commits)
  uint64_t* s_full = bars + 13;      // [2] (both CTAs)
  uint64_t* s_empty = bars + 15;     // [2] (leader: 8 warp arrivals)
  uint64_t* p_full = bars + 17;      // [2] (leader: 8 warp arrivals)
  uint64_t* o_ready = bars + 19;     // [2] (both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const uint32_t rank = cl_rank();
  const bool leader = rank == 0;
  const int item = blockIdx.x >> 1, e = blockIdx.y, head = blockIdx.z;
  if (prm.q_lo[e] + item * 4 * kRows >= prm.q_hi[e]) return;  // same decision in both CTAs
  const int q0 = prm.q_lo[e] + (item * 4 + (int)rank * 2) * kRows;  // this CTA's tile A (B = +128)
  const int n_vis = prm.n_vis[e];
  const int tiles_per_slot = (prm.kv_tokens + kKeys - 1) / kKeys;
  const int n_tiles = n_vis * tiles_per_slot;
  const uint32_t warp = warp_id();

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_kh);
    tma_prefetch(&map_kv);
    mbar_init(q_full, 1);
    for (int i = 0; i < kRingP; ++i) {
      mbar_init(&ring_full[i], 1);
      mbar_init(&ring_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&o_ready[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cl_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
  if (warp == 0) {
    if (lane_id() == 0) {
      // Q: both CTAs' two tiles complete on the leader's q_full (absent
      // tiles load rows past the entry, or TMA's zero fill, and are never
      // stored)
      const uint32_t lq = cl_map(q_full, 0);
      if (leader) mbar_arrive_expect_tx(q_full, 2 * 2 * kTile);
      const int qrow = prm.q_row[e] + (q0 - prm.q_lo[e]);
      tma_load_3d_pair(smem + Smem::qa, &map_q, lq, 0, head, qrow);
      tma_load_3d_pair(smem + Smem::qa + kHalf, &map_q, lq, 64, head, qrow);
      tma_load_3d_pair(smem + Smem::qb, &map_q, lq, 0, head, qrow + kRows);
      tma_load_3d_pair(smem + Smem::qb + kHalf, &map_q, lq, 64, head, qrow + kRows);
      for (int i = 0; i < 2 * n_tiles; ++i) {
        int j, is_v;
        ring_item(i, n_tiles, j, is_v);
        const int slot = i % kRingP;
        const uint32_t ph = (i / kRingP) & 1;
        const int kv_slot = prm.vis_slot[e][j / tiles_per_slot];
        const int t0 = (j % tiles_per_slot) * kKeys;
        const int mat = prm.mat_base + kv_slot * prm.mat_stride + (is_v ? prm.v_offset : 0);
        if (!is_v && prm.flags && (j % tiles_per_slot) == 0) {
          const uint32_t need = prm.need[e][j / tiles_per_slot];
          if (need) {  // K/V rows of this block come from peer GPUs: wait for each producer
            const uint32_t ep = need >> 8;
            const uint32_t* f = prm.flags + (size_t)(prm.flag_base + kv_slot) * prm.n_ranks;
            for (uint32_t m = need & 0xffu; m; m &= m - 1) spin_until_geq(f + (__ffs(m) - 1), ep, 256);
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        }
        mbar_wait(&ring_empty[slot], ph ^ 1);
        const uint32_t lb = cl_map(&ring_full[slot], 0);
        if (leader) mbar_arrive_expect_tx(&ring_full[slot], 2 * kItemP);
        uint8_t* dst = smem + Smem::ring + slot * kItemP;
        if (!is_v) {  // K: this CTA's 64 keys, both d halves
          tma_load_4d_pair(dst, &map_kh, lb, 0, head, t0 + 64 * (int)rank, mat);
          tma_load_4d_pair(dst + kHalfK, &map_kh, lb, 64, head, t0 + 64 * (int)rank, mat);
        } else {      // V: all 128 keys, this CTA's 64 head-dim columns
          tma_load_4d_pair(dst, &map_kv, lb, 64 * (int)rank, head, t0, mat);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc_qk = idesc_bf16(2 * kRows, kKeys);
      constexpr uint32_t idesc_pv = idesc_bf16(2 * kRows, kHd, 0, 1);  // B (= V) MN-major
      const uint32_t sq[2] = {smem_u32(smem + Smem::qa), smem_u32(smem + Smem::qb)};
      const uint32_t sp[2] = {smem_u32(smem + Smem::pa), smem_u32(smem + Smem::pb)};
      auto ring_slot = [&](int i) { return smem_u32(smem + Smem::ring + (i % kRingP) * kItemP); };
      auto issue_qk = [&](int x, int j) {
        if (elect_one()) {
          const uint32_t sk = ring_slot(kpos(j));
#pragma unroll
          for (int k = 0; k < kHd / 16; ++k) {
            const uint32_t aoff = (k >> 2) * kHalf + (k & 3) * 32;
            const uint32_t boff = (k >> 2) * kHalfK + (k & 3) * 32;
            mma2_bf16_ss(tmem + x * 128, desc_sw128(sq[x] + aoff, 16, 1024), desc_sw128(sk + boff, 16, 1024),
                         idesc_qk, k != 0);
          }
          mma2_commit(&s_full[x]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int x, int j) {
        if (elect_one()) {
          const uint32_t sv = ring_slot(vpos(j, n_tiles));
#pragma unroll
          for (int k = 0; k < kKeys / 16; ++k) {
            const uint32_t aoff = (k >> 2) * kHalf + (k & 3) * 32;
            mma2_bf16_ss(tmem + 256 + x * 128, desc_sw128(sp[x] + aoff, 16, 1024),
                         desc_sw128(sv + k * 2048, 16, 1024), idesc_pv, (j | k) != 0);
          }
          mma2_commit(&o_ready[x]);
        }
        __syncwarp();
      };
      auto release = [&](int i) {
        if (elect_one()) mma2_commit(&ring_empty[i % kRingP]);
        __syncwarp();
      };
      auto ring_wait = [&](int i) { mbar_wait(&ring_full[i % kRingP], (i / kRingP) & 1); };
#ifdef BC_ATTN_TRACE
      const long long trc0 = clock64();
      long long tw_se = 0, tw_p = 0, tw_k = 0, tw_v = 0, t_iq = 0, t_ip = 0;
#define PT(v) const long long v = clock64()
#define PA(acc, v) acc += clock64() - v
#else
#define PT(v)
#define PA(acc, v)
#endif
      mbar_wait(q_full, 0);
      if (n_tiles > 0) {
        ring_wait(0);
        tc_fence_after();
        for (int x = 0; x < 2; ++x) issue_qk(x, 0);
        release(0);
      }
      for (int j = 0; j < n_tiles; ++j) {
        const bool next = j + 1 < n_tiles;
        for (int x = 0; x < 2; ++x) {
          if (next) {
            PT(a0);
            cl_wait(&s_empty[x], j & 1);  // both CTAs' softmax x has read S_x(j)
            PA(tw_se, a0);
            PT(a1);
            if (x == 0) ring_wait(kpos(j + 1));
            PA(tw_k, a1);
            tc_fence_after();
            PT(a2);
            issue_qk(x, j + 1);
            PA(t_iq, a2);
            if (x == 1) release(kpos(j + 1));
          }
          PT(a3);
          cl_wait(&p_full[x], j & 1);
          PA(tw_p, a3);
          PT(a4);
          if (x == 0) ring_wait(vpos(j, n_tiles));
          PA(tw_v, a4);
          tc_fence_after();
          PT(a5);
          issue_pv(x, j);
          PA(t_ip, a5);
        }
        release(vpos(j, n_tiles));
      }
#ifdef BC_ATTN_TRACE
      const int cid = (blockIdx.z * gridDim.y + blockIdx.y) * (gridDim.x >> 1) + (blockIdx.x >> 1);
      if (prm.trace && lane_id() == 0 && cid < 256) {
        unsigned long long* r = prm.trace + 32 * 64 + cid * 8;
        r[0] = clock64() - trc0;
        r[1] = 0;
        r[2] = 4ull * n_tiles;  // (query tile, key tile) steps of the cluster
        r[3] = tw_p;
        r[4] = tw_k + tw_v;
        r[5] = tw_se;
        r[6] = t_iq;
        r[7] = t_ip;
      }
#endif
#undef PT
#undef PA
    }
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    const int x = (warp >= 8) ? 1 : 0;
    SoftmaxBars b{&s_full[x], &s_empty[x], &p_full[x], &o_ready[x]};
    b.s_empty_cl = cl_map(&s_empty[x], 0);
    b.p_full_cl = cl_map(&p_full[x], 0);
    softmax_tile<kPoly>(prm, tmem + x * 128, tmem + 256 + x * 128, smem + (x ? Smem::pb : Smem::pa), b, n_tiles,
                        tiles_per_slot, warp & 3, q0 + x * kRows, e, head, x);
  }
  tc_fence_before();
  cl_sync();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// Balanced persistent variant: one CTA per SM runs a
// host-built list of work items, each either a pair of 128-row query tiles
// (ping-pong, as attn_kernel) or a single tile.  With one item per CTA the
// last of ~7.7 waves leaves a third of the SMs idle; here the host assigns
// whole pairs round by round and splits the last round's pairs into single
// tiles when its cost model says that ends earlier (longest-processing-time
// first, build_sched).  The next item's Q load and first QK^T overlap the
// previous item's epilogue, which is what helps the 4-key-tile text
// cross-attention most (164 -> 138 ms per run).  Per-row arithmetic and key
// order are those of attn_kernel: results are bit-identical.
// Barrier phases run on across items: per-tile barriers of tile x count
// the tiles x has processed, q_full / q_empty count items, o_free[x] (the
// epilogue of x has read O_x) counts the items x took part in.
template <int kPoly>
__global__ void __launch_bounds__(kThreads, 1)
    attn_sched_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                      AttnParams prm, const __grid_constant__ AttnSched sch,
                      const __grid_constant__ CUtensorMap map_o, int tma_o) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* q_full = bars + 0;
  uint64_t* ring_full = bars + 1;   // [3]
  uint64_t* ring_empty = bars + 4;  // [3]
  uint64_t* s_full = bars + 7;      // [2]
  uint64_t* s_empty = bars + 9;     // [2]
  uint64_t* p_full = bars + 11;     // [2]
  uint64_t* o_ready = bars + 13;    // [2]
  uint64_t* q_empty = bars + 15;
  uint64_t* o_free = bars + 16;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int it0 = sch.start[blockIdx.x], it1 = sch.start[blockIdx.x + 1];
  if (it0 >= it1) return;
  const int tiles_per_slot = (prm.kv_tokens + kKeys - 1) / kKeys;
  const uint32_t warp = warp_id();
  // tile x of an item: query rows from token qx of entry ex (x = 0, 1); K/V
  // from entry e0's visible list (a cross-entry pair's entries have equal
  // lists).  Scalars, not arrays: a runtime-indexed array would live in
  // local memory.
  struct Item {
    int e0, e1, q0, q1, head, n_q, n_tiles;
    __device__ int e(int x) const { return x ? e1 : e0; }
    __device__ int q(int x) const { return x ? q1 : q0; }
  };
  auto item = [&](int i) {
    const uint32_t w = sch.items[i];
    Item r;
    r.e0 = (int)(w & 0xffu);
    r.head = (int)((w >> 8) & 0xffu);
    if (w & kItemCross) {  // the last query tiles of two entries
      r.e1 = (int)((w >> 16) & 0xffu);
      r.q0 = prm.q_lo[r.e0] + ((prm.q_hi[r.e0] - prm.q_lo[r.e0] - 1) / kRows) * kRows;
      r.q1 = prm.q_lo[r.e1] + ((prm.q_hi[r.e1] - prm.q_lo[r.e1] - 1) / kRows) * kRows;
      r.n_q = 2;
    } else {
      r.e1 = r.e0;
      r.q0 = prm.q_lo[r.e0] + (int)((w >> 16) & 0x3fffu) * kRows;
      r.q1 = r.q0 + kRows;
      r.n_q = (w & kItemPair) ? 2 : 1;
    }
    r.n_tiles = prm.n_vis[r.e0] * tiles_per_slot;
    return r;
  };

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_kv);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&ring_full[i], 1);
      mbar_init(&ring_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_ready[i], 1);
      mbar_init(&o_free[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
  if (warp == 0) {
    if (lane_id() == 0) {
      uint32_t g = 0;  // ring items issued so far
      for (int i = it0; i < it1; ++i) {
        const Item w = item(i);
        if (i > it0) mbar_wait(q_empty, (i - it0 - 1) & 1);  // previous item's QK^T are done with Q
        mbar_arrive_expect_tx(q_full, w.n_q * kTile);
        for (int x = 0; x < w.n_q; ++x) {
          const int qrow = prm.q_row[w.e(x)] + (w.q(x) - prm.q_lo[w.e(x)]);
          tma_load_3d(smem + Smem::qa + x * kTile, &map_q, q_full, 0, w.head, qrow);
          tma_load_3d(smem + Smem::qa + x * kTile + kHalf, &map_q, q_full, 64, w.head, qrow);
        }
        for (int r = 0; r < 2 * w.n_tiles; ++r, ++g) {
          int j, is_v;
          ring_item(r, w.n_tiles, j, is_v);
          const int slot = g % kRing;
          const uint32_t ph = (g / kRing) & 1;
          const int kv_slot = prm.vis_slot[w.e0][j / tiles_per_slot];
          const int t0 = (j % tiles_per_slot) * kKeys;
          const int mat = prm.mat_base + kv_slot * prm.mat_stride + (is_v ? prm.v_offset : 0);
          if (!is_v && prm.flags && (j % tiles_per_slot) == 0) {
            const uint32_t need = prm.need[w.e0][j / tiles_per_slot];
            if (need) {  // K/V rows of this block come from peer GPUs: wait for each producer
              const uint32_t ep = need >> 8;
              const uint32_t* f = prm.flags + (size_t)(prm.flag_base + kv_slot) * prm.n_ranks;
              for (uint32_t m = need & 0xffu; m; m &= m - 1) spin_until_geq(f + (__ffs(m) - 1), ep, 256);
              asm volatile("fence.proxy.async.global;" ::: "memory");
            }
          }
          mbar_wait(&ring_empty[slot], ph ^ 1);
#ifdef BC_ABL_HALFKV  // timing experiment only (wrong numerics): half the K/V bytes from L2
          mbar_arrive_expect_tx(&ring_full[slot], kHalf);
          uint8_t* dst = smem + Smem::ring + slot * kTile;
          tma_load_4d(dst, &map_kv, &ring_full[slot], 0, w.head, t0, mat);
#else
          mbar_arrive_expect_tx(&ring_full[slot], kTile);
          uint8_t* dst = smem + Smem::ring + slot * kTile;
          tma_load_4d(dst, &map_kv, &ring_full[slot], 0, w.head, t0, mat);
          tma_load_4d(dst + kHalf, &map_kv, &ring_full[slot], 64, w.head, t0, mat);
#endif
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_qk = idesc_bf16(kRows, kKeys);
    constexpr uint32_t idesc_pv = idesc_bf16(kRows, kHd, 0, 1);  // B (= V) MN-major
    const uint32_t sq[2] = {smem_u32(smem + Smem::qa), smem_u32(smem + Smem::qb)};
    const uint32_t sp[2] = {smem_u32(smem + Smem::pa), smem_u32(smem + Smem::pb)};
    auto slot_of = [&](uint32_t g) { return smem_u32(smem + Smem::ring + (g % kRing) * kTile); };
    auto ring_wait = [&](uint32_t g) { mbar_wait(&ring_full[g % kRing], (g / kRing) & 1); };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) mma_commit(bar);
      __syncwarp();
    };
    auto issue_qk = [&](int x, uint32_t g) {
      if (elect_one()) {
        const uint32_t sk = slot_of(g);
#pragma unroll
        for (int k = 0; k < kHd / 16; ++k) {
          const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
          mma_bf16_ss(tmem + x * 128, desc_sw128(sq[x] + off, 16, 1024), desc_sw128(sk + off, 16, 1024), idesc_qk,
                      k != 0);
        }
        mma_commit(&s_full[x]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int x, uint32_t g, bool first) {
      if (elect_one()) {
        const uint32_t sv = slot_of(g);
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          const uint32_t aoff = (k >> 2) * kHalf + (k & 3) * 32;
          mma_bf16_ss(tmem + 256 + x * 128, desc_sw128(sp[x] + aoff, 16, 1024),
                      desc_sw128(sv + k * 2048, kHalf, 1024), idesc_pv, !(first && k == 0));
        }
        mma_commit(&o_ready[x]);
      }
      __syncwarp();
    };
#ifdef BC_ATTN_TRACE
    // per-CTA summary (scripts/attn_trace.sh): cycles, key steps, and where
    // the issuer spent them
    const long long trc0 = clock64();
    unsigned long long trg0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trg0));
    long long tr_wait = 0, tr_kv = 0, tr_se = 0, tr_iqk = 0, tr_ipv = 0;
#define TR_T(v) const long long v = clock64()
#define TR_ADD(acc, v) acc += clock64() - v
#else
#define TR_T(v)
#define TR_ADD(acc, v)
#endif
    uint32_t ib = 0;                // ring items consumed before this item
    uint32_t tb[2] = {0u, 0u};      // tiles processed by x before this item
    uint32_t nb[2] = {0u, 0u};      // items x took part in before this item
    for (int i = it0; i < it1; ++i) {
      const Item w = item(i);
      const int n = w.n_tiles;
      mbar_wait(q_full, (i - it0) & 1);
      if (n > 0) {
        ring_wait(ib + kpos(0));
        tc_fence_after();
        for (int x = 0; x < w.n_q; ++x) {
          if (tb[x] > 0) mbar_wait(&s_empty[x], (tb[x] - 1) & 1);  // x read its previous S
          tc_fence_after();
          issue_qk(x, ib + kpos(0));
        }
        commit(&ring_empty[(ib + kpos(0)) % kRing]);
        if (n == 1) commit(q_empty);
        for (int j = 0; j < n; ++j) {
          const bool next = j + 1 < n;
          for (int x = 0; x < w.n_q; ++x) {
            if (next) {
              TR_T(ts0);
              mbar_wait(&s_empty[x], (tb[x] + j) & 1);
              TR_ADD(tr_se, ts0);
              if (x == 0) ring_wait(ib + kpos(j + 1));
              tc_fence_after();
              TR_T(tq0);
              issue_qk(x, ib + kpos(j + 1));
              TR_ADD(tr_iqk, tq0);
              if (x == w.n_q - 1) {
                commit(&ring_empty[(ib + kpos(j + 1)) % kRing]);
                if (j + 1 == n - 1) commit(q_empty);  // the item's last QK^T
              }
            }
            TR_T(tw0);
            mbar_wait(&p_full[x], (tb[x] + j) & 1);
            TR_ADD(tr_wait, tw0);
            TR_T(tw1);
            if (x == 0) ring_wait(ib + vpos(j, n));
            TR_ADD(tr_kv, tw1);
            if (j == 0 && nb[x] > 0) mbar_wait(&o_free[x], (nb[x] - 1) & 1);  // previous O read out
            tc_fence_after();
            TR_T(tp0);
            issue_pv(x, ib + vpos(j, n), j == 0);
            TR_ADD(tr_ipv, tp0);
          }
          commit(&ring_empty[(ib + vpos(j, n)) % kRing]);
        }
      } else {
        commit(q_empty);
      }
      ib += 2 * n;
      for (int x = 0; x < w.n_q; ++x) {
        tb[x] += n;
        nb[x] += 1;
      }
    }
#undef TR_T
#undef TR_ADD
#ifdef BC_ATTN_TRACE
    if (prm.trace && lane_id() == 0 && blockIdx.x < 256) {
      unsigned long long trg1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trg1));
      unsigned long long* r = prm.trace + 32 * 64 + blockIdx.x * 8;
      r[0] = clock64() - trc0;
      r[1] = trg1 - trg0;
      r[2] = tb[0] + tb[1];  // (query tile, key tile) steps processed
      r[3] = tr_wait;
      r[4] = tr_kv;
      r[5] = tr_se;
      r[6] = tr_iqk;
      r[7] = tr_ipv;
    }
#endif
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    const int x = (warp >= 8) ? 1 : 0;
    SoftmaxBars b{&s_full[x], &s_empty[x], &p_full[x], &o_ready[x]};
    uint32_t tb = 0;
    for (int i = it0; i < it1; ++i) {
      const Item w = item(i);
      if (x >= w.n_q) continue;
      softmax_tile<kPoly>(prm, tmem + x * 128, tmem + 256 + x * 128, smem + (x ? Smem::pb : Smem::pa), b,
                          w.n_tiles, tiles_per_slot, warp & 3, w.q(x), w.e(x), w.head, x, tb, &o_free[x],
                          tma_o ? &map_o : nullptr);
      tb += w.n_tiles;
    }
    if (tma_o && (warp & 3) == 0 && lane_id() == 0) bulk_wait<0>();  // O stores complete before exit
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    return (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p)
               : nullptr;
  }();
  return fn;
}

int encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
           const cuuint32_t* box) {
  auto fn = encoder();
  if (!fn) return bc_fail(BC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return bc_fail(BC_ERR_CUDA, "attention tensor map encode failed (%d)", (int)r);
  return BC_OK;
}

}  // namespace

int g_attn_balance = -1;  // -1: BC_ATTN_BALANCE env (default on)

namespace {

int sm_count_attn() { return current_sm_count(); }

// Cost of a single-tile item per key tile, in units of one tile of a pair
// (a pair costs 2).  Without a ping-pong partner the tile's softmax latency
// (MUFU-bound: 128 exps per thread) is exposed every key tile: measured
// ~0.9 of a whole pair.  BC_ATTN_SINGLE_COST (percent) overrides.
double single_cost() {
  static const double c = [] {
    const char* e = getenv("BC_ATTN_SINGLE_COST");
    return e ? atof(e) / 100.0 : 1.8;
  }();
  return c;
}

struct SchedKey {
  int n_entries, heads, kv_tokens, ctas;
  int n_vis[BC_MAX_ENTRIES], q_lo[BC_MAX_ENTRIES], q_hi[BC_MAX_ENTRIES];
  int group[BC_MAX_ENTRIES];  // first entry with an identical visible list
  bool operator==(const SchedKey& o) const { return memcmp(this, &o, sizeof(SchedKey)) == 0; }
};

struct WorkItem {
  uint32_t code;
  double cost;
  int order;  // tie-break: head-major, so concurrently running items share K/V in L2
};

// Longest-processing-time-first onto `bins` CTAs; returns the makespan and
// appends each bin's items (in assignment order) to lists[bin].
double lpt(std::vector<WorkItem>& items, std::vector<double>& load, std::vector<std::vector<uint32_t>>& lists) {
  std::stable_sort(items.begin(), items.end(), [](const WorkItem& a, const WorkItem& b) {
    return a.cost != b.cost ? a.cost > b.cost : a.order < b.order;
  });
  using Bin = std::pair<double, int>;
  std::priority_queue<Bin, std::vector<Bin>, std::greater<Bin>> heap;
  for (int b = 0; b < (int)load.size(); ++b) heap.push({load[b], b});
  for (const WorkItem& w : items) {
    Bin bin = heap.top();
    heap.pop();
    load[bin.second] += w.cost;
    lists[bin.second].push_back(w.code);
    heap.push({load[bin.second], bin.second});
  }
  return *std::max_element(load.begin(), load.end());
}

// Build the balanced work list (nullptr: does not fit, use attn_kernel).
// Whole pairs are placed first; the pairs that would form the last,
// partial round are either kept whole or split into two single-tile items,
// whichever the cost model says finishes earlier.
std::shared_ptr<const AttnSched> build_sched(const AttnArgs& a, const AttnParams& p, int* n_ctas) {
  static std::vector<std::pair<SchedKey, std::shared_ptr<const AttnSched>>> cache;
  static std::mutex mu;  // contexts may step from several host threads
  std::lock_guard<std::mutex> lock(mu);
  SchedKey key;
  memset(&key, 0, sizeof(key));
  key.n_entries = a.n_entries;
  key.heads = a.heads;
  key.kv_tokens = a.kv_tokens;
  key.ctas = std::min(sm_count_attn(), kSchedCtas);
  for (int e = 0; e < a.n_entries; ++e) {
    key.n_vis[e] = p.n_vis[e];
    key.q_lo[e] = p.q_lo[e];
    key.q_hi[e] = p.q_hi[e];
    key.group[e] = e;
    for (int f = 0; f < e; ++f)
      if (p.n_vis[f] == p.n_vis[e] && !memcmp(p.vis_slot[f], p.vis_slot[e], sizeof(int) * p.n_vis[e]) &&
          !memcmp(p.need[f], p.need[e], sizeof(uint32_t) * p.n_vis[e])) {
        key.group[e] = f;
        break;
      }
  }
  for (auto& c : cache)
    if (c.first == key) {
      *n_ctas = key.ctas;
      return c.second;
    }
  const int tps = (a.kv_tokens + kKeys - 1) / kKeys;
  auto n_qtiles = [&](int e) { return (p.q_hi[e] - p.q_lo[e] + kRows - 1) / kRows; };
  std::vector<WorkItem> pairs, singles;
  for (int h = 0; h < a.heads; ++h) {
    int open_single[BC_MAX_ENTRIES];  // per visible-list group: an unpaired last tile (-1: none)
    for (int e = 0; e < a.n_entries; ++e) open_single[e] = -1;
    for (int e = 0; e < a.n_entries; ++e) {
      const int nq = n_qtiles(e);
      const double nt = (double)p.n_vis[e] * tps;
      for (int t = 0; t < nq; t += 2) {
        const uint32_t code = (uint32_t)e | ((uint32_t)h << 8) | ((uint32_t)t << 16);
        const int order = (h * BC_MAX_ENTRIES + e) * 4096 + t;
        if (t + 1 < nq) {
          pairs.push_back({code | kItemPair, 2.0 * nt, order});
        } else if (open_single[key.group[e]] >= 0) {  // pair it with an earlier entry's last tile
          const int f = open_single[key.group[e]];
          open_single[key.group[e]] = -1;
          pairs.push_back({(uint32_t)f | ((uint32_t)h << 8) | ((uint32_t)e << 16) | kItemCross, 2.0 * nt, order});
        } else {
          open_single[key.group[e]] = e;
        }
      }
    }
    for (int e = 0; e < a.n_entries; ++e)  // last tiles left without a partner
      if (open_single[e] >= 0) {
        const int f = open_single[e];
        const uint32_t t = (uint32_t)(n_qtiles(f) - 1);
        singles.push_back({(uint32_t)f | ((uint32_t)h << 8) | (t << 16), single_cost() * p.n_vis[f] * tps,
                           (h * BC_MAX_ENTRIES + f) * 4096 + (int)t});
      }
  }
  const int G = key.ctas;
  // items emitted: every pair once, plus at most one extra per pair of the
  // last partial round when it is split into single tiles, plus the singles
  if (pairs.size() + pairs.size() % G + singles.size() > (size_t)kSchedItems || a.heads > 255 ||
      a.n_entries > 255)
    return nullptr;
  std::stable_sort(pairs.begin(), pairs.end(), [](const WorkItem& x, const WorkItem& y) {
    return x.cost != y.cost ? x.cost > y.cost : x.order < y.order;
  });
  const size_t whole = pairs.size() - pairs.size() % G;  // complete rounds of pairs
  auto plan = [&](bool split, std::vector<std::vector<uint32_t>>& lists) {
    std::vector<double> load(G, 0.0);
    lists.assign(G, {});
    std::vector<WorkItem> first(pairs.begin(), pairs.begin() + (split ? whole : pairs.size()));
    lpt(first, load, lists);
    std::vector<WorkItem> rest = singles;
    if (split)
      for (size_t i = whole; i < pairs.size(); ++i) {
        const WorkItem& w = pairs[i];
        const double c = single_cost() * w.cost / 2.0;
        const uint32_t h8 = w.code & 0xff00u;
        if (w.code & kItemCross) {  // the two entries' last tiles
          const uint32_t e1 = w.code & 0xffu, e2 = (w.code >> 16) & 0xffu;
          rest.push_back({e1 | h8 | ((uint32_t)(n_qtiles((int)e1) - 1) << 16), c, w.order});
          rest.push_back({e2 | h8 | ((uint32_t)(n_qtiles((int)e2) - 1) << 16), c, w.order + 1});
        } else {
          const uint32_t base = w.code & ~kItemPair;
          rest.push_back({base, c, w.order});
          rest.push_back({base + (1u << 16), c, w.order + 1});  // the pair's second tile
        }
      }
    return lpt(rest, load, lists);
  };
  std::vector<std::vector<uint32_t>> keep, split;
  const double m_keep = plan(false, keep);
  const double m_split = plan(true, split);
  const auto& lists = (m_split < m_keep) ? split : keep;
  auto sched = std::make_unique<AttnSched>();
  memset(sched.get(), 0, sizeof(AttnSched));
  size_t total = 0;
  for (const auto& l : lists) total += l.size();
  if (total > (size_t)kSchedItems) return nullptr;  // (cannot happen given the bound above)
  int n = 0;
  for (int b = 0; b < G; ++b) {
    sched->start[b] = (uint16_t)n;
    for (uint32_t c : lists[b]) sched->items[n++] = c;
  }
  sched->start[G] = (uint16_t)n;
  if (cache.size() >= 64) cache.erase(cache.begin());  // callers hold their own reference
  cache.emplace_back(key, std::shared_ptr<const AttnSched>(std::move(sched)));
  *n_ctas = G;
  return cache.back().second;
}

}  // namespace

int attention_run(const AttnArgs& a, cudaStream_t st) {
  if (a.head_dim != kHd) return bc_fail(BC_ERR_CONTRACT, "attention: head_dim must be 128");
  if (a.n_entries < 1 || a.n_entries > BC_MAX_ENTRIES)
    return bc_fail(BC_ERR_CONTRACT, "attention: bad entry count %d", a.n_entries);
  const uint64_t row_bytes = (uint64_t)a.heads * kHd * 2;
  CUtensorMap mq, mkv;
  {
    cuuint64_t dims[3] = {kHd, (cuuint64_t)a.heads,
                          (cuuint64_t)(a.ranged ? a.q_rows : a.n_entries * a.q_tokens)};
    cuuint64_t strides[2] = {kHd * 2, row_bytes};
    cuuint32_t box[3] = {64, 1, kRows};
    int rc = encode(&mq, a.q, 3, dims, strides, box);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[4] = {kHd, (cuuint64_t)a.heads, (cuuint64_t)a.kv_tokens, (cuuint64_t)a.n_mats};
    cuuint64_t strides[3] = {kHd * 2, row_bytes, row_bytes * (uint64_t)a.kv_tokens};
    cuuint32_t box[4] = {64, 1, kKeys, 1};
    int rc = encode(&mkv, a.kv_base, 4, dims, strides, box);
    if (rc) return rc;
  }
  AttnParams p{};
  p.q_tokens = a.q_tokens;
  p.kv_tokens = a.kv_tokens;
  p.heads = a.heads;
  p.mat_base = a.mat_base;
  p.mat_stride = a.mat_stride;
  p.v_offset = a.v_offset;
  p.scale = a.scale;
  p.out = a.out;
  p.n_ranks = a.n_ranks > 0 ? a.n_ranks : 1;
  int max_pairs = 0;
  for (int e = 0; e < a.n_entries; ++e) {
    if (a.n_vis[e] < 0 || a.n_vis[e] > BC_MAX_VIS) return bc_fail(BC_ERR_CONTRACT, "attention: bad visible count");
    if (a.ranged) {
      if (a.q_lo[e] < 0 || a.q_hi[e] > a.q_tokens || a.q_row[e] + (a.q_hi[e] - a.q_lo[e]) > a.q_rows)
        return bc_fail(BC_ERR_CONTRACT, "attention: bad query row range (entry %d)", e);
      p.q_lo[e] = a.q_lo[e];
      p.q_hi[e] = a.q_hi[e];
      p.q_row[e] = a.q_row[e];
    } else {
      p.q_lo[e] = 0;
      p.q_hi[e] = a.q_tokens;
      p.q_row[e] = e * a.q_tokens;
    }
    const int pairs = (p.q_hi[e] - p.q_lo[e] + 2 * kRows - 1) / (2 * kRows);
    max_pairs = pairs > max_pairs ? pairs : max_pairs;
    p.n_vis[e] = a.n_vis[e];
    for (int v = 0; v < a.n_vis[e]; ++v) {
      p.vis_slot[e][v] = a.vis_slot[e][v];
      p.need[e][v] = a.flags ? a.need[e][v] : 0u;
    }
  }
  p.flags = a.flags;
  p.flag_base = a.flag_base;
  p.trace = nullptr;
#ifdef BC_ATTN_TRACE
  {
    static unsigned long long* buf = nullptr;
    if (!buf) cudaMalloc(&buf, (32 * 64 + 256 * 8) * sizeof(unsigned long long));
    p.trace = buf;
    bc_attn_trace_ptr = buf;
  }
#endif
  // tuning knob: pairs of exponentials (of every 8) evaluated by the FMA-pipe
  // polynomial instead of MUFU.EX2
  static const int poly = [] {
    const char* env = getenv("BC_ATTN_POLY");
    const int v = env ? atoi(env) : kDefaultPoly;
    return (v != 0 && v != 2 && v != 3 && v != 4 && v != 8) ? kDefaultPoly : v;
  }();
  static PerDeviceOnce grid_attrs;
  BC_RC(per_device_once(grid_attrs, [&]() -> int {
    BC_CUDA(cudaFuncSetAttribute(attn_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::total + 1024));
    BC_CUDA(cudaFuncSetAttribute(attn_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::total + 1024));
    BC_CUDA(cudaFuncSetAttribute(attn_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::total + 1024));
    BC_CUDA(cudaFuncSetAttribute(attn_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::total + 1024));
    BC_CUDA(cudaFuncSetAttribute(attn_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::total + 1024));
    cudaFuncAttributes fa;
    BC_CUDA(cudaFuncGetAttributes(&fa, attn_kernel<0>));
    if (fa.numRegs != kRegsLaunch)  // the setmaxnreg split assumes this allocation (else: deadlock)
      return bc_fail(BC_ERR_CUDA, "attention kernel built with %d registers, expected %d", fa.numRegs, kRegsLaunch);
    return BC_OK;
  }));
  if (max_pairs == 0) return BC_OK;  // no query rows in this slice
  // CTA-pair kernel (BC_ATTN_PAIR=1): clusters of 2 sharing each K/V tile
  static const int pair_env = [] {
    const char* env = getenv("BC_ATTN_PAIR");
    return env ? atoi(env) : 0;
  }();
  if (pair_env && poly == 0) {
    static PerDeviceOnce pair_attrs;
    BC_RC(per_device_once(pair_attrs, [&]() -> int {
      BC_CUDA(cudaFuncSetAttribute(attn_pair_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   Smem::total + 1024));
      return BC_OK;
    }));
    CUtensorMap mkh;
    {
      cuuint64_t dims[4] = {kHd, (cuuint64_t)a.heads, (cuuint64_t)a.kv_tokens, (cuuint64_t)a.n_mats};
      cuuint64_t strides[3] = {kHd * 2, row_bytes, row_bytes * (uint64_t)a.kv_tokens};
      cuuint32_t box[4] = {64, 1, kKeys / 2, 1};
      int rc = encode(&mkh, a.kv_base, 4, dims, strides, box);
      if (rc) return rc;
    }
    int max_items = 0;
    for (int e = 0; e < a.n_entries; ++e) {
      const int items = (p.q_hi[e] - p.q_lo[e] + 4 * kRows - 1) / (4 * kRows);
      max_items = items > max_items ? items : max_items;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * max_items, a.n_entries, a.heads);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Smem::total + 1024;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    BC_CUDA(cudaLaunchKernelEx(&cfg, attn_pair_kernel<0>, mq, mkh, mkv, p));
    BC_LAUNCHED();
    return BC_OK;
  }
  if (g_attn_balance < 0) {
    const char* env = getenv("BC_ATTN_BALANCE");
    g_attn_balance = env ? atoi(env) : 1;
  }
  if (a.balance && g_attn_balance && poly == 0) {
    static PerDeviceOnce sched_attrs;
    BC_RC(per_device_once(sched_attrs, [&]() -> int {
      BC_CUDA(cudaFuncSetAttribute(attn_sched_kernel<kSchedPoly>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   Smem::total + 1024));
      return BC_OK;
    }));
    int ctas = 0;
    const std::shared_ptr<const AttnSched> sch = build_sched(a, p, &ctas);
    if (sch) {
      // O leaves by TMA (BC_ATTN_TMA_O=0: per-thread global stores)
      static int tma_o = -1;
      if (tma_o < 0) {
        const char* env = getenv("BC_ATTN_TMA_O");
        tma_o = env ? atoi(env) != 0 : 1;
      }
      CUtensorMap mo = mq;
      if (tma_o) {
        cuuint64_t dims[3] = {kHd, (cuuint64_t)a.heads,
                              (cuuint64_t)(a.ranged ? a.q_rows : a.n_entries * a.q_tokens)};
        cuuint64_t strides[2] = {kHd * 2, row_bytes};
        cuuint32_t box[3] = {64, 1, kRows};
        int rc = encode(&mo, a.out, 3, dims, strides, box);
        if (rc) return rc;
      }
      attn_sched_kernel<kSchedPoly><<<ctas, kThreads, Smem::total + 1024, st>>>(mq, mkv, p, *sch, mo, tma_o);
      BC_LAUNCHED();
      return BC_OK;
    }
  }
  dim3 grid(max_pairs, a.n_entries, a.heads);
  switch (poly) {
    case 2: attn_kernel<2><<<grid, kThreads, Smem::total + 1024, st>>>(mq, mkv, p); break;
    case 3: attn_kernel<3><<<grid, kThreads, Smem::total + 1024, st>>>(mq, mkv, p); break;
    case 4: attn_kernel<4><<<grid, kThreads, Smem::total + 1024, st>>>(mq, mkv, p); break;
    case 8: attn_kernel<8><<<grid, kThreads, Smem::total + 1024, st>>>(mq, mkv, p); break;
    default: attn_kernel<0><<<grid, kThreads, Smem::total + 1024, st>>>(mq, mkv, p);
  }
  BC_LAUNCHED();
  return BC_OK;
}

}  // namespace bc

// Select the attention kernel: 1 = balanced persistent work lists (default),
// 0 = one CTA per (query-tile pair, entry, head).  Results are identical.
extern "C" int bc_attention_set_balance(int on) {
  bc::g_attn_balance = on ? 1 : 0;
  return BC_OK;
}

// Host-side view of the balanced kernel's work list for a paged launch (the
// same arguments as bc_attention_paged, every entry's full q_per_entry rows):
// items[] / start[] as the kernel receives them (attention.h, AttnSched).
// Returns the item count, or -1 when the launch would use the grid kernel.
// Host logic only (no device work), so the CPU tests check coverage and
// pairing rules with it.
extern "C" int bc_attention_plan(const bc_batch* batch, int32_t q_per_entry, int32_t kv_tokens, int32_t heads,
                                 uint32_t* items, int32_t items_cap, uint16_t* start, int32_t* n_ctas) {
  if (!batch || !items || !start || !n_ctas) return bc_fail(BC_ERR_CONTRACT, "attention plan: null argument");
  if (batch->n_entries < 1 || batch->n_entries > BC_MAX_ENTRIES)
    return bc_fail(BC_ERR_CONTRACT, "attention plan: bad entry count");
  if (heads < 1 || heads > 255 || kv_tokens < 1 || q_per_entry < 1 || items_cap < 0)
    return bc_fail(BC_ERR_CONTRACT, "attention plan: bad heads / kv_tokens / q_per_entry / items_cap");
  for (int e = 0; e < batch->n_entries; ++e)
    if (batch->n_vis[e] < 0 || batch->n_vis[e] > BC_MAX_VIS)
      return bc_fail(BC_ERR_CONTRACT, "attention plan: bad visible count %d (entry %d)", batch->n_vis[e], e);
  bc::AttnArgs a{};
  bc::AttnParams p{};
  a.n_entries = batch->n_entries;
  a.heads = heads;
  a.kv_tokens = kv_tokens;
  for (int e = 0; e < a.n_entries; ++e) {
    p.n_vis[e] = batch->n_vis[e];
    for (int v = 0; v < batch->n_vis[e]; ++v) p.vis_slot[e][v] = batch->vis_slot[e][v];
    p.q_lo[e] = 0;
    p.q_hi[e] = q_per_entry;
  }
  int ctas = 0;
  const std::shared_ptr<const bc::AttnSched> sch = bc::build_sched(a, p, &ctas);
  if (!sch) return -1;
  const int n = sch->start[ctas];
  if (n > items_cap) return bc_fail(BC_ERR_CONTRACT, "attention plan: %d items exceed the buffer", n);
  for (int i = 0; i < n; ++i) items[i] = sch->items[i];
  for (int c = 0; c <= ctas; ++c) start[c] = sch->start[c];
  *n_ctas = ctas;
  return n;
}

// Self-attention over KV-arena slots.  k_arena points at layer 0 of an
// arena laid out [L][n_slots][2][T][heads*128]; slot_stride_elems is the
// distance between consecutive slots' K matrices in elements.
extern "C" int bc_attention_paged(const void* q, const void* k_arena, const void* v_arena,
                                  int64_t slot_stride_elems, int32_t kv_tokens, const bc_batch* batch,
                                  int32_t q_per_entry, int32_t heads, void* out, void* stream) {
  if (!q || !k_arena || !batch || !out) return bc_fail(BC_ERR_CONTRACT, "attention: null argument");
  const int64_t mat_elems = (int64_t)kv_tokens * heads * 128;
  if (slot_stride_elems % mat_elems) return bc_fail(BC_ERR_CONTRACT, "attention: bad slot stride");
  bc::AttnArgs a{};
  a.q = q;
  a.kv_base = k_arena;
  a.n_entries = batch->n_entries;
  a.q_tokens = q_per_entry;
  a.kv_tokens = kv_tokens;
  a.heads = heads;
  a.head_dim = 128;
  a.mat_stride = (int)(slot_stride_elems / mat_elems);
  a.v_offset = (int)(((const char*)v_arena - (const char*)k_arena) / (mat_elems * 2));
  a.mat_base = 0;
  int max_slot = 0;
  for (int e = 0; e < batch->n_entries; ++e) {
    a.n_vis[e] = batch->n_vis[e];
    for (int v = 0; v < batch->n_vis[e]; ++v) {
      a.vis_slot[e][v] = batch->vis_slot[e][v];
      max_slot = batch->vis_slot[e][v] > max_slot ? batch->vis_slot[e][v] : max_slot;
    }
  }
  a.n_mats = (max_slot + 1) * a.mat_stride + a.v_offset;
  a.scale = 1.0f / sqrtf(128.0f);
  a.out = out;
  a.balance = 1;
  return bc::attention_run(a, (cudaStream_t)stream);
}
