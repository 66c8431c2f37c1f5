// tcgen05 bf16 GEMM with fused epilogues -- the QKV / O / cross-attn /
// FFN / patch-embed / head / text projections of the Wan2.1-shaped DiT.
//
//   C[M,N] = epi( A[M,K] . B[N,K]^T + bias )      A, B bf16, K-major
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer  (A tile 128x64, B tile BNx64, 128B swizzle)
//   warp 1      MMA issuer    (tcgen05.mma kind::f16, M=128, N=BN, K=16)
//               + TMEM owner  (2 accumulators x BN fp32 columns)
//   warps 2..5  epilogue      (tcgen05.ld 32x32b -> fused op -> global)
// Pipelines: smem ring full/empty (TMA <-> MMA), TMEM full/empty
// (MMA <-> epilogue) so the epilogue of tile i overlaps the MMAs of i+1.
// Tile order is M-fastest inside an N band so the 148 concurrent tiles
// share B (weights) and stream A (activations) once from L2.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>

#include "bc_common.h"
#include "gemm.h"
#include "sm100.cuh"

namespace bc {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle atom row
constexpr int kEpiWarps = 8;      // 2 per TMEM lane quadrant (column halves)
constexpr int kResWarp = 2 + kEpiWarps;  // residual-tile TMA loader (gated-residual mode)
constexpr int kThreads = 64 + 32 * kEpiWarps + 32;
constexpr int kChunk = 16;        // columns per TMEM load / staging round
constexpr int kStagePitch = 20;   // floats per staged row (16 + 4 pad, 16 B aligned)
constexpr int kEpiStageBytes = kEpiWarps * 32 * kStagePitch * 4;

// CG = 1: one CTA per tile (M=128 MMA).  CG = 2: a CTA pair (cluster of 2
// on one TPC) shares a 256 x BN tile -- tcgen05.mma.cta_group::2 with M=256,
// each CTA holding 128 rows of A and BN/2 rows of B in its own smem and its
// own 128 x BN accumulator in TMEM; the leader CTA issues the MMAs, both
// CTAs' TMA loads complete on the leader's mbarrier, commits multicast to
// both CTAs.  Halves the B traffic per CTA and the smem operand bandwidth.
//
// RES (the gated-residual fp32 mode): the C tile is read and written by TMA
// through a ring of kResSlots slots, each two 128-row x kResCols fp32 boxes
// (one per epilogue column half, swizzled): a loader warp streams the
// residual ahead of the epilogue, the epilogue combines in place and
// TMA-stores the box.  The residual tile's DRAM read no longer sits on the
// epilogue's critical path (register prefetch one 16-column chunk ahead
// left the short-K residual GEMMs at ~60% tensor-active).  16-column boxes
// x 3 slots (48 KB) keep the mainloop ring at 6 stages for 192-wide pair
// tiles; measured in the step (scripts/bw_breakdown.py): 16 x 3 -3.6% on
// the residual GEMMs, 16 x 4 and 32 x 2 / 3 (5 / 4 stages) no gain.
#ifndef BC_GEMM_RES_COLS
#define BC_GEMM_RES_COLS 16
#endif
#ifndef BC_GEMM_RES_SLOTS
#define BC_GEMM_RES_SLOTS 3
#endif
constexpr int kResCols = BC_GEMM_RES_COLS;         // columns per residual box (16 or 32 fp32)
constexpr int kResSwz = kResCols * 4;              // box row bytes = swizzle span (64 or 128 B)
constexpr int kResBoxBytes = BM * kResCols * 4;
constexpr int kResSlots = BC_GEMM_RES_SLOTS;
static_assert(kResCols == 16 || kResCols == 32, "residual box width");
template <int BN, int CG, bool RES = false>
struct GemmCfg {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = (BN / CG) * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kResBytes = RES ? kResSlots * 2 * kResBoxBytes : 0;
  static constexpr int kEpiStage = RES ? 0 : kEpiStageBytes;
  static constexpr int kRingBudget = RES ? 227 * 1024 - 1024 - 256 - kResBytes : 192 * 1024;
  static constexpr int kStages = kRingBudget / kStageBytes > 8 ? 8 : kRingBudget / kStageBytes;
  // two accumulators, rounded up to the power-of-two column count
  // tcgen05.alloc requires (BN = 192 -> 512)
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr size_t kSmem = 1024 /*align slack*/ + (size_t)kStages * kStageBytes + kResBytes + 256 + kEpiStage;
  static_assert(!RES || (BN / 2) % kResCols == 0, "residual boxes tile each column half");
  static_assert(kSmem <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

// Grouped rasterisation: tiles run in bands of kGroupM M-tiles with N
// fastest inside a band, so the ~148 concurrent tiles cover a compact
// (M x N) rectangle and both operand panels stay L2-resident (with plain
// M-fastest order a K=8960 GEMM re-reads A once per N column).
constexpr int kGroupM = 16;

#ifdef BC_GEMM_TRACE
// debug timeline (scripts/gemm_trace.cu): [cta 0..3][event][kb] globaltimer
__device__ unsigned long long g_gemm_trace[4][3][256];
__device__ __forceinline__ void gemm_trace(int ev, int kb) {
  if (blockIdx.x < 4 && kb < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_trace[blockIdx.x][ev][kb] = t;
  }
}
#define GEMM_TRACE(ev, kb) gemm_trace(ev, kb)
#else
#define GEMM_TRACE(ev, kb)
#endif
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int& m_blk, int& n_blk) {
  const int per_group = kGroupM * num_n;
  const int g = tile / per_group;
  const int first = g * kGroupM;
  const int gm = min(kGroupM, num_m - first);
  const int r = tile - g * per_group;
  m_blk = first + r % gm;
  n_blk = r / gm;
}

// GELU (tanh form) with the MUFU tanh (tanh.approx.f32, rel. error ~2^-11,
// well below the bf16 output's 2^-8): libm tanhf made the FFN1 epilogue
// ~27 instructions per output and capped the tensor pipe at 79% (ncu)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_fast(k0 * fmaf(k1 * x, x * x, x)), hx);
}

template <int BN, int MODE, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ CUtensorMap map_c, void* __restrict__ c_ptr, int M, int N, int K,
                const float* __restrict__ bias, const float* __restrict__ gate, int gate_stride, int rows_per_gate,
                int gate_row0) {
  constexpr bool RES = MODE == kEpiResidualF32;
  using Cfg = GemmCfg<BN, CG, RES>;
  constexpr int S = Cfg::kStages;
  constexpr int TM = BM * CG;  // rows per (cluster) tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + S * Cfg::kABytes;
  uint8_t* res_buf = smem + S * Cfg::kStageBytes;  // RES: [slot][half] 128 x 32 fp32 boxes, SW128
  float* epi_stage = reinterpret_cast<float*>(smem + S * Cfg::kStageBytes + Cfg::kResBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes + Cfg::kResBytes + Cfg::kEpiStage);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* res_full = tempty + 2;
  uint64_t* res_empty = res_full + kResSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_empty + kResSlots);

  const uint32_t warp = warp_id();
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // cluster index
  const int n_units = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int num_m = (M + TM - 1) / TM;
  const int num_n = (N + BN - 1) / BN;  // a ragged last column tile (BN = 224) is masked
  const int num_tiles = num_m * num_n;
  const int num_kb = K / BK;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);  // the leader producer's arrival (+ tx bytes of both CTAs)
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CG == 2 ? CG * kEpiWarps : 32 * kEpiWarps);
    }
    if (RES) {
      tma_prefetch(&map_c);
      for (int i = 0; i < kResSlots; ++i) {
        mbar_init(&res_full[i], 1);   // the loader's arrival + both boxes' bytes
        mbar_init(&res_empty[i], 2);  // each column half's storing thread
      }
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(Cfg::kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane_id() == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = unit; tile < num_tiles; tile += n_units) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb);
        const int m0 = mb * TM + (int)rank * BM, n0 = nb * BN + (int)rank * (BN / CG);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (tile == unit) GEMM_TRACE(0, kb);
          if (CG == 2) {
            // only the leader arrives (expecting both CTAs' bytes); the
            // peer's loads just complete their tx on the leader's barrier.
            // A remote arrive per stage costs ~0.5 us of issue latency.
            const uint32_t lb = map_rank(&full[stage], 0);
            if (leader) mbar_arrive_expect_tx(&full[stage], CG * Cfg::kStageBytes);
            tma_load_2d_pair(sa + stage * Cfg::kABytes, &map_a, lb, kb * BK, m0);
            tma_load_2d_pair(sb + stage * Cfg::kBBytes, &map_b, lb, kb * BK, n0);
          } else {
            mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
            tma_load_2d(sa + stage * Cfg::kABytes, &map_a, &full[stage], kb * BK, m0);
            tma_load_2d(sb + stage * Cfg::kBBytes, &map_b, &full[stage], kb * BK, n0);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (CG == 2 && !leader) goto teardown;  // the leader issues the pair's MMAs
    constexpr uint32_t idesc = idesc_bf16(TM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = unit; tile < num_tiles; tile += n_units, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (it < 2 && lane_id() == 0) GEMM_TRACE(1, kb + it * num_kb);
        if (elect_one()) {
          const uint32_t a0 = smem_u32(sa + stage * Cfg::kABytes);
          const uint32_t b0 = smem_u32(sb + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = desc_sw128(a0 + k * 32, 16, 1024);
            const uint64_t bd = desc_sw128(b0 + k * 32, 16, 1024);
            if (CG == 2) mma_bf16_ss_pair(d_tmem, ad, bd, idesc, (kb | k) != 0);
            else mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          if (CG == 2) {
            mma_commit_pair(&empty[stage]);
            if (kb == num_kb - 1) mma_commit_pair(&tfull[acc]);
          } else {
            mma_commit(&empty[stage]);
            if (kb == num_kb - 1) mma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == kResWarp) {
    if (RES && lane_id() == 0) {
      // residual loader: box (tile, step, half) = C[m0 .. +128, n0 + half * BN/2 + step * 32 .. +32]
      int slot = 0;
      uint32_t ph = 0;
      for (int tile = unit; tile < num_tiles; tile += n_units) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb);
        const int m0 = mb * TM + (int)rank * BM, n0 = nb * BN;
        for (int step = 0; step < BN / 2 / kResCols; ++step) {
          mbar_wait(&res_empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&res_full[slot], 2 * kResBoxBytes);
          uint8_t* dst = res_buf + slot * 2 * kResBoxBytes;
          tma_load_2d(dst, &map_c, &res_full[slot], n0 + step * kResCols, m0);
          tma_load_2d(dst + kResBoxBytes, &map_c, &res_full[slot], n0 + BN / 2 + step * kResCols, m0);
          if (++slot == kResSlots) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (RES) {
    // gated-residual epilogue: warp w covers TMEM lanes 32*(w%4)..+31 (one
    // tile row per thread) and one column half; per 32-column step it reads
    // its row of the residual box from shared memory (swizzled: 16-byte
    // chunk j of row r at chunk j ^ (r & 7), conflict-free), writes
    // C = resid + gate * (acc + bias) back in place, and one thread per half
    // TMA-stores the box once the half's 128 threads are done with it.
    const int ew = (int)warp - 2;
    const uint32_t quad = warp & 3;
    const int half = ew >> 2;
    const uint32_t row = quad * 32 + lane_id();  // tile row
    const bool storer = quad == 0 && lane_id() == 0;
    int slot = 0, pend = -1;
    uint32_t ph = 0;
    int it = 0;
    for (int tile = unit; tile < num_tiles; tile += n_units, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb);
      const int m0 = mb * TM + (int)rank * BM, n0 = nb * BN;
      const int grow = min(m0 + (int)row, M - 1);
      const float* grow_ptr = gate ? gate + (size_t)((gate_row0 + grow) / rows_per_gate) * gate_stride : nullptr;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int step = 0; step < BN / 2 / kResCols; ++step) {
        const int c = half * (BN / 2) + step * kResCols;  // column within the tile
        const int col = n0 + c;
        const bool col_in = col < N;  // boxes past N: TMA loads zeros, the store is clipped
        uint32_t r[kResCols];
        if constexpr (kResCols == 32)
          tmem_ld32(tmem_base + ((quad * 32) << 16) + acc * BN + c, *reinterpret_cast<uint32_t(*)[32]>(r));
        else
          tmem_ld16(tmem_base + ((quad * 32) << 16) + acc * BN + c, *reinterpret_cast<uint32_t(*)[16]>(r));
        mbar_wait(&res_full[slot], ph);
        tmem_ld_wait();
        const uint32_t box = smem_u32(res_buf + slot * 2 * kResBoxBytes + half * kResBoxBytes) + row * kResSwz;
        // 128-byte swizzle: chunk j ^ (r & 7); 64-byte: chunk j ^ ((r >> 1) & 3)
        const uint32_t swz = kResCols == 32 ? (row & 7) : ((row >> 1) & 3);
#pragma unroll
        for (int j = 0; j < kResCols / 4; ++j) {
          const uint32_t a = box + ((j ^ swz) << 4);
          const float4 res = lds128f(a);
          const float4 g = grow_ptr && col_in ? __ldg(reinterpret_cast<const float4*>(grow_ptr + col) + j)
                                              : make_float4(1.f, 1.f, 1.f, 1.f);
          const float4 b = bias && col_in ? __ldg(reinterpret_cast<const float4*>(bias + col) + j)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          float4 o;
          o.x = fmaf(g.x, __uint_as_float(r[4 * j + 0]) + b.x, res.x);
          o.y = fmaf(g.y, __uint_as_float(r[4 * j + 1]) + b.y, res.y);
          o.z = fmaf(g.z, __uint_as_float(r[4 * j + 2]) + b.z, res.z);
          o.w = fmaf(g.w, __uint_as_float(r[4 * j + 3]) + b.w, res.w);
          sts128f(a, o);
        }
        fence_async_shared();
        named_bar_sync(1 + half, 128);
        if (storer) {
          tma_store_2d(&map_c, res_buf + slot * 2 * kResBoxBytes + half * kResBoxBytes, col, m0);
          bulk_commit();
          // release the previous box once its store has read shared memory
          if (pend >= 0) {
            bulk_wait_read<1>();
            mbar_arrive(&res_empty[pend]);
          }
          pend = slot;
        }
        if (++slot == kResSlots) {
          slot = 0;
          ph ^= 1;
        }
      }
      tc_fence_before();
      if (CG == 2) {
        __syncwarp();
        if (lane_id() == 0) mbar_arrive_remote(map_rank(&tempty[acc], 0));  // leader's barrier
      } else {
        mbar_arrive(&tempty[acc]);
      }
    }
    if (storer) bulk_wait<0>();  // C written before the CTA retires
  } else {
    // epilogue: 8 warps; warp w covers TMEM lanes 32*(w%4)..+31 (tile rows)
    // and one column half.  Each 32x16 chunk goes TMEM -> registers (row per
    // lane, + bias / GELU) -> a padded per-warp smem stage -> coalesced
    // global stores (8 rows x 64 B per warp instruction).
    const int ew = (int)warp - 2;
    const uint32_t quad = warp & 3;
    const int c_begin = (ew >> 2) * (BN / 2);
    float* stage = epi_stage + ew * (32 * kStagePitch);
    const int sub_row = lane_id() >> 2;        // 0..7
    const int sub_col = (lane_id() & 3) * 4;   // 0..12
    int it = 0;
    for (int tile = unit; tile < num_tiles; tile += n_units, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb);
      const int m0 = mb * TM + (int)rank * BM, n0 = nb * BN;
      const int row_base = m0 + (int)quad * 32;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (ew == 0 && lane_id() == 0) GEMM_TRACE(2, it);
#pragma unroll 1
      for (int c = c_begin; c < c_begin + BN / 2; c += kChunk) {
        if (n0 + c >= N) break;  // ragged last column tile (warp-uniform; N % 64 == 0)
        uint32_t r[16];
        __syncwarp();
        tmem_ld16(tmem_base + ((quad * 32) << 16) + acc * BN + c, r);
        tmem_ld_wait();
        const int col = n0 + c;
        float* srow = stage + lane_id() * kStagePitch;
#pragma unroll
        for (int j = 0; j < kChunk; j += 4) {
          float4 v;
          v.x = __uint_as_float(r[j]) + (bias ? __ldg(bias + col + j) : 0.0f);
          v.y = __uint_as_float(r[j + 1]) + (bias ? __ldg(bias + col + j + 1) : 0.0f);
          v.z = __uint_as_float(r[j + 2]) + (bias ? __ldg(bias + col + j + 2) : 0.0f);
          v.w = __uint_as_float(r[j + 3]) + (bias ? __ldg(bias + col + j + 3) : 0.0f);
          if (MODE == kEpiGeluBf16) {
            v.x = gelu_tanh(v.x);
            v.y = gelu_tanh(v.y);
            v.z = gelu_tanh(v.z);
            v.w = gelu_tanh(v.w);
          }
          *reinterpret_cast<float4*>(srow + j) = v;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int lr = i * 8 + sub_row;
          const int row = row_base + lr;
          const float4 v = *reinterpret_cast<const float4*>(stage + lr * kStagePitch + sub_col);
          if (row < M) {
            if (MODE == kEpiStoreF32) {
              *reinterpret_cast<float4*>(static_cast<float*>(c_ptr) + (size_t)row * N + col + sub_col) = v;
            } else {
              uint2 pk;
              pk.x = pack_bf16(v.x, v.y);
              pk.y = pack_bf16(v.z, v.w);
              *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(c_ptr) + (size_t)row * N + col + sub_col) = pk;
            }
          }
        }
      }
      tc_fence_before();
      if (CG == 2) {
        __syncwarp();
        if (lane_id() == 0) mbar_arrive_remote(map_rank(&tempty[acc], 0));  // leader's barrier
      } else {
        mbar_arrive(&tempty[acc]);
      }
    }
  }
teardown:
  tc_fence_before();
  if (CG == 2) cluster_sync_all(); else __syncthreads();
  if (warp == 1) {
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::kTmemCols)
                   : "memory");
    else
      tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

int sm_count() { return current_sm_count(); }

template <int BN, int MODE, int CG>
int launch(const CUtensorMap& ma, const CUtensorMap& mb, void* C, int M, int N, int K,
           const float* bias, const float* gate, int gate_stride, int rows_per_gate, int gate_row0,
           cudaStream_t st) {
  using Cfg = GemmCfg<BN, CG, MODE == kEpiResidualF32>;
  // the residual mode reads / writes C through TMA: fp32 [M][N], 128 x 32 boxes
  CUtensorMap mc = ma;
  if (MODE == kEpiResidualF32)
    BC_RC(make_tmap_2d_f32(&mc, C, (uint64_t)N, (uint64_t)M, (uint64_t)N * 4, kResCols, BM, kResSwz));
  static PerDeviceOnce attrs_once;
  BC_RC(per_device_once(attrs_once, [&]() -> int {
    BC_CUDA(cudaFuncSetAttribute(gemm_kernel<BN, MODE, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Cfg::kSmem));
    return BC_OK;
  }));
  const int tiles = ((M + BM * CG - 1) / (BM * CG)) * ((N + BN - 1) / BN);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CG;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  // A persistent grid must be fully co-resident: the tiles are pre-assigned
  // per unit, so a unit that only starts when another finishes doubles the
  // kernel time.  Pairs need both CTAs on one TPC, and not every TPC of the
  // part is whole, so ask the occupancy calculator how many clusters fit.
  static PerDeviceOnce units_once;
  static int units_of[PerDeviceOnce::kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  const int slot = (dev >= 0 && dev < PerDeviceOnce::kMaxDevices) ? dev : 0;
  per_device_once(units_once, [&]() -> int {
    int units = sm_count() / CG;
    if (CG > 1) {
      cfg.gridDim = dim3(units * CG);
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, gemm_kernel<BN, MODE, CG>, &cfg) == cudaSuccess && n > 0 &&
          n < units)
        units = n;
      (void)cudaGetLastError();
    }
    units_of[slot] = units;
    return BC_OK;
  });
  const int units = units_of[slot] > 0 ? units_of[slot] : sm_count() / CG;
  const int grid = (tiles < units ? tiles : units) * CG;
  cfg.gridDim = dim3(grid);
  BC_CUDA(cudaLaunchKernelEx(&cfg, gemm_kernel<BN, MODE, CG>, ma, mb, mc, C, M, N, K, bias, gate, gate_stride,
                             rows_per_gate, gate_row0));
  BC_LAUNCHED();
  return BC_OK;
}

template <int BN, int CG>
int dispatch_mode(int mode, const CUtensorMap& ma, const CUtensorMap& mb, void* C, int M, int N,
                  int K, const float* bias, const float* gate, int gs, int rpg, int gr0, cudaStream_t st) {
  switch (mode) {
    case kEpiStoreBf16: return launch<BN, kEpiStoreBf16, CG>(ma, mb, C, M, N, K, bias, gate, gs, rpg, gr0, st);
    case kEpiGeluBf16: return launch<BN, kEpiGeluBf16, CG>(ma, mb, C, M, N, K, bias, gate, gs, rpg, gr0, st);
    case kEpiStoreF32: return launch<BN, kEpiStoreF32, CG>(ma, mb, C, M, N, K, bias, gate, gs, rpg, gr0, st);
    case kEpiResidualF32: return launch<BN, kEpiResidualF32, CG>(ma, mb, C, M, N, K, bias, gate, gs, rpg, gr0, st);
  }
  return bc_fail(BC_ERR_CONTRACT, "gemm: unknown epilogue mode %d", mode);
}

}  // namespace

static int make_tmap_2d_typed(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t inner,
                              uint64_t outer, uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                              int swizzle_bytes) {
  auto fn = encode_fn();
  if (!fn) return bc_fail(BC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old or no GPU)");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle swz = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return bc_fail(BC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BC_OK;
}

int make_tmap_2d_swz(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  return make_tmap_2d_typed(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, inner, outer, row_stride_bytes, box_inner,
                            box_outer, swizzle_bytes);
}

int make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  return make_tmap_2d_typed(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, inner, outer, row_stride_bytes, box_inner,
                            box_outer, swizzle_bytes);
}

int make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d_swz(map, base, inner, outer, row_stride_bytes, box_inner, box_outer, 128);
}

int num_sms() { return sm_count(); }

// Automatic tiling: (tile width, CTAs per tile) minimising
//   waves x (per-SM columns per tile) x relative cost per column,
// waves = ceil(tiles / units) over 148 single CTAs or 74 CTA pairs.  The
// relative costs are measured (scripts/gemm_tiling.py, profiles/
// r2_gemm_tiling.txt): 256-wide pair tiles amortise best; narrower or
// single-CTA tiles pay for more A/B panel traffic per column, least when a
// short-K gated-residual epilogue dominates.  Small M is where the choice
// matters: the width-1 sequential rows (4680) quantise to 2 waves of pair
// tiles at N = 1536 but exactly 3 waves of 128-wide single tiles (-13%); a
// 2925-row G = 8 slice fits one wave of pairs at N = 1536, K = 8960 (-21% vs
// the previous choice).  224-wide pair tiles (7 column tiles over N = 1536,
// the last one 192 wide and masked) turn the 19 x 6 = 114 pair tiles of a
// 4680-row, N = 1536 GEMM (1.54 waves of 256) into 133 (1.80 waves of 224):
// 2 waves either way, 12.5% fewer columns per wave.  Every tiling gives
// bit-identical results.
struct Tiling {
  int bn, cg;
};
Tiling gemm_plan(int M, int N, int K, int mode, int only_cg) {
  const bool epi_bound = mode == kEpiResidualF32 && K <= 2048;
  struct Cand {
    int bn, cg;
    double cost_compute, cost_epi;
  };
  static const Cand cands[] = {{256, 2, 1.00, 1.00}, {224, 2, 1.05, 1.00}, {192, 2, 1.04, 0.99},
                                {256, 1, 1.10, 1.05}, {128, 1, 1.50, 1.18}};
  const int sms = sm_count();
  Tiling best{N % 128 == 0 ? 128 : 64, 1};
  double best_cost = 1e300;
  for (const Cand& c : cands) {
    // 224-wide pair tiles may end in a ragged (masked) column tile; the
    // cost counts the padded width
    if ((c.bn != 224 && N % c.bn) || (only_cg && c.cg != only_cg)) continue;
    const long units = c.cg == 2 ? sms / 2 : sms;
    const long tiles = (long)((M + BM * c.cg - 1) / (BM * c.cg)) * ((N + c.bn - 1) / c.bn);
    const long waves = (tiles + units - 1) / units;
    const double cost = (double)waves * c.bn * (epi_bound ? c.cost_epi : c.cost_compute);
    if (cost < best_cost) {
      best_cost = cost;
      best = Tiling{c.bn, c.cg};
    }
  }
  return best;
}

int gemm_run(const GemmArgs& g, cudaStream_t st) {
  if (g.K % BK || g.N % 64 || g.M < 1)
    return bc_fail(BC_ERR_CONTRACT, "gemm: need K %% 64 == 0, N %% 64 == 0 (M=%d N=%d K=%d)", g.M, g.N, g.K);
  int bn = g.bn, cg = g.cg;
  if (!bn) {
    const Tiling t = gemm_plan(g.M, g.N, g.K, g.mode, g.cg);
    bn = t.bn;
    if (!cg) cg = t.cg;
  }
  // a forced width without a forced pairing: pairs for the widths that have them
  if (!cg) cg = (bn == 256 || bn == 224 || bn == 192) ? 2 : 1;
  if (cg == 2 && bn != 256 && bn != 224 && bn != 192) cg = 1;
  if (cg == 1 && (bn == 192 || bn == 224))
    return bc_fail(BC_ERR_CONTRACT, "gemm: %d-wide tiles need CTA pairs", bn);
  if (bn != 224 && g.N % bn)
    return bc_fail(BC_ERR_CONTRACT, "gemm: tile width %d does not fit N=%d", bn, g.N);
  CUtensorMap ma, mb;
  int rc = make_tmap_2d(&ma, g.A, g.K, g.M, (uint64_t)g.K * 2, BK, BM);
  if (rc) return rc;
  rc = make_tmap_2d(&mb, g.B, g.K, g.N, (uint64_t)g.K * 2, BK, bn / cg);
  if (rc) return rc;
  if (cg == 2 && bn == 224)
    return dispatch_mode<224, 2>(g.mode, ma, mb, g.C, g.M, g.N, g.K, g.bias, g.gate, g.gate_stride, g.rows_per_gate, g.gate_row0, st);
  if (cg == 2 && bn == 192)
    return dispatch_mode<192, 2>(g.mode, ma, mb, g.C, g.M, g.N, g.K, g.bias, g.gate, g.gate_stride, g.rows_per_gate, g.gate_row0, st);
  if (cg == 2)
    return dispatch_mode<256, 2>(g.mode, ma, mb, g.C, g.M, g.N, g.K, g.bias, g.gate, g.gate_stride, g.rows_per_gate, g.gate_row0, st);
  switch (bn) {
    case 256: return dispatch_mode<256, 1>(g.mode, ma, mb, g.C, g.M, g.N, g.K, g.bias, g.gate, g.gate_stride, g.rows_per_gate, g.gate_row0, st);
    case 128: return dispatch_mode<128, 1>(g.mode, ma, mb, g.C, g.M, g.N, g.K, g.bias, g.gate, g.gate_stride, g.rows_per_gate, g.gate_row0, st);
    case 64: return dispatch_mode<64, 1>(g.mode, ma, mb, g.C, g.M, g.N, g.K, g.bias, g.gate, g.gate_stride, g.rows_per_gate, g.gate_row0, st);
  }
  return bc_fail(BC_ERR_CONTRACT, "gemm: bad tile width %d", bn);
}

}  // namespace bc

// The automatic tiling bc_gemm_bf16 would use (host logic only: the CPU
// tests pin the choices for the DiT's shapes).
extern "C" int bc_gemm_plan(int32_t M, int32_t N, int32_t K, int32_t mode, int32_t* bn, int32_t* cg) {
  if (!bn || !cg || M < 1 || N % 64 || K % 64) return bc_fail(BC_ERR_CONTRACT, "bc_gemm_plan: bad arguments");
  const bc::Tiling t = bc::gemm_plan(M, N, K, mode & 0xff, 0);
  *bn = t.bn;
  *cg = t.cg;
  return BC_OK;
}

extern "C" int bc_gemm_bf16(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                            int32_t mode, const float* bias, const float* gate, int32_t gate_stride,
                            int32_t rows_per_gate, void* stream) {
  // mode bits 0-7: epilogue; bits 8-15: forced tile width (0 = auto) in
  // units of 64 columns, or of 32 when bit 18 is set (224 = 7 << 8 | 1 << 18);
  // bits 16-17: 1 = single-CTA tiles only, 2 = CTA pairs when possible
  const int width_unit = (mode >> 18) & 1 ? 32 : 64;
  bc::GemmArgs g{A, B, C, M, N, K, mode & 0xff, bias, gate, gate_stride,
                 rows_per_gate > 0 ? rows_per_gate : 1, ((mode >> 8) & 0xff) * width_unit,
                 (mode >> 16) & 3, 0};
  return bc::gemm_run(g, (cudaStream_t)stream);
}
