// Wan2.1-shaped causal 3-D VAE decoder on sm_100a (SURVEY.md §8f rank 1:
// "VAE decode on a separate GPU, overlapped with the next iteration").
// The reference decodes through a linear stand-in (executor.py:189-212)
// charged by a cost model (engine.py:151-158); the paper's streaming FPS
// includes decoding.  The network restated here is the public
// Wan2.1 VAE decoder (oracle/vae.py is the fp32 checker).
//
// Activation layout ("padded frames"): bf16 / fp32 channels-last
//   [n_frames][H + 2][W + 2][C]
// with a zero border one pixel wide that nothing ever writes, and the first
// two frames of a conv input holding that conv's causal history (the last
// two input frames of the previous block; zeros before the first block).
// Flat row index o = (frame * (H + 2) + y + 1) * (W + 2) + x + 1.  Because
// the border is zero, EVERY tap (kt, kh, kw) of a causal 3x3x3 conv is a
// uniform row shift of the same flat 2-D tensor [rows][C]:
//   o + (kt - 2) * F + (kh - 1) * (W + 2) + (kw - 1),   F = (H + 2)(W + 2)
// so the implicit-GEMM A operand of a tap is 128 consecutive rows.
//
// conv_kernel (tcgen05 implicit GEMM): one CTA per SM, persistent over
// units of R consecutive 128-row output tiles x `ncol` output channels.
//   warp 0  TMA: per (kt, kh, channel chunk) ONE A strip of R*128 + 8 rows
//           (the +2 rows of the kw halo), then per kw the weight tile of
//           that tap [ncol][CK] -- two rings (A strips, B taps).
//   warp 1  MMA: the three kw taps read the same strip through descriptors
//           shifted by kw rows (the swizzle is applied on absolute smem
//           addresses, so a row shift needs no base offset -- measured,
//           scripts/shift_desc_probe.cu), so each A byte from L2 feeds 3 taps.
//           R accumulators of ncol fp32 columns in TMEM.
//   warps 2-5 epilogue, one output row per thread: + bias (+ fp32 residual),
//           stores fp32 / bf16, and the NEXT layer's input fused in:
//           silu(RMS_norm(y) * gamma) (F.normalize over channels * sqrt(C)),
//           computed with a second TMEM pass (y is written back to TMEM);
//           the head mode writes the clamped video frame channel-first.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "bc_common.h"
#include "gemm.h"
#include "sm100.cuh"

namespace bc {
namespace {

constexpr int kConvThreads = 320;  // TMA warp, MMA warp, 8 epilogue warps

template <int CK, int R, int NMAX>
struct ConvCfg {
  static constexpr int kRowBytes = CK * 2;  // 64 (SW64) or 128 (SW128)
  static constexpr int kStripRows = R * 128 + 8;
  static constexpr int kABytes = ((kStripRows * kRowBytes + 1023) / 1024) * 1024;
  static constexpr int kBBytes = ((NMAX * kRowBytes + 1023) / 1024) * 1024;
  static constexpr int kBudget = 200 * 1024;
#ifndef BC_VAE_SA_MAX
#define BC_VAE_SA_MAX 4
#endif
#ifndef BC_VAE_SB_MAX
#define BC_VAE_SB_MAX 8
#endif
  // one B stage holds the weights of all kw taps of a (kt, kh, channel
  // chunk): the MMA issuer then runs kw x R x CK/16 MMAs per barrier wait.
  // With one tap per stage a group was only R x CK/16 = 4 MMAs (192 cycles
  // of tensor work at N = 96) and the ~150-cycle issue gap between groups
  // (commits, the next stage's wait, descriptor setup) left the tensor pipe
  // ~50% idle -- the pipe queues barely more than one instruction.
  static constexpr int kTapsPerB = 3;
  static constexpr int kBStage = kTapsPerB * kBBytes;
  static constexpr int kSB0 = (96 * 1024) / kBStage;
  static constexpr int kSB = kSB0 < 2 ? 2 : kSB0 > BC_VAE_SB_MAX ? BC_VAE_SB_MAX : kSB0;
  static constexpr int kSA0 = (kBudget - kSB * kBStage) / kABytes;
  static constexpr int kSA = kSA0 < 2 ? 2 : kSA0 > BC_VAE_SA_MAX ? BC_VAE_SA_MAX : kSA0;
  static constexpr int kAcc = 2 * R * NMAX <= 512 ? 2 : 1;  // double-buffered accumulators when they fit
  static constexpr int kCols = kAcc * R * NMAX;
  static constexpr int kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
  static constexpr size_t kSmem = 1024 + (size_t)kSA * kABytes + (size_t)kSB * kBStage + 512 + 1024;
  static_assert(kCols <= 512, "TMEM holds 512 fp32 columns");
  static_assert(kSmem <= 227 * 1024, "shared memory");
};

struct ConvParams {
  int H, W, Wp, F;      // valid extent, padded width, rows per frame
  int row0, rows;       // output flat rows [row0, row0 + rows)
  int cin, cout, ncol;  // ncol: output channels per unit (<= NMAX)
  int kt, kh, kw, n_cc;
  int num_mg, num_ng;
  int ilv_t, ilv_per;   // unit order: ilv_t frame slots of ilv_per row groups (see unit_of)
  const float* bias;
  const float* res;
  float* out32;
  __nv_bfloat16* out16;
  __nv_bfloat16* act;
  const float* gamma;
  int act_silu;
  float* video;
  int video_ch, video_frame0;
};

__device__ __forceinline__ uint64_t desc_swz(uint32_t addr, uint32_t row_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                                   // LBO (unused, swizzled K-major)
  d |= (uint64_t)(((8 * row_bytes) >> 4) & 0x3FFF) << 32;   // SBO: 8-row atom
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(row_bytes == 128 ? 2 : 4) << 61;          // SWIZZLE_128B / SWIZZLE_64B
  return d;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ float silu(float a) { return a * __frcp_rn(1.0f + __expf(-a)); }
// 256-bit global accesses (sm_100: one full 32-byte sector per lane)
__device__ __forceinline__ void ld8f(const float* p, float (&r)[8]) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void st8f(float* p, const float* r) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]),
               "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
               : "memory");
}
__device__ __forceinline__ void st8bf16x2(void* p, const float* r) {  // 16 floats -> 16 bf16 (32 B)
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(pack_bf16(r[0], r[1])),
               "r"(pack_bf16(r[2], r[3])), "r"(pack_bf16(r[4], r[5])), "r"(pack_bf16(r[6], r[7])),
               "r"(pack_bf16(r[8], r[9])), "r"(pack_bf16(r[10], r[11])), "r"(pack_bf16(r[12], r[13])),
               "r"(pack_bf16(r[14], r[15]))
               : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Execution order of the units (R 128-row tiles x ncol channels): unit u
// -> row group mg = (u_m % ilv_t) * ilv_per + u_m / ilv_t.  With ilv_t = the
// conv's output frames and ilv_per ~ row groups per frame, the ~148 units in
// flight cover the same spatial rows of EVERY frame, so the kt = 0/1/2 taps
// (frames f-2, f-1, f of the input) are read while the neighbouring frames'
// units still hold them in L2 -- in plain row order the three input windows
// are a frame (40-80 MB) apart and each input row came from DRAM once per
// kt.  Returns false for the padding slots of the last frame.
__device__ __forceinline__ bool unit_of(const ConvParams& p, int u, int& mg, int& ng) {
  const int um = u / p.num_ng;
  ng = u - um * p.num_ng;
  mg = (um % p.ilv_t) * p.ilv_per + um / p.ilv_t;
  return mg < p.num_mg;
}

template <int CK, int R, int NMAX>
__global__ void __launch_bounds__(kConvThreads, 1)
    conv_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_a8,
                const __grid_constant__ CUtensorMap map_b, const __grid_constant__ ConvParams p) {
  using Cfg = ConvCfg<CK, R, NMAX>;
  constexpr int SA = Cfg::kSA, SB = Cfg::kSB, RB = Cfg::kRowBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + SA * Cfg::kABytes;
  uint64_t* afull = reinterpret_cast<uint64_t*>(sb + SB * Cfg::kBStage);
  uint64_t* aempty = afull + SA;
  uint64_t* bfull = aempty + SA;
  uint64_t* bempty = bfull + SB;
  uint64_t* tfull = bempty + SB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* ss_part = reinterpret_cast<float*>(smem + SA * Cfg::kABytes + SB * Cfg::kBStage + 512);  // [4][2][32]

  const uint32_t warp = warp_id();
  const int n_units = p.ilv_t * p.ilv_per * p.num_ng;
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_a8);
    tma_prefetch(&map_b);
    for (int i = 0; i < SA; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < SB; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane_id() == 0) {
      int ia = 0, ib = 0;
      uint32_t pa = 0, pb = 0;
      const uint32_t a_bytes = (R * 128 + 8) * RB, b_bytes = p.ncol * RB;
      for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
        int mg, ng;
        if (!unit_of(p, unit, mg, ng)) continue;
        const int o0 = p.row0 + mg * R * 128, n0 = ng * p.ncol;
        for (int kt = 0; kt < p.kt; ++kt)
          for (int kh = 0; kh < p.kh; ++kh)
            for (int cc = 0; cc < p.n_cc; ++cc) {
              mbar_wait(&aempty[ia], pa ^ 1);
              mbar_arrive_expect_tx(&afull[ia], a_bytes);
              const int base = o0 + (kt - (p.kt - 1)) * p.F + (kh - (p.kh - 1) / 2) * p.Wp - (p.kw - 1) / 2;
              uint8_t* dst = sa + ia * Cfg::kABytes;
#pragma unroll
              for (int r = 0; r < R; ++r) tma_load_2d(dst + r * 128 * RB, &map_a, &afull[ia], cc * CK, base + r * 128);
              tma_load_2d(dst + R * 128 * RB, &map_a8, &afull[ia], cc * CK, base + R * 128);
              if (++ia == SA) {
                ia = 0;
                pa ^= 1;
              }
              mbar_wait(&bempty[ib], pb ^ 1);
              mbar_arrive_expect_tx(&bfull[ib], p.kw * b_bytes);
              for (int kw = 0; kw < p.kw; ++kw) {
                const int tap = (kt * p.kh + kh) * p.kw + kw;
                tma_load_2d(sb + ib * Cfg::kBStage + kw * Cfg::kBBytes, &map_b, &bfull[ib], tap * p.cin + cc * CK,
                            n0);
              }
              if (++ib == SB) {
                ib = 0;
                pb ^= 1;
              }
            }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16(128, p.ncol);
    const int stages = p.kt * p.kh * p.n_cc;
    int ia = 0, ib = 0, it = 0;
    uint32_t pa = 0, pb = 0;
    for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
      int mg, ng;
      if (!unit_of(p, unit, mg, ng)) continue;
      const int acc = Cfg::kAcc == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = Cfg::kAcc == 2 ? ((it >> 1) & 1) : (it & 1);
      ++it;
      const uint32_t d_base = tmem_base + acc * (R * NMAX);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      for (int s = 0; s < stages; ++s) {
        mbar_wait(&afull[ia], pa);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sa + ia * Cfg::kABytes);
        mbar_wait(&bfull[ib], pb);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t b0 = smem_u32(sb + ib * Cfg::kBStage);
          for (int kw = 0; kw < p.kw; ++kw)
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
              for (int k = 0; k < CK / 16; ++k)
                mma_bf16_ss(d_base + r * NMAX, desc_swz(a0 + (r * 128 + kw) * RB + k * 32, RB),
                            desc_swz(b0 + kw * Cfg::kBBytes + k * 32, RB), idesc, (s | kw | k) != 0);
          mma_commit(&bempty[ib]);
          mma_commit(&aempty[ia]);
          if (s == stages - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++ib == SB) {
          ib = 0;
          pb ^= 1;
        }
        if (++ia == SA) {
          ia = 0;
          pa ^= 1;
        }
      }
    }
  } else {
    // 8 epilogue warps: two per TMEM lane quadrant, interleaved 16-column
    // chunks (even chunks to the first, odd to the second).  A row's
    // residual loads are all issued before its first TMEM load; the fused
    // norm's sum of squares is combined across the pair through shared
    // memory and a 64-thread named barrier per quadrant.
    constexpr int kMaxMine = (NMAX / 16 + 1) / 2;  // chunks per warp of the pair
    const uint32_t quad = warp & 3;
    const int half = ((int)warp - 2) >> 2;
    const int n_chunks = p.ncol / 16;
    const int mine = (n_chunks - half + 1) / 2;
    const int row_end = p.row0 + p.rows;
    const float norm_scale = sqrtf((float)p.cout);
    float* ssx = ss_part + quad * 64;
    int it = 0;
    for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
      int mg, ng;
      if (!unit_of(p, unit, mg, ng)) continue;
      const int o0 = p.row0 + mg * R * 128, n0 = ng * p.ncol;
      const int acc = Cfg::kAcc == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = Cfg::kAcc == 2 ? ((it >> 1) & 1) : (it & 1);
      ++it;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const int row = o0 + r * 128 + (int)quad * 32 + (int)lane_id();
        const int f = row / p.F;
        const int rem = row - f * p.F;
        const int yy = rem / p.Wp, xx = rem - (rem / p.Wp) * p.Wp;
        const bool valid = row < row_end && yy >= 1 && yy <= p.H && xx >= 1 && xx <= p.W;
        const uint32_t taddr = tmem_base + ((quad * 32) << 16) + (acc * R + r) * NMAX;
        // residual loads run kPre chunks ahead of their use (rolling buffer)
        constexpr int kPre = kMaxMine <= 3 ? kMaxMine : 2;
        float rq[kPre][16];
        const bool do_res = p.res && valid;
        auto load_res = [&](int i) {
          const float* src = p.res + (size_t)row * p.cout + n0 + (2 * i + half) * 16;
          float t0[8], t1[8];
          ld8f(src, t0);
          ld8f(src + 8, t1);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            rq[i % kPre][j] = t0[j];
            rq[i % kPre][8 + j] = t1[j];
          }
        };
        if (do_res) {
#pragma unroll
          for (int i = 0; i < kPre; ++i)
            if (i < mine) load_res(i);
        }
        float y[kMaxMine][16];
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < kMaxMine; ++i) {
          if (i < mine) {
            const int c = (2 * i + half) * 16;
            uint32_t v[16];
            tmem_ld16(taddr + c, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) y[i][j] = __uint_as_float(v[j]) + __ldg(p.bias + n0 + c + j);
            const size_t off = (size_t)row * p.cout + n0 + c;
            if (do_res) {
#pragma unroll
              for (int j = 0; j < 16; ++j) y[i][j] += rq[i % kPre][j];
              if (i + kPre < mine) load_res(i + kPre);
            }
            if (valid) {
              if (p.out32) {
                st8f(p.out32 + off, &y[i][0]);
                st8f(p.out32 + off + 8, &y[i][8]);
              }
              if (p.out16) st8bf16x2(p.out16 + off, &y[i][0]);
              if (p.video && c == 0) {
                const int vf = f - p.row0 / p.F + p.video_frame0;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (j < p.video_ch)
                    p.video[(((size_t)vf * p.video_ch + j) * p.H + (yy - 1)) * p.W + (xx - 1)] =
                        fminf(1.0f, fmaxf(-1.0f, y[i][j]));
              }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) ss = fmaf(y[i][j], y[i][j], ss);
          }
        }
        if (p.act) {
          ssx[half * 32 + lane_id()] = ss;
          named_bar_sync(1 + quad, 64);
          const float tot = ssx[lane_id()] + ssx[32 + lane_id()];
          named_bar_sync(1 + quad, 64);       // both read before the next row writes
          const float inv = norm_scale / fmaxf(sqrtf(tot), 1e-12f);
#pragma unroll
          for (int i = 0; i < kMaxMine; ++i) {
            if (i < mine) {
              const int c = (2 * i + half) * 16;
              float a[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                a[j] = y[i][j] * inv * __ldg(p.gamma + n0 + c + j);
                if (p.act_silu) a[j] = silu(a[j]);
              }
              if (valid) st8bf16x2(p.act + (size_t)row * p.cout + n0 + c, a);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
}

template <int CK, int R, int NMAX>
int conv_launch(const bc_vae_conv_args& a, int ncol, cudaStream_t st) {
  using Cfg = ConvCfg<CK, R, NMAX>;
  ConvParams p{};
  p.H = a.H;
  p.W = a.W;
  p.Wp = a.W + 2;
  p.F = (a.H + 2) * (a.W + 2);
  p.row0 = a.frame0 * p.F;
  p.rows = a.n_out_frames * p.F;
  p.cin = a.cin;
  p.cout = a.cout;
  p.ncol = ncol;
  p.kt = a.kt;
  p.kh = a.kh;
  p.kw = a.kw;
  p.n_cc = a.cin / CK;
  const int tiles = (p.rows + 127) / 128;
  p.num_mg = (tiles + R - 1) / R;
  p.num_ng = a.cout / ncol;
  static const int ilv_env = [] {
    const char* e = getenv("BC_VAE_ILV");
    return e ? atoi(e) : 1;
  }();
  p.ilv_t = (ilv_env && a.kt > 1 && a.n_out_frames > 1 && p.num_mg >= a.n_out_frames) ? a.n_out_frames : 1;
  p.ilv_per = (p.num_mg + p.ilv_t - 1) / p.ilv_t;
  p.bias = a.bias;
  p.res = a.res;
  p.out32 = a.out32;
  p.out16 = static_cast<__nv_bfloat16*>(a.out16);
  p.act = static_cast<__nv_bfloat16*>(a.act);
  p.gamma = a.gamma;
  p.act_silu = a.act_silu;
  p.video = a.video;
  p.video_ch = a.video_channels;
  p.video_frame0 = a.video_frame0;
  const uint64_t total_rows = (uint64_t)a.n_frames * p.F;
  const int taps = a.kt * a.kh * a.kw;
  CUtensorMap ma, ma8, mb;
  BC_RC(make_tmap_2d_swz(&ma, a.in, a.cin, total_rows, (uint64_t)a.cin * 2, CK, 128, CK * 2));
  BC_RC(make_tmap_2d_swz(&ma8, a.in, a.cin, total_rows, (uint64_t)a.cin * 2, CK, 8, CK * 2));
  BC_RC(make_tmap_2d_swz(&mb, a.w, (uint64_t)taps * a.cin, a.cout, (uint64_t)taps * a.cin * 2, CK, ncol, CK * 2));
  static PerDeviceOnce once;
  BC_RC(per_device_once(once, [&]() -> int {
    BC_CUDA(cudaFuncSetAttribute(conv_kernel<CK, R, NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Cfg::kSmem));
    return BC_OK;
  }));
  const int units = p.ilv_t * p.ilv_per * p.num_ng;
  const int sms = current_sm_count();
  conv_kernel<CK, R, NMAX><<<units < sms ? units : sms, kConvThreads, Cfg::kSmem, st>>>(ma, ma8, mb, p);
  BC_LAUNCHED();
  return BC_OK;
}

// ------------------------------------------------------------ bandwidth ops

// z [T][zc][H][W] fp32 (channel-first, the engine's block latents) ->
// z * std + mean -> conv2 (1x1x1, zc -> zc, fp32) -> bf16 padded frames
// [frame0 + t][..][cpad] (channels zc..cpad-1 stay zero).
__global__ void prep_kernel(const float* __restrict__ z, const float* __restrict__ w2, const float* __restrict__ b2,
                            const float* __restrict__ mean, const float* __restrict__ stdv,
                            __nv_bfloat16* __restrict__ out, int T, int zc, int H, int W, int frame0, int cpad) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int hw = H * W;
  if (idx >= T * hw) return;
  const int t = idx / hw, pix = idx - t * hw, y = pix / W, x = pix - (pix / W) * W;
  float zz[16];
  for (int c = 0; c < zc; ++c) zz[c] = z[((size_t)t * zc + c) * hw + pix] * stdv[c] + mean[c];
  const size_t row = ((size_t)(frame0 + t) * (H + 2) + y + 1) * (W + 2) + x + 1;
  for (int o = 0; o < zc; ++o) {
    float acc = b2[o];
    for (int c = 0; c < zc; ++c) acc = fmaf(w2[o * zc + c], zz[c], acc);
    out[row * cpad + o] = __float2bfloat16_rn(acc);
  }
}

// nearest-exact x2 upsample of fp32 source frames into bf16 padded frames of
// the next level.  Output frame j reads source frame map->frame[j] of source
// map->src[j] (0: a, channel stride C; 1: b, channel stride 2C at channel
// offset map->chan[j]) -- the time-conv output's two halves interleaved in
// time (Resample 'upsample3d'), or the plain stream (first frame /
// 'upsample2d').
__global__ void upsample_kernel(const float* __restrict__ a, const float* __restrict__ b, bc_vae_frame_map map,
                                int C, int H, int W, __nv_bfloat16* __restrict__ out, int out_frame0, int n_out) {
  const int groups = C / 8;
  const int H2 = 2 * H, W2 = 2 * W;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)n_out * H2 * W2 * groups;
  if (idx >= total) return;
  const int g = (int)(idx % groups);
  long long r = idx / groups;
  const int x2 = (int)(r % W2);
  r /= W2;
  const int y2 = (int)(r % H2);
  const int j = (int)(r / H2);
  const int src = map.src[j];
  const float* s = src ? b : a;
  const int stride = src ? 2 * C : C;
  const size_t srow = ((size_t)map.frame[j] * (H + 2) + (y2 >> 1) + 1) * (W + 2) + (x2 >> 1) + 1;
  const float4* sp = reinterpret_cast<const float4*>(s + srow * stride + map.chan[j] + g * 8);
  const float4 u = sp[0], v = sp[1];
  uint4 o;
  o.x = pack_bf16(u.x, u.y);
  o.y = pack_bf16(u.z, u.w);
  o.z = pack_bf16(v.x, v.y);
  o.w = pack_bf16(v.z, v.w);
  const size_t orow = ((size_t)(out_frame0 + j) * (H2 + 2) + y2 + 1) * (W2 + 2) + x2 + 1;
  *reinterpret_cast<uint4*>(out + orow * C + g * 8) = o;
}

// AttentionBlock operands of one frame from the padded qkv rows [..][3C]:
// q, k [np][C] and v^T [C][np] (tokens in h*w order, rows >= H*W zero).
__global__ void attn_gather_kernel(const __nv_bfloat16* __restrict__ qkv, int frame, int H, int W, int C, int np,
                                   __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                                   __nv_bfloat16* __restrict__ vt) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int groups = C / 8;
  if (idx >= np * groups) return;
  const int t = idx % np, g = idx / np;
  uint4 qa = make_uint4(0, 0, 0, 0), ka = qa, va = qa;
  if (t < H * W) {
    const int y = t / W, x = t - (t / W) * W;
    const size_t row = ((size_t)frame * (H + 2) + y + 1) * (W + 2) + x + 1;
    const uint4* src = reinterpret_cast<const uint4*>(qkv + row * 3 * C);
    qa = src[g];
    ka = src[groups + g];
    va = src[2 * groups + g];
  }
  reinterpret_cast<uint4*>(q + (size_t)t * C)[g] = qa;
  reinterpret_cast<uint4*>(k + (size_t)t * C)[g] = ka;
  const __nv_bfloat16* vv = reinterpret_cast<const __nv_bfloat16*>(&va);
#pragma unroll
  for (int i = 0; i < 8; ++i) vt[(size_t)(g * 8 + i) * np + t] = vv[i];
}

// row softmax of S [rows][np] (first n_valid columns), scaled; P bf16
__global__ void softmax_kernel(const float* __restrict__ S, __nv_bfloat16* __restrict__ P, int np, int n_valid,
                               float scale) {
  const float* s = S + (size_t)blockIdx.x * np;
  __nv_bfloat16* o = P + (size_t)blockIdx.x * np;
  __shared__ float red[32];
  float m = -INFINITY;
  for (int c = threadIdx.x; c < n_valid; c += blockDim.x) m = fmaxf(m, s[c]);
  for (int sh = 16; sh; sh >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, sh));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
    for (int sh = 16; sh; sh >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, sh));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int c = threadIdx.x; c < n_valid; c += blockDim.x) sum += __expf((s[c] - m) * scale);
  for (int sh = 16; sh; sh >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, sh);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int sh = 16; sh; sh >>= 1) v += __shfl_xor_sync(0xffffffffu, v, sh);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.0f / red[0];
  for (int c = threadIdx.x; c < np; c += blockDim.x)
    o[c] = __float2bfloat16_rn(c < n_valid ? __expf((s[c] - m) * scale) * inv : 0.f);
}

// AttentionBlock residual: x[row] += proj[t] (bias already in proj), then the
// next conv's input act = silu(RMS_norm(x) * gamma).  One warp per pixel.
__global__ void attn_out_kernel(float* __restrict__ x, const float* __restrict__ proj,
                                const float* __restrict__ gamma, __nv_bfloat16* __restrict__ act, int frame, int H,
                                int W, int C) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= H * W) return;
  const int y = warp / W, xx = warp - (warp / W) * W;
  const size_t row = ((size_t)frame * (H + 2) + y + 1) * (W + 2) + xx + 1;
  float* xr = x + row * C;
  const float* pr = proj + (size_t)warp * C;
  float ss = 0.f;
  for (int c = lane; c < C; c += 32) {
    const float v = xr[c] + pr[c];
    xr[c] = v;
    ss = fmaf(v, v, ss);
  }
  for (int sh = 16; sh; sh >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, sh);
  const float inv = sqrtf((float)C) / fmaxf(sqrtf(ss), 1e-12f);
  for (int c = lane; c < C; c += 32) act[row * C + c] = __float2bfloat16_rn(silu(xr[c] * inv * gamma[c]));
}

// silu?(RMS_norm(x) * gamma) of fp32 padded frames [frame0, frame0 + n)
// into bf16 (the next conv's input) -- for convs whose output row does not
// fit one unit (cout 384), where the norm cannot be fused.  Warp per pixel.
__global__ void norm_act_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                                __nv_bfloat16* __restrict__ act, int frame0, int n, int H, int W, int C,
                                int use_silu) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n * H * W) return;
  const int f = warp / (H * W), pix = warp - f * (H * W), y = pix / W, xx = pix - (pix / W) * W;
  const size_t row = ((size_t)(frame0 + f) * (H + 2) + y + 1) * (W + 2) + xx + 1;
  const float* xr = x + row * C;
  float ss = 0.f;
  for (int c = lane * 4; c < C; c += 128) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
  }
  for (int sh = 16; sh; sh >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, sh);
  const float inv = sqrtf((float)C) / fmaxf(sqrtf(ss), 1e-12f);
  for (int c = lane * 4; c < C; c += 128) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    float a0 = v.x * inv * gamma[c], a1 = v.y * inv * gamma[c + 1], a2 = v.z * inv * gamma[c + 2],
          a3 = v.w * inv * gamma[c + 3];
    if (use_silu) {
      a0 = silu(a0);
      a1 = silu(a1);
      a2 = silu(a2);
      a3 = silu(a3);
    }
    uint2 o;
    o.x = pack_bf16(a0, a1);
    o.y = pack_bf16(a2, a3);
    *reinterpret_cast<uint2*>(act + row * C + c) = o;
  }
}

}  // namespace
}  // namespace bc

using namespace bc;

extern "C" int bc_vae_norm_act(const float* x, const float* gamma, void* act, int32_t frame0, int32_t n_frames,
                               int32_t H, int32_t W, int32_t C, int32_t use_silu, void* stream) {
  if (C % 4) return bc_fail(BC_ERR_CONTRACT, "vae_norm_act: C %d", C);
  const long long threads = (long long)n_frames * H * W * 32;
  norm_act_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      x, gamma, static_cast<__nv_bfloat16*>(act), frame0, n_frames, H, W, C, use_silu);
  BC_LAUNCHED();
  return BC_OK;
}

extern "C" int bc_vae_conv(const bc_vae_conv_args* a, void* stream) {
  if (!a || !a->in || !a->w || !a->bias) return bc_fail(BC_ERR_CONTRACT, "vae_conv: null operand");
  if (a->cin % 32 || a->cout % 16 || a->H < 1 || a->W < 1 || a->n_out_frames < 1 || a->frame0 < a->kt - 1 ||
      a->frame0 + a->n_out_frames > a->n_frames || (a->kh != 1 && a->kh != 3) || (a->kw != 1 && a->kw != 3) ||
      (a->kt != 1 && a->kt != 3))
    return bc_fail(BC_ERR_CONTRACT, "vae_conv: bad geometry (cin %d cout %d kt %d kh %d kw %d frames %d+%d of %d)",
                   a->cin, a->cout, a->kt, a->kh, a->kw, a->frame0, a->n_out_frames, a->n_frames);
  if (a->video && a->video_channels > 16) return bc_fail(BC_ERR_CONTRACT, "vae_conv: video channels > 16");
  cudaStream_t st = (cudaStream_t)stream;
  // unit shape: >= 128 output channels -> 2 row tiles x (up to 192) columns,
  // else 4 row tiles x cout columns (TMEM: R * columns <= 384 of 512)
  if (a->cout >= 128) {
    const int ncol = a->cout % 192 == 0 ? 192 : a->cout % 128 == 0 ? 128 : a->cout % 96 == 0 ? 96 : 64;
    if (a->cout % ncol) return bc_fail(BC_ERR_CONTRACT, "vae_conv: cout %d has no tile width", a->cout);
    if ((a->act || a->video) && ncol != a->cout)
      return bc_fail(BC_ERR_CONTRACT, "vae_conv: fused norm needs the whole row in one unit (cout %d)", a->cout);
    // a unit holding a whole 192-channel row with a fused norm: one row tile,
    // double-buffered accumulators (the epilogue overlaps the next mainloop)
    static const int r1 = [] {
      const char* e = getenv("BC_VAE_R1");
      return e ? atoi(e) : 1;
    }();
    if (r1 && a->cin % 64 == 0 && ncol == a->cout && a->act) return conv_launch<64, 1, 192>(*a, ncol, st);
    return a->cin % 64 == 0 ? conv_launch<64, 2, 192>(*a, ncol, st) : conv_launch<32, 2, 192>(*a, ncol, st);
  }
  static const int r4 = [] {
    const char* e = getenv("BC_VAE_R4");
    return e ? atoi(e) : 0;
  }();
  if (r4) return conv_launch<32, 4, 96>(*a, a->cout, st);
  return conv_launch<32, 2, 96>(*a, a->cout, st);
}

extern "C" int bc_vae_prep(const float* z, const float* w2, const float* b2, const float* mean, const float* stdv,
                           void* out, int32_t T, int32_t zc, int32_t H, int32_t W, int32_t frame0, int32_t cpad,
                           void* stream) {
  if (zc > 16 || zc > cpad) return bc_fail(BC_ERR_CONTRACT, "vae_prep: z channels %d (cpad %d)", zc, cpad);
  const int n = T * H * W;
  prep_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(z, w2, b2, mean, stdv,
                                                                   static_cast<__nv_bfloat16*>(out), T, zc, H, W,
                                                                   frame0, cpad);
  BC_LAUNCHED();
  return BC_OK;
}

extern "C" int bc_vae_upsample(const float* a, const float* b, const bc_vae_frame_map* map, int32_t C, int32_t H,
                               int32_t W, void* out, int32_t out_frame0, int32_t n_out, void* stream) {
  if (!map || n_out < 1 || n_out > BC_VAE_MAX_FRAMES || C % 8)
    return bc_fail(BC_ERR_CONTRACT, "vae_upsample: bad frame map (n_out %d, C %d)", n_out, C);
  const long long total = (long long)n_out * 4 * H * W * (C / 8);
  upsample_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      a, b, *map, C, H, W, static_cast<__nv_bfloat16*>(out), out_frame0, n_out);
  BC_LAUNCHED();
  return BC_OK;
}

extern "C" int bc_vae_attn_gather(const void* qkv, int32_t frame, int32_t H, int32_t W, int32_t C, int32_t np,
                                  void* q, void* k, void* vt, void* stream) {
  if (np < H * W || C % 8) return bc_fail(BC_ERR_CONTRACT, "vae_attn_gather: np %d < %d tokens", np, H * W);
  const int n = np * (C / 8);
  attn_gather_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const __nv_bfloat16*>(qkv), frame, H, W, C, np, static_cast<__nv_bfloat16*>(q),
      static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(vt));
  BC_LAUNCHED();
  return BC_OK;
}

extern "C" int bc_vae_softmax(const float* S, void* P, int32_t rows, int32_t np, int32_t n_valid, float scale,
                              void* stream) {
  softmax_kernel<<<rows, 256, 0, (cudaStream_t)stream>>>(S, static_cast<__nv_bfloat16*>(P), np, n_valid, scale);
  BC_LAUNCHED();
  return BC_OK;
}

extern "C" int bc_vae_attn_out(float* x, const float* proj, const float* gamma, void* act, int32_t frame, int32_t H,
                               int32_t W, int32_t C, void* stream) {
  const long long threads = (long long)H * W * 32;
  attn_out_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      x, proj, gamma, static_cast<__nv_bfloat16*>(act), frame, H, W, C);
  BC_LAUNCHED();
  return BC_OK;
}
