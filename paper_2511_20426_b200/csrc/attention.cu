// tcgen05 flash attention over the paged KV arena (self-attention of the
// cascade) or a dense K/V (text cross-attention).
//
// Semantics = reference layer_attend + _gather (denoiser.py:264-296):
// for the queries of batch entry e, keys/values are the concatenation of the
// visible blocks' K/V in ascending block order -- here the arena slots
// vis_slot[e][0..n_vis) in that order -- and softmax runs over exactly those
// keys.  Key tiles are consumed strictly in that order (no split-K, no
// atomics), so results are independent of how many entries share a launch.
//
// One CTA = one 128-row query tile x one head x one entry.
//   warp 0     TMA: Q once, then K_j / V_j (128 keys x 128 dims, 2 stages)
//   warp 1     MMA: S_j = Q K_j^T into TMEM (double-buffered),
//                   O += P_j V_j into TMEM (P from smem, V MN-major)
//   warps 2-5  softmax: thread = query row; S row from TMEM, online softmax
//              with lazy rescale (only when the running max grows by > 2^8),
//              P_j (bf16) written to smem in the UMMA K-major SW128 layout.
// TMEM: S0 [0,128) S1 [128,256) O [256,384).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdint.h>

#include "attention.h"
#include "bc_common.h"
#include "gemm.h"
#include "sm100.cuh"

namespace bc {
namespace {

constexpr int kRows = 128;     // query rows per CTA
constexpr int kKeys = 128;     // keys per tile
constexpr int kHd = 128;       // head dim
constexpr int kHalf = 128 * 64 * 2;   // one 64-column half tile (16 KB)
constexpr int kTile = 2 * kHalf;      // 128 x 128 bf16 (32 KB)
constexpr int kStages = 2;
constexpr int kThreads = 192;
constexpr float kRescaleThresh = 8.0f;  // log2 domain

struct AttnSmem {
  static constexpr int q = 0;
  static constexpr int k = q + kTile;
  static constexpr int v = k + kStages * kTile;
  static constexpr int p = v + kStages * kTile;
  static constexpr int bars = p + kTile;
  static constexpr int total = bars + 256;
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                AttnParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + AttnSmem::bars);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_empty = bars + 11; // [2]
  uint64_t* p_full = bars + 13;
  uint64_t* o_ready = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int qt = blockIdx.x, head = blockIdx.y, e = blockIdx.z;
  const int q0 = qt * kRows;
  if (q0 >= prm.q_tokens) return;
  const int n_vis = prm.n_vis[e];
  const int tiles_per_slot = (prm.kv_tokens + kKeys - 1) / kKeys;
  const int n_tiles = n_vis * tiles_per_slot;
  const uint32_t warp = warp_id();

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_kv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(o_ready, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem + 256;

  if (warp == 0) {
    if (lane_id() == 0) {
      const int qrow = e * prm.q_tokens + q0;
      mbar_arrive_expect_tx(q_full, kTile);
      tma_load_3d(smem + AttnSmem::q, &map_q, q_full, 0, head, qrow);
      tma_load_3d(smem + AttnSmem::q + kHalf, &map_q, q_full, 64, head, qrow);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const int slot = prm.vis_slot[e][j / tiles_per_slot];
        const int t0 = (j % tiles_per_slot) * kKeys;
        const int kmat = prm.mat_base + slot * prm.mat_stride;
        const int vmat = kmat + prm.v_offset;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[st], kTile);
        tma_load_4d(smem + AttnSmem::k + st * kTile, &map_kv, &k_full[st], 0, head, t0, kmat);
        tma_load_4d(smem + AttnSmem::k + st * kTile + kHalf, &map_kv, &k_full[st], 64, head, t0, kmat);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[st], kTile);
        tma_load_4d(smem + AttnSmem::v + st * kTile, &map_kv, &v_full[st], 0, head, t0, vmat);
        tma_load_4d(smem + AttnSmem::v + st * kTile + kHalf, &map_kv, &v_full[st], 64, head, t0, vmat);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_qk = idesc_bf16(kRows, kKeys);
    constexpr uint32_t idesc_pv = idesc_bf16(kRows, kHd, 0, 1);  // B (=V) MN-major
    const uint32_t sq = smem_u32(smem + AttnSmem::q);
    const uint32_t sp = smem_u32(smem + AttnSmem::p);
    auto issue_qk = [&](int j) {
      const int st = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      mbar_wait(&s_empty[st], ph ^ 1);
      mbar_wait(&k_full[st], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sk = smem_u32(smem + AttnSmem::k + st * kTile);
#pragma unroll
        for (int k = 0; k < kHd / 16; ++k) {
          const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
          mma_bf16_ss(tmem + st * 128, desc_sw128(sq + off, 16, 1024), desc_sw128(sk + off, 16, 1024),
                      idesc_qk, k != 0);
        }
        mma_commit(&k_empty[st]);
        mma_commit(&s_full[st]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    if (n_tiles > 0) issue_qk(0);
    for (int j = 0; j < n_tiles; ++j) {
      if (j + 1 < n_tiles) issue_qk(j + 1);
      const int st = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      mbar_wait(p_full, j & 1);
      mbar_wait(&v_full[st], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sv = smem_u32(smem + AttnSmem::v + st * kTile);
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          // A = P [128 rows x 128 keys] K-major; B = V [128 keys x 128 dims] MN-major
          const uint32_t aoff = (k >> 2) * kHalf + (k & 3) * 32;
          const uint64_t ad = desc_sw128(sp + aoff, 16, 1024);
          const uint64_t bd = desc_sw128(sv + k * 2048, kHalf, 1024);
          mma_bf16_ss(t_o, ad, bd, idesc_pv, (j | k) != 0);
        }
        mma_commit(&v_empty[st]);
        mma_commit(o_ready);
      }
      __syncwarp();
    }
  } else {
    // softmax / correction / epilogue: 128 threads, thread <-> query row
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane_id();
    const uint32_t lane_base = (quad * 32) << 16;
    const float scale_log2 = prm.scale * 1.4426950408889634f;
    float m_used = -INFINITY, l_sum = 0.0f;
    uint8_t* sp = smem + AttnSmem::p;
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      const int t0 = (j % tiles_per_slot) * kKeys;
      const int valid = min(kKeys, prm.kv_tokens - t0);
      mbar_wait(&s_full[st], ph);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + st * 128 + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      mbar_arrive(&s_empty[st]);
      float mt = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        s[i] = (i < valid) ? s[i] * scale_log2 : -INFINITY;
        mt = fmaxf(mt, s[i]);
      }
      // lazy rescale: move the reference max only when it grows by > 2^8
      float alpha = 1.0f;
      const bool bump = (j == 0) || (mt > m_used + kRescaleThresh);
      if (bump) {
        const float m_new = fmaxf(m_used, mt);
        alpha = (j == 0) ? 0.0f : exp2f(m_used - m_new);
        m_used = m_new;
      }
      float tsum = 0.0f;
      uint32_t pk[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float p0 = exp2f(s[2 * i] - m_used);
        const float p1 = exp2f(s[2 * i + 1] - m_used);
        tsum += p0 + p1;
        pk[i] = pack_bf16(p0, p1);
      }
      l_sum = l_sum * alpha + tsum;
      // PV(j-1) must be complete before O is rescaled or P is overwritten
      if (j > 0) {
        mbar_wait(o_ready, (j - 1) & 1);
        tc_fence_after();
        const bool any_bump = __any_sync(0xffffffffu, bump && alpha != 1.0f);
        if (any_bump) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(t_o + lane_base + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(t_o + lane_base + c * 32, r);
          }
          tmem_st_wait();
        }
      }
      // P row -> smem, K-major SW128: half h holds keys [64h, 64h+64),
      // 16-byte chunk c of row r lands at chunk (c ^ (r & 7)).
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int half = c >> 3, ch = c & 7;
        uint8_t* dst = sp + half * kHalf + row * 128 + ((ch ^ (row & 7)) << 4);
        *reinterpret_cast<uint4*>(dst) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      fence_async_shared();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 out
    if (n_tiles > 0) {
      mbar_wait(o_ready, (n_tiles - 1) & 1);
      tc_fence_after();
    }
    const int qrow = q0 + (int)row;
    const bool live = qrow < prm.q_tokens;
    const float inv = (l_sum > 0.0f) ? 1.0f / l_sum : 0.0f;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(prm.out) +
                         ((size_t)(e * prm.q_tokens + qrow) * prm.heads + head) * kHd;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(t_o + lane_base + c * 32, r);
      tmem_ld_wait();
      if (live) {
        uint4* dst = reinterpret_cast<uint4*>(out + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 v;
          v.x = pack_bf16(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
          v.y = pack_bf16(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
          v.z = pack_bf16(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
          v.w = pack_bf16(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
          dst[q] = v;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims,
           const cuuint64_t* strides, const cuuint32_t* box) {
  auto fn = encoder();
  if (!fn) return bc_fail(BC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return bc_fail(BC_ERR_CUDA, "attention tensor map encode failed (%d)", (int)r);
  return BC_OK;
}

}  // namespace

int attention_run(const AttnArgs& a, cudaStream_t st) {
  if (a.head_dim != kHd) return bc_fail(BC_ERR_CONTRACT, "attention: head_dim must be 128");
  if (a.n_entries < 1 || a.n_entries > BC_MAX_ENTRIES)
    return bc_fail(BC_ERR_CONTRACT, "attention: bad entry count %d", a.n_entries);
  const uint64_t row_bytes = (uint64_t)a.heads * kHd * 2;
  CUtensorMap mq, mkv;
  {
    cuuint64_t dims[3] = {kHd, (cuuint64_t)a.heads, (cuuint64_t)a.n_entries * a.q_tokens};
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
  for (int e = 0; e < a.n_entries; ++e) {
    if (a.n_vis[e] < 0 || a.n_vis[e] > BC_MAX_VIS)
      return bc_fail(BC_ERR_CONTRACT, "attention: bad visible count");
    p.n_vis[e] = a.n_vis[e];
    for (int v = 0; v < a.n_vis[e]; ++v) p.vis_slot[e][v] = a.vis_slot[e][v];
  }
  static bool attr = false;
  if (!attr) {
    BC_CUDA(cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 AttnSmem::total + 1024));
    attr = true;
  }
  dim3 grid((a.q_tokens + kRows - 1) / kRows, a.heads, a.n_entries);
  attn_kernel<<<grid, kThreads, AttnSmem::total + 1024, st>>>(mq, mkv, p);
  BC_LAUNCHED();
  return BC_OK;
}

}  // namespace bc

// Self-attention over KV-arena slots.  k_arena points at layer 0 of an
// arena laid out [L][n_slots][2][T][heads*128]; slot_stride_elems is the
// distance between consecutive (K or V) matrices in elements (T*heads*128).
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
  return bc::attention_run(a, (cudaStream_t)stream);
}
