// Probe: tcgen05.mma throughput by operand source and shape (cycles per
// instruction vs the tensor-pipe floor of 128*N/256 cycles for M=128 per
// SM), and whether concurrent st.shared stores / bulk copies slow it.
// One CTA (or CTA pair) per SM; warp 0 (the leader's) issues `groups` x 8
// MMAs back to back; optional store warps (4-7) hammer a 32 KB region with
// st.shared.v4; optional warp 2 streams 32 KB bulk copies global->smem.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/smem_bw_probe scripts/smem_bw_probe.cu
// Round-2 result: profiles/r2_mma_operand_probe.txt
#include <cstdio>
#include "../paper_2511_20426_b200/csrc/sm100.cuh"
using namespace bc;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// mode bits: 1 = A from TMEM (TS), 2 = store warps, 4 = bulk-copy warp, 8 = A and B at the same smem tile
template <int N, int CG, int mode>
__global__ void __launch_bounds__(256, 1) k(long long* out, const uint8_t* gsrc, int groups) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar, cbar;
  __shared__ volatile int done;
  const uint32_t warp = threadIdx.x >> 5;
  const bool leader = CG == 1 || cta_rank() == 0;
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<512>(&tslot);
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&cbar, 1);
    done = 0;
    fence_barrier_init();
  }
  if (mode & 256) {  // fill the operand tiles with small finite bf16 values
    for (int i = threadIdx.x; i < 196 * 1024 / 4; i += blockDim.x) {
      const uint32_t h = (uint32_t)i * 2654435761u;
      reinterpret_cast<uint32_t*>(smem)[i] = (0x3c00u + ((h >> 8) & 0xff)) | ((0x3c00u + ((h >> 20) & 0xff)) << 16);
    }
  } else if (mode & 512) {
    for (int i = threadIdx.x; i < 196 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  }
  fence_async_shared();
  tc_fence_before();
  if (CG == 2) cl_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t base = smem_u32(smem);
  if (warp == 0) {
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16(128 * CG, N);
      const uint32_t b0 = (mode & 8) ? base : base + 32768;
      uint64_t ad[8], bd[8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        ad[kk] = desc_sw128(base + off, 16, 1024);
        bd[kk] = desc_sw128(b0 + off, 16, 1024);
      }
      long long t0 = clock64(), t_issue = 0;
      for (int g = 0; g < groups; ++g) {
        const long long ts = clock64();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t d = tmem + (N <= 128 ? (g & 1) * 128 : 0);
            const uint32_t acc = kk != 0;
            if (CG == 1) {
              if (mode & 1) mma_bf16_ts(d, tmem + 256 + kk * 8, bd[kk], idesc, acc);
              else mma_bf16_ss(d, ad[kk], bd[kk], idesc, acc);
            } else if (mode & 1) {
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                           "r"(tmem + 256 + kk * 8), "l"(bd[kk]), "r"(idesc), "r"(acc) : "memory");
            } else {
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                           "l"(ad[kk]), "l"(bd[kk]), "r"(idesc), "r"(acc) : "memory");
            }
          }
        }
        __syncwarp();
        t_issue += clock64() - ts;
      }
      if (elect_one()) {
        if (CG == 2)
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                           smem_u32(&bar)), "h"((uint16_t)0x3) : "memory");
        else
          mma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, 0);
      long long t1 = clock64();
      if (lane_id() == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[3] = t_issue; }
    } else {
      mbar_wait(&bar, 0);
    }
    if (lane_id() == 0) done = 1;
  } else if (warp == 2 && (mode & 4)) {
    long long bytes = 0;
    uint32_t ph = 0;
    while (!done) {
      if (elect_one()) {
        mbar_arrive_expect_tx(&cbar, 32768);
        bulk_g2s(base + 131072 + (ph & 1) * 32768, gsrc + ((size_t)(blockIdx.x * 7 + ph) % 512) * 32768, 32768, &cbar);
      }
      __syncwarp();
      mbar_wait(&cbar, ph & 1);
      ++ph;
      bytes += 32768;
    }
    if (lane_id() == 0 && blockIdx.x == 0) out[2] = bytes;
  } else if (warp >= 4 && (mode & 2)) {
    const uint32_t t = threadIdx.x - 128;
    long long n = 0;
    while (!done) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const uint32_t a = base + 98304 + (q >> 3) * 16384 + t * 128 + (((q & 7) ^ (t & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(q), "r"(t), "r"(q), "r"(t) : "memory");
      }
      n += 16 * 16;
    }
    if (t == 0 && blockIdx.x == 0) out[1] = n * 128;
  }
  tc_fence_before();
  if (CG == 2) cl_sync(); else __syncthreads();
  if (warp == 0) {
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      tmem_dealloc<512>(tmem);
  }
}

template <int N, int CG, int mode>
void run1(long long* out, const uint8_t* src) {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k<N, CG, mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  {
    const int groups = 512;
    long long h[4] = {0, 0, 0, 0};
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(out, 0, 32);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CG;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k<N, CG, mode>, out, src, groups);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    const double floor_cyc = 128.0 * N / 256.0;  // per instruction, per SM (M = 128 rows per SM)
    const double per = (double)h[0] / (groups * 8);
    printf("mode %3d CG=%d M=%3d N=%3d %s%s%s%s%s%s: %6.1f cyc/MMA (issue %6.1f, floor %5.1f) -> %5.1f%% of tensor peak; sts %5.1f B/clk, bulk %5.1f B/clk (%s)\n",
           mode, CG, 128 * CG, N, (mode & 1) ? "TS" : "SS", (mode & 8) ? "(A=B)" : "", (mode & 2) ? "+sts" : "",
           (mode & 4) ? "+bulk" : "", (mode & 16) ? "+Bshift3K" : "", (mode & 32) ? "+2acc" : "", per, (double)h[3] / (groups * 8), floor_cyc, 100.0 * floor_cyc / per, (double)h[1] / h[0], (double)h[2] / h[0],
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  long long* out;
  uint8_t* src;
  cudaMalloc(&out, 64);
  cudaMalloc(&src, 512 * 32768);
  cudaMemset(src, 0, 512 * 32768);
  run1<64, 1, 0>(out, src);
  run1<64, 1, 1>(out, src);
  run1<128, 1, 0>(out, src);
  run1<128, 1, 1>(out, src);
  run1<128, 1, 6>(out, src);
  run1<128, 1, 7>(out, src);
  run1<256, 1, 0>(out, src);
  run1<256, 1, 1>(out, src);
  run1<128, 2, 0>(out, src);
  run1<128, 2, 1>(out, src);
  run1<128, 2, 6>(out, src);
  run1<256, 2, 0>(out, src);
  run1<256, 2, 1>(out, src);
  return 0;
}
