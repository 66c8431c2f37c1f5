// Probe: can a tcgen05 K-major SW128 / SW64 A operand start at an arbitrary
// ROW of a TMA-written swizzled tile (row shift = kw tap of an implicit-GEMM
// convolution), and is the descriptor's base-offset field needed for it?
// D = A[s .. s+127, 0:K] . B[0:64, 0:K]^T for shifts s = 0..9, compared with
// a host fp32 reference.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -I paper_2511_20426_b200/csrc scripts/shift_desc_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "sm100.cuh"

using namespace bc;

constexpr int ROWS = 144;  // A rows in smem (128 + shift room)

__device__ __forceinline__ uint64_t desc_sw(uint32_t addr, uint32_t sbo, uint32_t swz, uint32_t base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;  // LBO (unused for swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)swz << 61;  // 2 = 128B, 4 = 64B
  return d;
}

// KB = bytes per row (128 -> SW128, K = 64; 64 -> SW64, K = 32)
template <int KB>
__global__ void probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int shift,
                      int bo_mode, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;
  uint8_t* sb = sm + ROWS * KB;  // ROWS*KB is a multiple of 1024
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<64>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, ROWS * KB + 64 * KB);
    tma_load_2d(sa, &ma, &bar, 0, 0);
    tma_load_2d(sb, &mb, &bar, 0, 0);
    mbar_wait(&bar, 0);
    tc_fence_after();
    constexpr uint32_t swz = KB == 128 ? 2 : 4;
    constexpr uint32_t sbo = 8 * KB;
    const uint32_t a0 = smem_u32(sa) + shift * KB;
    const uint32_t b0 = smem_u32(sb);
    const uint32_t idesc = idesc_bf16(128, 64);
    for (int k = 0; k < KB / 32; ++k) {
      const uint32_t aa = a0 + k * 32;
      const uint32_t bo = bo_mode == 0 ? 0 : bo_mode == 1 ? ((aa >> 7) & 7) : ((aa >> 7) & 3);
      const uint64_t ad = desc_sw(aa, sbo, swz, bo);
      const uint64_t bd = desc_sw(b0 + k * 32, sbo, swz, 0);
      mma_bf16_ss(tbase, ad, bd, idesc, k != 0);
    }
    mma_commit(&mbar);
  }
  __syncwarp();
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t r[32];
  for (int c = 0; c < 64; c += 32) {
    tmem_ld32(tbase + ((warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(warp * 32 + (threadIdx.x & 31)) * 64 + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tbase);
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static void map2d(CUtensorMap* m, void* base, int inner, int outer, int box_outer, CUtensorMapSwizzle swz) {
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t str[1] = {(cuuint64_t)inner * 2};
  cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", (int)r);
}

template <int KB>
static void run() {
  const int K = KB / 2;
  std::vector<__nv_bfloat16> ha(ROWS * K), hb(64 * K);
  std::vector<float> fa(ROWS * K), fb(64 * K);
  srand(1);
  for (int i = 0; i < ROWS * K; ++i) {
    ha[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
    fa[i] = __bfloat162float(ha[i]);
  }
  for (int i = 0; i < 64 * K; ++i) {
    hb[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
    fb[i] = __bfloat162float(hb[i]);
  }
  void *da, *db;
  float* dout;
  cudaMalloc(&da, ha.size() * 2);
  cudaMalloc(&db, hb.size() * 2);
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap ma, mb;
  const auto swz = KB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  map2d(&ma, da, K, ROWS, ROWS, swz);
  map2d(&mb, db, K, 64, 64, swz);
  const int smem = 1024 + ROWS * KB + 64 * KB;
  cudaFuncSetAttribute(probe<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> out(128 * 64);
  for (int bo_mode = 0; bo_mode < 3; ++bo_mode) {
    for (int s = 0; s <= 9; ++s) {
      cudaMemset(dout, 0, 128 * 64 * 4);
      probe<KB><<<1, 128, smem>>>(ma, mb, s, bo_mode, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) {
        printf("KB=%d bo=%d s=%d: CUDA error %s\n", KB, bo_mode, s, cudaGetErrorString(e));
        return;
      }
      cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)fa[(m + s) * K + k] * fb[n * K + k];
          maxerr = fmax(maxerr, fabs(ref - out[m * 64 + n]));
        }
      printf("KB=%3d (%s) base_offset_mode=%d shift=%d rows: max abs err %.3g %s\n", KB, KB == 128 ? "SW128" : "SW64",
             bo_mode, s, maxerr, maxerr < 1e-3 ? "OK" : "WRONG");
    }
  }
}

int main() {
  run<128>();
  run<64>();
  return 0;
}
