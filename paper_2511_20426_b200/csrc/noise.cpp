// Counter-keyed Gaussian noise, bit-identical to the reference NoiseStream
// (blockcascade/core.py:161-186), which draws
//   np.random.Generator(np.random.Philox(key=seed, counter=[b,p,f,0]))
//     .standard_normal(D).
// numpy pinned here: 2.3.x (the reference's `numpy>=1.24` dependency,
// pkg/pyproject.toml:11).  The bit generator is Philox4x64-10 (Salmon et al.,
// SC'11) with numpy's buffering convention: the 256-bit counter is
// incremented BEFORE each 4-word block is produced and words are consumed in
// order.  The normal transform is numpy's own ziggurat, linked from
// numpy/random/lib/libnpyrandom.a, so no re-derived constants are involved.
//
// Host code: runs without the GIL (ctypes releases it), one std::thread per
// stream, so a Wan-sized block (3 frames x 99,840) costs one stream's time.
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include <algorithm>

#include "../../include/bcb200.h"
#include "bc_common.h"

extern "C" {
typedef struct bitgen {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
} bitgen_t;
// from libnpyrandom.a (numpy/random/src/distributions/distributions.c)
void random_standard_normal_fill(bitgen_t* state, intptr_t cnt, double* out);
}

namespace {

constexpr uint64_t kMul0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t kMul1 = 0xCA5A826395121157ULL;
constexpr uint64_t kWeyl0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kWeyl1 = 0xBB67AE8584CAA73BULL;

inline void philox_block(const uint64_t in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t x0 = in[0], x1 = in[1], x2 = in[2], x3 = in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += kWeyl0;
      k1 += kWeyl1;
    }
    const unsigned __int128 p0 = (unsigned __int128)kMul0 * x0;
    const unsigned __int128 p1 = (unsigned __int128)kMul1 * x2;
    const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    const uint64_t y0 = hi1 ^ x1 ^ k0;
    const uint64_t y2 = hi0 ^ x3 ^ k1;
    x0 = y0;
    x1 = lo1;
    x2 = y2;
    x3 = lo0;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

struct PhiloxStream {
  uint64_t ctr[4];
  uint64_t key[2];
  uint64_t words[4];
  int next = 4;  // consumed all buffered words -> refill on first use

  uint64_t u64() {
    if (next == 4) {
      // 256-bit increment with carry, then one Philox block
      for (int i = 0; i < 4; ++i)
        if (++ctr[i] != 0) break;
      philox_block(ctr, key, words);
      next = 0;
    }
    return words[next++];
  }
};

uint64_t s_u64(void* st) { return static_cast<PhiloxStream*>(st)->u64(); }
uint32_t s_u32(void* st) { return (uint32_t)static_cast<PhiloxStream*>(st)->u64(); }
double s_f64(void* st) {
  return (double)(static_cast<PhiloxStream*>(st)->u64() >> 11) * (1.0 / 9007199254740992.0);
}

void run_task(const bc_noise_task& t, int dtype, std::vector<double>& scratch) {
  PhiloxStream s;
  std::memcpy(s.ctr, t.counter, sizeof(s.ctr));
  std::memcpy(s.key, t.key, sizeof(s.key));
  bitgen_t bg{&s, s_u64, s_u32, s_f64, s_u64};
  if (dtype == 0) {
    random_standard_normal_fill(&bg, (intptr_t)t.n, static_cast<double*>(t.out));
    return;
  }
  float* dst = static_cast<float*>(t.out);
  constexpr int64_t kChunk = 8192;
  scratch.resize(kChunk);
  for (int64_t off = 0; off < t.n; off += kChunk) {
    const int64_t m = std::min(kChunk, t.n - off);
    random_standard_normal_fill(&bg, (intptr_t)m, scratch.data());
    for (int64_t i = 0; i < m; ++i) dst[off + i] = (float)scratch[i];
  }
}

}  // namespace

extern "C" int bc_philox4x64(const uint64_t key[2], const uint64_t counter[4], uint64_t out[4]) {
  philox_block(counter, key, out);
  return BC_OK;
}

extern "C" int bc_noise_run(const bc_noise_task* tasks, int n_tasks, int dtype, int n_threads) {
  if (n_tasks < 0 || (dtype != 0 && dtype != 1)) return bc_fail(BC_ERR_CONTRACT, "bc_noise_run: bad arguments");
  if (n_tasks == 0) return BC_OK;
  for (int i = 0; i < n_tasks; ++i)
    if (tasks[i].n < 0 || (tasks[i].n > 0 && tasks[i].out == nullptr))
      return bc_fail(BC_ERR_CONTRACT, "bc_noise_run: bad task");
  int workers = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  workers = std::max(1, std::min(workers, n_tasks));
  if (workers == 1) {
    std::vector<double> scratch;
    for (int i = 0; i < n_tasks; ++i) run_task(tasks[i], dtype, scratch);
    return BC_OK;
  }
  std::vector<std::thread> pool;
  pool.reserve(workers);
  for (int w = 0; w < workers; ++w) {
    pool.emplace_back([=]() {
      std::vector<double> scratch;
      for (int i = w; i < n_tasks; i += workers) run_task(tasks[i], dtype, scratch);
    });
  }
  for (auto& th : pool) th.join();
  return BC_OK;
}
