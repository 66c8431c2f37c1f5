// Shared host-side helpers: status codes, last-error text, CUDA checks.
#pragma once
#include <cstdarg>
#include <cstdio>

#include "../../include/bcb200.h"

// Records a formatted message for bc_last_error() and returns `code`.
int bc_fail(int code, const char* fmt, ...);
// Counts every kernel this library launches (bc_launch_count()).
void bc_count_launch();

#ifdef __CUDACC__
#include <cuda_runtime.h>
#define BC_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return bc_fail(BC_ERR_CUDA, "%s:%d %s -> %s", __FILE__, __LINE__, #call,     \
                     cudaGetErrorString(_e));                                      \
  } while (0)
#define BC_LAUNCHED()                                                              \
  do {                                                                             \
    bc_count_launch();                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess)                                                         \
      return bc_fail(BC_ERR_CUDA, "%s:%d launch -> %s", __FILE__, __LINE__,        \
                     cudaGetErrorString(_e));                                      \
  } while (0)
#endif

#ifdef __CUDACC__
#include <mutex>
// Propagate a non-zero status code.
#define BC_RC(x)               \
  do {                         \
    const int _rc = (x);       \
    if (_rc) return _rc;       \
  } while (0)
// One-time per-device setup (cudaFuncSetAttribute applies per device; the
// first launch on each device must set it), safe under concurrent callers.
struct PerDeviceOnce {
  static constexpr int kMaxDevices = 64;
  std::once_flag flag[kMaxDevices];
};
template <class F>
int per_device_once(PerDeviceOnce& once, F&& fn) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= PerDeviceOnce::kMaxDevices) return fn();
  int rc = 0;
  std::call_once(once.flag[dev], [&] { rc = fn(); });
  return rc;
}
// SM count of the current device (queried per call: cheap, no shared state).
inline int current_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}
#endif
