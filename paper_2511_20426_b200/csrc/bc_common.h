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
