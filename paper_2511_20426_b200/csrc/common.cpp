// Last-error bookkeeping for the C-ABI (thread-local, like errno).
#include <cstdarg>
#include <cstdio>

#include "bc_common.h"

namespace {
thread_local char g_last_error[512] = "";
}

int bc_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

extern "C" const char* bc_last_error(void) { return g_last_error; }

extern "C" const char* bc_version(void) {
  return "bcb200 0.1 sm_100a (tcgen05/TMEM/TMA), noise=numpy-philox4x64+ziggurat";
}
