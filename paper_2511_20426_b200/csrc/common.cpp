// Last-error bookkeeping for the C-ABI (thread-local, like errno).
#include <cstdarg>
#include <cstdio>

#include "bc_common.h"

#include <atomic>

namespace {
thread_local char g_last_error[512] = "";
std::atomic<long long> g_launches{0};
}

void bc_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" long long bc_launch_count(void) { return g_launches.load(); }

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
