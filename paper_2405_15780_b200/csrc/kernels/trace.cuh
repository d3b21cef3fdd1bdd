// trace.cuh — optional per-event clock64 tracing of one CTA (tuning aid).
// Compiled in only with -DUA_TRACE=1 (a variant build, see build.py); the
// shipped library contains none of it.  Records (clock64, role, tile, event)
// for the CTA with blockIdx.x == UA_TRACE_CTA into a device buffer that the
// host dumps to $UA_TRACE_FILE after the launch.
#pragma once
#include <cstdint>

#ifndef UA_TRACE
#define UA_TRACE 0
#endif
#ifndef UA_TRACE_CTA
#define UA_TRACE_CTA 100
#endif

#if UA_TRACE
#include <cstdio>
#include <cstdlib>
namespace ua {
constexpr int kTraceCap = 1 << 16;
__device__ unsigned long long g_trace[kTraceCap * 2];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace_ev(int role, int tile, int ev) {
  if (blockIdx.x != UA_TRACE_CTA || blockIdx.y != 0 || blockIdx.z != 0) return;
  unsigned int i = atomicAdd(&g_trace_n, 1u);
  if (i < kTraceCap) {
    g_trace[2 * i] = clock64();
    g_trace[2 * i + 1] = (unsigned long long)((role << 24) | (tile << 8) | ev);
  }
}
inline void trace_reset() {
  unsigned int z = 0;
  cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z));
}
inline void trace_dump(const char* tag) {
  cudaDeviceSynchronize();
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(n));
  if (n > kTraceCap) n = kTraceCap;
  static unsigned long long buf[kTraceCap * 2];
  cudaMemcpyFromSymbol(buf, g_trace, sizeof(unsigned long long) * 2 * n);
  const char* path = std::getenv("UA_TRACE_FILE");
  FILE* f = std::fopen(path ? path : "ua_trace.txt", "a");
  if (!f) return;
  for (unsigned int i = 0; i < n; ++i)
    std::fprintf(f, "%s %llu %llu %llu %llu\n", tag, buf[2 * i], buf[2 * i + 1] >> 24, (buf[2 * i + 1] >> 8) & 0xFFFF,
                 buf[2 * i + 1] & 0xFF);
  std::fclose(f);
}
}  // namespace ua
#define UA_TEV(role, tile, ev) ::ua::trace_ev(role, tile, ev)
#else
#define UA_TEV(role, tile, ev) ((void)0)
#endif
