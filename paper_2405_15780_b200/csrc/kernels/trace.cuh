// trace.cuh — optional per-event clock64 tracing of one CTA (tuning aid).
// Compiled in only with -DUA_TRACE=1 (a variant build, see build.py); the
// shipped library contains none of it.  Each (role, tile, event) of the CTA
// with blockIdx == (UA_TRACE_CTA, 0, 0) stores clock64() into its own slot of
// a device buffer (plain stores, no atomics, so the timeline is not
// perturbed); the host dumps the non-zero slots to $UA_TRACE_FILE.
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
#include <vector>
namespace ua {
constexpr int kTraceRoles = 8, kTraceTiles = 4096, kTraceEvents = 32;
constexpr int kTraceSlots = kTraceRoles * kTraceTiles * kTraceEvents;
__device__ unsigned long long g_trace[kTraceSlots];
__device__ __forceinline__ void trace_ev(int role, int tile, int ev) {
  if (blockIdx.x != UA_TRACE_CTA || blockIdx.y != 0 || blockIdx.z != 0 || tile >= kTraceTiles) return;
  g_trace[(role * kTraceTiles + tile) * kTraceEvents + ev] = clock64();
}
inline void trace_reset() {
  static std::vector<unsigned long long> z(kTraceSlots, 0ull);
  cudaMemcpyToSymbol(g_trace, z.data(), sizeof(unsigned long long) * kTraceSlots);
}
inline void trace_dump(const char* tag) {
  cudaDeviceSynchronize();
  static std::vector<unsigned long long> buf(kTraceSlots);
  cudaMemcpyFromSymbol(buf.data(), g_trace, sizeof(unsigned long long) * kTraceSlots);
  const char* path = std::getenv("UA_TRACE_FILE");
  FILE* f = std::fopen(path ? path : "ua_trace.txt", "a");
  if (!f) return;
  for (int i = 0; i < kTraceSlots; ++i)
    if (buf[i])
      std::fprintf(f, "%s %llu %d %d %d\n", tag, buf[i], i / (kTraceTiles * kTraceEvents),
                   (i / kTraceEvents) % kTraceTiles, i % kTraceEvents);
  std::fclose(f);
}
}  // namespace ua
#define UA_TEV(role, tile, ev) ::ua::trace_ev(role, tile, ev)
#else
#define UA_TEV(role, tile, ev) ((void)0)
#endif
