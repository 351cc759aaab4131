// Library-level entry points of the ts_b200 C ABI.
#include <atomic>

#include "ts_common.cuh"

namespace ts {
static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace ts

extern "C" uint64_t ts_launch_count(void) { return ts::g_launches.load(); }

extern "C" const char* ts_version(void) { return "ts_b200 0.1 (sm_100a)"; }

extern "C" int ts_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
