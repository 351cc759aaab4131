// Library-level entry points of the ts_b200 C ABI.
#include "ts_common.cuh"

extern "C" const char* ts_version(void) { return "ts_b200 0.1 (sm_100a)"; }

extern "C" int ts_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
