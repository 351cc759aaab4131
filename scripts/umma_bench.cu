// Micro-benchmark: cycles per tcgen05.mma (kind::f16, M = 128, K = 16,
// bf16 operands from shared memory, fp32 accumulate in TMEM) for the
// SWIZZLE_64B and SWIZZLE_128B K-major layouts and several N, with the A
// descriptor fixed or sliding by one row per MMA (the halo kernels' tap
// walk).  One CTA per SM; one elected thread issues the MMAs back to back.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/umma_bench \
//        scripts/umma_bench.cu && scripts/umma_bench
#include <cstdio>
#include <cstdint>
#include <vector>

#include "../paper_2509_20198_b200/csrc/tc_ptx.cuh"

using namespace ts::tcx;

constexpr int kIters = 8192;

__global__ void __launch_bounds__(128, 1) umma_kernel(int sw, int n, int slide, int kind2,
                                                      unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  // A: 256 rows, B: 256 rows, each row 128 bytes (enough for both layouts)
  uint8_t* a = smem;
  uint8_t* b = smem + 256 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(a)[i] = 0x3F803F80u;
    reinterpret_cast<uint32_t*>(b)[i] = 0x3F803F80u;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint64_t da = sw == 128 ? sw128_desc(su32(a)) : sw64_desc(su32(a));
    const uint64_t db = sw == 128 ? sw128_desc(su32(b)) : sw64_desc(su32(b));
    const uint32_t idesc = make_idesc(1u, n);
    const int ksteps = sw == 128 ? 4 : 2;   // 32-byte K steps per row
    const uint32_t row16 = (uint32_t)sw >> 4;  // descriptor units per row
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < kIters; ++i) {
        const int k = i % ksteps;
        const uint64_t ao = (uint64_t)(2 * k) + (slide ? (uint64_t)((i / ksteps) % 64) * row16 : 0);
        const uint32_t d = kind2 ? tmem + (uint32_t)((i & 1) * 256) : tmem;
        umma<false>(d, da + ao, db + (uint64_t)(2 * k), idesc, i ? 1u : 0u);
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_out;
  cudaMalloc(&d_out, sms * sizeof(unsigned long long));
  const int smem = 2 * 256 * 128 + 1024;
  cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<unsigned long long> h(sms);
  printf("layout N slide : cycles/MMA (CTA 0, median over SMs)  ideal = N/2\n");
  for (int sw : {64, 128})
    for (int n : {32, 64, 128, 256})
      for (int slide : {0, 1}) {
        for (int rep = 0; rep < 2; ++rep) {
          umma_kernel<<<sms, 128, smem>>>(sw, n, slide, 0, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        }
        cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
        std::vector<unsigned long long> s(h);
        std::sort(s.begin(), s.end());
        printf("SW%-3d N=%-3d slide=%d : %.1f\n", sw, n, slide,
               (double)s[sms / 2] / kIters);
      }
  return 0;
}
