// Micro-benchmark: the FP16X3 halo kernel's MMA issue pattern on a CTA pair
// (tcgen05.mma.cta_group::2, M = 256: each SM its own 128 rows of A, the B
// columns split between the two CTAs' shared memory) against one CTA per SM
// (cta_group::1, scripts/umma_pattern.cu).  Per stage and sub-tile u, two K
// steps of { a0 . [b0 | b1] (N = 2 BN), a1 . b0 (N = BN) }, a commit per
// stage (multicast to both CTAs).  Prints cycles per stage, i.e. per
// SUB x 128 positions x BN channels PER SM in both modes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/umma_pair \
//        scripts/umma_pair.cu && scripts/umma_pair
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2509_20198_b200/csrc/tc_ptx.cuh"

using namespace ts::tcx;

constexpr int kStages = 2048;

// cluster_rank, cluster_sync_all, umma2, umma_commit2: tc_ptx.cuh

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(int bn, int sub, int ring, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* a = smem;                 // 2 planes x 640 rows x 64 B
  uint8_t* b = smem + 2 * 640 * 64;  // this CTA's half of B
  __shared__ uint64_t bar[2];
  __shared__ uint64_t rbar[8];  // ring: stage st waits for the commit of st - ring
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (2 * 640 + 2 * 128) * 64 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(&slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool leader = cluster_rank() == 0;
  if (threadIdx.x < 32 && leader) {
    const uint64_t da = sw64_desc(su32(a)), db = sw64_desc(su32(b));
    const uint32_t pa = (640 * 64) >> 4;
    const uint32_t idesc = make_idesc(0u, 2 * bn, 256), idesc_b0 = make_idesc(0u, bn, 256);
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int st = 0; st < kStages; ++st) {
        if (ring && st >= ring) mbar_wait(&rbar[(st - ring) % ring], (uint32_t)(((st - ring) / ring) & 1));
        const uint64_t a0 = da + (uint64_t)((st % 9) / 3 * 70 + (st % 3)) * 4;  // tap slide
#pragma unroll 1
        for (int k = 0; k < 2; ++k)
          for (int u = 0; u < sub; ++u) {
            const uint64_t ak = a0 + (uint64_t)(u * (128 * 64 >> 4) + 2 * k);
            const uint32_t du = tmem + u * 2 * bn;
            umma2(du, ak, db + 2 * k, idesc, (st | k) ? 1u : 0u);
            umma2(du + bn, ak + pa, db + 2 * k, idesc_b0, 1u);
          }
        if (ring) umma_commit2(&rbar[st % ring]);
        else umma_commit2(&bar[st & 1]);
      }
      umma_commit2(&bar[0]);
    }
    __syncwarp();
    const int n0 = ring ? 1 : (kStages + 1) / 2 + 1;
    mbar_wait(&bar[0], (uint32_t)((n0 - 1) & 1));
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x / 2] = t1 - t0;
  } else if (threadIdx.x < 32) {
    // the peer's barrier receives the same multicast arrivals
    const int n0 = ring ? 1 : (kStages + 1) / 2 + 1;
    mbar_wait(&bar[0], (uint32_t)((n0 - 1) & 1));
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int pairs = sms / 2;
  unsigned long long* d_out;
  cudaMalloc(&d_out, pairs * sizeof(unsigned long long));
  const int smem = (2 * 640 + 2 * 128) * 64 + 1024;
  cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<unsigned long long> h(pairs);
  printf("cta_group::2  BN SUB : cycles/stage (median pair; per SM: SUB x 128 rows x BN)\n");
  const int cfg[][2] = {{32, 4}, {64, 2}, {96, 1}, {128, 1}};
  for (int ring : {0, 4, 8})
  for (auto& c : cfg) {
    const int bn = c[0], sub = c[1];
    for (int rep = 0; rep < 2; ++rep) {
      pair_kernel<<<2 * pairs, 128, smem>>>(bn, sub, ring, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h.data(), d_out, pairs * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    printf("  ring %d  %3d %d : %8.1f\n", ring, bn, sub, (double)h[pairs / 2] / kStages);
  }
  return 0;
}
