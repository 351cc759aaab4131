// Micro-benchmark of the FP16X3 halo kernel's MMA issue pattern: per stage
// (one tap of one 32-channel chunk) and per sub-tile u, two K steps of
// { a0 . [b0 | b1] (N = 2 BN), a1 . b0 (N = BN) }, a commit per stage.
// SWIZZLE_64B operands, sliding A descriptor, one CTA per SM, one elected
// thread issuing.  Prints cycles per stage against the model
// 2 x SUB x (max(BN, 32 + BN/2) + max(BN/2, 32 + BN/4)).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/umma_pattern \
//        scripts/umma_pattern.cu && scripts/umma_pattern
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2509_20198_b200/csrc/tc_ptx.cuh"

using namespace ts::tcx;

constexpr int kStages = 2048;

// align: tap slides of whole 8-row swizzle atoms instead of the 3x3
// pattern; sts: warps 1..10 store 16-byte pieces to a separate region while
// the MMAs run (the producers' halo stores)
__global__ void __launch_bounds__(352, 1) pat_kernel(int bn, int sub, int commit_each, int align,
                                                     int sts, int ring, int spin, int every,
                                                     int plain, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* a = smem;                    // 2 planes x 640 rows x 64 B
  uint8_t* b = smem + 2 * 640 * 64;     // 2 planes x 128 rows x 64 B
  __shared__ uint64_t bar[2];
  __shared__ uint64_t rbar[32];
  __shared__ uint64_t pbar;  // completed once at init (phase 0 done)
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  uint8_t* scratch = smem + (2 * 640 + 2 * 128) * 64;  // 400 rows x 128 B
  for (int i = threadIdx.x; i < (2 * 640 + 2 * 128) * 64 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    for (int i = 0; i < 32; ++i) mbar_init(&rbar[i], 1);
    mbar_init(&pbar, 1);
    mbar_arrive(&pbar);
    fence_barrier_init();
    done = 0;
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint64_t da = sw64_desc(su32(a)), db = sw64_desc(su32(b));
    const uint32_t pa = (640 * 64) >> 4, pb = (uint32_t)(bn * 64) >> 4;
    const uint32_t idesc = make_idesc(0u, 2 * bn), idesc_b0 = make_idesc(0u, bn);
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int st = 0; st < kStages; ++st) {
        if (ring && st >= ring && st % every == 0) {
          uint64_t* rb = plain ? &pbar : &rbar[(st - ring) % ring];
          const uint32_t par = plain ? 0u : (uint32_t)(((st - ring) / ring) & 1);
          if (spin) {  // non-suspending polls
            uint32_t done = 0;
            while (!done)
              asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                           : "=r"(done) : "r"(su32(rb)), "r"(par) : "memory");
          } else {
            mbar_wait(rb, par);
          }
        }
        const uint64_t a0 = da + (uint64_t)((align ? (st % 9) * 8 : (st % 9) / 3 * 70 + (st % 3))) * 4;  // tap slide
#pragma unroll 1
        for (int k = 0; k < 2; ++k)
          for (int u = 0; u < sub; ++u) {
            const uint64_t ak = a0 + (uint64_t)(u * (128 * 64 >> 4) + 2 * k);
            const uint32_t du = tmem + u * 2 * bn;
            umma<false>(du, ak, db + 2 * k, idesc, (st | k) ? 1u : 0u);
            umma<false>(du + bn, ak + pa, db + 2 * k, idesc_b0, 1u);
          }
        if (ring) umma_commit(&rbar[st % ring]);
        else if (commit_each) umma_commit(&bar[st & 1]);
      }
      umma_commit(&bar[0]);
    }
    __syncwarp();
    // wait for the final commit (phase count depends on commits per barrier)
    unsigned long long t1;
    {
      const int n0 = (commit_each && !ring) ? (kStages + 1) / 2 + 1 : 1;
      mbar_wait(&bar[0], (uint32_t)((n0 - 1) & 1));
      t1 = clock64();
    }
    (void)pb;
    if (threadIdx.x == 0) {
      out[blockIdx.x] = t1 - t0;
      done = 1;
    }
  } else if (sts) {
    const int t = threadIdx.x - 32;
    uint4 v = make_uint4(t, t + 1, t + 2, t + 3);
    while (!done) {
#pragma unroll 4
      for (int r = t; r < 400 * 8; r += 320) {
        *reinterpret_cast<uint4*>(scratch + r * 16) = v;
        v.x += 1;
      }
    }
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
  const int smem = (2 * 640 + 2 * 128) * 64 + 400 * 128 + 1024;
  cudaFuncSetAttribute(pat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<unsigned long long> h(sms);
  printf("BN SUB commit align sts : cycles/stage (median SM)   model\n");
  const int cfg[][2] = {{32, 4}, {64, 2}, {96, 1}, {128, 1}};
  const int var[][4] = {{0, 0, 1, 0}, {8, 0, 1, 0}, {8, 0, 2, 0}, {8, 0, 4, 0}, {8, 0, 9, 0},
                        {8, 0, 1, 1}, {8, 1, 1, 1}};
  for (auto& vv : var)
  for (auto& c : cfg)
    for (int v = 0; v < 1; ++v) {
      const int ring = vv[0], spin = vv[1], every = vv[2], plain = vv[3];
      if (c[0] != 64) continue;
      const int bn = c[0], sub = c[1], ce = 1, al = v & 1, sts = v >> 1;
      for (int rep = 0; rep < 2; ++rep) {
        pat_kernel<<<sms, 352, smem>>>(bn, sub, ce, al, sts, ring, spin, every, plain, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      }
      cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.end());
      const double model = 2.0 * sub * (std::max(bn, 32 + bn / 2) + std::max(bn / 2, 32 + bn / 4));
      printf("ring %2d spin %d every %d plain %d %3d %d %d %d %d : %8.1f   %6.1f\n", ring, spin,
             every, plain, bn, sub, ce, al, sts,
             (double)h[sms / 2] / kStages, model);
    }
  return 0;
}
