// Numerics probe for tcgen05.mma kind::f16 (bf16 in, fp32 accumulate in
// TMEM): how large and how biased is the accumulation error, and which
// operand-split / accumulator layouts reach fp32 (CUDA-core FMA) accuracy?
//
// One CTA.  A: 128 rows x K, B: N = 64 rows x K (K-major, SWIZZLE_128B
// images of 64 bf16 per row).  A ~ |N(0,1)| (post-ReLU activations), B ~
// N(0, 1/K) (He-scaled weights).  Every variant is a list of MMAs
// (A image, B image, TMEM column block, accumulate flag); the host sums the
// column blocks in fp32 (RN) the way an epilogue would and compares with the
// fp64 dot product of the fp32 operands.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_numerics \
//        scripts/mma_numerics.cu && scripts/mma_numerics
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include <cuda_fp16.h>

#include "../paper_2509_20198_b200/csrc/tc_ptx.cuh"

using namespace ts::tcx;

constexpr int M = 128, N = 64;
constexpr int KB = 2;            // K blocks of 64 held in shared memory
constexpr int K = KB * 64;
constexpr int kAImg = M * 128;   // bytes per A image (one K block, one plane)
constexpr int kBImg = N * 128;
constexpr int kPlanes = 3;       // bf16 planes per operand

struct Op {
  int aimg, bimg, kstep, col, acc;  // kstep: 16-element step inside the 64-wide block
};

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const uint8_t* ga, const uint8_t* gb, const Op* ops, int nops, int ncolblk,
                 float* out, int f16) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* a = smem;                                  // kPlanes * KB A images
  uint8_t* b = smem + kPlanes * KB * kAImg;           // kPlanes * KB B images
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int abytes = kPlanes * KB * kAImg, bbytes = kPlanes * KB * kBImg;
  for (int i = threadIdx.x; i < abytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(a)[i] = reinterpret_cast<const uint4*>(ga)[i];
  for (int i = threadIdx.x; i < bbytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(b)[i] = reinterpret_cast<const uint4*>(gb)[i];
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
    const uint32_t idesc = make_idesc(f16 ? 0u : 1u, N);
    if (elect_one()) {
      for (int i = 0; i < nops; ++i) {
        const Op o = ops[i];
        const uint64_t da = sw128_desc(su32(a + o.aimg * kAImg)) + (uint64_t)(2 * o.kstep);
        const uint64_t db = sw128_desc(su32(b + o.bimg * kBImg)) + (uint64_t)(2 * o.kstep);
        umma<false>(tmem + (uint32_t)(o.col * N), da, db, idesc, (uint32_t)o.acc);
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row = warp * 32 + lane;
  for (int c = 0; c < ncolblk * N; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
    for (int j = 0; j < 16; ++j) out[(size_t)row * 512 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static uint16_t bf16_rn(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float bf2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t f16_rn(float x) {
  __half h = __float2half_rn(x);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static float f162f(uint16_t u) {
  __half h;
  memcpy(&h, &u, 2);
  return __half2float(h);
}
// element (r, k) of a SW128 K-major image with 64 bf16 per row
static size_t sw128_off(int r, int k) {
  const int chunk = (k * 2) / 16, inner = (k * 2) % 16;
  return (size_t)r * 128 + (size_t)((chunk ^ (r & 7)) * 16 + inner);
}

// fmt 0: bf16 planes p_i = rn(residual) (unscaled); fmt 1: fp16 planes,
// plane i scaled by 2^(11 i) (so every plane is in the normal range)
static void split(float x, int fmt, uint16_t* p) {
  float r = x;
  for (int i = 0; i < kPlanes; ++i) {
    if (fmt == 0) {
      p[i] = bf16_rn(r);
      r = r - bf2f(p[i]);
    } else {
      p[i] = f16_rn(r);
      r = (r - f162f(p[i])) * 2048.f;
    }
  }
}

struct Var {
  const char* name;
  int fmt;
  std::vector<std::pair<int, int>> prods;
  int sep;    // 1: products grouped by class i+j into their own accumulators
  int chunk;  // K steps per main accumulator block (0 = one block)
};

int main() {
  uint8_t *da, *db;
  Op* dops;
  float* dout;
  cudaMalloc(&da, (size_t)kPlanes * KB * kAImg);
  cudaMalloc(&db, (size_t)kPlanes * KB * kBImg);
  cudaMalloc(&dops, 65536 * sizeof(Op));
  cudaMalloc(&dout, (size_t)M * 512 * 4);
  const int smem = kPlanes * KB * (kAImg + kBImg) + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const std::vector<std::pair<int, int>> P1 = {{0, 0}};
  const std::vector<std::pair<int, int>> P3 = {{0, 0}, {0, 1}, {1, 0}};
  const std::vector<std::pair<int, int>> P4 = {{0, 0}, {0, 1}, {1, 0}, {1, 1}};
  const std::vector<std::pair<int, int>> P6 = {{0, 0}, {0, 1}, {1, 0}, {1, 1}, {0, 2}, {2, 0}};
  const std::vector<Var> vars = {
      {"bf16 1 product", 0, P1, 0, 0},
      {"bf16 3 products, one acc (r01 default)", 0, P3, 0, 0},
      {"bf16 3 products, corr sep", 0, P3, 1, 0},
      {"bf16 6 products, corr sep", 0, P6, 1, 0},
      {"bf16 6 products, corr sep, main 4 blocks", 0, P6, 1, -4},
      {"fp16 1 product", 1, P1, 0, 0},
      {"fp16 3 scaled, corr sep", 1, P3, 1, 0},
      {"fp16 3 scaled, corr sep, main 2 blocks", 1, P3, 1, -2},
      {"fp16 3 scaled, corr sep, main 4 blocks", 1, P3, 1, -4},
      {"fp16 3 scaled, corr sep, main chunks of 8", 1, P3, 1, 8},
      {"fp16 3 scaled, corr sep, main chunks of 4", 1, P3, 1, 4},
      {"fp16 4 scaled, corr sep", 1, P4, 1, 0},
      {"fp16 4 scaled, corr sep, main 4 blocks", 1, P4, 1, -4},
  };
  for (int R : {1, 5, 22}) {
    for (int dist = 0; dist < 2; ++dist) {
      std::mt19937_64 rng(7 + R);
      std::normal_distribution<float> nd(0.f, 1.f);
      std::vector<float> A((size_t)M * K), B((size_t)N * K);
      // dist 0: |N(0,1)| activations; dist 1: 0.05 |N(0,1)| with 5% spikes x40
      for (auto& x : A) {
        x = std::fabs(nd(rng));
        if (dist == 1) x *= (rng() % 20 == 0) ? 2.f : 0.05f;
      }
      for (auto& x : B) x = nd(rng) / std::sqrt((float)(K * R));
      std::vector<double> ref((size_t)M * N), mag((size_t)M * N);
      std::vector<float> fma32((size_t)M * N);
      for (int r = 0; r < M; ++r)
        for (int c = 0; c < N; ++c) {
          double s = 0, m = 0;
          float f = 0.f;
          for (int rep = 0; rep < R; ++rep)
            for (int k = 0; k < K; ++k) {
              const double p = (double)A[(size_t)r * K + k] * B[(size_t)c * K + k];
              s += p;
              m += std::fabs(p);
              f = std::fmaf(A[(size_t)r * K + k], B[(size_t)c * K + k], f);
            }
          ref[(size_t)r * N + c] = s;
          mag[(size_t)r * N + c] = m;
          fma32[(size_t)r * N + c] = f;
        }
      auto report = [&](const char* name, const std::vector<float>& got) {
        double se = 0, sa = 0, mx = 0, bias = 0;
        for (size_t i = 0; i < got.size(); ++i) {
          const double e = (double)got[i] - ref[i];
          const double rel = e / mag[i];
          se += rel;
          sa += rel * rel;
          mx = std::max(mx, std::fabs(rel));
          bias += (ref[i] >= 0 ? rel : -rel);
        }
        const double n = (double)got.size();
        printf("  %-44s err/sum|ab|: outward %+.2e rms %.2e max %.2e\n", name, bias / n,
               std::sqrt(sa / n), mx);
      };
      printf("K = %d, activations %s\n", K * R, dist ? "0.05|N| + 5%% spikes" : "|N(0,1)|");
      report("fp32 CUDA-core FMA chain (target)", fma32);
      for (const Var& v : vars) {
        std::vector<uint8_t> ha((size_t)kPlanes * KB * kAImg), hb((size_t)kPlanes * KB * kBImg);
        for (int r = 0; r < M; ++r)
          for (int k = 0; k < K; ++k) {
            uint16_t p[kPlanes];
            split(A[(size_t)r * K + k], v.fmt, p);
            for (int i = 0; i < kPlanes; ++i)
              memcpy(&ha[(size_t)(i * KB + k / 64) * kAImg + sw128_off(r, k % 64)], &p[i], 2);
          }
        for (int r = 0; r < N; ++r)
          for (int k = 0; k < K; ++k) {
            uint16_t p[kPlanes];
            split(B[(size_t)r * K + k], v.fmt, p);
            for (int i = 0; i < kPlanes; ++i)
              memcpy(&hb[(size_t)(i * KB + k / 64) * kBImg + sw128_off(r, k % 64)], &p[i], 2);
          }
        cudaMemcpy(da, ha.data(), ha.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(db, hb.data(), hb.size(), cudaMemcpyHostToDevice);
        const int ksteps = R * K / 16;
        // main blocks: chunk < 0 => -chunk interleaved blocks; chunk > 0 =>
        // consecutive runs of `chunk` K steps cycling over 2 blocks (the
        // epilogue would drain one while the other fills)
        const int nmain = v.chunk < 0 ? -v.chunk : v.chunk > 0 ? 2 : 1;
        std::vector<Op> ops;
        std::vector<int> started(8, 0);
        std::vector<int> blk_class(8, 0);
        int maxclass = 0;
        for (const auto& pr : v.prods) maxclass = std::max(maxclass, pr.first + pr.second);
        // drained: host accumulates finished chunk sums (emulating the epilogue)
        for (int s = 0; s < ksteps; ++s) {
          const int kb = (s / 4) % KB, ks = s % 4;
          for (const auto& pr : v.prods) {
            const int cls = pr.first + pr.second;
            int blk;
            if (cls == 0 || !v.sep) {
              blk = v.chunk < 0 ? s % nmain : v.chunk > 0 ? (s / v.chunk) % 2 : 0;
            } else {
              blk = nmain + cls - 1;
            }
            blk_class[blk] = v.sep ? cls : 0;
            Op o{pr.first * KB + kb, pr.second * KB + kb, ks, blk, started[blk]};
            started[blk] = 1;
            ops.push_back(o);
          }
          if (v.chunk > 0 && (s + 1) % v.chunk == 0) {
            // next chunk of the same block restarts its accumulator: mark a
            // drain point (encoded as an op with aimg = -1)
            ops.push_back(Op{-1, 0, 0, (s / v.chunk) % 2, 0});
            started[(s / v.chunk) % 2] = 0;
          }
        }
        const int ncol = v.sep ? nmain + maxclass : nmain;
        // run segment by segment (drain points split the op list)
        std::vector<float> chunk_acc((size_t)M * N, 0.f);
        std::vector<float> out((size_t)M * 512);
        size_t i0 = 0;
        bool ok = true;
        auto run = [&](size_t a, size_t b) {
          if (b == a) return;
          cudaMemcpy(dops, ops.data() + a, (b - a) * sizeof(Op), cudaMemcpyHostToDevice);
          probe_kernel<<<1, 128, smem>>>(da, db, dops, (int)(b - a), ncol, dout, v.fmt);
          if (cudaDeviceSynchronize() != cudaSuccess) ok = false;
          cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
        };
        std::vector<float> got((size_t)M * N, 0.f);
        if (v.chunk > 0) {
          // emulate: each chunk is its own fresh accumulation; the epilogue
          // adds the chunk result into an fp32 register total (RN)
          std::vector<Op> seg;
          std::vector<float> tot((size_t)M * N, 0.f);
          std::vector<Op> corr;
          for (const Op& o : ops) {
            if (o.aimg < 0) {
              cudaMemcpy(dops, seg.data(), seg.size() * sizeof(Op), cudaMemcpyHostToDevice);
              probe_kernel<<<1, 128, smem>>>(da, db, dops, (int)seg.size(), ncol, dout, v.fmt);
              cudaDeviceSynchronize();
              cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
              for (int r = 0; r < M; ++r)
                for (int c = 0; c < N; ++c) tot[(size_t)r * N + c] += out[(size_t)r * 512 + o.col * N + c];
              seg.clear();
              continue;
            }
            if (o.col >= nmain) corr.push_back(o);
            else {
              Op q = o;
              q.acc = seg.empty() ? 0 : q.acc;
              seg.push_back(q);
            }
          }
          // fix accumulate flags inside chunks: every op after the first accumulates
          // (seg handling above sets acc=0 only on the first op of a chunk)
          (void)i0;
          // corrections in one run
          for (size_t j = 0; j < corr.size(); ++j) corr[j].acc = j < (size_t)maxclass ? 0 : 1;
          std::vector<int> st(8, 0);
          for (auto& o : corr) { o.acc = st[o.col]; st[o.col] = 1; }
          run(0, 0);
          cudaMemcpy(dops, corr.data(), corr.size() * sizeof(Op), cudaMemcpyHostToDevice);
          probe_kernel<<<1, 128, smem>>>(da, db, dops, (int)corr.size(), ncol, dout, v.fmt);
          cudaDeviceSynchronize();
          cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
          for (int r = 0; r < M; ++r)
            for (int c = 0; c < N; ++c) {
              float s = 0.f;
              for (int b = ncol - 1; b >= nmain; --b) {
                const float sc = v.fmt ? std::ldexp(1.f, -11 * blk_class[b]) : 1.f;
                s += sc * out[(size_t)r * 512 + b * N + c];
              }
              got[(size_t)r * N + c] = s + tot[(size_t)r * N + c];
            }
        } else {
          run(0, ops.size());
          for (int r = 0; r < M; ++r)
            for (int c = 0; c < N; ++c) {
              float s = 0.f;  // smallest class first, then the main blocks
              for (int b = ncol - 1; b >= 0; --b) {
                const float sc = v.fmt ? std::ldexp(1.f, -11 * blk_class[b]) : 1.f;
                s += sc * out[(size_t)r * 512 + b * N + c];
              }
              got[(size_t)r * N + c] = s;
            }
        }
        if (!ok) {
          printf("error\n");
          return 1;
        }
        report(v.name, got);
      }
    }
  }
  return 0;
}
