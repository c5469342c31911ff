// bulk_probe.cu -- kernel-design probe (not product code): read throughput of
// cp.async.bulk global->shared as a function of copy size, copies per ring
// stage, ring depth and issuing warps.  One CTA per SM; warp w of PW issuing
// warps issues its share of the K copies of every stage; stage s is reused
// once its mbarrier phase has completed (no consumer: pure load path).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1603_02297_b200/csrc \
//        scripts/bulk_probe.cu -o scripts/_bin/bulk_probe
#include <cstdio>
#include <cstdint>

#include "btile.cuh"

using namespace ttb;

__global__ void bulk_ring(const unsigned char* src, uint64_t span, uint32_t R, uint32_t K,
                          uint32_t NS, uint32_t rounds, uint32_t stride, int PW) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t bar[16];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NS; ++s) mbar_init(&bar[s], 32 * PW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t stage_bytes = K * R;
  uint32_t s = 0, ph = 0;
  // every copy reads its own R bytes: copy j of the grid sits at j*R scattered
  // by a fixed odd multiplier over the span (no L2 reuse across CTAs)
  const uint64_t nslots = span / R;
  for (uint32_t r = 0; r < rounds; ++r) {
    if (r >= NS) mbar_wait(&bar[s], ph ^ 1);  // previous use of this stage has landed
    uint32_t bytes = 0;
    for (uint32_t k = warp * 32 + lane; k < K; k += 32 * PW) {
      const uint64_t j = (uint64_t(r) * gridDim.x + blockIdx.x) * K + k;
      const uint64_t off = ((j * stride) % nslots) * R;
      bulk_g2s(sm + s * stage_bytes + k * R, src + (off & ~uint64_t{15}), R, &bar[s]);
      bytes += R;
    }
    mbar_arrive_expect_tx(&bar[s], bytes);
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
  // drain
  for (uint32_t i = 0; i < NS && i < rounds; ++i) {
    mbar_wait(&bar[s], ph ^ 1);
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
}

int main() {
  const uint64_t span = 3ull << 30;
  unsigned char* src;
  cudaMalloc(&src, span + 65536);
  cudaMemset(src, 1, span + 65536);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { uint32_t R, K, NS; int PW; int CPS; };
  const Cfg cfgs[] = {
      {256, 64, 2, 2, 1}, {256, 64, 2, 2, 2}, {256, 64, 2, 2, 4}, {256, 64, 2, 2, 6},
      {512, 32, 2, 2, 1}, {512, 32, 2, 2, 2}, {512, 32, 2, 2, 4}, {512, 32, 2, 2, 6},
      {1024, 16, 2, 2, 2}, {1024, 16, 2, 2, 4}, {2048, 16, 2, 2, 4}, {128, 64, 2, 2, 6},
  };
  for (const Cfg& c : cfgs) {
    const uint32_t smem = c.R * c.K * c.NS;
    if (smem > 200 * 1024) continue;
    cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // ~1.5 GB read in total, rows scattered with a 64 KB stride
    const uint32_t rounds = static_cast<uint32_t>((1500ull << 20) / (148ull * c.CPS * c.R * c.K));
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
      cudaEventRecord(e0);
      bulk_ring<<<148 * c.CPS, 32 * c.PW, smem>>>(src, span, c.R, c.K, c.NS, rounds, 40503u, c.PW);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it && ms < best) best = ms;
    }
    const double bytes = 148.0 * c.CPS * rounds * c.R * c.K;
    printf("R=%5u K=%3u NS=%2u PW=%d CTAs/SM=%d: %8.1f GB/s read  (%.2f us per stage per CTA) %s\n", c.R, c.K,
           c.NS, c.PW, c.CPS, bytes / (best * 1e6), best * 1e3 / rounds,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
