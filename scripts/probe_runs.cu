// probe_runs.cu -- HBM efficiency versus contiguous run length (kernel-design probe,
// not product code).  A 1.6 GB buffer is cut into chunks of R bytes laid out as
// an M x K chunk grid; chunk (i, j) moves to (j, i) of the destination grid.
// mode 0: contiguous reads, chunk-scattered writes; mode 1: scattered reads,
// contiguous writes; mode 2: both contiguous (plain copy).  16-B accesses,
// 4 in flight per thread.  Prints GB/s (read + write bytes / event time).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/probe_runs.cu -o probe_runs
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void perm_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t units,
                          uint32_t upc /*units per chunk*/, uint64_t M, uint64_t K, int mode) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t u0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u0 < units; u0 += 4 * stride) {
    uint4 v[4];
    uint64_t d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t u = u0 + k * stride;
      if (u >= units) break;
      const uint64_t c = u / upc, o = u - c * upc;
      const uint64_t i = c % M, j = c / M;
      const uint64_t t = (j + K * i) * upc + o;
      uint64_t s = u;
      d[k] = u;
      if (mode == 0) d[k] = t;
      if (mode == 1) s = t;
      v[k] = __ldcs(src + s);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t u = u0 + k * stride;
      if (u >= units) break;
      __stcs(dst + d[k], v[k]);
    }
  }
}

int main() {
  const uint64_t bytes = 1600ull << 20;
  uint4 *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  const int runs[] = {32, 64, 128, 256, 384, 512, 1024, 2048, 4096};
  for (int mode = 0; mode < 3; ++mode) {
    for (int R : runs) {
      if (R < 16) continue;
      const uint32_t upc = R / 16;
      const uint64_t chunks = bytes / R;
      uint64_t M = 1;
      while (M * M < chunks) M <<= 1;
      const uint64_t K = chunks / M;
      const uint64_t units = M * K * upc;
      float best = 1e30f;
      for (int it = 0; it < 6; ++it) {
        cudaEventRecord(e0);
        perm_copy<<<sms * 8, 256>>>(a, b, units, upc, M, K, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 && ms < best) best = ms;
      }
      printf("mode %d run %5d B: %8.1f GB/s\n", mode, R, 2.0 * units * 16 / (best * 1e6));
      if (mode == 2) break;
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
