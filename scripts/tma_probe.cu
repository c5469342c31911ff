// tma_probe.cu -- what the driver's tensor-map encoder accepts and how TMA
// lays boxes out in shared memory (development probe, not product code).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/_bin/tma_probe scripts/tma_probe.cu
//
// Each case encodes a map over a u32 buffer holding its own element index,
// loads one box into shared memory with cp.async.bulk.tensor, copies the
// shared bytes out verbatim and compares them with the box the host expects
// (row-major over the box dims, dim 0 fastest; swizzle cases are printed).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int R>
__global__ void load_box(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int c3, int c4,
                         uint32_t bytes, uint32_t* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0xdeadbeefu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("{ .reg .b64 s; mbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1; }" ::"r"(su32(&bar)),
                 "r"(bytes)
                 : "memory");
    if constexpr (R == 2)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(sm)),
          "l"(&m), "r"(c0), "r"(c1), "r"(su32(&bar))
          : "memory");
    if constexpr (R == 3)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su32(sm)),
          "l"(&m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&bar))
          : "memory");
    if constexpr (R == 4)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
              su32(sm)),
          "l"(&m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(&bar))
          : "memory");
  }
  asm volatile(
      "{ .reg .pred d; W: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0; @!d bra W; }" ::"r"(su32(&bar))
      : "memory");
  for (uint32_t i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<uint32_t*>(sm)[i];
}

struct Case {
  const char* name;
  int rank;
  std::vector<cuuint64_t> dim, stride_el;  // stride_el: element strides of dims 1..rank-1
  std::vector<cuuint32_t> box;
  std::vector<int> coord;
  CUtensorMapSwizzle sw;
};

int main() {
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
          cudaSuccess ||
      !encode) {
    std::printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  const size_t N = size_t{1} << 24;
  uint32_t* buf;
  cudaMalloc(&buf, N * 4);
  std::vector<uint32_t> h(N);
  for (size_t i = 0; i < N; ++i) h[i] = static_cast<uint32_t>(i);
  cudaMemcpy(buf, h.data(), N * 4, cudaMemcpyHostToDevice);
  uint32_t* out;
  cudaMalloc(&out, 1 << 20);
  cudaFuncSetAttribute(load_box<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(load_box<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(load_box<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);

  std::vector<Case> cases = {
      // monotone reference: [16 x 8 x 4] of a (64, 32, ...) array
      {"monotone3", 3, {64, 32, 64}, {64, 64 * 32}, {16, 8, 4}, {4, 2, 1}, CU_TENSOR_MAP_SWIZZLE_NONE},
      // non-monotone strides: dim1 stride > dim2 stride
      {"nonmono3", 3, {64, 64, 32}, {64 * 32, 64}, {16, 4, 8}, {4, 1, 2}, CU_TENSOR_MAP_SWIZZLE_NONE},
      // carrier dim with a huge extent in the middle (overlapping view)
      {"carrier_mid", 3, {16, 1u << 20, 8}, {64, 256}, {16, 1, 8}, {0, 77, 3}, CU_TENSOR_MAP_SWIZZLE_NONE},
      // odd-quad inner box (36 x 20), no swizzle
      {"box36x20", 2, {4000, 4000}, {4000}, {36, 20}, {8, 5}, CU_TENSOR_MAP_SWIZZLE_NONE},
      // partial box at the end (OOB fill)
      {"oob", 2, {50, 40}, {64}, {16, 8}, {40, 36}, CU_TENSOR_MAP_SWIZZLE_NONE},
      // swizzle 128B with a 32-byte inner box (layout printed)
      // a box whose dim-0 start is not 16-byte aligned (coordinate 1, 3, 5)
      {"start1", 2, {4000, 4000}, {4000}, {36, 20}, {1, 5}, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"start3", 2, {4003, 4000}, {4000}, {40, 4}, {3, 7}, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"start5", 3, {1001, 20, 40}, {1004, 1004 * 20}, {8, 3, 2}, {5, 4, 3}, CU_TENSOR_MAP_SWIZZLE_NONE},
      // a row stride of 4 elements' phase: class view (every 4th row, base at row 1)
      {"classrow", 2, {283 + 3, 100}, {283 * 4}, {96, 8}, {3, 2}, CU_TENSOR_MAP_SWIZZLE_NONE},
      // 4D non-monotone
      {"nonmono4", 4, {8, 16, 16, 16}, {8 * 16 * 16, 8, 8 * 16}, {8, 4, 4, 2}, {0, 1, 2, 3},
       CU_TENSOR_MAP_SWIZZLE_NONE},
  };
  for (const Case& c : cases) {
    CUtensorMap m;
    std::vector<cuuint64_t> gs;
    for (cuuint64_t s : c.stride_el) gs.push_back(s * 4);
    std::vector<cuuint32_t> es(c.rank, 1);
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, c.rank, buf, c.dim.data(), gs.data(), c.box.data(),
                        es.data(), CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      std::printf("%-12s encode rc=%d\n", c.name, static_cast<int>(r));
      continue;
    }
    uint32_t cnt = 1;
    for (cuuint32_t b : c.box) cnt *= b;
    const uint32_t bytes = cnt * 4;
    int cc[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < c.rank; ++i) cc[i] = c.coord[i];
    if (c.rank == 2) load_box<2><<<1, 128, bytes>>>(m, cc[0], cc[1], 0, 0, 0, bytes, out);
    if (c.rank == 3) load_box<3><<<1, 128, bytes>>>(m, cc[0], cc[1], cc[2], 0, 0, bytes, out);
    if (c.rank == 4) load_box<4><<<1, 128, bytes>>>(m, cc[0], cc[1], cc[2], cc[3], 0, bytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      std::printf("%-12s kernel error %s\n", c.name, cudaGetErrorString(e));
      return 2;
    }
    std::vector<uint32_t> got(cnt);
    cudaMemcpy(got.data(), out, bytes, cudaMemcpyDeviceToHost);
    // expected, dense box order
    int bad = 0;
    for (uint32_t i = 0; i < cnt; ++i) {
      uint32_t rem = i;
      int64_t off = 0;
      bool oob = false;
      for (int d = 0; d < c.rank; ++d) {
        const uint32_t k = rem % c.box[d];
        rem /= c.box[d];
        const int64_t co = c.coord[d] + k;
        if (co >= static_cast<int64_t>(c.dim[d])) oob = true;
        off += co * (d == 0 ? 1 : static_cast<int64_t>(c.stride_el[d - 1]));
      }
      const uint32_t want = oob ? 0u : static_cast<uint32_t>(off);
      if (got[i] != want) ++bad;
    }
    std::printf("%-12s encode ok, %u elements, %d differ from the dense box order\n", c.name, cnt, bad);
    if (c.sw != CU_TENSOR_MAP_SWIZZLE_NONE) {
      for (uint32_t i = 0; i < std::min<uint32_t>(cnt, 256); ++i)
        std::printf("%u%c", got[i], (i % 16 == 15) ? '\n' : ' ');
    }
  }
  return 0;
}
