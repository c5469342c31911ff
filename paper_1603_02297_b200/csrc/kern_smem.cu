// kern_smem.cu -- instantiation and launch of smem_kernel (staged tiles).
#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace ttb {

namespace {
template <class F>
cudaError_t with_smem(int ka, int kb, int mode, bool dense, int ept, F&& f) {
  return with_types(ka, kb, [&](auto t) {
    using T = decltype(t);
    return with_mode(mode, [&](auto m) {
      constexpr int M = decltype(m)::value;
      using SA = typename T::SA;
      using SB = typename T::SB;
      if (dense) {
        switch (ept) {
          case 4: return f(&smem_dense_kernel<SA, SB, T::C, M, 4>);
          case 8: return f(&smem_dense_kernel<SA, SB, T::C, M, 8>);
          case 16: return f(&smem_dense_kernel<SA, SB, T::C, M, 16>);
          default: return f(&smem_dense_kernel<SA, SB, T::C, M, 0>);
        }
      }
      return f(&smem_kernel<typename T::SA, typename T::SB, T::C, decltype(m)::value>);
    });
  });
}
}  // namespace

cudaError_t launch_smem(int ka, int kb, int mode, const SmemParams& p, const Launch& l,
                        cudaStream_t s) {
  return with_smem(ka, kb, mode, p.dense != 0, p.ept, [&](auto fn) {
    if (l.smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
      if (e != cudaSuccess) return e;
    }
    fn<<<l.grid, l.block, l.smem, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_smem(int ka, int kb, int mode, bool dense, int ept, int block, int smem) {
  int n = 0;
  with_smem(ka, kb, mode, dense, ept, [&](auto fn) {
    // staged tiles want the whole unified L1/shared array as shared memory
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem);
  });
  return n;
}

}  // namespace ttb
