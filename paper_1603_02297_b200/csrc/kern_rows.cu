// kern_rows.cu -- instantiation, launch and occupancy of rowcopy_kernel
// (rows.cuh): the eight kind pairs, update modes 0-2.
#include "dispatch.cuh"
#include "launch.hpp"
#include "rows.cuh"

namespace ttb {

namespace {
template <class F>
cudaError_t with_rows(int ka, int kb, int mode, F&& f) {
  return with_types(ka, kb, [&](auto t) {
    using T = decltype(t);
    return with_mode(mode, [&](auto m) {
      return f(&rowcopy_kernel<typename T::SA, typename T::SB, T::C, decltype(m)::value>);
    });
  });
}
}  // namespace

cudaError_t launch_rowcopy(int ka, int kb, int mode, const CopyParams& p, const Launch& l, cudaStream_t s) {
  return with_rows(ka, kb, mode, [&](auto fn) {
    if (l.smem > kSmemOptIn) {
      const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
      if (e != cudaSuccess) return e;
    }
    fn<<<l.grid, l.block, l.smem, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_rowcopy(int ka, int kb, int mode, int block, int smem) {
  int n = 0;
  with_rows(ka, kb, mode, [&](auto fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (smem > kSmemOptIn) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem);
  });
  return n;
}

}  // namespace ttb
