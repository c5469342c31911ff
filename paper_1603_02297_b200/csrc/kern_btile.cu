// kern_btile.cu -- instantiation and launch of btile_kernel (btile.cuh): the
// four same-kind pairs (mixed pairs run on the other staged tiles), update
// modes 0-3 (3: beta != 0 with B read directly, not through the ring), 1-16
// column elements per consumer lane or the linear walk (0).
#include <type_traits>

#include "btile.cuh"
#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace ttb {

namespace {
template <class F>
cudaError_t with_btile(int ka, int kb, int mode, int jy, F&& f) {
  if (ka != kb || mode < 0 || mode > 3) return cudaErrorInvalidValue;
  return with_types(ka, kb, [&](auto t) -> cudaError_t {
    using T = decltype(t);
    if constexpr (!std::is_same<typename T::SA, typename T::SB>::value) {
      return cudaErrorInvalidValue;
    } else {
      auto modes = [&](auto&& g) -> cudaError_t {
        if (mode == 3) return g(std::integral_constant<int, 3>{});
        return with_mode(mode, g);
      };
      return modes([&](auto m) {
        constexpr int M = decltype(m)::value;
        using SA = typename T::SA;
        switch (jy) {
          case 0: return f(&btile_kernel<SA, SA, T::C, M, 0>);
          case 1: return f(&btile_kernel<SA, SA, T::C, M, 1>);
          case 2: return f(&btile_kernel<SA, SA, T::C, M, 2>);
          case 4: return f(&btile_kernel<SA, SA, T::C, M, 4>);
          case 8: return f(&btile_kernel<SA, SA, T::C, M, 8>);
          case 16: return f(&btile_kernel<SA, SA, T::C, M, 16>);
          default: return cudaErrorInvalidValue;
        }
      });
    }
  });
}
}  // namespace

cudaError_t launch_btile(int ka, int kb, int mode, const SmemParams& p, const Launch& l,
                         cudaStream_t s) {
  const int jy = p.ly == 0 ? 0 : btile_rows_per_lane(p.S * p.ty, p.ly);  // ly 0: linear walk
  return with_btile(ka, kb, mode, jy, [&](auto fn) {
    if (l.smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
      if (e != cudaSuccess) return e;
    }
    fn<<<l.grid, l.block, l.smem, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_btile(int ka, int kb, int mode, int jy, int block, int smem) {
  int n = 0;
  with_btile(ka, kb, mode, jy, [&](auto fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem);
  });
  return n;
}

}  // namespace ttb
