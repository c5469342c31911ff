// kern_copy.cu -- instantiation and launch of the shared-stride-1 copy kernels.
#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace ttb {

namespace {
template <class F>
cudaError_t with_copy(int ka, int kb, int v, int mode, bool long_rows, F&& f) {
  return with_types(ka, kb, [&](auto t) {
    using T = decltype(t);
    constexpr int EA = sizeof(typename T::SA) * T::C, EB = sizeof(typename T::SB) * T::C;
    constexpr int EMIN = EA < EB ? EA : EB;
    return with_width<EMIN>(v, [&](auto vw) {
      return with_mode(mode, [&](auto m) {
        constexpr int V = decltype(vw)::value, M = decltype(m)::value;
        if (long_rows) return f(&copy_rows_kernel<typename T::SA, typename T::SB, T::C, V, M>);
        return f(&copy_kernel<typename T::SA, typename T::SB, T::C, V, M>);
      });
    });
  });
}
}  // namespace

cudaError_t launch_copy(int ka, int kb, int v, int mode, const CopyParams& p, const Launch& l,
                        cudaStream_t s) {
  if (p.bulk) return launch_rowcopy(ka, kb, mode, p, l, s);
  return with_copy(ka, kb, v, mode, p.long_rows != 0, [&](auto fn) {
    fn<<<l.grid, l.block, 0, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_copy(int ka, int kb, int v, int mode, bool long_rows, int block) {
  int n = 0;
  with_copy(ka, kb, v, mode, long_rows, [&](auto fn) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, 0);
  });
  return n;
}

}  // namespace ttb
