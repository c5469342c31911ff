// kern_copy.cu -- instantiation and launch of copy_kernel (shared stride-1 index).
#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace ttb {

namespace {
template <class T, int V, int MODE>
auto copy_fn() {
  return &copy_kernel<typename T::SA, typename T::SB, T::C, V, MODE>;
}

template <class F>
cudaError_t with_copy(int ka, int kb, int v, int mode, F&& f) {
  return with_types(ka, kb, [&](auto t) {
    using T = decltype(t);
    constexpr int EA = sizeof(typename T::SA) * T::C, EB = sizeof(typename T::SB) * T::C;
    constexpr int EMIN = EA < EB ? EA : EB;
    return with_width<EMIN>(v, [&](auto vw) {
      return with_mode(mode, [&](auto m) { return f(copy_fn<T, decltype(vw)::value, decltype(m)::value>()); });
    });
  });
}
}  // namespace

cudaError_t launch_copy(int ka, int kb, int v, int mode, const CopyParams& p, const Launch& l,
                        cudaStream_t s) {
  return with_copy(ka, kb, v, mode, [&](auto fn) {
    fn<<<l.grid, l.block, 0, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_copy(int ka, int kb, int v, int mode, int block) {
  int n = 0;
  with_copy(ka, kb, v, mode, [&](auto fn) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, 0);
  });
  return n;
}

}  // namespace ttb
