// kern_rt.cu -- instantiation and launch of rt_kernel (in-register micro-tiles).
#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace ttb {

namespace {
template <class F>
cudaError_t with_rt(int ka, int kb, int mx, int my, int mode, F&& f) {
  return with_types(ka, kb, [&](auto t) {
    using T = decltype(t);
    constexpr int EA = sizeof(typename T::SA) * T::C, EB = sizeof(typename T::SB) * T::C;
    return with_width<EA>(mx, [&](auto x) {
      return with_width<EB>(my, [&](auto y) {
        return with_mode(mode, [&](auto m) {
          return f(&rt_kernel<typename T::SA, typename T::SB, T::C, decltype(x)::value,
                              decltype(y)::value, decltype(m)::value>);
        });
      });
    });
  });
}
}  // namespace

cudaError_t launch_rt(int ka, int kb, int mx, int my, int mode, const RtParams& p,
                      const Launch& l, cudaStream_t s) {
  return with_rt(ka, kb, mx, my, mode, [&](auto fn) {
    fn<<<l.grid, l.block, 0, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_rt(int ka, int kb, int mx, int my, int mode, int block) {
  int n = 0;
  with_rt(ka, kb, mx, my, mode, [&](auto fn) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, 0);
  });
  return n;
}

}  // namespace ttb
