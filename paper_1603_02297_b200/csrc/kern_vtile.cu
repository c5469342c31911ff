// kern_vtile.cu -- instantiation and launch of vtile_kernel (vtile.cuh): equal
// kinds s/d/c, every update mode, vector widths VA, VB of 1/2/4 elements that
// fit 16 bytes (not both 1 -- that shape runs on dense_kernel / tile_kernel).
#include <type_traits>

#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"
#include "vtile.cuh"

namespace ttb {

namespace {
template <class F>
cudaError_t with_vtile(int ka, int kb, int mode, int va, int vb, int sh, F&& f) {
  if (ka != kb || ka > 2 || (va == 1 && vb == 1)) return cudaErrorInvalidValue;
  if (sh < 0 || sh > 3) return cudaErrorInvalidValue;
  return with_types(ka, kb, [&](auto t) -> cudaError_t {
    using T = decltype(t);
    using SA = typename T::SA;
    using SB = typename T::SB;
    constexpr int EB = static_cast<int>(sizeof(SA)) * T::C;
    if constexpr (!std::is_same<SA, SB>::value) {
      return cudaErrorInvalidValue;
    } else {
    auto modes = [&](auto&& g) -> cudaError_t {
      if (mode == 3) return g(std::integral_constant<int, 3>{});
      return with_mode(mode, g);
    };
    return modes([&](auto m) {
      constexpr int M = decltype(m)::value;
      if (sh != 0) {  // shifted sides: full 16-byte vectors on both sides
        constexpr int V = 16 / EB;
        if (va != V || vb != V) return cudaErrorInvalidValue;
        switch (sh) {
          case 1: return f(&vtile_kernel<SA, SB, T::C, M, V, V, 1>);
          case 2: return f(&vtile_kernel<SA, SB, T::C, M, V, V, 2>);
          default: return f(&vtile_kernel<SA, SB, T::C, M, V, V, 3>);
        }
      }
      return with_width<EB>(va, [&](auto a) {
        return with_width<EB>(vb, [&](auto b) {
          constexpr int VA = decltype(a)::value, VB = decltype(b)::value;
          if constexpr (VA == 1 && VB == 1)
            return cudaErrorInvalidValue;
          else
            return f(&vtile_kernel<SA, SB, T::C, M, VA, VB, 0>);
        });
      });
    });
    }
  });
}
}  // namespace

cudaError_t launch_vtile(int ka, int kb, int mode, const SmemParams& p, const Launch& l,
                         cudaStream_t s) {
  return with_vtile(ka, kb, mode, p.va, p.vb, p.sh, [&](auto fn) {
    if (l.smem > kSmemOptIn) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
      if (e != cudaSuccess) return e;
    }
    fn<<<l.grid, l.block, l.smem, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_vtile(int ka, int kb, int mode, int va, int vb, int sh, int block, int smem) {
  int n = 0;
  with_vtile(ka, kb, mode, va, vb, sh, [&](auto fn) {
    if (smem_carveout() >= 0)
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, smem_carveout());
    if (smem > kSmemOptIn) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem);
  });
  return n;
}

}  // namespace ttb
