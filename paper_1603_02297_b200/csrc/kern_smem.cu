// kern_smem.cu -- instantiation and launch of the staged-tile kernels:
// tile_kernel (32-bit tables, the common case) and smem_kernel (64-bit).
#include <cstdlib>

#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace ttb {

namespace {
// dense: 2 -> dense_kernel (power-of-two fast path, kk = EPT), 1 -> tile_kernel
// (kk = compile-time walk length or 0), 0 -> smem_kernel (64-bit offsets)
template <class F>
cudaError_t with_smem(int ka, int kb, int mode, int dense, int kk, F&& f) {
  return with_types(ka, kb, [&](auto t) {
    using T = decltype(t);
    using SA = typename T::SA;
    using SB = typename T::SB;
    // mode 3 (update with direct B reads) exists for the staged-tile kernels
    // only; the 64-bit smem_kernel always reads B directly under mode 2
    auto modes = [&](auto&& g) -> cudaError_t {
      if (mode == 3) return g(std::integral_constant<int, 3>{});
      return with_mode(mode, g);
    };
    return modes([&](auto m) {
      constexpr int M = decltype(m)::value;
      if (dense == 2 || dense == 3) {  // 3: three-stage cp.async ring
        const bool s3 = dense == 3;
        switch (kk) {
          case 4:
            return s3 ? f(&dense_kernel<SA, SB, T::C, M, 4, 3>) : f(&dense_kernel<SA, SB, T::C, M, 4, 2>);
          case 8:
            return s3 ? f(&dense_kernel<SA, SB, T::C, M, 8, 3>) : f(&dense_kernel<SA, SB, T::C, M, 8, 2>);
          default:
            return s3 ? f(&dense_kernel<SA, SB, T::C, M, 16, 3>)
                      : f(&dense_kernel<SA, SB, T::C, M, 16, 2>);
        }
      }
      if (dense == 1) {
        switch (kk) {
          case 4: return f(&tile_kernel<SA, SB, T::C, M, 4>);
          case 8: return f(&tile_kernel<SA, SB, T::C, M, 8>);
          case 16: return f(&tile_kernel<SA, SB, T::C, M, 16>);
          default: return f(&tile_kernel<SA, SB, T::C, M, 0>);
        }
      }
      return f(&smem_kernel<SA, SB, T::C, (M == 3 ? 2 : M)>);
    });
  });
}

}  // namespace

int smem_carveout() {
  // shared/L1 split of the unified array (percent shared).  Half leaves L1 room
  // for the cp.async (.ca) line allocations; TTB_CARVEOUT overrides, < 0 keeps
  // the driver default.
  static const int c = [] {
    const char* e = std::getenv("TTB_CARVEOUT");
    return e ? std::atoi(e) : 50;
  }();
  return c;
}

cudaError_t launch_smem(int ka, int kb, int mode, const SmemParams& p, const Launch& l,
                        cudaStream_t s) {
  if (p.dense == 4) return launch_vtile(ka, kb, mode, p, l, s);
  if (p.dense == 5 && !p.tma) return launch_btile(ka, kb, mode, p, BtileTma{}, l, s);
  if (p.dense == 5) return cudaErrorInvalidValue;  // tensor-map sides: launch_btile with the plan's views
  return with_smem(ka, kb, mode, p.dense, p.ept, [&](auto fn) {
    if (l.smem > kSmemOptIn) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
      if (e != cudaSuccess) return e;
    }
    fn<<<l.grid, l.block, l.smem, s>>>(p);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_smem(int ka, int kb, int mode, int dense, int ept, int block, int smem) {
  int n = 0;
  with_smem(ka, kb, mode, dense, ept, [&](auto fn) {
    if (smem_carveout() >= 0)
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, smem_carveout());
    if (smem > kSmemOptIn) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem);
  });
  return n;
}

}  // namespace ttb
