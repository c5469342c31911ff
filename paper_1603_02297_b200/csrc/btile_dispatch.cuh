// btile_dispatch.cuh -- run-time -> template dispatch of btile_kernel for one
// warp-role configuration (NC consumer warps, PW producer warps), shared by
// kern_btile.cu (the default roles) and kern_btile_big.cu (large tiles).
#pragma once

#include <type_traits>

#include "btile.cuh"
#include "dispatch.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace ttb {

// JYS: the column-walk depths instantiated (0 = linear walk)
template <int NC, int PW, int... JYS>
struct BtileCfg {
  template <class F>
  static cudaError_t with(int ka, int kb, int mode, int jy, F&& f) {
    if (mode < 0 || mode > 3) return cudaErrorInvalidValue;
    // every kind pair: A rows and B columns are fetched with their own element
    // sizes, the epilogue converts (executor.hpp:18-31)
    return with_types(ka, kb, [&](auto t) -> cudaError_t {
      using T = decltype(t);
      auto modes = [&](auto&& g) -> cudaError_t {
        if (mode == 3) return g(std::integral_constant<int, 3>{});
        return with_mode(mode, g);
      };
      return modes([&](auto m) {
        constexpr int M = decltype(m)::value;
        using SA = typename T::SA;
        using SB = typename T::SB;
        cudaError_t r = cudaErrorInvalidValue;
        ((jy == JYS ? (r = f(&btile_kernel<SA, SB, T::C, M, JYS, PW, NC>), true) : false) || ...);
        return r;
      });
    });
  }

  static cudaError_t launch(int ka, int kb, int mode, const SmemParams& p, const TmaPlan& tp,
                            const Launch& l, cudaStream_t s) {
    const int jy = p.ly == 0 ? 0 : btile_rows_per_lane(p.S * p.ty, p.ly);  // ly 0: linear walk
    BtileParams q;
    q.p = p;
    q.p.ctr = btile_counter(s);  // null: static tile order
    if (p.tma & 1) {
      const cudaError_t e = tma_encode(&q.ma, tp.va, p.A);
      if (e != cudaSuccess) return e;
    }
    if (p.tma & 2) {
      const cudaError_t e = tma_encode(&q.mb, tp.vb, p.B);
      if (e != cudaSuccess) return e;
    }
    return with(ka, kb, mode, jy, [&](auto fn) {
      if (l.smem > kSmemOptIn) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
        if (e != cudaSuccess) return e;
      }
      fn<<<l.grid, l.block, l.smem, s>>>(q);
      count_launch();
      return cudaGetLastError();
    });
  }

  static int occupancy(int ka, int kb, int mode, int jy, int block, int smem) {
    int n = 0;
    with(ka, kb, mode, jy, [&](auto fn) {
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (smem > kSmemOptIn) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem);
    });
    return n;
  }
};

}  // namespace ttb
