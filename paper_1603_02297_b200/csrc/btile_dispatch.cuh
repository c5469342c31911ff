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

  // one phase class's map: its rows start `row` rows into the buffer; the
  // map's base is the 16-byte aligned address at or before that, the shift
  // (elements) tells the kernel where the rows begin inside a box
  static cudaError_t encode_class(CUtensorMap* m, int* shift, TmaView v, const void* base, int64_t row_bytes,
                                  uint32_t r, int e) {
    const uintptr_t at = reinterpret_cast<uintptr_t>(base) + static_cast<uintptr_t>(row_bytes) * r;
    const uintptr_t lo = at & ~static_cast<uintptr_t>(15);
    *shift = static_cast<int>((at - lo) / static_cast<uintptr_t>(e));
    const uint64_t per16 = 16u / static_cast<uint64_t>(v.esz);
    v.dim[0] = (v.dim[0] + static_cast<uint64_t>(at - lo) / static_cast<uint64_t>(v.esz) + per16 - 1) / per16 * per16;
    return tma_encode(m, v, reinterpret_cast<const void*>(lo));
  }

  static cudaError_t launch(int ka, int kb, int mode, const SmemParams& p, const BtileTma& bt,
                            const Launch& l, cudaStream_t s) {
    const int jy = p.ly == 0 ? 0 : btile_rows_per_lane(p.S * p.ty, p.ly);  // ly 0: linear walk
    BtileParams q;
    q.p = p;
    q.p.ctr = btile_counter(s);  // null: static tile order
    if (p.tma & 1)
      for (uint32_t r = 0; r < p.ca; ++r) {
        const cudaError_t e = encode_class(&q.ma[r], &q.sha[r], bt.a[r], p.A, bt.row_bytes_a, r, bt.ea);
        if (e != cudaSuccess) return e;
      }
    if (p.tma & 2)
      for (uint32_t r = 0; r < p.cb; ++r) {
        const cudaError_t e = encode_class(&q.mb[r], &q.shb[r], bt.b[r], p.B, bt.row_bytes_b, r, bt.eb);
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
