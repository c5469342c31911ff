// kern_tma.cu -- tensor-map encoding, instantiation and launch of tma_kernel
// (tma.cuh): the eight kind pairs, update modes 0-2, micro-tile (case 2) or
// run-chunk (case 1) consumers.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "dispatch.cuh"
#include "launch.hpp"
#include "tma.cuh"

namespace ttb {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

// L2 fetch size of the maps' loads (experiment switch TTB_TMA_L2: 0, 64, 128, 256)
CUtensorMapL2promotion l2_promotion() {
  static const CUtensorMapL2promotion p = [] {
    const char* e = std::getenv("TTB_TMA_L2");
    const int v = e ? std::atoi(e) : 256;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                            : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  return p;
}

}  // namespace

cudaError_t tma_encode(CUtensorMap* m, const TmaView& v, const void* base) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = encoder();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dim[kTmaMaxRank], str[kTmaMaxRank];
  cuuint32_t box[kTmaMaxRank], es[kTmaMaxRank];
  for (int k = 0; k < v.rank; ++k) {
    dim[k] = v.dim[k];
    box[k] = v.box[k];
    es[k] = 1;
    if (k) str[k - 1] = v.stride[k];
  }
  const CUresult r = fn(m, v.esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64,
                        static_cast<cuuint32_t>(v.rank), const_cast<void*>(base), dim, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

namespace {

template <class F>
cudaError_t with_tma(int ka, int kb, int mode, bool runs, F&& f) {
  return with_types(ka, kb, [&](auto t) {
    using T = decltype(t);
    return with_mode(mode, [&](auto m) {
      constexpr int M = decltype(m)::value;
      if (runs) {
        if constexpr (std::is_same<typename T::SA, typename T::SB>::value)
          return f(&tma_kernel<typename T::SA, typename T::SB, T::C, M, true>);
        return cudaErrorInvalidValue;
      }
      return f(&tma_kernel<typename T::SA, typename T::SB, T::C, M, false>);
    });
  });
}

}  // namespace

bool tma_available() { return encoder() != nullptr; }

cudaError_t launch_tma(int ka, int kb, int mode, const TmaPlan& p, const void* A, void* B, const Launch& l,
                       cudaStream_t s) {
  TmaParams q;
  q.t = p;
  cudaError_t e = tma_encode(&q.ma, p.va, A);
  if (e == cudaSuccess) e = tma_encode(&q.mb, p.vb, B);
  if (e != cudaSuccess) return e;
  return with_tma(ka, kb, mode, p.kch > 0, [&](auto fn) {
    if (l.smem > kSmemOptIn) {
      cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
      if (r != cudaSuccess) return r;
    }
    fn<<<l.grid, l.block, l.smem, s>>>(q);
    count_launch();
    return cudaGetLastError();
  });
}

int occupancy_tma(int ka, int kb, int mode, bool runs, int block, int smem) {
  int n = 0;
  with_tma(ka, kb, mode, runs, [&](auto fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (smem > kSmemOptIn) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem);
  });
  return n;
}

}  // namespace ttb
