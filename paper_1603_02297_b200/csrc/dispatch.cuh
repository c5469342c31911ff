// dispatch.cuh -- run-time (kind_a, kind_b) -> (SA, SB, C) template dispatch.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

namespace ttb {

template <class A_, class B_, int C_>
struct Types {
  using SA = A_;
  using SB = B_;
  static constexpr int C = C_;
};

// the eight kind pairs ttune accepts (problem.cpp:45-52)
template <class F>
cudaError_t with_types(int ka, int kb, F&& f) {
  switch (ka * 4 + kb) {
    case 0 * 4 + 0: return f(Types<float, float, 1>{});
    case 1 * 4 + 1: return f(Types<double, double, 1>{});
    case 2 * 4 + 2: return f(Types<float, float, 2>{});
    case 3 * 4 + 3: return f(Types<double, double, 2>{});
    case 0 * 4 + 1: return f(Types<float, double, 1>{});
    case 1 * 4 + 0: return f(Types<double, float, 1>{});
    case 2 * 4 + 3: return f(Types<float, double, 2>{});
    case 3 * 4 + 2: return f(Types<double, float, 2>{});
    default: return cudaErrorInvalidValue;
  }
}

template <class F>
cudaError_t with_mode(int mode, F&& f) {
  switch (mode) {
    case 0: return f(std::integral_constant<int, 0>{});
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    default: return cudaErrorInvalidValue;
  }
}

// vector widths 1/2/4 elements, only those that fit 16 bytes (per element size)
template <int EB, class F>
cudaError_t with_width(int w, F&& f) {
  switch (w) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2:
      if constexpr (2 * EB <= 16) return f(std::integral_constant<int, 2>{});
      break;
    case 4:
      if constexpr (4 * EB <= 16) return f(std::integral_constant<int, 4>{});
      break;
    default: break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace ttb
