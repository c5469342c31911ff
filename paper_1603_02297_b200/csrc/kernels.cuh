// kernels.cuh -- sm_100a device code of the engine (templated; instantiated
// per element-kind pair and update mode in kern_*.cu).
//
// Three data-movement kernels replace ttune's CPU executor paths
// (proj/core/src/executor.cpp):
//   copy_kernel  <- run_case1 / run_copy_1d   (shared stride-1 index)
//   rt_kernel    <- run_case2 + micro_tile_staged (w x w in-register tiles)
//   smem_kernel  <- run_case2 for unaligned / tiny leading extents
// and the element update of every kernel is ttune's arithmetic contract
// (executor.hpp:18-40) with explicit round-to-nearest intrinsics so nvcc can
// never contract it into an FMA.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "params.hpp"

namespace ttb {

// ------------------------------------------------------------ arithmetic --

template <class SA, class SB>
struct WideOf {
  using type = float;
};
template <>
struct WideOf<double, float> {
  using type = double;
};
template <>
struct WideOf<float, double> {
  using type = double;
};
template <>
struct WideOf<double, double> {
  using type = double;
};

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <class T>
__device__ __forceinline__ T narrow(float x);
template <>
__device__ __forceinline__ float narrow<float>(float x) { return x; }
template <>
__device__ __forceinline__ double narrow<double>(float x) { return static_cast<double>(x); }
template <class T>
__device__ __forceinline__ T narrow(double x);
template <>
__device__ __forceinline__ float narrow<float>(double x) { return __double2float_rn(x); }
template <>
__device__ __forceinline__ double narrow<double>(double x) { return x; }

// Update modes: 0 = move (alpha == 1, beta == 0: SB(W(a)), no arithmetic),
// 1 = scale (beta == 0: SB(alpha*W(a)), B never read),
// 2 = update (SB(alpha*W(a) + beta*W(b)), two products, one sum).
template <class SA, class SB, int MODE>
struct Update {
  using W = typename WideOf<SA, SB>::type;
  W al, be;
  __device__ __forceinline__ explicit Update(const Scale& s)
      : al(static_cast<W>(s.alpha)), be(static_cast<W>(s.beta)) {}
  __device__ __forceinline__ SB operator()(SA a, SB b) const {
    const W wa = static_cast<W>(a);
    if constexpr (MODE == 0) {
      return narrow<SB>(wa);
    } else if constexpr (MODE == 1) {
      return narrow<SB>(mul_rn(al, wa));
    } else {
      return narrow<SB>(add_rn(mul_rn(al, wa), mul_rn(be, static_cast<W>(b))));
    }
  }
};

// ------------------------------------------------------------- vectors --

template <class T, int N>
struct alignas((sizeof(T) * N) >= 16 ? 16 : (sizeof(T) * N)) Vec {
  T v[N];
};

// streaming read-only load of one <=16-byte chunk (A is never written)
template <int BYTES>
__device__ __forceinline__ void ld_nc(const void* p, void* out) {
  if constexpr (BYTES == 16) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    *reinterpret_cast<uint4*>(out) = r;
  } else if constexpr (BYTES == 8) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p));
    *reinterpret_cast<uint2*>(out) = r;
  } else {
    static_assert(BYTES == 4, "chunk");
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    *reinterpret_cast<uint32_t*>(out) = r;
  }
}

// load of B for the beta != 0 update (B is read once, then overwritten)
template <int BYTES>
__device__ __forceinline__ void ld_b(const void* p, void* out) {
  if constexpr (BYTES == 16) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    *reinterpret_cast<uint4*>(out) = r;
  } else if constexpr (BYTES == 8) {
    uint2 r;
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    *reinterpret_cast<uint2*>(out) = r;
  } else {
    static_assert(BYTES == 4, "chunk");
    uint32_t r;
    asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    *reinterpret_cast<uint32_t*>(out) = r;
  }
}

template <int BYTES>
__device__ __forceinline__ void st_g(void* p, const void* in) {
  if constexpr (BYTES == 16) {
    const uint4 r = *reinterpret_cast<const uint4*>(in);
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(r.x), "r"(r.y), "r"(r.z),
                 "r"(r.w)
                 : "memory");
  } else if constexpr (BYTES == 8) {
    const uint2 r = *reinterpret_cast<const uint2*>(in);
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(r.x), "r"(r.y) : "memory");
  } else {
    static_assert(BYTES == 4, "chunk");
    const uint32_t r = *reinterpret_cast<const uint32_t*>(in);
    asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(r) : "memory");
  }
}

// whole-vector helpers: vectors of up to 32 bytes move as <=16-byte chunks
template <class T, int N>
__device__ __forceinline__ void vload_a(Vec<T, N>& v, const T* p) {
  constexpr int BYTES = sizeof(T) * N;
  constexpr int CH = BYTES > 16 ? 16 : BYTES;
#pragma unroll
  for (int c = 0; c < BYTES / CH; ++c)
    ld_nc<CH>(reinterpret_cast<const char*>(p) + c * CH, reinterpret_cast<char*>(v.v) + c * CH);
}

template <class T, int N>
__device__ __forceinline__ void vload_b(Vec<T, N>& v, const T* p) {
  constexpr int BYTES = sizeof(T) * N;
  constexpr int CH = BYTES > 16 ? 16 : BYTES;
#pragma unroll
  for (int c = 0; c < BYTES / CH; ++c)
    ld_b<CH>(reinterpret_cast<const char*>(p) + c * CH, reinterpret_cast<char*>(v.v) + c * CH);
}

template <class T, int N>
__device__ __forceinline__ void vstore(T* p, const Vec<T, N>& v) {
  constexpr int BYTES = sizeof(T) * N;
  constexpr int CH = BYTES > 16 ? 16 : BYTES;
#pragma unroll
  for (int c = 0; c < BYTES / CH; ++c)
    st_g<CH>(reinterpret_cast<char*>(p) + c * CH, reinterpret_cast<const char*>(v.v) + c * CH);
}

// --------------------------------------------------------- index decode --

// flat index of a Space -> element offsets in A and in B
__device__ __forceinline__ void decode(const Space& s, uint32_t idx, int64_t& oa, int64_t& ob) {
  oa = 0;
  ob = 0;
  for (int d = 0; d < s.nd; ++d) {
    const uint32_t q = udiv(idx, s.ext[d]);
    const int64_t r = static_cast<int64_t>(idx - q * s.ext[d].d);
    oa += r * s.sa[d];
    ob += r * s.sb[d];
    idx = q;
  }
}

// ------------------------------------------------------------- kernels --

// Shared stride-1 index: each vector of V elements is contiguous in A and B.
template <class SA, class SB, int C, int V, int MODE>
__global__ void __launch_bounds__(256) copy_kernel(const CopyParams P) {
  const Update<SA, SB, MODE> up(P.sc);
  const SA* __restrict__ A = static_cast<const SA*>(P.A);
  SB* __restrict__ B = static_cast<SB*>(P.B);
  constexpr int U = 4;  // independent vectors in flight per thread
  const uint32_t nth = gridDim.x * blockDim.x;
  for (uint32_t f0 = blockIdx.x * blockDim.x + threadIdx.x; f0 < P.total_vec; f0 += U * nth) {
    Vec<SA, V * C> a[U];
    Vec<SB, V * C> b[U];
    SB* pb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t f = f0 + u * nth;
      pb[u] = nullptr;
      if (f < P.total_vec) {
        const uint32_t row = udiv(f, P.vpr);
        const uint32_t v = f - row * P.vec_per_row;
        int64_t oa, ob;
        decode(P.rows, row, oa, ob);
        vload_a(a[u], A + (oa + static_cast<int64_t>(v) * V) * C);
        pb[u] = B + (ob + static_cast<int64_t>(v) * V) * C;
        if constexpr (MODE == 2) vload_b(b[u], pb[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!pb[u]) continue;
#pragma unroll
      for (int i = 0; i < V * C; ++i) b[u].v[i] = up(a[u].v[i], b[u].v[i]);
      vstore(pb[u], b[u]);
    }
  }
}

// In-register micro-tile transpose.  A warp covers (lx*MX) x ((32/lx)*MY)
// elements of the X-by-Y plane per item: lane (i, j) loads MY vectors of MX
// elements (rows y..y+MY-1, contiguous in A), transposes them in registers
// and stores MX vectors of MY elements (columns x..x+MX-1, contiguous in B).
// The paper's w x w micro-kernel (executor.hpp:101-128) mapped to one thread.
template <class SA, class SB, int C, int MX, int MY, int MODE>
__global__ void __launch_bounds__(256) rt_kernel(const RtParams P) {
  const Update<SA, SB, MODE> up(P.sc);
  const SA* __restrict__ A = static_cast<const SA*>(P.A);
  SB* __restrict__ B = static_cast<SB*>(P.B);
  const int lane = threadIdx.x & 31;
  const uint32_t li = static_cast<uint32_t>(lane % P.lx);
  const uint32_t lj = static_cast<uint32_t>(lane / P.lx);
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < P.items; it += nwarps) {
    uint32_t xc, yc, o;
    if (P.order == 0) {
      const uint32_t t = udiv(it, P.dnx);
      xc = it - t * P.nxc;
      o = udiv(t, P.dny);
      yc = t - o * P.nyc;
    } else {
      const uint32_t t = udiv(it, P.dny);
      yc = it - t * P.nyc;
      o = udiv(t, P.dnx);
      xc = t - o * P.nxc;
    }
    const uint32_t x = xc * P.wx + li * MX;
    const uint32_t y = yc * P.wy + lj * MY;
    if (x >= P.X.total || y >= P.Y.total) continue;
    int64_t aO, bO, aX, bX, aY, bY;
    decode(P.O, o, aO, bO);
    decode(P.X, x, aX, bX);
    decode(P.Y, y, aY, bY);
    const SA* pa = A + (aO + aX + aY) * C;
    Vec<SA, MX * C> r[MY];
#pragma unroll
    for (int k = 0; k < MY; ++k) vload_a(r[k], pa + k * P.sa_y0 * C);
    SB* pb = B + (bO + bX + bY) * C;
#pragma unroll
    for (int j = 0; j < MX; ++j) {
      Vec<SB, MY * C> w;
      SB* q = pb + j * P.sb_x0 * C;
      if constexpr (MODE == 2) vload_b(w, q);
#pragma unroll
      for (int k = 0; k < MY; ++k)
#pragma unroll
        for (int c = 0; c < C; ++c) w.v[k * C + c] = up(r[k].v[j * C + c], w.v[k * C + c]);
      vstore(q, w);
    }
  }
}

// Shared-memory staged tile for any shape (unaligned or tiny leading
// extents).  Tile = S (shared stride-1 extent, 1 if none) x TX x TY.  Loads
// walk the tile in A order (s, x, y) and stores in B order (s, y, x), so both
// sides are warp-contiguous; rows of `rl` elements are padded so neither walk
// has shared-memory bank conflicts (pad chosen on the host).
template <class SA, class SB, int C, int MODE>
__global__ void __launch_bounds__(256) smem_kernel(const SmemParams P) {
  using E = Vec<SA, C>;  // one element (C scalars) moves as a unit
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t* offAX = reinterpret_cast<int64_t*>(smem_raw);
  int64_t* offBX = offAX + P.tx;
  int64_t* offAY = offBX + P.tx;
  int64_t* offBY = offAY + P.ty;
  E* tile = reinterpret_cast<E*>(offBY + P.ty);

  const Update<SA, SB, MODE> up(P.sc);
  const SA* __restrict__ A = static_cast<const SA*>(P.A);
  SB* __restrict__ B = static_cast<SB*>(P.B);
  const uint32_t L = P.S * P.tx * P.ty;

  for (uint32_t it = blockIdx.x; it < P.items; it += gridDim.x) {
    uint32_t xc, yc, o;
    if (P.order == 0) {
      const uint32_t t = udiv(it, P.dnx);
      xc = it - t * P.nxc;
      o = udiv(t, P.dny);
      yc = t - o * P.nyc;
    } else {
      const uint32_t t = udiv(it, P.dny);
      yc = it - t * P.nyc;
      o = udiv(t, P.dnx);
      xc = t - o * P.nxc;
    }
    const uint32_t x0 = xc * P.tx, y0 = yc * P.ty;
    const uint32_t nx = min(P.tx, P.X.total - x0), ny = min(P.ty, P.Y.total - y0);
    int64_t aO, bO;
    decode(P.O, o, aO, bO);
    for (uint32_t i = threadIdx.x; i < nx; i += blockDim.x) {
      int64_t a, b;
      decode(P.X, x0 + i, a, b);
      offAX[i] = a + aO;
      offBX[i] = b + bO;
    }
    for (uint32_t i = threadIdx.x; i < ny; i += blockDim.x) {
      int64_t a, b;
      decode(P.Y, y0 + i, a, b);
      offAY[i] = a;
      offBY[i] = b;
    }
    __syncthreads();

    // A -> smem, A-contiguous walk (s fastest, then x, then y)
    constexpr int U = 8;
    for (uint32_t f0 = threadIdx.x; f0 < L; f0 += U * blockDim.x) {
      E v[U];
      int dst[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = f0 + u * blockDim.x;
        dst[u] = -1;
        if (f < L) {
          const uint32_t r = udiv(f, P.dS);
          const uint32_t s = f - r * P.S;
          const uint32_t y = udiv(r, P.dtx);
          const uint32_t x = r - y * P.tx;
          if (x < nx && y < ny) {
            vload_a(v[u], A + (offAX[x] + offAY[y] + s) * C);
            dst[u] = static_cast<int>(y * P.rl + x * P.S + s);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (dst[u] >= 0) tile[dst[u]] = v[u];
    }
    __syncthreads();

    // smem -> B, B-contiguous walk (s fastest, then y, then x)
    for (uint32_t f0 = threadIdx.x; f0 < L; f0 += U * blockDim.x) {
      Vec<SB, C> w[U];
      E a[U];
      SB* q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = f0 + u * blockDim.x;
        q[u] = nullptr;
        if (f < L) {
          const uint32_t r = udiv(f, P.dS);
          const uint32_t s = f - r * P.S;
          const uint32_t x = udiv(r, P.dty);
          const uint32_t y = r - x * P.ty;
          if (x < nx && y < ny) {
            q[u] = B + (offBX[x] + offBY[y] + s) * C;
            if constexpr (MODE == 2) vload_b(w[u], q[u]);
            a[u] = tile[y * P.rl + x * P.S + s];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!q[u]) continue;
#pragma unroll
        for (int c = 0; c < C; ++c) w[u].v[c] = up(a[u].v[c], w[u].v[c]);
        vstore(q[u], w[u]);
      }
    }
    __syncthreads();
  }
}

}  // namespace ttb
