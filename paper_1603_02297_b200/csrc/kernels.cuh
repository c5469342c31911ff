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
// 2 = update (SB(alpha*W(a) + beta*W(b)), two products, one sum);
// 3 = update as well -- the staged-tile kernels use it for "read B directly
// instead of through the cp.async ring".
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

// N elements moved as one aligned unit (16 or 32 bytes: LDS/STS/STG.128)
template <class T, int N>
struct alignas(16) Piece {
  T e[N];
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

// Row r (tile-ordered linear row index) -> element offsets of the row start
// in A and in B; false for the masked rows of partial tiles.
__device__ __forceinline__ bool copy_row(const CopyParams& P, uint32_t r, int64_t& oa,
                                         int64_t& ob) {
  const uint32_t rit = r & ((1u << (P.ltx + P.lty)) - 1);
  const uint32_t tile = r >> (P.ltx + P.lty);
  uint32_t xc, yc, o;
  if (P.order == 0) {
    const uint32_t t = udiv(tile, P.dnx);
    xc = tile - t * P.nxc;
    o = udiv(t, P.dny);
    yc = t - o * P.nyc;
  } else {
    const uint32_t t = udiv(tile, P.dny);
    yc = tile - t * P.nyc;
    o = udiv(t, P.dnx);
    xc = t - o * P.nxc;
  }
  const uint32_t x = xc * P.tx + (rit & (P.tx - 1));
  const uint32_t y = yc * P.ty + (rit >> P.ltx);
  if (x >= P.X.total || y >= P.Y.total) return false;
  int64_t a1, b1, a2, b2;
  decode(P.O, o, oa, ob);
  decode(P.X, x, a1, b1);
  decode(P.Y, y, a2, b2);
  oa += a1 + a2;
  ob += b1 + b2;
  return true;
}

// Shared stride-1 index, short rows: a warp owns 32 consecutive rows (in tile
// order).  Lane l decodes row l's offsets once; the warp then streams the
// 32 * lvec vectors of those rows with consecutive lanes on consecutive
// vectors, fetching each vector's row offsets by warp shuffle -- no per-vector
// index decode.  U vectors per lane in flight.
template <class SA, class SB, int C, int V, int MODE>
__global__ void __launch_bounds__(256) copy_kernel(const CopyParams P) {
  const Update<SA, SB, MODE> up(P.sc);
  const SA* __restrict__ A = static_cast<const SA*>(P.A);
  SB* __restrict__ B = static_cast<SB*>(P.B);
  constexpr int U = 4;  // vectors per lane in flight
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < P.items; it += nwarps) {
    const uint32_t r = it * 32 + lane;
    int64_t roa = 0, rob = 0;
    const bool rok = r < P.rows && copy_row(P, r, roa, rob);
    for (uint32_t k0 = 0; k0 < P.lvec; k0 += U) {
      Vec<SA, V * C> a[U];
      Vec<SB, V * C> b[U];
      SB* pb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = (k0 + u) * 32 + lane;  // vector index within the 32 rows
        const uint32_t rl = udiv(f, P.dl);          // row within the group (< 32 when valid)
        const uint32_t v = f - rl * P.lvec;
        const uint32_t src = rl & 31;
        const int64_t oa = __shfl_sync(0xffffffffu, roa, src);
        const int64_t ob = __shfl_sync(0xffffffffu, rob, src);
        const bool ok = __shfl_sync(0xffffffffu, rok, src) && k0 + u < P.lvec;
        pb[u] = nullptr;
        if (ok) {
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
}

// Shared stride-1 index, long rows: a warp streams one segment of 32*U
// vectors of a row per item (row offsets decoded once per item).
// Resident CTAs per SM: 4 without B loads (more warps hide the load latency),
// 2 with them (twice the registers in flight; 4 would spill).
template <class SA, class SB, int C, int V, int MODE>
__global__ void __launch_bounds__(256, MODE == 2 ? 2 : 4) copy_rows_kernel(const CopyParams P) {
  const Update<SA, SB, MODE> up(P.sc);
  const SA* __restrict__ A = static_cast<const SA*>(P.A);
  SB* __restrict__ B = static_cast<SB*>(P.B);
  // an item is 4 KB of the row per warp: IT vectors per lane (rows_item_vectors),
  // all of them in flight at once (x2 loads with beta)
  constexpr int IT = rows_item_vectors(V * C * static_cast<int>(sizeof(SA) > sizeof(SB) ? sizeof(SA) : sizeof(SB)));
  constexpr int U = IT;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < P.items; it += nwarps) {
    const uint32_t row = udiv(it, P.dseg);
    const uint32_t seg = it - row * P.nseg;
    int64_t oa, ob;
    if (!copy_row(P, row, oa, ob)) continue;
    // segments start on 128-byte lines of the aligned side (P.align: 1 B, 2 A):
    // the row's first segment is shortened by the row start's offset in its line
    uint32_t sh = 0;
    if (P.align) {
      const uint64_t addr = P.align == 1 ? reinterpret_cast<uint64_t>(B + ob * C)
                                         : reinterpret_cast<uint64_t>(A + oa * C);
      const uint32_t vb = static_cast<uint32_t>((P.align == 1 ? sizeof(SB) : sizeof(SA)) * V * C);
      sh = static_cast<uint32_t>((addr & 127u) / vb);
    }
#pragma unroll 1
    for (int c = 0; c < IT / U; ++c) {
      const uint32_t v0 = (seg * IT + c * U) * 32 + lane - sh;  // wraps below 0: masked by v < lvec
      Vec<SA, V * C> a[U];
      Vec<SB, V * C> b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = v0 + u * 32;
        if (v < P.lvec) {
          vload_a(a[u], A + (oa + static_cast<int64_t>(v) * V) * C);
          if constexpr (MODE == 2)
            vload_b(b[u], B + (ob + static_cast<int64_t>(v) * V) * C);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = v0 + u * 32;
        if (v < P.lvec) {
#pragma unroll
          for (int i = 0; i < V * C; ++i) b[u].v[i] = up(a[u].v[i], b[u].v[i]);
          vstore(B + (ob + static_cast<int64_t>(v) * V) * C, b[u]);
        }
      }
    }
  }
}

// In-register micro-tile transpose.  A warp covers (lx*MX) x ((32/lx)*MY)
// elements of the X-by-Y plane per item: lane (i, j) loads MY vectors of MX
// elements (rows y..y+MY-1, contiguous in A), transposes them in registers
// and stores MX vectors of MY elements (columns x..x+MX-1, contiguous in B).
// The paper's w x w micro-kernel (executor.hpp:101-128) mapped to one thread.
// Software-pipelined: the loads of a warp's next item are in flight while the
// current item is transposed and stored, so HBM sees a continuous stream.
template <class SA, class SB, int C, int MX, int MY, int MODE>
struct RtItem {
  const SA* pa;
  SB* pb;
  bool valid;
  Vec<SA, MX * C> r[MY];   // MY rows of MX elements (A side)
  Vec<SB, MY * C> w[MX];   // MX columns of MY elements (B side; loaded when beta != 0)
};

template <class SA, class SB, int C, int MX, int MY, int MODE>
__device__ __forceinline__ void rt_fetch(const RtParams& P, uint32_t it, uint32_t li, uint32_t lj,
                                         RtItem<SA, SB, C, MX, MY, MODE>& I) {
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
  I.valid = x < P.X.total && y < P.Y.total;
  if (!I.valid) return;
  int64_t aO, bO, aX, bX, aY, bY;
  decode(P.O, o, aO, bO);
  decode(P.X, x, aX, bX);
  decode(P.Y, y, aY, bY);
  I.pa = static_cast<const SA*>(P.A) + (aO + aX + aY) * C;
  I.pb = static_cast<SB*>(P.B) + (bO + bX + bY) * C;
#pragma unroll
  for (int k = 0; k < MY; ++k) vload_a(I.r[k], I.pa + k * P.sa_y0 * C);
  if constexpr (MODE == 2) {
#pragma unroll
    for (int j = 0; j < MX; ++j) vload_b(I.w[j], I.pb + j * P.sb_x0 * C);
  }
}

template <class SA, class SB, int C, int MX, int MY, int MODE>
__device__ __forceinline__ void rt_commit(const RtParams& P, const Update<SA, SB, MODE>& up,
                                          RtItem<SA, SB, C, MX, MY, MODE>& I) {
  if (!I.valid) return;
#pragma unroll
  for (int j = 0; j < MX; ++j) {
#pragma unroll
    for (int k = 0; k < MY; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c) I.w[j].v[k * C + c] = up(I.r[k].v[j * C + c], I.w[j].v[k * C + c]);
    vstore(I.pb + j * P.sb_x0 * C, I.w[j]);
  }
}

template <class SA, class SB, int C, int MX, int MY, int MODE>
__global__ void __launch_bounds__(256, 4) rt_kernel(const RtParams P) {
  using Item = RtItem<SA, SB, C, MX, MY, MODE>;
  const Update<SA, SB, MODE> up(P.sc);
  const int lane = threadIdx.x & 31;
  const uint32_t li = static_cast<uint32_t>(lane & (P.lx - 1));
  const uint32_t lj = static_cast<uint32_t>(lane >> P.lx_log2);
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (it >= P.items) return;
  Item a, b;
  rt_fetch(P, it, li, lj, a);
  // ping-pong between two register sets: fetch(next) overlaps commit(current)
  for (;;) {
    it += nwarps;
    if (it >= P.items) {
      rt_commit(P, up, a);
      return;
    }
    rt_fetch(P, it, li, lj, b);
    rt_commit(P, up, a);
    it += nwarps;
    if (it >= P.items) {
      rt_commit(P, up, b);
      return;
    }
    rt_fetch(P, it, li, lj, a);
    rt_commit(P, up, b);
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

namespace ttb {

// asynchronous global -> shared copy of one element (LDGSTS): no register
// staging, so a thread can keep its whole share of a tile in flight
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gsrc) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gsrc), "n"(BYTES)
                 : "memory");
}
// predicated forms: nothing is touched when pred == 0 (masked tile edges)
template <int BYTES>
__device__ __forceinline__ void cp_async_pred(void* smem_dst, const void* gsrc, bool pred) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  if constexpr (BYTES == 16)
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %2, 0; @p cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(s),
        "l"(gsrc), "r"(static_cast<int>(pred))
        : "memory");
  else
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %2, 0; @p cp.async.ca.shared.global [%0], [%1], %3; }" ::"r"(s),
        "l"(gsrc), "r"(static_cast<int>(pred)), "n"(BYTES)
        : "memory");
}

template <class T, int N>
__device__ __forceinline__ void vstore_pred(T* p, const Vec<T, N>& v, bool pred) {
  constexpr int BYTES = sizeof(T) * N;
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "element store");
  const int pr = static_cast<int>(pred);
  if constexpr (BYTES == 16) {
    const uint4 r = *reinterpret_cast<const uint4*>(v.v);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %5, 0; @p st.global.v4.u32 [%0], {%1,%2,%3,%4}; }" ::"l"(p),
                 "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(pr)
                 : "memory");
  } else if constexpr (BYTES == 8) {
    const uint2 r = *reinterpret_cast<const uint2*>(v.v);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %3, 0; @p st.global.v2.u32 [%0], {%1,%2}; }" ::"l"(p),
                 "r"(r.x), "r"(r.y), "r"(pr)
                 : "memory");
  } else {
    const uint32_t r = *reinterpret_cast<const uint32_t*>(v.v);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p st.global.u32 [%0], %1; }" ::"l"(p), "r"(r),
                 "r"(pr)
                 : "memory");
  }
}

template <class T, int N>
__device__ __forceinline__ void vload_b_pred(Vec<T, N>& v, const T* p, bool pred) {
  constexpr int BYTES = sizeof(T) * N;
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "element load");
  const int pr = static_cast<int>(pred);
  if constexpr (BYTES == 16) {
    uint4 r = make_uint4(0, 0, 0, 0);
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %5, 0; @p ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4]; }"
        : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
        : "l"(p), "r"(pr));
    *reinterpret_cast<uint4*>(v.v) = r;
  } else if constexpr (BYTES == 8) {
    uint2 r = make_uint2(0, 0);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %3, 0; @p ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2]; }"
                 : "+r"(r.x), "+r"(r.y)
                 : "l"(p), "r"(pr));
    *reinterpret_cast<uint2*>(v.v) = r;
  } else {
    uint32_t r = 0;
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p ld.global.L1::no_allocate.u32 %0, [%1]; }"
                 : "+r"(r)
                 : "l"(p), "r"(pr));
    *reinterpret_cast<uint32_t*>(v.v) = r;
  }
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace ttb

#include "tile.cuh"
#include "dense.cuh"
