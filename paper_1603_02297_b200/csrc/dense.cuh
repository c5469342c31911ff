// dense.cuh -- power-of-two fast path of the staged tile (S == 1, X group
// contiguous in A, Y group contiguous in B, tx, ty <= 256 powers of two with
// tx*ty = 256*EPT).  A thread's column (load walk) and row (store walk) are
// fixed for the whole kernel and its EPT elements per walk sit at constant
// strides: each element costs one table read, one address add and one
// predicated cp.async / store.  Two tile stages: the next tile's cp.async
// stream is in flight while the current tile is written out.  Measured the
// fastest variant for these shapes (see profiles/); everything else runs on
// tile_kernel (tile.cuh).
#pragma once

#include "kernels.cuh"

namespace ttb {

struct DenseTile {
  uint32_t x0, y0, nx, ny, o;
};

__device__ __forceinline__ DenseTile dense_tile(const SmemParams& P, uint32_t it) {
  DenseTile t;
  uint32_t xc, yc;
  if (P.order == 0) {
    const uint32_t q = udiv(it, P.dnx);
    xc = it - q * P.nxc;
    t.o = udiv(q, P.dny);
    yc = q - t.o * P.nyc;
  } else {
    const uint32_t q = udiv(it, P.dny);
    yc = it - q * P.nyc;
    t.o = udiv(q, P.dnx);
    xc = q - t.o * P.nxc;
  }
  t.x0 = xc * P.tx;
  t.y0 = yc * P.ty;
  t.nx = min(P.tx, P.X.total - t.x0);
  t.ny = min(P.ty, P.Y.total - t.y0);
  return t;
}

// Dense fast path of the staged tile (the common case after index merging):
// no shared stride-1 index, the X group is one contiguous run of A and the Y
// group one contiguous run of B.  Per tile the A offset of every row (y) and
// the B offset of every column (x) go to shared memory, so an element costs a
// split of its tile position and one warp-broadcast table read on either
// walk.  Two tile buffers: the cp.async loads of the next tile are in flight
// while the current tile is written out.
//
// EPT > 0: tx, ty <= 256 are powers of two and tx*ty = 256*EPT, so a thread's
// column (load walk) and row (store walk) are fixed for the whole kernel and
// its EPT elements per walk sit at constant strides: each element costs one
// table read, one address add and one predicated LDGSTS / STG.
// EPT == 0: any tile shape, positions split per element.
template <class SA, class SB, int C, int MODE, int EPT>
__global__ void __launch_bounds__(256, (MODE < 2 && C == 1 && sizeof(SA) == sizeof(SB))
                                           ? 1
                                           : 4) dense_kernel(const SmemParams P) {
  using E = Vec<SA, C>;
  constexpr int EB = static_cast<int>(sizeof(E));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // offsets are 32-bit: the planner only picks this kernel for tensors whose
  // footprints stay below 2^31 elements
  const uint32_t table_bytes = ((P.tx + P.ty) * 4 + 15) & ~15u;
  const uint32_t stage_bytes = table_bytes + ((P.ty * P.rl * EB + 15) & ~15u);
  auto rowA = [&](int s) { return reinterpret_cast<uint32_t*>(smem_raw + s * stage_bytes); };
  auto colB = [&](int s) { return rowA(s) + P.ty; };
  auto tile = [&](int s) { return reinterpret_cast<E*>(smem_raw + s * stage_bytes + table_bytes); };

  const Update<SA, SB, MODE> up(P.sc);
  const SA* __restrict__ A = static_cast<const SA*>(P.A);
  SB* __restrict__ B = static_cast<SB*>(P.B);
  const uint32_t L = P.tx * P.ty;

  auto tables = [&](const DenseTile& t, int s) {
    int64_t aO, bO;
    decode(P.O, t.o, aO, bO);
    uint32_t* ra = rowA(s);
    uint32_t* cb = colB(s);
    for (uint32_t i = threadIdx.x; i < t.ny; i += blockDim.x) {
      int64_t a, b;
      decode(P.Y, t.y0 + i, a, b);
      ra[i] = static_cast<uint32_t>(a + aO + t.x0);
    }
    for (uint32_t i = threadIdx.x; i < t.nx; i += blockDim.x) {
      int64_t a, b;
      decode(P.X, t.x0 + i, a, b);
      cb[i] = static_cast<uint32_t>(b + bO + t.y0);
    }
  };
  // A -> smem: A-contiguous walk (x fastest), all of it asynchronous
  auto loads = [&](const DenseTile& t, int s) {
    const uint32_t* ra = rowA(s);
    E* tl = tile(s);
    if constexpr (EPT > 0) {
      const uint32_t xt = threadIdx.x & (P.tx - 1), yt = threadIdx.x >> P.ltx;
      const uint32_t R = 256u >> P.ltx;
      const bool xv = xt < t.nx;
      const E* ax = reinterpret_cast<const E*>(A) + xt;
      E* tx0 = tl + yt * P.rl + xt;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const uint32_t y = yt + k * R;  // < ty: the table read is in bounds even when masked
        cp_async_pred<EB>(tx0 + k * R * P.rl, ax + ra[y], xv && y < t.ny);
      }
      return;
    }
    for (uint32_t f = threadIdx.x; f < L; f += blockDim.x) {
      uint32_t x, y;
      if (P.dense == 2) {
        x = f & (P.tx - 1);
        y = f >> P.ltx;
      } else {
        y = udiv(f, P.dtx);
        x = f - y * P.tx;
      }
      if (x < t.nx && y < t.ny) cp_async<EB>(tl + y * P.rl + x, A + (ra[y] + x) * C);
    }
  };

  uint32_t it = blockIdx.x;
  if (it >= P.items) return;
  DenseTile cur = dense_tile(P, it);
  tables(cur, 0);
  __syncthreads();
  loads(cur, 0);
  cp_async_commit();
  for (int s = 0; it < P.items; it += gridDim.x, s ^= 1) {
    const uint32_t nxt = it + gridDim.x;
    DenseTile nt{};
    if (nxt < P.items) {
      nt = dense_tile(P, nxt);
      tables(nt, s ^ 1);
    }
    __syncthreads();
    if (nxt < P.items) loads(nt, s ^ 1);
    cp_async_commit();
    cp_async_wait<1>();  // this thread's copies of the current tile have landed
    __syncthreads();     // ... and everyone else's

    // smem -> B: B-contiguous walk (y fastest)
    const uint32_t* cb = colB(s);
    const E* tl = tile(s);
    constexpr int U = 8;
    if constexpr (EPT > 0) {
      const uint32_t yt = threadIdx.x & (P.ty - 1), xt = threadIdx.x >> P.lty;
      const uint32_t Q = 256u >> P.lty;
      const bool yv = yt < cur.ny;
      using EBv = Vec<SB, C>;
      EBv* by = reinterpret_cast<EBv*>(B) + yt;
      const E* ty0 = tl + yt * P.rl + xt;
#pragma unroll
      for (int k0 = 0; k0 < EPT; k0 += U) {
        EBv w[U];
        E a[U];
        EBv* q[U];
        bool v[U];
#pragma unroll
        for (int u = 0; u < U && k0 + u < EPT; ++u) {
          const uint32_t x = xt + (k0 + u) * Q;  // < tx: table read in bounds when masked
          v[u] = yv && x < cur.nx;
          q[u] = by + cb[x];
          if constexpr (MODE == 2) vload_b_pred(w[u], q[u]->v, v[u]);
          a[u] = ty0[(k0 + u) * Q];
        }
#pragma unroll
        for (int u = 0; u < U && k0 + u < EPT; ++u) {
#pragma unroll
          for (int c = 0; c < C; ++c) w[u].v[c] = up(a[u].v[c], w[u].v[c]);
          vstore_pred(q[u]->v, w[u], v[u]);
        }
      }
      __syncthreads();
      cur = nt;
      continue;
    }
    for (uint32_t f0 = threadIdx.x; f0 < L; f0 += U * blockDim.x) {
      Vec<SB, C> w[U];
      E a[U];
      SB* q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = f0 + u * blockDim.x;
        uint32_t x, y;
        if (P.dense == 2) {
          y = f & (P.ty - 1);
          x = f >> P.lty;
        } else {
          x = udiv(f, P.dty);
          y = f - x * P.ty;
        }
        q[u] = nullptr;
        if (f < L && x < cur.nx && y < cur.ny) {
          q[u] = B + (cb[x] + y) * C;
          if constexpr (MODE == 2) vload_b(w[u], q[u]);
          a[u] = tl[y * P.rl + x];
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
    cur = nt;
  }
}


}  // namespace ttb
