// dense.cuh -- power-of-two fast path of the staged tile (S == 1, X group
// contiguous in A, Y group contiguous in B, tx, ty <= 256 powers of two with
// tx*ty = 256*EPT).  A thread's column (load walk) and row (store walk) are
// fixed for the whole kernel and its EPT elements per walk sit at constant
// strides: each element costs one table read, one address add and one
// predicated cp.async (load) or store.  NS tile stages form a cp.async ring:
// the loads of the next NS-1 tiles are in flight while the current tile is
// written out, which is what keeps enough bytes in flight per SM (Little's
// law) at the low occupancy these unrolled walks allow.  With beta != 0 the
// tile's B elements ride the same ring (second smem buffer), so the
// read-modify-write of B never waits on HBM latency.  Everything that is not
// a power-of-two dense tile runs on tile_kernel (tile.cuh).
#pragma once

#include "kernels.cuh"

namespace ttb {

struct DenseTile {
  uint32_t x0, y0, nx, ny, o;
};

__device__ __forceinline__ DenseTile dense_tile(const SmemParams& P, uint32_t it) {
  DenseTile t;
  uint32_t xc, yc;
  smem_tile_coords(P, it, xc, yc, t.o);
  t.x0 = xc * P.tx;
  t.y0 = yc * P.ty;
  t.nx = min(P.tx, P.X.total - t.x0);
  t.ny = min(P.ty, P.Y.total - t.y0);
  return t;
}

// bytes of one pipeline stage; must match plan.cpp's shared-memory size
__host__ __device__ inline uint32_t dense_stage_bytes(uint32_t tx, uint32_t ty, uint32_t rl,
                                                      uint32_t ea, uint32_t eb, int mode) {
  const uint32_t tables = ((tx + ty) * 4 + 15) & ~15u;
  const uint32_t tile_a = (ty * rl * ea + 15) & ~15u;
  const uint32_t tile_b = mode == 2 ? ((tx * ty * eb + 15) & ~15u) : 0u;
  return tables + tile_a + tile_b;
}

template <class SA, class SB, int C, int MODE, int EPT, int NS>
__global__ void __launch_bounds__(256, (MODE < 2 && C == 1 && sizeof(SA) == sizeof(SB))
                                           ? 1
                                           : 4) dense_kernel(const SmemParams P) {
  static_assert(EPT > 0 && NS >= 2, "dense tile");
  using E = Vec<SA, C>;
  using EBv = Vec<SB, C>;
  constexpr int EB = static_cast<int>(sizeof(E));
  constexpr int EBB = static_cast<int>(sizeof(EBv));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // offsets are 32-bit: the planner only picks this kernel for tensors whose
  // footprints stay below 2^31 elements
  const uint32_t table_bytes = ((P.tx + P.ty) * 4 + 15) & ~15u;
  const uint32_t tile_a_bytes = (P.ty * P.rl * EB + 15) & ~15u;
  const uint32_t stage_bytes = dense_stage_bytes(P.tx, P.ty, P.rl, EB, EBB, MODE);
  auto rowA = [&](int s) { return reinterpret_cast<uint32_t*>(smem_raw + s * stage_bytes); };
  auto colB = [&](int s) { return rowA(s) + P.ty; };
  auto tile = [&](int s) { return reinterpret_cast<E*>(smem_raw + s * stage_bytes + table_bytes); };
  auto tileB = [&](int s) {  // [x][y], column-major like B
    return reinterpret_cast<EBv*>(smem_raw + s * stage_bytes + table_bytes + tile_a_bytes);
  };

  const Update<SA, SB, MODE> up(P.sc);
  const E* __restrict__ A = static_cast<const E*>(P.A);
  EBv* __restrict__ B = static_cast<EBv*>(P.B);

  // per tile: A offset of every row y, B offset of every column x
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
  // load walk: thread column xl, rows yl + k*R (A-contiguous along x)
  const uint32_t xl = threadIdx.x & (P.tx - 1), yl = threadIdx.x >> P.ltx;
  const uint32_t R = 256u >> P.ltx;
  // store walk: thread row yt, columns xt + k*Q (B-contiguous along y)
  const uint32_t yt = threadIdx.x & (P.ty - 1), xt = threadIdx.x >> P.lty;
  const uint32_t Q = 256u >> P.lty;
  auto loads = [&](const DenseTile& t, int s) {
    const uint32_t* ra = rowA(s);
    const bool xv = xl < t.nx;
    const E* ax = A + xl;
    E* dst = tile(s) + yl * P.rl + xl;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint32_t y = yl + k * R;  // < ty: the table read is in bounds even when masked
      cp_async_pred<EB>(dst + k * R * P.rl, ax + ra[y], xv && y < t.ny);
    }
    if constexpr (MODE == 2) {  // the tile's B elements, in the store walk's layout
      const uint32_t* cb = colB(s);
      const bool yv = yt < t.ny;
      EBv* bdst = tileB(s) + yt;
      const EBv* by = B + yt;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const uint32_t x = xt + k * Q;
        cp_async_pred<EBB>(bdst + x * P.ty, by + cb[x], yv && x < t.nx);
      }
    }
  };

  const uint32_t g = gridDim.x;
  uint32_t it = blockIdx.x;
  if (it >= P.items) return;
  // prologue: tables and loads of the first NS-1 tiles
#pragma unroll
  for (int p = 0; p < NS - 1; ++p)
    if (it + p * g < P.items) tables(dense_tile(P, it + p * g), p);
  __syncthreads();
#pragma unroll
  for (int p = 0; p < NS - 1; ++p) {
    if (it + p * g < P.items) loads(dense_tile(P, it + p * g), p);
    cp_async_commit();
  }

  for (int s = 0; it < P.items; it += g, s = (s + 1 == NS) ? 0 : s + 1) {
    const uint32_t nxt = it + (NS - 1) * g;
    const int sn = (s + NS - 1) % NS;  // the stage tile it - g used
    if (nxt < P.items) tables(dense_tile(P, nxt), sn);
    __syncthreads();
    if (nxt < P.items) loads(dense_tile(P, nxt), sn);
    cp_async_commit();
    cp_async_wait<NS - 1>();  // this thread's copies of tile `it` have landed
    __syncthreads();          // ... and everybody's

    // smem -> B: B-contiguous walk (y fastest)
    const DenseTile cur = dense_tile(P, it);
    const uint32_t* cb = colB(s);
    const bool yv = yt < cur.ny;
    EBv* by = B + yt;
    const E* src = tile(s) + yt * P.rl + xt;
    const EBv* bsrc = tileB(s) + yt;
    constexpr int U = EPT < 8 ? EPT : 8;
#pragma unroll
    for (int k0 = 0; k0 < EPT; k0 += U) {
      EBv w[U];
      E a[U];
      EBv* q[U];
      bool v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t x = xt + (k0 + u) * Q;  // < tx: table read in bounds when masked
        v[u] = yv && x < cur.nx;
        q[u] = by + cb[x];
        if constexpr (MODE == 2) w[u] = bsrc[x * P.ty];             // prefetched
        if constexpr (MODE == 3) vload_b_pred(w[u], q[u]->v, v[u]);  // direct (no B ring)
        a[u] = src[(k0 + u) * Q];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int c = 0; c < C; ++c) w[u].v[c] = up(a[u].v[c], w[u].v[c]);
        vstore_pred(q[u]->v, w[u], v[u]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

}  // namespace ttb
