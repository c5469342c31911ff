// tile.cuh -- the staged-tile transpose (ttune's run_case2 / run_case1 for
// shapes whose stride-1 runs are short or unaligned, executor.cpp:172-281).
//
// Tile = S x TX x TY elements: S the shared stride-1 extent (1 unless A's and
// B's stride-1 index coincide), TX a chunk of the X group (A axes after it,
// contiguous-ish in A), TY a chunk of the Y group (B positions after it).
// A is read along (s, x) rows, B written along (s, y) columns, so both HBM
// streams are warp-contiguous; shared memory does the transposition.
//
// Every thread owns a fixed position in a tile row (load walk) and in a tile
// column (store walk), worked out once per kernel; per tile it reads one
// offset from a small per-tile table, and per element it adds one
// warp-broadcast table entry and issues one predicated cp.async (load) or
// one predicated store.  The next tile's cp.async stream is in flight while
// the current tile is written out (two stages).
#pragma once

#include "kernels.cuh"

namespace ttb {

struct TileBox {
  uint32_t x0, y0, nx, ny, o;
};

// tile index -> (X chunk, Y chunk, outer index) in the plan's tile order:
// 0 X chunks fastest, 1 Y chunks fastest, >= 2 groups of P.grp Y chunks
// (Y fastest inside a group, then X, then the next group)
__device__ __forceinline__ void smem_tile_coords(const SmemParams& P, uint32_t it, uint32_t& xc,
                                                 uint32_t& yc, uint32_t& o) {
  if (P.order == 0) {
    const uint32_t q = udiv(it, P.dnx);
    xc = it - q * P.nxc;
    o = udiv(q, P.dny);
    yc = q - o * P.nyc;
  } else if (P.order == 1) {
    const uint32_t q = udiv(it, P.dny);
    yc = it - q * P.nyc;
    o = udiv(q, P.dnx);
    xc = q - o * P.nxc;
  } else {
    o = udiv(it, P.dplane);
    const uint32_t r = it - o * (P.nxc * P.nyc);
    const uint32_t g = udiv(r, P.dgrp);
    const uint32_t rr = r - g * (P.grp * P.nxc);
    const uint32_t y0 = g * P.grp;
    const uint32_t gh = min(P.grp, P.nyc - y0);
    const uint32_t q = gh == P.grp ? udiv(rr, P.dG) : rr / gh;
    xc = q;
    yc = y0 + (rr - q * gh);
  }
}

__device__ __forceinline__ TileBox tile_box(const SmemParams& P, uint32_t it) {
  TileBox t;
  uint32_t xc, yc;
  smem_tile_coords(P, it, xc, yc, t.o);
  t.x0 = xc * P.tx;
  t.y0 = yc * P.ty;
  t.nx = min(P.tx, P.X.total - t.x0);
  t.ny = min(P.ty, P.Y.total - t.y0);
  return t;
}

// KK > 0: both walks have exactly KK steps covering the tile (S*tx and S*ty
// divide 256 and tx*ty*S = 256*KK), so the loops unroll completely and need
// neither a step bound nor a table clamp.  KK == 0: any shape.
template <class SA, class SB, int C, int MODE, int KK>
__global__ void __launch_bounds__(256, 1) tile_kernel(const SmemParams P) {
  using EA = Vec<SA, C>;
  using EBv = Vec<SB, C>;
  constexpr int EAB = static_cast<int>(sizeof(EA));
  constexpr int EBB = static_cast<int>(sizeof(EBv));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // per stage: offAX[tx] offBX[tx] offAY[ty] offBY[ty] (uint32), the A tile,
  // and with beta != 0 the tile's B elements ([x][s, y], prefetched by cp.async)
  const uint32_t table_bytes = ((P.tx + P.ty) * 8 + 15) & ~15u;
  const uint32_t tile_a_bytes = (P.ty * P.rl * EAB + 15) & ~15u;
  const uint32_t stage_bytes =
      table_bytes + tile_a_bytes + (MODE == 2 ? ((P.S * P.tx * P.ty * EBB + 15) & ~15u) : 0u);
  auto tab = [&](int s) { return reinterpret_cast<uint32_t*>(smem_raw + s * stage_bytes); };
  auto tile = [&](int s) { return reinterpret_cast<EA*>(smem_raw + s * stage_bytes + table_bytes); };
  auto tileB = [&](int s) {
    return reinterpret_cast<EBv*>(smem_raw + s * stage_bytes + table_bytes + tile_a_bytes);
  };

  const Update<SA, SB, MODE> up(P.sc);
  const EA* __restrict__ A = static_cast<const EA*>(P.A);
  EBv* __restrict__ B = static_cast<EBv*>(P.B);
  const uint32_t tid = threadIdx.x;

  // fixed per-thread positions (one division each, once per kernel)
  const uint32_t LR = P.S * P.tx, LC = P.S * P.ty;
  const uint32_t R = 256u / LR, Q = 256u / LC;  // rows / columns per step
  const bool act_l = tid < R * LR, act_s = tid < Q * LC;
  const uint32_t i_l = tid % LR, r0 = tid / LR;
  const uint32_t s_l = i_l % P.S, x_l = i_l / P.S;
  const uint32_t j_s = tid % LC, c0 = tid / LC;
  const uint32_t s_s = j_s % P.S, y_s = j_s / P.S;
  const uint32_t K1 = KK > 0 ? KK : (P.ty + R - 1) / R;
  const uint32_t K2 = KK > 0 ? KK : (P.tx + Q - 1) / Q;
  constexpr uint32_t UN = KK > 0 ? KK : 4;  // unroll of the walks

  auto tables = [&](const TileBox& t, int s) {
    int64_t aO, bO;
    decode(P.O, t.o, aO, bO);
    uint32_t* T = tab(s);
    for (uint32_t i = tid; i < t.nx; i += 256) {
      int64_t a, b;
      decode(P.X, t.x0 + i, a, b);
      T[i] = static_cast<uint32_t>(a + aO);
      T[P.tx + i] = static_cast<uint32_t>(b + bO);
    }
    for (uint32_t i = tid; i < t.ny; i += 256) {
      int64_t a, b;
      decode(P.Y, t.y0 + i, a, b);
      T[2 * P.tx + i] = static_cast<uint32_t>(a);
      T[2 * P.tx + P.ty + i] = static_cast<uint32_t>(b);
    }
  };
  // A -> smem along (s, x) rows
  auto loads = [&](const TileBox& t, int s) {
    const uint32_t* T = tab(s);
    const bool vx = act_l && x_l < t.nx;
    const EA* a0 = A + (vx ? T[x_l] : 0u) + s_l;
    const uint32_t* offAY = T + 2 * P.tx;
    EA* dst = tile(s) + r0 * P.rl + i_l;
    for (uint32_t k0 = 0; k0 < K1; k0 += UN) {
#pragma unroll
      for (uint32_t u = 0; u < UN; ++u) {
        const uint32_t k = k0 + u;
        const uint32_t y = r0 + k * R;
        const bool v = vx && (KK > 0 || k < K1) && y < t.ny;
        cp_async_pred<EAB>(dst + k * R * P.rl, a0 + offAY[KK > 0 ? y : min(y, P.ty - 1)], v);
      }
    }
    if constexpr (MODE == 2) {  // B elements of the tile, in the store walk's layout
      const bool vy = act_s && y_s < t.ny;
      const EBv* b0 = B + (vy ? T[2 * P.tx + P.ty + y_s] : 0u) + s_s;
      const uint32_t* offBX = T + P.tx;
      EBv* bdst = tileB(s) + j_s;
      for (uint32_t k0 = 0; k0 < K2; k0 += UN) {
#pragma unroll
        for (uint32_t u = 0; u < UN; ++u) {
          const uint32_t k = k0 + u;
          const uint32_t x = c0 + k * Q;
          const uint32_t xc = KK > 0 ? x : min(x, P.tx - 1);
          cp_async_pred<EBB>(bdst + xc * LC, b0 + offBX[xc], vy && (KK > 0 || k < K2) && x < t.nx);
        }
      }
    }
  };

  uint32_t it = blockIdx.x;
  if (it >= P.items) return;
  TileBox cur = tile_box(P, it);
  tables(cur, 0);
  __syncthreads();
  loads(cur, 0);
  cp_async_commit();
  for (int s = 0; it < P.items; it += gridDim.x, s ^= 1) {
    const uint32_t nxt = it + gridDim.x;
    TileBox nt{};
    if (nxt < P.items) {
      nt = tile_box(P, nxt);
      tables(nt, s ^ 1);
    }
    __syncthreads();
    if (nxt < P.items) loads(nt, s ^ 1);
    cp_async_commit();
    cp_async_wait<1>();  // this thread's copies of the current tile have landed
    __syncthreads();     // ... and everybody's

    // smem -> B along (s, y) columns
    {
      const uint32_t* T = tab(s);
      const bool vy = act_s && y_s < cur.ny;
      EBv* b0 = B + (vy ? T[2 * P.tx + P.ty + y_s] : 0u) + s_s;
      const uint32_t* offBX = T + P.tx;
      const EA* src = tile(s) + y_s * P.rl + s_s;
      const EBv* bsrc = tileB(s) + j_s;
      constexpr uint32_t U2 = UN > 8 ? 8 : UN;  // stores per batch
      for (uint32_t k0 = 0; k0 < K2; k0 += U2) {
        EBv w[U2];
        EA a[U2];
        EBv* q[U2];
        bool v[U2];
#pragma unroll
        for (uint32_t u = 0; u < U2; ++u) {
          const uint32_t k = k0 + u;
          const uint32_t x = c0 + k * Q;
          const uint32_t xc = KK > 0 ? x : min(x, P.tx - 1);
          v[u] = vy && (KK > 0 || k < K2) && x < cur.nx;
          q[u] = b0 + offBX[xc];
          if constexpr (MODE == 2) w[u] = bsrc[xc * LC];               // prefetched
          if constexpr (MODE == 3) vload_b_pred(w[u], q[u]->v, v[u]);  // direct (no B ring)
          a[u] = src[xc * P.S];
        }
#pragma unroll
        for (uint32_t u = 0; u < U2; ++u) {
#pragma unroll
          for (int c = 0; c < C; ++c) w[u].v[c] = up(a[u].v[c], w[u].v[c]);
          vstore_pred(q[u]->v, w[u], v[u]);
        }
      }
    }
    __syncthreads();
    cur = nt;
  }
}

}  // namespace ttb
