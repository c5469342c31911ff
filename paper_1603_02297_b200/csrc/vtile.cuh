// vtile.cuh -- the staged tile with vector memory accesses on both HBM sides.
//
// Same tile as dense_kernel / tile_kernel (S == 1, X group contiguous in A,
// Y group contiguous in B, any tx x ty), for the shapes where every tile row
// of A starts on a VA-element boundary and every tile column of B on a
// VB-element boundary (the planner checks the strides, plan.cpp).  A rows are
// fetched as VA-element cp.async chunks (16 bytes for fp32 x4 / fp64 x2), B
// columns written as VB-element vector stores, so a warp instruction moves
// 4x (fp32) the bytes of the element-wise kernels -- those were issue-bound
// (~1 warp instruction per element) on the generic tile shapes.  Ragged tile
// edges: the last chunk of a row is a zero-filling partial cp.async (only the
// valid source bytes are read), the last vector of a column is written
// element by element.
#pragma once

#include "kernels.cuh"

namespace ttb {

// cp.async of the first `src_bytes` (1..BYTES) bytes of a BYTES chunk, the rest
// of the shared-memory chunk zero-filled; nothing happens when pred == 0
template <int BYTES>
__device__ __forceinline__ void cp_async_part(void* smem_dst, const void* gsrc, uint32_t src_bytes,
                                              bool pred) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  if constexpr (BYTES == 16)
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %3, 0; @p cp.async.cg.shared.global [%0], [%1], 16, %2; }" ::"r"(s),
        "l"(gsrc), "r"(src_bytes), "r"(static_cast<int>(pred))
        : "memory");
  else
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %3, 0; @p cp.async.ca.shared.global [%0], [%1], %4, %2; }" ::"r"(s),
        "l"(gsrc), "r"(src_bytes), "r"(static_cast<int>(pred)), "n"(BYTES)
        : "memory");
}

// bytes of one pipeline stage; must match plan.cpp's shared-memory size
__host__ __device__ inline uint32_t vtile_stage_bytes(uint32_t tx, uint32_t ty, uint32_t rl,
                                                      uint32_t ea, uint32_t eb, int mode,
                                                      uint32_t vb, int shb) {
  const uint32_t tables = ((tx + ty) * 4 + 15) & ~15u;
  const uint32_t tile_a = (ty * rl * ea + 15) & ~15u;
  const uint32_t tile_b = mode == 2 ? ((tx * (ty + (shb ? vb : 0u)) * eb + 15) & ~15u) : 0u;
  return tables + tile_a + tile_b;
}

// SH bit 0 (SHA): A tile rows may start anywhere -- each row is fetched as the
// aligned VA-chunks that cover it and lands in shared memory shifted by its
// misalignment d(y) = row offset mod VA (read back at y*rl + d(y) + x).
// SH bit 1 (SHB): B tile columns may start anywhere -- the store walk writes
// the aligned VB-vectors that cover a column (full vectors as one store, the
// two ragged ends element by element) and picks each vector's elements out
// of the tile at the column's own shift.  Chunks that straddle a row / column
// end are read whole (same 16-byte block, so never a fault) but only the
// valid elements are ever written.  Requires 16-byte aligned A and B.
template <class SA, class SB, int C, int MODE, int VA, int VB, int SH>
__global__ void __launch_bounds__(256, 2) vtile_kernel(const SmemParams P) {
  using E = Vec<SA, C>;
  using EBv = Vec<SB, C>;
  using VBv = Vec<SB, C * VB>;
  constexpr int EAB = static_cast<int>(sizeof(E));
  constexpr int EBB = static_cast<int>(sizeof(EBv));
  constexpr int NS = 2;
  constexpr bool SHA = (SH & 1) != 0, SHB = (SH & 2) != 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // stage: A offset per tile row, B offset per tile column (uint32), the A tile
  // [ty][rl], and with beta != 0 the tile's B elements [tx][bpitch]
  const uint32_t bpitch = P.ty + (SHB ? VB : 0);
  const uint32_t table_bytes = ((P.tx + P.ty) * 4 + 15) & ~15u;
  const uint32_t tile_a_bytes = (P.ty * P.rl * EAB + 15) & ~15u;
  const uint32_t stage_bytes = vtile_stage_bytes(P.tx, P.ty, P.rl, EAB, EBB, MODE, VB, SHB);
  auto rowA = [&](int s) { return reinterpret_cast<uint32_t*>(smem_raw + s * stage_bytes); };
  auto colB = [&](int s) { return rowA(s) + P.ty; };
  auto tile = [&](int s) { return reinterpret_cast<E*>(smem_raw + s * stage_bytes + table_bytes); };
  auto tileB = [&](int s) {
    return reinterpret_cast<EBv*>(smem_raw + s * stage_bytes + table_bytes + tile_a_bytes);
  };

  const Update<SA, SB, MODE> up(P.sc);
  const E* __restrict__ A = static_cast<const E*>(P.A);
  EBv* __restrict__ B = static_cast<EBv*>(P.B);
  const uint32_t tid = threadIdx.x;

  // load walk: LRv chunks per tile row, R rows per step; store walk: LCv
  // vectors per tile column, Q columns per step (one division each, once);
  // a shifted side needs one chunk / vector more per row / column
  const uint32_t LRv = P.tx / VA + (SHA ? 1 : 0), LCv = P.ty / VB + (SHB ? 1 : 0);
  const uint32_t R = 256u / LRv, Q = 256u / LCv;
  const uint32_t r0 = tid / LRv, xl = (tid - r0 * LRv) * VA;
  const uint32_t c0 = tid / LCv, yl = (tid - c0 * LCv) * VB;
  const bool act_l = r0 < R, act_s = c0 < Q;
  const uint32_t K1 = (P.ty + R - 1) / R, K2 = (P.tx + Q - 1) / Q;

  auto tables = [&](const DenseTile& t, int s) {
    int64_t aO, bO;
    decode(P.O, t.o, aO, bO);
    uint32_t* ra = rowA(s);
    uint32_t* cb = colB(s);
    for (uint32_t i = tid; i < t.ny; i += 256) {
      int64_t a, b;
      decode(P.Y, t.y0 + i, a, b);
      ra[i] = static_cast<uint32_t>(a + aO + t.x0);
    }
    for (uint32_t i = tid; i < t.nx; i += 256) {
      int64_t a, b;
      decode(P.X, t.x0 + i, a, b);
      cb[i] = static_cast<uint32_t>(b + bO + t.y0);
    }
  };
  auto loads = [&](const DenseTile& t, int s) {
    const uint32_t* ra = rowA(s);
    E* dst = tile(s) + r0 * P.rl + xl;
    if constexpr (SHA) {
#pragma unroll 4
      for (uint32_t k = 0; k < K1; ++k) {
        const uint32_t y = r0 + k * R;
        const uint32_t ga = ra[min(y, P.ty - 1)];
        const uint32_t d = ga & (VA - 1), end = t.nx + d;  // row = chunk elements [d, end)
        const bool v = act_l && y < t.ny && xl < end;
        const uint32_t nbytes = v ? min(static_cast<uint32_t>(VA), end - xl) * EAB : 0u;
        cp_async_part<VA * EAB>(dst + k * R * P.rl, A + (ga - d) + xl, nbytes, v);
      }
    } else {
      const bool xv = act_l && xl < t.nx;
      const uint32_t nbytes = xv ? min(static_cast<uint32_t>(VA), t.nx - xl) * EAB : 0u;
      const E* ax = A + xl;
#pragma unroll 4
      for (uint32_t k = 0; k < K1; ++k) {
        const uint32_t y = r0 + k * R;
        cp_async_part<VA * EAB>(dst + k * R * P.rl, ax + ra[min(y, P.ty - 1)], nbytes,
                                xv && y < t.ny);
      }
    }
    if constexpr (MODE == 2) {  // the tile's B elements, column-major like B
      const uint32_t* cb = colB(s);
      EBv* bdst = tileB(s) + yl;
#pragma unroll 4
      for (uint32_t k = 0; k < K2; ++k) {
        const uint32_t x = c0 + k * Q;
        const uint32_t xc = min(x, P.tx - 1);
        const uint32_t gb = cb[xc];
        const uint32_t d = SHB ? (gb & (VB - 1)) : 0u, end = t.ny + d;
        const bool v = act_s && x < t.nx && yl < end;
        const uint32_t bbytes = v ? min(static_cast<uint32_t>(VB), end - yl) * EBB : 0u;
        cp_async_part<VB * EBB>(bdst + xc * bpitch, B + (gb - d) + yl, bbytes, v);
      }
    }
  };

  const uint32_t g = gridDim.x;
  uint32_t it = blockIdx.x;
  if (it >= P.items) return;
  tables(dense_tile(P, it), 0);
  __syncthreads();
  loads(dense_tile(P, it), 0);
  cp_async_commit();

  for (int s = 0; it < P.items; it += g, s ^= 1) {
    const uint32_t nxt = it + g;
    if (nxt < P.items) tables(dense_tile(P, nxt), s ^ 1);
    __syncthreads();
    if (nxt < P.items) loads(dense_tile(P, nxt), s ^ 1);
    cp_async_commit();
    cp_async_wait<NS - 1>();
    __syncthreads();

    // smem -> B: each thread writes VB consecutive elements of a column; U
    // columns per batch so the batch's B reads (mode 3) are in flight together
    const DenseTile cur = dense_tile(P, it);
    const uint32_t* cb = colB(s);
    const uint32_t* ra = rowA(s);
    const E* T = tile(s);
    const EBv* bsrc = tileB(s) + yl;
    // unshifted columns: this thread's VB tile rows are fixed for the tile
    uint32_t rb[VB];
    if constexpr (!SHB) {
#pragma unroll
      for (int m = 0; m < VB; ++m) {
        const uint32_t y = yl + m;
        rb[m] = y * P.rl + (SHA ? (ra[min(y, P.ty - 1)] & (VA - 1)) : 0u);
      }
    }
    constexpr uint32_t U = MODE == 3 ? 4 : 1;  // batching only pays for the B reads
#pragma unroll(MODE == 3 ? 1 : 2)
    for (uint32_t k0 = 0; k0 < K2; k0 += U) {
      VBv w[U];
      E a[U][VB];
      EBv* q[U];
      bool v[U];
      uint32_t vm[U];  // per-element validity bits of the vector
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) {
        const uint32_t x = c0 + (k0 + u) * Q;
        const uint32_t xc = min(x, P.tx - 1);
        const uint32_t gb = cb[xc];
        const uint32_t d = SHB ? (gb & (VB - 1)) : 0u;
        v[u] = act_s && k0 + u < K2 && x < cur.nx;
        q[u] = B + (gb - d) + yl;
        vm[u] = 0;
#pragma unroll
        for (int m = 0; m < VB; ++m) {
          const int y = static_cast<int>(yl + m) - static_cast<int>(d);  // tile row of element m
          const bool ok = y >= 0 && y < static_cast<int>(cur.ny);
          vm[u] |= (ok ? 1u : 0u) << m;
          if constexpr (SHB) {
            const uint32_t yc = static_cast<uint32_t>(min(max(y, 0), static_cast<int>(P.ty) - 1));
            a[u][m] = T[yc * P.rl + (SHA ? (ra[yc] & (VA - 1)) : 0u) + xc];
          } else {
            a[u][m] = T[rb[m] + xc];
          }
        }
        if (!v[u]) vm[u] = 0;
        if constexpr (MODE == 2) {
#pragma unroll
          for (int m = 0; m < VB; ++m) {
            const EBv b = bsrc[xc * bpitch + m];
#pragma unroll
            for (int c = 0; c < C; ++c) w[u].v[m * C + c] = b.v[c];
          }
        }
        if constexpr (MODE == 3) {
          if (vm[u] == (1u << VB) - 1) {
            vload_b_pred(w[u], q[u]->v, true);
          } else {
#pragma unroll
            for (int m = 0; m < VB; ++m) {
              EBv b;
              vload_b_pred(b, q[u][m].v, (vm[u] >> m) & 1u);
#pragma unroll
              for (int c = 0; c < C; ++c) w[u].v[m * C + c] = b.v[c];
            }
          }
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) {
#pragma unroll
        for (int m = 0; m < VB; ++m)
#pragma unroll
          for (int c = 0; c < C; ++c) w[u].v[m * C + c] = up(a[u][m].v[c], w[u].v[m * C + c]);
        if (vm[u] == (1u << VB) - 1) {
          vstore_pred(q[u]->v, w[u], true);
        } else if (vm[u]) {
#pragma unroll
          for (int m = 0; m < VB; ++m) {
            EBv e;
#pragma unroll
            for (int c = 0; c < C; ++c) e.v[c] = w[u].v[m * C + c];
            vstore_pred(q[u][m].v, e, (vm[u] >> m) & 1u);
          }
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

}  // namespace ttb
