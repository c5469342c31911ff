// tma.cuh -- the tensor-map tile: TMA box in, transpose through shared
// memory, TMA box out.
//
// ttune's run_case2 (executor.cpp:213-281) walks tiles of (A's stride-1 axis)
// x (B's stride-1 axis) and moves each through a w x w micro-tile
// (micro_tile_staged, executor.hpp:101-118).  Here a tile is one TMA box per
// side: the A box [by][bx] arrives in shared memory with a single
// cp.async.bulk.tensor (SASS UTMALDG), the consumer warps transpose it in
// registers, w x w elements per lane with 16-byte shared loads and stores,
// into the B box [bx][by], and a single cp.async.bulk.tensor store (UTMASTG)
// writes it back.  With beta != 0 the B box is loaded first through the same
// map and updated in place.  Partial tiles need no masking: the tensor maps
// zero-fill loads and clip stores outside the tensor.  With a shared
// stride-1 run (run_case1, executor.cpp:172-211) each (x, y) is an S-element
// run moved as 16-byte chunks.
//
// Warp roles (one elected lane each): warp 0 loads A boxes into the A ring,
// warp 1 (beta != 0) loads B boxes into the B ring, warps 2..2+SW-1 store
// finished B boxes -- each store warp takes every SW-th tile and waits for
// its store to have read shared memory before it hands the B slot back, so
// SW stores are in flight -- and the remaining warps are the consumers.  An
// A slot is refilled as soon as the consumers have read it; a B slot only
// once its store has read it.  Every role walks the same static tile
// sequence (blockIdx.x, + gridDim.x, ...).
//
// Bank conflicts: the 4 x 8 micro-tiles of a warp are assigned so that every
// 8-lane phase of a 16-byte shared access touches 8 distinct 16-byte bank
// groups when the tile rows are an odd number of 16-byte chunks long (the
// planner prefers such tiles); see the lane map in tma_lane().
#pragma once

#include <cuda.h>

#include "btile.cuh"
#include "kernels.cuh"

namespace ttb {

struct TmaParams {
  CUtensorMap ma;  // A, as seen from the A side
  CUtensorMap mb;  // B, as seen from the B side
  TmaPlan t;
};

// tile index -> box coordinates of both maps (mixed-radix digits, each
// feeding one dim of each map with a multiplier)
__device__ __forceinline__ void tma_coords(const TmaPlan& P, uint32_t t, int* ca, int* cb) {
#pragma unroll
  for (int k = 0; k < kTmaMaxRank; ++k) ca[k] = cb[k] = 0;
#pragma unroll
  for (int l = 0; l < kTmaLevels; ++l) {
    if (l >= P.nlev) break;
    const uint32_t q = udiv(t, P.lev[l]);
    const int d = static_cast<int>(t - q * P.lev[l].d);
    t = q;
#pragma unroll
    for (int k = 0; k < kTmaMaxRank; ++k) {
      if (P.dimA[l] == k) ca[k] += d * P.mulA[l];
      if (P.dimB[l] == k) cb[k] += d * P.mulB[l];
    }
  }
}

// lane -> micro-tile (i along x, j along y) of the warp's 4 x 8 block.  For
// 16-byte elements (w = 1) a phase is 8 consecutive j.  Otherwise phase h of
// 16-lane group g holds the 8 pairs with (i >> 1) == (j >> 1) (h = 0) or !=
// (h = 1): with odd row lengths (in 16-byte chunks) the loads of a phase hit
// ((4j' + i) mod 8) distinct chunks for w = 4 and ((2 pi(j) + i) mod 8) for
// w = 2, and the stores the same with i and j swapped.
template <int WM>
__device__ __forceinline__ void tma_lane(uint32_t lane, uint32_t wxl, uint32_t& i, uint32_t& j) {
  if (wxl == kTmaDiagonal) {  // i = k (x within the 8 x 8 block), j = d (the lane's diagonal)
    i = lane & 7;
    j = lane >> 3;
  } else if (wxl != 2) {  // warp tiles of 8, 16 or 32 micro-tiles along x (short tiles along y)
    i = lane & ((1u << wxl) - 1);
    j = lane >> wxl;
  } else if constexpr (WM == 1) {
    i = lane >> 3;
    j = lane & 7;
  } else {
    const uint32_t g = lane >> 4, h = (lane >> 3) & 1, m = lane & 7;
    const uint32_t c = m >> 2;
    i = 2 * c + (m & 1);
    j = 4 * g + 2 * (c ^ h) + ((m >> 1) & 1);
  }
}


template <class SA, class SB, int C, int MODE, bool RUNS, int NC = kTmaConsumerWarps,
          int SW = kTmaStoreWarps>
__global__ void __launch_bounds__(32 * (NC + 2 + SW)) tma_kernel(const __grid_constant__ TmaParams Q) {
  const TmaPlan& P = Q.t;
  using EA = Vec<SA, C>;
  using EB = Vec<SB, C>;
  constexpr int eA = sizeof(SA) * C, eB = sizeof(SB) * C;
  constexpr int emin = eA < eB ? eA : eB;
  constexpr int WM = 16 / emin > 0 ? 16 / emin : 1;  // micro-tile side (elements)
  constexpr bool UPD = MODE >= 2;
  extern __shared__ __align__(128) unsigned char smem[];
  // A ring: fa (A box landed), ea (consumers done with it)
  // B ring: fb (beta: B box landed), db (consumers wrote it), fr (its store has read it)
  __shared__ uint64_t fa[kTmaMaxStages], ea[kTmaMaxStages];
  __shared__ uint64_t fb[kTmaMaxStages], db[kTmaMaxStages], fr[kTmaMaxStages];

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t NA = P.ns, NB = P.nsb;  // A ring / B ring slots
  unsigned char* ring_a = smem;
  unsigned char* ring_b = smem + NA * P.tile_a;
  if (tid == 0) {
    for (uint32_t s = 0; s < NA; ++s) {
      mbar_init(&fa[s], 1);
      mbar_init(&ea[s], NC);
    }
    for (uint32_t s = 0; s < NB; ++s) {
      mbar_init(&fb[s], 1);
      mbar_init(&db[s], NC);
      mbar_init(&fr[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t g = gridDim.x;

  if (warp == 0 || warp == 1) {
    // ------------------------------------------- loads: A (warp 0), B (warp 1)
    const bool is_a = warp == 0;
    if (lane != 0 || (!is_a && !UPD)) return;
    const CUtensorMap* m = is_a ? &Q.ma : &Q.mb;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
    const uint32_t bytes = P.bx * P.by * P.S * (is_a ? eA : eB);
    const uint32_t N = is_a ? NA : NB;
    uint32_t s = 0, ph = 0;
    for (uint32_t t = blockIdx.x; t < P.items; t += g) {
      mbar_wait(is_a ? &ea[s] : &fr[s], ph ^ 1);  // a fresh barrier passes parity 1 at once
      int ca[kTmaMaxRank], cb[kTmaMaxRank];
      tma_coords(P, t, ca, cb);
      uint64_t* bar = is_a ? &fa[s] : &fb[s];
      mbar_arrive_expect_tx(bar, bytes);
      if (is_a)
        tma_load(m, P.va.rank, ring_a + s * P.tile_a, ca, bar);
      else
        tma_load(m, P.vb.rank, ring_b + s * P.tile_b, cb, bar);
      if (++s == N) {
        s = 0;
        ph ^= 1;
      }
    }
    return;
  }
  if (warp < 2 + SW) {
    // ------------------------------------------------------------ stores --
    // store warp q takes every SW-th tile and waits for its store to have
    // read shared memory before handing the B slot back: SW stores in flight
    if (lane != 0) return;
    const uint32_t q = warp - 2;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&Q.mb)) : "memory");
    uint32_t k = q;
    for (uint32_t t = blockIdx.x + q * g; t < P.items; t += SW * g, k += SW) {
      const uint32_t s = k % NB, ph = (k / NB) & 1;
      mbar_wait(&db[s], ph);
      int ca[kTmaMaxRank], cb[kTmaMaxRank];
      tma_coords(P, t, ca, cb);
      tma_store(&Q.mb, P.vb.rank, ring_b + s * P.tile_b, cb);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_arrive(&fr[s]);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    return;
  }

  // ------------------------------------------------------------ consumers --
  const Update<SA, SB, MODE> up(P.sc);
  const uint32_t cw = warp - 2 - SW;
  uint32_t s = 0, ph = 0, sb = 0, phb = 0;
  uint32_t i = 0, j = 0;
  if (!RUNS) tma_lane<WM>(lane, P.wxl, i, j);
  for (uint32_t t = blockIdx.x; t < P.items; t += g) {
    mbar_wait(&fa[s], ph);
    mbar_wait(UPD ? &fb[sb] : &fr[sb], UPD ? phb : phb ^ 1);  // beta: B landed; else: slot free
    const unsigned char* ta = ring_a + s * P.tile_a;
    unsigned char* tb = ring_b + sb * P.tile_b;
    if constexpr (RUNS) {
      // (x, y) runs of S elements, K 16-byte chunks each, walked in B order
      const uint32_t total = P.bx * P.by * P.kch;
      constexpr int PE = 16 / eA;  // elements per chunk (equal kinds)
      for (uint32_t e = cw * 32 + lane; e < total; e += NC * 32) {
        const uint32_t pr = udiv(e, P.dk);
        const uint32_t kk = e - pr * P.kch;
        const uint32_t x = udiv(pr, P.dby);
        const uint32_t y = pr - x * P.by;
        const Piece<EA, PE> a =
            *reinterpret_cast<const Piece<EA, PE>*>(ta + ((y * P.bx + x) * P.kch + kk) * 16);
        Piece<EB, PE>* dst = reinterpret_cast<Piece<EB, PE>*>(tb + ((x * P.by + y) * P.kch + kk) * 16);
        Piece<EB, PE> b;
        if constexpr (UPD) b = *dst;
#pragma unroll
        for (int u = 0; u < PE; ++u)
#pragma unroll
          for (int c = 0; c < C; ++c) b.e[u].v[c] = up(a.e[u].v[c], UPD ? b.e[u].v[c] : SB(0));
        *dst = b;
      }
    } else {
      const bool diag = P.wxl == kTmaDiagonal;
      const uint32_t wxn = diag ? 8u : 1u << P.wxl, wyn = diag ? 8u : 32u >> P.wxl;
      for (uint32_t w = cw; w < P.nwt; w += NC) {
        const uint32_t blk = diag ? w >> 1 : w;
        const uint32_t wy = udiv(blk, P.dnwx);
        const uint32_t wx = blk - wy * P.nwx;
        uint32_t xb = wxn * wx + i, ya = wyn * wy + j;
        // diagonal map: an 8-lane phase holds (x + k, y + (k + d) mod 8), k = 0..7,
        // distinct x for the loads and distinct y for the stores whatever the
        // row lengths (bank group k (W q + 1) + const with W q even, likewise W p)
        if (diag) ya = wyn * wy + ((i + 4 * (w & 1) + j) & 7);
        if (xb >= P.mx || ya >= P.my) continue;
        // WM rows of the A tile (y = WM*ya + r), WM elements each (x = WM*xb + q)
        Piece<EA, WM> a[WM];
#pragma unroll
        for (int r = 0; r < WM; ++r)
          a[r] = *reinterpret_cast<const Piece<EA, WM>*>(ta + ((WM * ya + r) * P.bx + WM * xb) * eA);
#pragma unroll
        for (int qq = 0; qq < WM; ++qq) {
          Piece<EB, WM>* dst = reinterpret_cast<Piece<EB, WM>*>(tb + ((WM * xb + qq) * P.by + WM * ya) * eB);
          Piece<EB, WM> b;
          if constexpr (UPD) b = *dst;
#pragma unroll
          for (int r = 0; r < WM; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) b.e[r].v[c] = up(a[r].e[qq].v[c], UPD ? b.e[r].v[c] : SB(0));
          *dst = b;
        }
      }
    }
    // this warp is done reading the A slot; its B writes go to the async
    // proxy (the store) once every consumer warp has arrived
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&ea[s]);
      mbar_arrive(&db[sb]);
    }
    if (++s == NA) {
      s = 0;
      ph ^= 1;
    }
    if (++sb == NB) {
      sb = 0;
      phb ^= 1;
    }
  }
}

}  // namespace ttb
