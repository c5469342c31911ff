// btile.cuh -- the staged tile fed by the Blackwell bulk-copy (TMA) engine.
//
// Same tile as dense_kernel / vtile_kernel (X group contiguous in A, Y group
// contiguous in B -- ttune's run_case2, executor.cpp:213-281; with a shared
// stride-1 extent S > 1 the tile is S x tx x ty, run_case1 at 172-211), but the
// global -> shared side is one cp.async.bulk per tile row instead of one
// LDGSTS per element or 16-byte chunk, and the kernel is warp specialised:
//
//   warps NC..NC+PW-1   (producers) claim the next tile (a global counter:
//                       whole-tile work stealing), wait until the ring stage
//                       is free, decode the tile's row / column offsets (one
//                       lane per row / column), issue a bulk copy per A tile
//                       row -- and with beta != 0 per B tile column; rows or
//                       columns that continue each other go as one copy --
//                       write the offset tables and the tile index into the
//                       stage, and arrive on its `full` mbarrier with the bytes.
//   warps 0..NC-1       wait on `full`, write the tile to B with lanes along
//                       B's stride-1 run (column walk) or along the whole tile
//                       in B order (linear walk), alpha/beta fused (MODE 3: B
//                       read directly, not through the ring), release `empty`.
//
// Bulk copies need 16-byte aligned addresses and sizes: a row that starts or
// ends inside a 16-byte block is fetched as the aligned superset of blocks that
// covers it (at most 12 bytes either side, never outside the blocks that hold
// the row's own first and last element, so never outside the allocation) and
// its elements land in shared memory shifted by d(y) = (row start mod 16) /
// element bytes; the consumer reads element x of row y at y*pitch + d(y) + x.
// Bytes of the superset outside the logical row are never used.
//
// Measured on B200: copies are issued one lane at a time through
// the uniform datapath and a CTA keeps about one stage of them moving, so the
// throughput comes from producer warps (4) and CTAs per SM (3-6, 2-3 stages
// each), or from large tiles (kern_btile_big.cu) -- not from deeper rings.
#pragma once

#include <cuda.h>

#include "kernels.cuh"

namespace ttb {

constexpr int kBtileMaxStages = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// arrive and add `bytes` to the phase's expected transaction count (the
// copies it covers may already have completed: tx-count may go negative)
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{ .reg .b64 st; mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1; }" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// wait for a phase with mbarrier.try_wait: the warp sleeps in hardware until
// the phase completes (or a time limit passes, then it asks again) instead of
// spinning on test_wait -- the spinning warps took issue slots from the
// working ones (whole sweep +1.4%, c5_t06 +9%, t07 / t22 +4% on B200;
// -DTTB_SPIN_WAIT builds the spinning form for comparison)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred done;\n"
#ifdef TTB_SPIN_WAIT
      "W: mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n"
#else
      "W: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n"
#endif
      " @!done bra W;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy (TMA engine, no tensor map), completion counted
// in bytes on `bar`; dst, src and bytes are multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// tensor-map box load (SASS UTMALDG) into shared memory, completion counted
// in bytes on `bar`, and the box store (UTMASTG) in the thread's bulk group;
// c[] holds one coordinate per map dim
__device__ __forceinline__ void tma_load(const CUtensorMap* m, int rank, void* dst, const int* c,
                                         uint64_t* bar) {
  const uint32_t d = smem_u32(dst), b = smem_u32(bar);
  const uint64_t mp = reinterpret_cast<uint64_t>(m);
  switch (rank) {
    case 1:
      asm volatile(
          "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(d),
          "l"(mp), "r"(c[0]), "r"(b)
          : "memory");
      break;
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              d),
          "l"(mp), "r"(c[0]), "r"(c[1]), "r"(b)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              d),
          "l"(mp), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
              d),
          "l"(mp), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
              d),
          "l"(mp), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
          : "memory");
      break;
  }
}

__device__ __forceinline__ void tma_store(const CUtensorMap* m, int rank, const void* src, const int* c) {
  const uint32_t s = smem_u32(src);
  const uint64_t mp = reinterpret_cast<uint64_t>(m);
  switch (rank) {
    case 1:
      asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];" ::"l"(mp), "r"(c[0]),
                   "r"(s)
                   : "memory");
      break;
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(mp),
                   "r"(c[0]), "r"(c[1]), "r"(s)
                   : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(mp),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(s)
                   : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(mp),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(s)
                   : "memory");
      break;
    default:
      asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                       mp),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(s)
                   : "memory");
      break;
  }
}

// (stage layout: btile_stage_bytes, params.hpp)

// P.ns stages, P.pa / P.pb row / column pitches (bytes), P.ly lanes along a
// tile column (power of two <= 32; 32 / ly columns per warp step), JY = column
// elements per lane (S*ty <= JY * ly; JY == 0: the linear walk, any S*ty,
// P.ly == 0).  P.S is the shared stride-1 extent (1
// when A's and B's stride-1 indices differ): an A tile row is then S*tx
// elements, a B tile column S*ty.  MODE 0-3 as Update (3: B read directly
// by the consumers, not through the ring).
// kernel parameters: the tile plan plus, when P.tma is set, the tensor maps
// of the side(s) that arrive as one box (param space, __grid_constant__)
struct BtileParams {
  CUtensorMap ma[kBtileMaxClasses], mb[kBtileMaxClasses];  // per phase class (P.ca / P.cb)
  int sha[kBtileMaxClasses], shb[kBtileMaxClasses];          // class row start within its 16 bytes (elements)
  SmemParams p;
};

template <class SA, class SB, int C, int MODE, int JY, int PW = kBtileProducerWarps,
          int NC = kBtileConsumerWarps>
__global__ void __launch_bounds__(32 * (NC + PW)) btile_kernel(const __grid_constant__ BtileParams Q) {
  const SmemParams& P = Q.p;
  using E = Vec<SA, C>;
  using EBv = Vec<SB, C>;
  constexpr uint32_t EA = sizeof(E), EB = sizeof(EBv);
  constexpr bool UPD = MODE == 2;  // B staged through the ring (MODE 3 reads B directly)
  // columns per consumer step: ~4 words of loads in flight per tile row
  constexpr int UX = EB <= 4 ? 4 : EB <= 8 ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full[kBtileMaxStages], empty[kBtileMaxStages];

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t NS = P.ns;
  const uint32_t al = P.tma ? 128u : 16u;  // a box lands 128-byte aligned
  const uint32_t tables = btile_tables_bytes(P.tx, P.ty, UPD, al);
  const uint32_t stage_bytes = btile_stage_bytes(P.tx, P.ty, P.abytes, P.bbytes, UPD, al);
  const uint32_t a_bytes = btile_round(P.abytes, al);
  // tensor-map sides: elements per 16 bytes (box starts), class region sizes
  constexpr uint32_t ALA = EA >= 16 ? 1u : 16u / EA, ALB = EB >= 16 ? 1u : 16u / EB;
  const uint32_t cla = btile_class_bytes(P.rowa, P.cola, EA), clb = btile_class_bytes(P.rowb, P.colb, EB);
  auto stage = [&](uint32_t s) { return smem_raw + s * stage_bytes; };

  if (tid == 0) {
    for (uint32_t s = 0; s < NS; ++s) {
      mbar_init(&full[s], 32 * PW);  // every producer lane arrives (with its bytes)
      mbar_init(&empty[s], NC);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint32_t g = gridDim.x;
  if (warp >= NC) {
    // ------------------------------------------------------------ producer --
    const unsigned char* A = static_cast<const unsigned char*>(P.A);
    const unsigned char* Bc = static_cast<const unsigned char*>(P.B);
    uint32_t s = 0, ph = 0;
    // tiles: blockIdx.x first, then (P.ctr) the next unclaimed one from a
    // global counter -- whole-tile work stealing, so one slow SM does not hold
    // up the launch -- or (no counter) every g-th.  The leader lane claims and
    // publishes the index in the stage header for the other producer warps
    // and the consumers; the counter resets itself when the last CTA is done.
    const bool leader = warp == NC && lane == 0;
    uint32_t it = blockIdx.x;
    for (uint32_t k = 0;; ++k) {
      mbar_wait(&empty[s], ph ^ 1);  // a fresh barrier passes parity 1 at once
      unsigned char* st = stage(s);
      volatile uint32_t* hdr = reinterpret_cast<volatile uint32_t*>(st);
      // (claiming the next tile one round early, to hide the counter's round
      // trip, measured 1% slower on c5_t00 / t13: the claim is not the bound)
      if (k > 0) it = P.ctr ? (leader ? g + atomicAdd(P.ctr, 1u) : 0u) : it + g;
      if (leader) *hdr = it;
      asm volatile("bar.sync 1, %0;" ::"r"(32 * PW) : "memory");
      it = *hdr;
      if (it >= P.items) {
        mbar_arrive(&full[s]);  // consumers find the end mark in the header
        if (leader && P.ctr) {
          __threadfence();
          if (atomicAdd(P.ctr + 1, 1u) == g - 1) {  // every CTA has made its last claim
            P.ctr[0] = 0;
            P.ctr[1] = 0;
          }
        }
        break;
      }
      const DenseTile t = dense_tile(P, it);
      int64_t aO, bO;
      decode(P.O, t.o, aO, bO);
      uint32_t* rbase = reinterpret_cast<uint32_t*>(st + 16);
      uint32_t* boff = rbase + P.ty;
      uint32_t* cbase = boff + P.tx;
      unsigned char* ta = st + tables;
      unsigned char* tb = ta + a_bytes;
      uint32_t bytes = 0;
      // a side that arrives by tensor map: per phase class r (rows y with
      // y mod ca == r; one class when the rows are 16-byte aligned apart) one
      // box of the class's rows in this tile, starting at the 16-byte aligned
      // element at or before x0, issued by the leader
      if (P.tma && leader) {
        // dim 0 counts map elements: 16-byte kinds are two 8-byte ones
        constexpr int SUBA = EA > 8 ? static_cast<int>(EA / 8) : 1, SUBB = EB > 8 ? static_cast<int>(EB / 8) : 1;
        if (P.tma & 1) {
          for (uint32_t r = 0; r < P.ca; ++r) {
            const uint32_t yr = t.y0 + (r + P.ca - t.y0 % P.ca) % P.ca;  // first row of class r
            if (yr >= t.y0 + t.ny) continue;
            const int x = static_cast<int>(t.x0) + Q.sha[r];
            const int c[3] = {(x & ~static_cast<int>(ALA - 1)) * SUBA, static_cast<int>((yr - r) / P.ca),
                              static_cast<int>(aO / P.tca)};
            tma_load(&Q.ma[r], P.tra, ta + r * cla, c, &full[s]);
            bytes += P.rowa * P.cola * EA;
          }
        }
        if (UPD && (P.tma & 2)) {
          for (uint32_t r = 0; r < P.cb; ++r) {
            const uint32_t xr = t.x0 + (r + P.cb - t.x0 % P.cb) % P.cb;  // first column of class r
            if (xr >= t.x0 + t.nx) continue;
            const int y = static_cast<int>(t.y0) + Q.shb[r];
            const int c[3] = {(y & ~static_cast<int>(ALB - 1)) * SUBB, static_cast<int>((xr - r) / P.cb),
                              static_cast<int>(bO / P.tcb)};
            tma_load(&Q.mb[r], P.trb, tb + r * clb, c, &full[s]);
            bytes += P.rowb * P.colb * EB;
          }
        }
      }
      auto copy = [&](unsigned char* dst, uint64_t src, uint32_t n) {
        bulk_g2s(dst, reinterpret_cast<const void*>(src), n, &full[s]);
      };
      // P.runs bit 0 / 1: A rows / B columns may continue each other (the
      // planner's static test); then items are handled 32 at a time per warp:
      // whose data continue each other in memory (a row right after the
      // previous row: the tile spans X completely and Y's first axis follows
      // X in A; likewise for B columns) are fetched as one bulk copy per run,
      // landing packed from the run's first slot; tab[i] = element index of
      // item i's first element in the region.
      auto fetch = [&](uint32_t base, uint32_t cnt, uint32_t len, int64_t off, const unsigned char* gbase,
                       uint32_t esz, unsigned char* region, uint32_t pitch, uint32_t* tab, uint32_t ti) {
        const uint32_t i = base + lane;  // slot; the table entry is tab[ti]
        const bool valid = i < cnt;
        const int64_t prev = __shfl_up_sync(0xffffffffu, off, 1);
        const bool start = valid && (lane == 0 || prev + len != off);
        const uint32_t smask = __ballot_sync(0xffffffffu, start);
        const uint32_t nvalid = __popc(__ballot_sync(0xffffffffu, valid));
        uint32_t shift = 0;
        if (start) {
          const uint32_t above = smask & ~((2u << lane) - 1u);
          const uint32_t end = min(above ? static_cast<uint32_t>(__ffs(above)) - 1u : 32u, nvalid);
          const uint64_t ga = reinterpret_cast<uint64_t>(gbase + off * esz);
          const uint64_t lo = ga & ~uint64_t{15};
          const uint64_t hi = (ga + static_cast<uint64_t>(end - lane) * len * esz + 15) & ~uint64_t{15};
          shift = static_cast<uint32_t>(ga - lo);
          copy(region + i * pitch, lo, static_cast<uint32_t>(hi - lo));
          bytes += static_cast<uint32_t>(hi - lo);
        }
        const uint32_t s0 = valid ? 31u - __clz(smask & ((2u << lane) - 1u)) : 0u;
        const uint32_t sh0 = __shfl_sync(0xffffffffu, shift, s0);
        if (valid) tab[ti] = ((base + s0) * pitch + sh0) / esz + (lane - s0) * len;
      };
      // one bulk copy per item (the common case: no item continues another)
      auto fetch1 = [&](uint32_t i, uint32_t len, int64_t off, const unsigned char* gbase, uint32_t esz,
                        unsigned char* region, uint32_t pitch, uint32_t* tab) {
        const uint64_t ga = reinterpret_cast<uint64_t>(gbase + off * esz);
        const uint64_t lo = ga & ~uint64_t{15};
        const uint64_t hi = (ga + static_cast<uint64_t>(len) * esz + 15) & ~uint64_t{15};
        copy(region + i * pitch, lo, static_cast<uint32_t>(hi - lo));
        bytes += static_cast<uint32_t>(hi - lo);
        tab[i] = (i * pitch + static_cast<uint32_t>(ga - lo)) / esz;
      };
      if (P.tma & 1) {
        for (uint32_t y = (warp - NC) * 32 + lane; y < t.ny; y += 32 * PW) {
          const uint32_t yy = t.y0 + y, r = yy % P.ca;
          const uint32_t yr = t.y0 + (r + P.ca - t.y0 % P.ca) % P.ca;
          const uint32_t off = (t.x0 + static_cast<uint32_t>(Q.sha[r])) & (ALA - 1);
          rbase[y] = r * (cla / EA) + (yy - yr) / P.ca * P.cola + off;
        }
      } else if (P.runs & 1) {
        for (uint32_t base = (warp - NC) * 32; base < t.ny; base += 32 * PW) {
          int64_t a = 0, b;
          const uint32_t y = base + lane;
          if (y < t.ny) decode(P.Y, t.y0 + y, a, b);
          fetch(base, t.ny, t.nx * P.S, a + aO + t.x0 * P.S, A, EA, ta, P.pa, rbase, y);
        }
      } else {
        for (uint32_t y = (warp - NC) * 32 + lane; y < t.ny; y += 32 * PW) {
          int64_t a, b;
          decode(P.Y, t.y0 + y, a, b);
          fetch1(y, t.nx * P.S, a + aO + t.x0 * P.S, A, EA, ta, P.pa, rbase);
        }
      }
      if (UPD && (P.tma & 2)) {
        // B box: column x at x*ty; the stores still need each column's offset
        for (uint32_t x = (warp - NC) * 32 + lane; x < t.nx; x += 32 * PW) {
          int64_t a, b;
          decode(P.X, t.x0 + x, a, b);
          boff[x] = static_cast<uint32_t>(b + bO + t.y0 * P.S);
          const uint32_t xx = t.x0 + x, r = xx % P.cb;
          const uint32_t xr = t.x0 + (r + P.cb - t.x0 % P.cb) % P.cb;
          const uint32_t off = (t.y0 + static_cast<uint32_t>(Q.shb[r])) & (ALB - 1);
          cbase[x] = r * (clb / EB) + (xx - xr) / P.cb * P.colb + off;
        }
      } else if (UPD && P.xp && t.nx == P.tx) {
        // column-permuted walk: fetch B columns in walk order j, where
        // consecutive columns continue each other in B
        for (uint32_t base = (warp - NC) * 32; base < t.nx; base += 32 * PW) {
          int64_t a, b = 0;
          const uint32_t j = base + lane;
          const uint32_t q2 = udiv(j, P.dxm);
          const uint32_t x = (j - q2 * P.xm) * P.xp + q2;
          if (j < t.nx) decode(P.X, t.x0 + x, a, b);
          const int64_t bo = b + bO + t.y0 * P.S;
          if (j < t.nx) boff[x] = static_cast<uint32_t>(bo);
          fetch(base, t.nx, t.ny * P.S, bo, Bc, EB, tb, P.pb, cbase, x);
        }
      } else if (UPD && (P.runs & 2)) {
        for (uint32_t base = (warp - NC) * 32; base < t.nx; base += 32 * PW) {
          int64_t a, b = 0;
          const uint32_t x = base + lane;
          if (x < t.nx) decode(P.X, t.x0 + x, a, b);
          const int64_t bo = b + bO + t.y0 * P.S;
          if (x < t.nx) boff[x] = static_cast<uint32_t>(bo);
          fetch(base, t.nx, t.ny * P.S, bo, Bc, EB, tb, P.pb, cbase, x);
        }
      } else {
        for (uint32_t x = (warp - NC) * 32 + lane; x < t.nx; x += 32 * PW) {
          int64_t a, b;
          decode(P.X, t.x0 + x, a, b);
          const int64_t bo = b + bO + t.y0 * P.S;
          boff[x] = static_cast<uint32_t>(bo);
          if constexpr (UPD) fetch1(x, t.ny * P.S, bo, Bc, EB, tb, P.pb, cbase);
        }
      }
      mbar_arrive_expect_tx(&full[s], bytes);
      if (++s == NS) {
        s = 0;
        ph ^= 1;
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers --
  const Update<SA, SB, MODE> up(P.sc);
  EBv* __restrict__ B = static_cast<EBv*>(P.B);
  const uint32_t ly = P.ly, lxn = 32u / ly;
  const uint32_t yi = lane & (ly - 1), xi = lane / ly;
  const uint32_t xstep = NC * lxn;
  uint32_t s = 0, ph = 0;
  for (;;) {
    mbar_wait(&full[s], ph);
    const unsigned char* st = stage(s);
    const uint32_t it = *reinterpret_cast<const volatile uint32_t*>(st);
    if (it >= P.items) break;
    const DenseTile t = dense_tile(P, it);
    const uint32_t* rbase = reinterpret_cast<const uint32_t*>(st + 16);
    const uint32_t* boff = rbase + P.ty;
    const uint32_t* cbase = boff + P.tx;
    const E* ta = reinterpret_cast<const E*>(st + tables);
    const EBv* tb = reinterpret_cast<const EBv*>(st + tables + a_bytes);
    if constexpr (JY == 0) {
      // linear walk of the tile in B order: element e of the tile index space
      // is column x = e / (S*ty), element c = e mod (S*ty) of that column; the
      // lanes of a warp cover consecutive B addresses even when a column is
      // shorter than a warp (small ty, or a column run that continues into
      // the next column)
      const uint32_t Lf = P.S * P.ty, Lv = P.S * t.ny, total = Lf * t.nx;
      // P.xp > 0 (full tiles only): a tile column is an (X0, X1) pair with X0
      // (extent xp) covered completely and B continuing from Y into X1;
      // walking X1 fastest keeps consecutive columns contiguous in B
      const bool xperm = P.xp != 0 && t.nx == P.tx;
      constexpr int U = 4;
      for (uint32_t e0 = warp * 32 + lane; e0 < total; e0 += U * 32 * NC) {
        EBv w[U];
        EBv* q[U];
        bool v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t e = e0 + u * 32 * NC;
          const uint32_t j = udiv(e, P.dcol);  // column in walk order
          const uint32_t c = e - j * Lf;
          v[u] = e < total && c < Lv;
          uint32_t x = j;
          if (xperm) {  // walk X's second axis before its first (B's order)
            const uint32_t q2 = udiv(j, P.dxm);
            x = (j - q2 * P.xm) * P.xp + q2;
          }
          const uint32_t xc = v[u] ? x : 0u, cc = v[u] ? c : 0u;
          const uint32_t y = P.S == 1 ? cc : udiv(cc, P.dS);
          const E a = ta[rbase[y] + xc * P.S + (cc - y * P.S)];
          q[u] = B + boff[xc] + cc;
          EBv b;
          if constexpr (UPD) b = tb[cbase[xc] + cc];
          if constexpr (MODE == 3) vload_b_pred(b, q[u]->v, v[u]);
#pragma unroll
          for (int k = 0; k < C; ++k) w[u].v[k] = up(a.v[k], MODE >= 2 ? b.v[k] : SB(0));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) vstore_pred(q[u]->v, w[u], v[u]);
      }
    } else {
    // a tile column is S*ny elements contiguous in B (element e = y*S + s);
    // this lane's JY column elements (e = yi + j*ly) are fixed for the tile,
    // rb[j] = where element e of column 0 sits in the A tile; UX columns per
    // step, all loads of a step issued before its stores
    const uint32_t L = t.ny * P.S;
    uint32_t rb[JY];
    bool yv[JY];
#pragma unroll
    for (int j = 0; j < JY; ++j) {
      const uint32_t e = yi + j * ly;
      yv[j] = e < L;
      const uint32_t y = P.S == 1 ? e : udiv(e, P.dS);
      rb[j] = yv[j] ? rbase[y] + (e - y * P.S) : 0u;
    }
    for (uint32_t x0 = warp * lxn + xi; x0 < t.nx; x0 += UX * xstep) {
      EBv* q[UX];
      uint32_t xs[UX], cb[UX];
      bool xv[UX];
#pragma unroll
      for (int u = 0; u < UX; ++u) {
        const uint32_t x = x0 + u * xstep;
        xv[u] = x < t.nx;
        xs[u] = xv[u] ? x : x0;
        q[u] = B + boff[xs[u]] + yi;
        if constexpr (UPD) cb[u] = cbase[xs[u]];
      }
      EBv w[UX][JY];
#pragma unroll
      for (int u = 0; u < UX; ++u)
#pragma unroll
        for (int j = 0; j < JY; ++j) {
          const E a = ta[rb[j] + xs[u] * P.S];
          if constexpr (UPD) {
            const EBv b = tb[cb[u] + (yv[j] ? yi + j * ly : 0u)];  // stay inside the column
#pragma unroll
            for (int c = 0; c < C; ++c) w[u][j].v[c] = up(a.v[c], b.v[c]);
          } else if constexpr (MODE == 3) {
            EBv b;
            vload_b_pred(b, q[u][j * ly].v, xv[u] && yv[j]);
#pragma unroll
            for (int c = 0; c < C; ++c) w[u][j].v[c] = up(a.v[c], b.v[c]);
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c) w[u][j].v[c] = up(a.v[c], SB(0));
          }
        }
#pragma unroll
      for (int u = 0; u < UX; ++u)
#pragma unroll
        for (int j = 0; j < JY; ++j) {
          vstore_pred(q[u][j * ly].v, w[u][j], xv[u] && yv[j]);
        }
    }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
}

}  // namespace ttb
