// rows.cuh -- bulk row copy: run_case1 / run_copy_1d (executor.cpp:164-211)
// for long shared stride-1 rows at any element alignment.
//
// copy_rows_kernel moves a row as V-element vectors that must be aligned on
// both sides, so rows whose A and B starts differ in 16-byte phase (c5_t04:
// 72.8 KB fp32 rows at a 4-byte phase; the suite's case-1 rows of 1496 bytes)
// fall back to element-wide loads and stores and stay latency-bound.  Here a
// row is cut into segments; one producer lane brings each segment into
// shared memory with a single cp.async.bulk (the 16-byte aligned superset of
// the segment, SASS UBLKCP; with beta != 0 also B's segment), so the bytes in
// flight sit in shared memory, not registers.  The consumer warps then write
// B with 16-byte stores at B's own alignment, gathering each chunk's A
// elements from shared memory at the phase difference (head and tail element
// by element), alpha / beta fused.
#pragma once

#include "btile.cuh"
#include "kernels.cuh"

namespace ttb {

struct RowSeg {  // per row of a stage
  int valid;
  uint32_t n, sha, shb;  // elements; byte offsets of the first element in its A / B slot
  int64_t ob;            // element offset of the row segment's first element in B
  int64_t pad;
};

template <class SA, class SB, int C, int MODE, int NC = kRowsConsumerWarps>
__global__ void __launch_bounds__(32 * (NC + 1)) rowcopy_kernel(const CopyParams P) {
  using EAv = Vec<SA, C>;
  using EBv = Vec<SB, C>;
  constexpr uint32_t EA = sizeof(EAv), EB = sizeof(EBv);
  constexpr uint32_t VB = EB >= 16 ? 1u : 16u / EB;  // elements per 16-byte chunk of B
  constexpr bool UPD = MODE == 2;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[kBtileMaxStages], empty[kBtileMaxStages];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t NS = P.bns, R = P.brows;
  const uint32_t seg = min(P.bseg, P.lvec);
  const uint32_t head_bytes = rowcopy_head_bytes(R);
  const uint32_t slot_a = rowcopy_slot_bytes(seg, EA), slot_b = rowcopy_slot_bytes(seg, EB);
  if (tid == 0) {
    for (uint32_t s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned char* A = static_cast<const unsigned char*>(P.A);
  unsigned char* Bb = static_cast<unsigned char*>(P.B);
  const uint32_t g = gridDim.x;

  if (warp == NC) {
    // ----------------------------------------------------------- producer --
    if (lane != 0) return;
    uint32_t s = 0, ph = 0;
    for (uint32_t it = blockIdx.x; it < P.bitems; it += g) {
      mbar_wait(&empty[s], ph ^ 1);
      unsigned char* st = smem + s * P.bstage;
      const uint32_t grp = udiv(it, P.dbnseg);
      const uint32_t e0 = (it - grp * P.bnseg) * P.bseg;
      uint32_t bytes = 0;
      for (uint32_t i = 0; i < R; ++i) {
        RowSeg* h = reinterpret_cast<RowSeg*>(st) + i;
        const uint32_t row = grp * R + i;
        int64_t oa = 0, ob = 0;
        const bool ok = row < P.rows && e0 < P.lvec && copy_row(P, row, oa, ob);
        h->valid = ok;
        if (!ok) continue;
        const uint32_t n = min(P.bseg, P.lvec - e0);
        const uint64_t ga = reinterpret_cast<uint64_t>(A + (oa + e0) * EA);
        const uint64_t lo = ga & ~uint64_t{15}, hi = (ga + uint64_t{n} * EA + 15) & ~uint64_t{15};
        bulk_g2s(st + head_bytes + i * slot_a, reinterpret_cast<const void*>(lo), static_cast<uint32_t>(hi - lo),
                 &full[s]);
        bytes += static_cast<uint32_t>(hi - lo);
        h->n = n;
        h->sha = static_cast<uint32_t>(ga - lo);
        h->ob = ob + e0;
        h->shb = 0;
        if constexpr (UPD) {
          const uint64_t gb = reinterpret_cast<uint64_t>(Bb + (ob + e0) * EB);
          const uint64_t blo = gb & ~uint64_t{15}, bhi = (gb + uint64_t{n} * EB + 15) & ~uint64_t{15};
          bulk_g2s(st + head_bytes + R * slot_a + i * slot_b, reinterpret_cast<const void*>(blo),
                   static_cast<uint32_t>(bhi - blo), &full[s]);
          bytes += static_cast<uint32_t>(bhi - blo);
          h->shb = static_cast<uint32_t>(gb - blo);
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
  uint32_t s = 0, ph = 0;
  const uint32_t ct = warp * 32 + lane;
  for (uint32_t it = blockIdx.x; it < P.bitems; it += g) {
    mbar_wait(&full[s], ph);
    const unsigned char* st = smem + s * P.bstage;
    for (uint32_t i = 0; i < R; ++i) {
      const RowSeg h = reinterpret_cast<const RowSeg*>(st)[i];
      if (!h.valid) continue;
      const unsigned char* sa = st + head_bytes + i * slot_a + h.sha;
      const unsigned char* sb = st + head_bytes + R * slot_a + i * slot_b + h.shb;
      unsigned char* out = Bb + h.ob * EB;
      // elements before B's first 16-byte boundary, whole chunks, the rest
      const uint32_t head =
          min(h.n, static_cast<uint32_t>(((16u - reinterpret_cast<uint64_t>(out) % 16u) % 16u) / EB));
      const uint32_t chunks = (h.n - head) / VB, body_end = head + chunks * VB;
      for (uint32_t j = ct; j < chunks; j += NC * 32) {
        const uint32_t i0 = head + j * VB;
        Piece<EBv, VB> w;
        if constexpr (UPD) w = *reinterpret_cast<const Piece<EBv, VB>*>(sb + i0 * EB);  // 16-byte aligned
#pragma unroll
        for (uint32_t k = 0; k < VB; ++k) {
          const EAv a = *reinterpret_cast<const EAv*>(sa + (i0 + k) * EA);
#pragma unroll
          for (int c = 0; c < C; ++c) w.e[k].v[c] = up(a.v[c], UPD ? w.e[k].v[c] : SB(0));
        }
        *reinterpret_cast<Piece<EBv, VB>*>(out + i0 * EB) = w;
      }
      // head and tail element by element (< 2 VB of them)
      const uint32_t edge = head + (h.n - body_end);
      for (uint32_t q = ct; q < edge; q += NC * 32) {
        const uint32_t e = q < head ? q : body_end + (q - head);
        const EAv a = *reinterpret_cast<const EAv*>(sa + e * EA);
        EBv b;
        if constexpr (UPD) b = *reinterpret_cast<const EBv*>(sb + e * EB);
        EBv w;
#pragma unroll
        for (int c = 0; c < C; ++c) w.v[c] = up(a.v[c], UPD ? b.v[c] : SB(0));
        *reinterpret_cast<EBv*>(out + e * EB) = w;
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
