// params.hpp -- launch parameter blocks shared by the host planner and the
// sm_100a kernels.  All in-kernel index spaces are 32-bit (the executor splits
// problems whose spaces would not fit, see api.cpp); memory offsets are 64-bit.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define TTB_HD __host__ __device__ __forceinline__
#else
#define TTB_HD inline
#endif

namespace ttb {

constexpr int kSpaceDims = 16;  // axes per flattened index space

// Unsigned 32-bit division by a run-time constant: q = (umulhi(n, m) + n) >> s
// (round-up multiplier; exact for every n < 2^32).
struct Div32 {
  uint32_t d = 1, m = 1, s = 0;

  static Div32 make(uint32_t d) {
    Div32 r;
    r.d = d;
    uint32_t s = 0;
    while ((uint64_t{1} << s) < d) ++s;
    r.s = s;
    r.m = static_cast<uint32_t>(((uint64_t{1} << 32) * ((uint64_t{1} << s) - d)) / d + 1);
    return r;
  }
};

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t udiv(uint32_t n, const Div32& f) {
  return static_cast<uint32_t>((static_cast<uint64_t>(__umulhi(n, f.m)) + n) >> f.s);
}
#endif

// A group of tensor axes flattened column-major into one index (first axis
// fastest), with each axis' element stride in A and in B.
struct Space {
  int nd = 0;
  uint32_t total = 1;
  Div32 ext[kSpaceDims];
  int64_t sa[kSpaceDims];
  int64_t sb[kSpaceDims];
};

enum Variant : int { kCopy = 0, kRt = 1, kSmem = 2, kTma = 3 };

// Element-wise update constants (the W-typed alpha/beta are formed in-kernel).
struct Scale {
  double alpha = 1.0, beta = 0.0;
};

// kCopy: rows of `lead` elements contiguous in both tensors (shared stride-1
// index, run_case1 / run_copy_1d analogue), rows enumerated by `rows`.
// Rows are enumerated in tiles of tx x ty rows over the X group (A axes after
// the shared one) and the Y group (B positions after it), so both the reads
// and the writes of neighbouring rows stay in a small address window.
struct CopyParams {
  const void* A;
  void* B;
  Scale sc;
  Space X, Y, O;
  uint32_t lvec;          // vectors per row (lead / V)
  Div32 dl;               // divisor lvec
  uint32_t tx, ty, ltx, lty;  // row tile, powers of two
  uint32_t nxc, nyc;
  Div32 dnx, dny;
  int order;
  uint32_t nseg;          // row segments of 32*U vectors (long-row kernel)
  Div32 dseg;
  uint32_t rows;          // rows including the masked rows of partial tiles
  uint32_t items;         // warp items: long rows (row, segment); short rows 32-row groups
  int long_rows;          // 1: copy_rows_kernel, 0: copy_kernel
  int align;              // copy_rows_kernel: segments on 128-byte lines of B (1) or A (2), 0 off
  // rowcopy_kernel (bulk rows): a row in segments of `bseg` elements, each
  // brought into shared memory by one bulk copy (its 16-byte aligned
  // superset) and written out with 16-byte stores at B's alignment; `bns`
  // ring stages of `bstage` bytes; items = rows * bnseg
  // rows shorter than a segment travel `brows` at a time (one copy each)
  int bulk;
  uint32_t bseg, bnseg, brows, bns, bstage, bitems;
  Div32 dbnseg;
};
constexpr int kRowsConsumerWarps = 4;
constexpr int kRowsMaxGroup = 32;
// rowcopy_kernel stage: `rows` 32-byte headers (128-byte multiple), then per
// row an A slot of `seg` elements (+16 for the aligned superset), then (beta
// != 0) the B slots; slot bytes 16-byte multiples
TTB_HD uint32_t rowcopy_slot_bytes(uint32_t seg, uint32_t e) { return (seg * e + 16u + 15u) & ~15u; }
TTB_HD uint32_t rowcopy_head_bytes(uint32_t rows) { return (rows * 32u + 127u) & ~127u; }
TTB_HD uint32_t rowcopy_stage_bytes(uint32_t seg, uint32_t rows, uint32_t ea, uint32_t eb, bool upd) {
  return (rowcopy_head_bytes(rows) + rows * (rowcopy_slot_bytes(seg, ea) + (upd ? rowcopy_slot_bytes(seg, eb) : 0u)) +
          127u) & ~127u;
}

// kRt: register micro-tile transpose between the X space (starts with A's
// stride-1 axis) and the Y space (starts with B's stride-1 axis), vectors of
// MX elements along X on load and MY elements along Y on store.
struct RtParams {
  const void* A;
  void* B;
  Scale sc;
  Space X, Y, O;
  int lx;                 // lanes along X per warp (32/lx along Y), power of two
  int lx_log2;
  uint32_t wx, wy;        // warp tile: lx*MX by (32/lx)*MY
  uint32_t nxc, nyc;      // chunk counts along X / Y
  Div32 dnx, dny;         // divisors nxc, nyc
  int order;              // 0: X chunks fastest, 1: Y chunks fastest
  uint32_t items;         // nxc * nyc * O.total
  int64_t sa_y0;          // A stride of Y's first axis
  int64_t sb_x0;          // B stride of X's first axis
};

// kSmem: shared-memory staged tile  S (shared lead) x TX x TY  with padded
// rows of `rl` elements; per-tile offset tables live in shared memory too.
struct SmemParams {
  const void* A;
  void* B;
  Scale sc;
  Space X, Y, O;
  uint32_t S, tx, ty, rl;
  Div32 dS, dtx, dty;
  uint32_t nxc, nyc;
  Div32 dnx, dny;
  int order;
  uint32_t items;
  // dense fast path: S == 1, X contiguous in A, Y contiguous in B, tx/ty powers
  // of two -> the walks need shifts and masks only, no per-element division
  int dense;              // 0 generic, 1 dense (any tile), 2/3 dense power-of-two tile, 4 vector tile,
                          // 5 bulk-copy tile
  uint32_t ltx, lty;
  int ept;                // dense with tx,ty <= 256 and tx*ty = 256*ept: fixed walks
  int va, vb;             // dense == 4 (vtile_kernel): vector widths along x in A / y in B
  int sh;                 // dense == 4: bit 0 A rows shifted, bit 1 B columns shifted (vtile.cuh)
  // dense == 5 (btile_kernel, bulk-copy ring): stages, A row / B column pitch
  // in shared memory (bytes, multiples of 16), consumer lanes along y
  uint32_t ns, pa, pb, ly;
  // order >= 2: tiles walked in groups of `order` tile rows (Y chunks), X
  // chunks next, so the tiles in flight at once form a block whose A rows and
  // B columns continue across tiles (longer DRAM runs on both sides)
  uint32_t grp;
  Div32 dplane, dgrp, dG;  // nxc*nyc, grp*nxc, grp
  Div32 dcol;              // dense == 5, linear walk: S*ty (tile column length)
  int runs;                // dense == 5: bit 0 A tile rows / bit 1 B tile columns may be contiguous
  unsigned int* ctr;       // dense == 5: [next tile, CTAs done] for dynamic tile scheduling, or null
  uint32_t xp, xm;         // dense == 5, linear walk: X0 extent and tx / xp (xp 0: natural column order)
  Div32 dxm;               // divisor xm
  // dense == 5: bit 0 the A tile arrives by tensor map, bit 1 (beta != 0) the B
  // tile.  A side: A seen as [X (contiguous, one dim), Y0, carrier]; when Y0's
  // stride is not a multiple of 16 bytes its rows split into `ca` phase
  // classes (y mod ca), each a map whose rows are 16-byte aligned apart, one
  // box per class per tile ([cola, rowa, 1]) landing in its own region of the
  // tile; B side likewise over columns ([colb, rowb, 1], `cb` classes).
  // Ranks of the maps and the element strides their carrier coordinates
  // divide the outer offsets by.
  int tma, tra, trb;
  int64_t tca, tcb;
  uint32_t ca, cola, rowa, cb, colb, rowb;
  uint32_t abytes, bbytes;  // dense == 5: bytes of the A tile / B tile regions of a stage
};

// kTma: the tensor-map tile (tma.cuh).  One TMA box per tile and side: the A
// tile [by][bx] (x fastest) is loaded from A's map, transposed through shared
// memory into the B tile [bx][by], and stored through B's map (with beta != 0
// the B tile is first loaded through the same map).  Each map is the tensor
// seen from one side: its dims are the tile's axes with box > 1 (runs that are
// contiguous in that tensor merged) plus one "carrier" dim that takes every
// axis the tile covers with extent 1, folded as coordinate multiples (a
// larger stride is always a whole multiple of the smallest one).
constexpr int kTmaMaxRank = 5;
constexpr int kTmaLevels = 12;
constexpr int kTmaMaxStages = 8;
struct TmaView {
  int rank = 0;
  int esz = 4;                 // map element bytes (4 or 8; 16-byte kinds as 2 x 8)
  uint64_t dim[kTmaMaxRank];   // elements
  uint64_t stride[kTmaMaxRank];  // bytes (stride[0] unused)
  uint32_t box[kTmaMaxRank];
};
struct TmaPlan {
  TmaView va, vb;
  Scale sc;
  uint32_t bx, by;          // tile extents along X / Y (flattened, OOB included)
  uint32_t S;               // case 1: shared stride-1 run per (x, y) (1 in case 2)
  uint32_t items;           // tiles
  int nlev;                 // tile-index levels (mixed radix, first fastest)
  Div32 lev[kTmaLevels];
  int dimA[kTmaLevels], dimB[kTmaLevels];  // map dim a level's digit feeds
  int32_t mulA[kTmaLevels], mulB[kTmaLevels];
  uint32_t ns, nsb;         // A ring / B ring slots
  uint32_t tile_a, tile_b;  // bytes of one A / B tile in shared memory (128-B rounded)
  // case 2: micro-tiles per tile and warp tiles (2^wxl x 2^(5-wxl) micro-tiles each)
  uint32_t mx, my, nwx, nwt, wxl;
  Div32 dnwx;
  // case 1: 16-byte chunks per run, divisors for the (chunk, y, x) walk
  uint32_t kch;
  Div32 dk, dby;
};
// the tensor-map sides of a bulk tile: per side up to 4 phase-class maps
constexpr int kBtileMaxClasses = 4;
struct BtileTma {
  // per class; dim[0] holds the row length (map elements) before the launch
  // adds the class's start shift and rounds up to 16 bytes
  TmaView a[kBtileMaxClasses], b[kBtileMaxClasses];
  int64_t row_bytes_a = 0, row_bytes_b = 0;  // A stride of Y0 / B stride of X0 (class r starts r rows in)
  int ea = 4, eb = 4;                        // tensor element bytes of A / B
};
constexpr int kTmaConsumerWarps = 4;
// TmaPlan::wxl value of the diagonal lane map (8 x 8 micro-tile blocks, half per warp step)
constexpr uint32_t kTmaDiagonal = 6;
constexpr int kTmaStoreWarps = 2;

// btile_kernel warp roles: consumer warps write B; producer warps issue the
// bulk copies (issued per warp through the uniform datapath, one lane's copy
// at a time, so the issue rate scales with producer warps, not lanes)
constexpr int kBtileConsumerWarps = 4;
constexpr int kBtileProducerWarps = 4;
// tiles of 32 KB and more (one CTA per SM): kern_btile_big.cu
constexpr int kBtileBigConsumerWarps = 8;
constexpr int kBtileBigProducerWarps = 4;
constexpr int kBtileBigTileBytes = 32 * 1024;

// btile_kernel shared-memory layout of one stage (offsets multiples of `al`:
// 16, or 128 when a tile side arrives by tensor map):
//   header     u32 tile index of the stage (>= items: no more tiles), 16 bytes
//   rbase[ty]  u32: element index of tile row y's first element in the A tile
//   boff[tx]   u32: B element offset of tile column x's first element
//   cbase[tx]  u32: (beta != 0) element index of column x in the B tile
//   A tile     ty rows of pa bytes
//   B tile     (beta != 0) tx columns of pb bytes
TTB_HD uint32_t btile_round(uint32_t v, uint32_t al) { return (v + al - 1u) & ~(al - 1u); }
TTB_HD uint32_t btile_tables_bytes(uint32_t tx, uint32_t ty, bool upd, uint32_t al = 16u) {
  return btile_round(16u + (ty + tx * (upd ? 2u : 1u)) * 4u, al);  // 16: tile-index header
}
TTB_HD uint32_t btile_a_bytes(uint32_t ty, uint32_t pa, uint32_t al = 16u) { return btile_round(ty * pa, al); }
// a side by tensor map: `classes` boxes of rows x cols elements of e bytes, each 128-byte aligned
TTB_HD uint32_t btile_class_bytes(uint32_t rows, uint32_t cols, uint32_t e) { return btile_round(rows * cols * e, 128u); }
// abytes / bbytes: the A tile / B tile regions (SmemParams::abytes, bbytes)
TTB_HD uint32_t btile_stage_bytes(uint32_t tx, uint32_t ty, uint32_t abytes, uint32_t bbytes, bool upd,
                                  uint32_t al = 16u) {
  return btile_round(btile_tables_bytes(tx, ty, upd, al) + btile_round(abytes, al) + (upd ? bbytes : 0u), al);
}

// btile_kernel column elements per consumer lane (template JY: 1, 2, 4, 8 or 16)
TTB_HD int btile_rows_per_lane(uint32_t col, uint32_t ly) {  // col = S*ty
  const uint32_t n = (col + ly - 1) / ly;
  return n <= 1 ? 1 : n <= 2 ? 2 : n <= 4 ? 4 : n <= 8 ? 8 : 16;
}

// copy_rows_kernel: vectors per lane in one warp item (4 KB per warp for
// vectors of up to 16 bytes; 8 for wider ones)
TTB_HD constexpr int rows_item_vectors(int vector_bytes) {
  return vector_bytes >= 16 ? 8 : 8 * (16 / vector_bytes);
}

// Launch shape chosen by the planner.
struct Launch {
  int grid = 0, block = 256;
  int smem = 0;
};

}  // namespace ttb
