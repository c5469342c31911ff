// shard.cpp -- multi-GPU partition of the output.
//
// Every element of B depends on exactly one element of A (executor.hpp:33-40),
// so any partition of B's index space is independent: no exchange, no
// collective on the data path.  Rank r receives a contiguous range of the
// flattened index over the k slowest "split axes", with k the smallest whose
// extent product splits across `world` ranks within 5% of perfect balance;
// the range decomposes into at most 2k-1 boxes of the original index space.
// Split axes are B's positions from the outermost, except that A's and B's
// stride-1 axes come last: cutting either one cuts the contiguous runs the
// tiles read and write (c5_t18's outermost B index is A's stride-1 axis of
// extent 10 -- pieces of 1-2 elements -- measured 3.6x at 8 ranks instead of
// 7x, scripts/predict_scaling.py).  An axis of that order that splits within
// 7% of perfect balance by itself is taken alone (one box per rank).  A rank's
// B region is a slab whenever the split axes are B's outermost positions.
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ttb.h"
#include "problem.hpp"

namespace {

struct Box {
  std::vector<int64_t> origin, extent;  // B position order
};

// boxes covering flattened range [lo, hi) over dims[d..] (slowest first)
void split(const std::vector<int64_t>& ext, size_t d, int64_t lo, int64_t hi, Box cur,
           std::vector<Box>& out) {
  if (lo >= hi) return;
  int64_t inner = 1;
  for (size_t j = d + 1; j < ext.size(); ++j) inner *= ext[j];
  if (d + 1 == ext.size()) {
    cur.origin[d] = lo;
    cur.extent[d] = hi - lo;
    out.push_back(cur);
    return;
  }
  int64_t a = lo / inner;
  const int64_t b = hi / inner;
  if (a == b) {
    cur.origin[d] = a;
    cur.extent[d] = 1;
    split(ext, d + 1, lo - a * inner, hi - a * inner, cur, out);
    return;
  }
  if (lo % inner) {
    Box head = cur;
    head.origin[d] = a;
    head.extent[d] = 1;
    split(ext, d + 1, lo % inner, inner, head, out);
    ++a;
  }
  if (a < b) {
    Box mid = cur;
    mid.origin[d] = a;
    mid.extent[d] = b - a;
    for (size_t j = d + 1; j < ext.size(); ++j) {
      mid.origin[j] = 0;
      mid.extent[j] = ext[j];
    }
    out.push_back(mid);
  }
  if (hi % inner) {
    Box tail = cur;
    tail.origin[d] = b;
    tail.extent[d] = 1;
    split(ext, d + 1, 0, hi % inner, tail, out);
  }
}

}  // namespace

extern "C" int ttb_shard_boxes(int rank, const int* perm, const int64_t* sizes, int world, int r,
                               int64_t* origins, int64_t* extents, int* n_boxes) {
  if (rank < 1 || rank > 64 || !perm || !sizes || world < 1 || r < 0 || r >= world || !n_boxes)
    return TTB_EINVAL;
  std::vector<int> inv(static_cast<size_t>(rank), -1);
  for (int a = 0; a < rank; ++a) {
    if (perm[a] < 1 || perm[a] > rank || inv[static_cast<size_t>(perm[a] - 1)] >= 0) return TTB_EINVAL;
    inv[static_cast<size_t>(perm[a] - 1)] = a;
  }
  // split axes (A axis ids), slowest first: B positions outermost first,
  // A's stride-1 axis (A axis 0) and B's (B position 0) moved to the end
  std::vector<int> order;
  for (int p = rank - 1; p >= 0; --p) {
    const int a = inv[static_cast<size_t>(p)];
    if (a != 0 && p != 0) order.push_back(a);
  }
  for (int p = rank - 1; p >= 0; --p) {
    const int a = inv[static_cast<size_t>(p)];
    if (a == 0 || p == 0) order.push_back(a);
  }
  // One axis that splits evenly on its own is preferred: one box (one launch)
  // per rank instead of up to 2k-1 small ones.  Candidates in the order above;
  // a stride-1 axis only when a rank's piece of it stays long (>= 512 elements).
  // Measured with scripts/predict_scaling.py at 8 ranks: c5_t09 cut along its
  // extent-1016 axis (127 each) instead of three boxes over (34, 1016), c5_t22
  // along 53 (7 or 6 each) instead of three boxes over (53, 542).
  // The outermost candidate within 2% of perfect balance, else the best
  // balanced one within 7%.
  {
    int pick = -1;
    double best = 1.07;
    for (int a : order) {
      const bool lead = a == 0 || perm[a] == 1;
      const int64_t n = sizes[a], per = (n + world - 1) / world;
      if (lead && n / world < 512) continue;
      const double imb = static_cast<double>(per) * world / static_cast<double>(n);
      if (imb <= 1.02) {
        pick = a;
        break;
      }
      if (imb < best) {
        best = imb;
        pick = a;
      }
    }
    if (pick >= 0) order.assign(1, pick);
  }
  std::vector<int64_t> outer;
  int k = 0;
  int64_t F = 1;
  for (int a : order) {
    F *= sizes[a];
    outer.push_back(sizes[a]);
    ++k;
    const int64_t per = (F + world - 1) / world;
    if (static_cast<double>(per) * world / static_cast<double>(F) <= (order.size() == 1 ? 1.07 : 1.05)) break;
  }
  const int64_t lo = F * r / world, hi = F * (r + 1) / world;
  Box base;
  base.origin.assign(outer.size(), 0);
  base.extent.assign(outer.size(), 0);
  std::vector<Box> boxes;
  split(outer, 0, lo, hi, base, boxes);
  *n_boxes = static_cast<int>(boxes.size());
  if (!origins || !extents) return TTB_OK;
  for (size_t i = 0; i < boxes.size(); ++i) {
    for (int a = 0; a < rank; ++a) {
      origins[i * rank + a] = 0;
      extents[i * rank + a] = sizes[a];
    }
    for (int j = 0; j < k; ++j) {
      const int a = order[static_cast<size_t>(j)];
      origins[i * rank + a] = boxes[i].origin[static_cast<size_t>(j)];
      extents[i * rank + a] = boxes[i].extent[static_cast<size_t>(j)];
    }
  }
  return TTB_OK;
}
