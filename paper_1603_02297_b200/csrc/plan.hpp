// plan.hpp -- the sm_100a planner.
//
// Replaces ttune's CPU search space (proj/core/src/search.cpp:81-303: blocking,
// loop order, prefetch distance, streaming stores) with a GPU plan space:
// kernel variant (copy / register-transpose / smem-staged), the index groups
// that form each tile side (the planner's "merge small leading extents until
// a tile is full"), vector widths from alignment, warp/tile shape and tile
// order.  Candidates are ranked by a heuristic; ttb_plan_autotune measures
// them (tuner.cpp:27-64 analogue).
#pragma once

#include <string>
#include <vector>

#include "params.hpp"
#include "problem.hpp"

namespace ttb {

// Geometry of the MERGED problem in A axis order.
struct Geo {
  int r = 0;
  int64_t n[kMaxRank] = {}, sa[kMaxRank] = {}, sb[kMaxRank] = {};
  int pos[kMaxRank] = {};  // 0-based B position of A axis a
  int at[kMaxRank] = {};   // A axis sitting at B position k
  int ka = 0, kb = 0, C = 1, eA = 4, eB = 4;
  int mode = 0;            // 0 move, 1 scale, 2 update
  double alpha = 1.0, beta = 0.0;
  int64_t elements = 1;
  int64_t foot_a = 1, foot_b = 1;  // required_elements of A and B
};
Geo make_geo(const Problem& merged);

// One point of the plan space (serializable like ttune's CandidatePlan).
struct Spec {
  Variant v = kSmem;
  int w1 = 1, w2 = 1;  // copy: V = w1; rt: MX = w1, MY = w2
  int lx = 4;          // rt: lanes along X
  int kx = 1, ky = 1;  // axes in the X / Y index groups
  int tx = 0, ty = 0;  // smem tile extents along X / Y
  int order = 0;       // 0: X chunks fastest, 1: Y chunks fastest
  int occ = 0;         // CTAs per SM (0: occupancy limit)
  int st = 2;          // smem: cp.async pipeline stages (dense tiles: 2 or 3)
  int bp = 1;          // smem, beta != 0: B through the cp.async ring (1) or direct (0)
  int vec = 1;         // smem: vector tile kernel where the strides allow it (0: element-wise)
  int xp = 0;          // smem, linear-walk bulk tile: walk X's second axis first (in the text only when 1)
  int ly = 0;          // smem, column-walk bulk tile: lanes along a column (0: up to 32; text only when set)
  int sb = 0;          // tma: B ring slots (0: as many as A stages `st`; text only when set)
  int ts = 0;          // bulk tile: sides that arrive as one tensor-map box (1 A, 2 B; text only when set)
  int bulk = 0;        // copy: bulk rows in segments of this many KB (rowcopy_kernel, `st` stages; text only when set)
  double cost = 0;     // heuristic rank (lower first)

  std::string text() const;
  static bool parse(const std::string& s, Spec* out);
};

// Ready-to-launch form of a Spec (buffer pointers are filled at execution).
struct Prepared {
  Spec spec;
  int mode = 0;
  Launch l;
  CopyParams cp{};
  RtParams rp{};
  SmemParams sp{};
  TmaPlan tp{};
  BtileTma bt{};  // bulk tile: the tensor-map sides' class views
  int a_align = 1, b_align = 1;  // required base alignment (bytes) of A and B
};

// ranked candidate list; the last entry is always an smem plan that needs
// only element alignment (the fallback for misaligned buffers)
std::vector<Spec> candidates(const Geo& g);

// builds launch parameters; false (with a reason) if the spec does not apply
bool prepare(const Geo& g, const Spec& s, int sms, Prepared* out, std::string* why);

}  // namespace ttb
