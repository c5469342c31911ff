// problem.hpp -- host-side problem model of the engine.
//
// B200 counterpart of ttune's problem layer (proj/core/include/ttune/problem.hpp):
// the same validation rules and messages, the same index-merging fixpoint and
// the same cache key, re-expressed as a small value type the planner and the
// kernels consume.  Everything here runs on the host.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace ttb {

constexpr int kMaxRank = 16;  // TTB_MAX_RANK

enum class Kind : int { S = 0, D = 1, C = 2, Z = 3 };

inline int kind_bytes(int k) { return k == 0 ? 4 : (k == 3 ? 16 : 8); }
inline int kind_components(int k) { return (k == 2 || k == 3) ? 2 : 1; }
inline bool kind_double(int k) { return k == 1 || k == 3; }
inline int scalar_bytes(int k) { return kind_double(k) ? 8 : 4; }
inline char kind_letter(int k) { return "sdcz?"[(k >= 0 && k < 4) ? k : 4]; }

// Thrown for anything ttune reports as std::invalid_argument; the C ABI maps it
// to TTB_EINVAL with the message preserved.
struct InvalidArgument {
  std::string what;
};

// A transposition problem exactly as ttune::TransposeProblem holds it
// (problem.hpp:37-49): scatter perm (1-based), sizes/lda in A order, ldb in B
// order, real alpha/beta, element kinds.
struct Problem {
  std::vector<int> perm;
  std::vector<int64_t> sizes, lda, ldb;
  int kind_a = 0, kind_b = 0;
  double alpha = 1.0, beta = 0.0;

  int rank() const { return static_cast<int>(perm.size()); }
  int64_t elements() const;                 // logical element count
  std::vector<int64_t> b_extents() const;   // sizes_b (problem.cpp:161-168)
  std::vector<int64_t> a_strides() const;   // element_strides_a
  std::vector<int64_t> b_strides_of_a() const;  // element_strides_b_for_a
  int64_t footprint_a() const;              // required_elements_a
  int64_t footprint_b() const;              // required_elements_b
};

// make_problem defaults (problem.cpp:85-105): empty lda -> sizes; empty ldb ->
// sizes_b when the perm is valid and sizes has the right length.
Problem make(std::vector<int> perm, std::vector<int64_t> sizes, int kind_a, int kind_b,
             double alpha, double beta, std::vector<int64_t> lda, std::vector<int64_t> ldb);

// validate (problem.cpp:107-159): throws InvalidArgument with the reference's text
void check(const Problem& p);

// canonical_key (problem.cpp:228-241)
std::string cache_key(const Problem& p);

// merge_indices (problem.cpp:270-340).  `runs` holds, per merged index, the
// 1-based first/last original A index it covers.
struct Merged {
  Problem p;
  std::vector<std::pair<int, int>> runs;
};
Merged fuse_indices(const Problem& p);

}  // namespace ttb
