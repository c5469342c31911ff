// problem.cpp -- validation, geometry, cache key and index fusion.
// Rules and messages follow ttune (proj/core/src/problem.cpp); the code is a
// fresh implementation over a per-index record list.
#include "problem.hpp"

#include <algorithm>
#include <cstdio>

namespace ttb {

namespace {

std::string fmt(const char* f, long long a, long long b = 0, long long c = 0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, f, a, b, c);
  return buf;
}

bool is_bijection(const std::vector<int>& perm) {
  const int n = static_cast<int>(perm.size());
  std::vector<char> hit(static_cast<size_t>(n), 0);
  for (int v : perm) {
    if (v < 1 || v > n || hit[static_cast<size_t>(v - 1)]) return false;
    hit[static_cast<size_t>(v - 1)] = 1;
  }
  return n > 0;
}

std::vector<int64_t> scatter(const std::vector<int>& perm, const std::vector<int64_t>& v) {
  std::vector<int64_t> out(perm.size());
  for (size_t a = 0; a < perm.size(); ++a) out[static_cast<size_t>(perm[a] - 1)] = v[a];
  return out;
}

std::vector<int64_t> column_major_strides(const std::vector<int64_t>& ld) {
  std::vector<int64_t> st(ld.size());
  int64_t acc = 1;
  for (size_t i = 0; i < ld.size(); ++i) {
    st[i] = acc;
    acc *= ld[i];
  }
  return st;
}

int64_t span_of(const std::vector<int64_t>& ext, const std::vector<int64_t>& st) {
  int64_t last = 0;
  for (size_t i = 0; i < ext.size(); ++i) last += (ext[i] - 1) * st[i];
  return last + 1;
}

}  // namespace

int64_t Problem::elements() const {
  int64_t n = 1;
  for (int64_t s : sizes) n *= s;
  return n;
}

std::vector<int64_t> Problem::b_extents() const { return scatter(perm, sizes); }

std::vector<int64_t> Problem::a_strides() const { return column_major_strides(lda); }

std::vector<int64_t> Problem::b_strides_of_a() const {
  const std::vector<int64_t> by_pos = column_major_strides(ldb);
  std::vector<int64_t> out(perm.size());
  for (size_t a = 0; a < perm.size(); ++a) out[a] = by_pos[static_cast<size_t>(perm[a] - 1)];
  return out;
}

int64_t Problem::footprint_a() const { return span_of(sizes, a_strides()); }

int64_t Problem::footprint_b() const { return span_of(b_extents(), column_major_strides(ldb)); }

Problem make(std::vector<int> perm, std::vector<int64_t> sizes, int kind_a, int kind_b,
             double alpha, double beta, std::vector<int64_t> lda, std::vector<int64_t> ldb) {
  Problem p;
  p.perm = std::move(perm);
  p.sizes = std::move(sizes);
  p.kind_a = kind_a;
  p.kind_b = kind_b;
  p.alpha = alpha;
  p.beta = beta;
  p.lda = lda.empty() ? p.sizes : std::move(lda);
  if (!ldb.empty())
    p.ldb = std::move(ldb);
  else if (is_bijection(p.perm) && p.sizes.size() == p.perm.size())
    p.ldb = p.b_extents();
  return p;
}

void check(const Problem& p) {
  const int n = p.rank();
  if (n < 1) throw InvalidArgument{"perm: empty permutation"};
  if (!is_bijection(p.perm)) throw InvalidArgument{fmt("perm: not a permutation of 1..%lld", n)};
  const struct {
    const char* name;
    size_t got;
  } lens[3] = {{"sizes", p.sizes.size()}, {"lda", p.lda.size()}, {"ldb", p.ldb.size()}};
  for (const auto& l : lens)
    if (static_cast<int>(l.got) != n) {
      char buf[128];
      std::snprintf(buf, sizeof buf, "%s: expected %d entries, got %zu", l.name, n, l.got);
      throw InvalidArgument{buf};
    }
  for (int m = 0; m < n; ++m) {
    if (p.sizes[m] < 1) throw InvalidArgument{fmt("sizes[%lld] = %lld < 1", m + 1, p.sizes[m])};
    if (p.lda[m] < p.sizes[m])
      throw InvalidArgument{fmt("lda[%lld] = %lld < size %lld", m + 1, p.lda[m], p.sizes[m])};
  }
  const std::vector<int64_t> eb = p.b_extents();
  for (int k = 0; k < n; ++k)
    if (p.ldb[k] < eb[k])
      throw InvalidArgument{fmt("ldb[%lld] = %lld < size %lld", k + 1, p.ldb[k], eb[k])};
  const bool kinds_ok = p.kind_a >= 0 && p.kind_a < 4 && p.kind_b >= 0 && p.kind_b < 4 &&
                        kind_components(p.kind_a) == kind_components(p.kind_b);
  if (!kinds_ok) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "dataType: unsupported kind pair %c%c", kind_letter(p.kind_a),
                  kind_letter(p.kind_b));
    throw InvalidArgument{buf};
  }
  int64_t volume = 1;
  const int64_t cap = int64_t{1} << 62;
  for (int m = 0; m < n; ++m) {
    if (p.lda[m] > cap / std::max<int64_t>(volume, 1)) throw InvalidArgument{"sizes: volume overflow"};
    volume *= p.lda[m];
  }
}

std::string cache_key(const Problem& p) {
  std::string s = "perm=";
  auto list = [&s](const auto& v) {
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) s += ',';
      s += std::to_string(v[i]);
    }
  };
  list(p.perm);
  s += ";size=";
  list(p.sizes);
  s += ";lda=";
  list(p.lda);
  s += ";ldb=";
  list(p.ldb);
  s += ";kinds=";
  s += kind_letter(p.kind_a);
  s += kind_letter(p.kind_b);
  s += p.beta == 0.0 ? ";beta=z" : ";beta=nz";
  return s;
}

namespace {

// one A index during fusion: extent, A leading dim, 1-based B position and
// the original A indices it stands for
struct Idx {
  int64_t ext, lda;
  int pos;
  int first, last;
};

struct Fusion {
  std::vector<Idx> a;          // A order
  std::vector<int64_t> ldb;    // B order

  // delete A index i, whose B position is a.pos; later B positions move down
  void remove(size_t i) {
    const int k = a[i].pos;
    a.erase(a.begin() + static_cast<long>(i));
    ldb.erase(ldb.begin() + (k - 1));
    for (Idx& x : a)
      if (x.pos > k) --x.pos;
  }
};

}  // namespace

Merged fuse_indices(const Problem& p) {
  check(p);
  Fusion f;
  for (int i = 0; i < p.rank(); ++i)
    f.a.push_back({p.sizes[i], p.lda[i], p.perm[i], i + 1, i + 1});
  f.ldb = p.ldb;

  // (1) extent-1 indices vanish (problem.cpp:282-304).  The stride-1 index of
  // a tensor may only go if it is unpadded; an interior index hands its
  // leading dimension to the next-inner index so outer strides are kept.
  for (bool again = true; again && f.a.size() > 1;) {
    again = false;
    for (size_t i = 0; i < f.a.size() && f.a.size() > 1; ++i) {
      const Idx& x = f.a[i];
      if (x.ext != 1) continue;
      const size_t n = f.a.size();
      const int k = x.pos;
      if (i == 0 && x.lda != 1) continue;
      if (k == 1 && f.ldb[0] != 1) continue;
      if (i > 0 && i + 1 < n) f.a[i - 1].lda *= x.lda;
      if (k > 1 && k < static_cast<int>(n)) f.ldb[static_cast<size_t>(k - 2)] *= f.ldb[static_cast<size_t>(k - 1)];
      if (i > 0)
        f.a[i - 1].last = x.last;
      else
        f.a[1].first = x.first;
      f.remove(i);
      again = true;
      break;
    }
  }

  // (2) fuse i with i+1 when they are also adjacent (and in order) in B and i
  // is unpadded in both tensors (problem.cpp:306-327); sweep to a fixpoint
  for (bool again = true; again;) {
    again = false;
    for (size_t i = 0; i + 1 < f.a.size();) {
      Idx& x = f.a[i];
      const Idx& y = f.a[i + 1];
      const size_t kb = static_cast<size_t>(x.pos - 1);
      if (y.pos == x.pos + 1 && x.lda == x.ext && f.ldb[kb] == x.ext) {
        x.ext *= y.ext;
        x.lda *= y.lda;
        f.ldb[kb] *= f.ldb[kb + 1];
        x.last = y.last;
        f.remove(i + 1);
        again = true;
      } else {
        ++i;
      }
    }
  }

  Merged m;
  m.p = p;
  m.p.perm.clear();
  m.p.sizes.clear();
  m.p.lda.clear();
  for (const Idx& x : f.a) {
    m.p.perm.push_back(x.pos);
    m.p.sizes.push_back(x.ext);
    m.p.lda.push_back(x.lda);
    m.runs.emplace_back(x.first, x.last);
  }
  m.p.ldb = f.ldb;
  check(m.p);
  return m;
}

}  // namespace ttb
