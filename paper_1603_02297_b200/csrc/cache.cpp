// cache.cpp -- the reference's SolutionCache file format (tuner.cpp:81-205)
// and its benchmark-suite generator (benchmark.cpp:17-220), restated for the
// engine's host side.
#include "cache.hpp"

#include <fcntl.h>
#include <sys/file.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>

#include "problem.hpp"

namespace ttb {

namespace {

constexpr char kSep = '\t';

bool single_line(const std::string& s) {
  return !s.empty() && s.find_first_of("\t\n\r") == std::string::npos;
}

bool parse_line(const std::string& line, CacheEntry* e) {
  std::vector<std::string> f;
  size_t start = 0;
  while (f.size() < 5) {
    const size_t pos = line.find(kSep, start);
    if (pos == std::string::npos) {
      f.push_back(line.substr(start));
      break;
    }
    f.push_back(line.substr(start, pos - start));
    start = pos + 1;
  }
  if (f.size() != 5) return false;
  for (const std::string& x : f)
    if (x.empty()) return false;
  errno = 0;
  char* end = nullptr;
  const double bw = std::strtod(f[3].c_str(), &end);
  if (end != f[3].c_str() + f[3].size() || errno != 0) return false;
  e->problem_key = f[0];
  e->hardware_key = f[1];
  e->plan = f[2];
  e->bandwidth_gibs = bw;
  e->timestamp = f[4];
  return true;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);  // also drops the flock
  }
};

}  // namespace

bool cache_lookup(const std::string& file, const std::string& problem_key,
                  const std::string& hardware_key, CacheEntry* out) {
  Fd f;
  f.fd = ::open(file.c_str(), O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return false;
  if (::flock(f.fd, LOCK_SH) != 0) throw std::runtime_error("cache: lock failed");
  std::string text;
  char buf[1 << 16];
  ssize_t got;
  while ((got = ::read(f.fd, buf, sizeof buf)) > 0) text.append(buf, static_cast<size_t>(got));
  if (got < 0) throw std::runtime_error("cache: read failed");
  bool found = false;
  int bad = 0;
  size_t start = 0;
  while (start < text.size()) {
    size_t nl = text.find('\n', start);
    if (nl == std::string::npos) nl = text.size();
    const std::string line = text.substr(start, nl - start);
    start = nl + 1;
    if (line.empty()) continue;
    CacheEntry e;
    if (!parse_line(line, &e)) {
      ++bad;
      continue;
    }
    if (e.problem_key == problem_key && e.hardware_key == hardware_key) {
      *out = e;
      found = true;
    }
  }
  if (bad > 0)
    std::fprintf(stderr, "warning: cache %s: skipped %d malformed line(s)\n", file.c_str(), bad);
  return found;
}

void cache_store(const std::string& file, const CacheEntry& e) {
  if (!single_line(e.problem_key) || !single_line(e.hardware_key) || !single_line(e.plan) ||
      !single_line(e.timestamp))
    throw InvalidArgument{"cache: entry fields must be non-empty single-line text"};
  char bw[64];
  std::snprintf(bw, sizeof bw, "%.17g", e.bandwidth_gibs);
  const std::string line = e.problem_key + kSep + e.hardware_key + kSep + e.plan + kSep + bw +
                           kSep + e.timestamp + '\n';
  Fd f;
  f.fd = ::open(file.c_str(), O_WRONLY | O_CREAT | O_APPEND | O_CLOEXEC, 0644);
  if (f.fd < 0) throw std::runtime_error("cache: cannot open " + file);
  if (::flock(f.fd, LOCK_EX) != 0) throw std::runtime_error("cache: lock failed");
  size_t off = 0;
  while (off < line.size()) {
    const ssize_t put = ::write(f.fd, line.data() + off, line.size() - off);
    if (put < 0) throw std::runtime_error("cache: write failed");
    off += static_cast<size_t>(put);
  }
}

std::string iso8601_utc_now() {
  const std::time_t now = std::time(nullptr);
  std::tm tm{};
  gmtime_r(&now, &tm);
  char buf[32];
  std::strftime(buf, sizeof buf, "%Y-%m-%dT%H:%M:%SZ", &tm);
  return buf;
}

// --------------------------------------------------------------- suite --

namespace {

// uniform draw in [0, n) by rejection (benchmark.cpp:19-24)
uint64_t below(std::mt19937_64& g, uint64_t n) {
  const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
  uint64_t v = g();
  while (v >= lim) v = g();
  return v % n;
}

std::vector<int> reversed(int d) {
  std::vector<int> p(static_cast<size_t>(d));
  for (int i = 0; i < d; ++i) p[static_cast<size_t>(i)] = d - i;
  return p;
}

// perms (1-based maps, lexicographic order) with no adjacent +1 pair, i.e.
// nothing merge_indices could fuse; stride-1 keepers start with 1 and are not
// the identity, the general ones move index 1 and are not the reversal
std::vector<std::vector<int>> candidates_of(int d, bool keep_stride1) {
  std::vector<int> p(static_cast<size_t>(d));
  std::iota(p.begin(), p.end(), 1);
  const std::vector<int> rev = reversed(d);
  std::vector<std::vector<int>> out;
  do {
    bool fusable = false;
    for (size_t a = 0; a + 1 < p.size(); ++a) fusable = fusable || p[a + 1] == p[a] + 1;
    if (fusable) continue;
    if (keep_stride1) {
      bool ident = true;
      for (size_t i = 0; i < p.size(); ++i) ident = ident && p[i] == static_cast<int>(i) + 1;
      if (p[0] == 1 && !ident) out.push_back(p);
    } else if (p[0] != 1 && p != rev) {
      out.push_back(p);
    }
  } while (std::next_permutation(p.begin(), p.end()));
  return out;
}

double deviation(const std::vector<int64_t>& s, int64_t target) {
  int64_t n = 1;
  for (int64_t e : s) n *= e;
  return std::fabs(static_cast<double>(n) / static_cast<double>(target) - 1.0);
}

// extents near the d-th root of the element count; `skew` (>= 0) is 6x the
// others; one axis absorbs the rounding (benchmark.cpp:73-99)
std::vector<int64_t> shape(int d, int64_t target, int skew) {
  const double scale = skew < 0 ? 1.0 : 6.0;
  const double root = std::pow(static_cast<double>(target) / scale, 1.0 / d);
  std::vector<int64_t> best;
  double best_dev = 1e300;
  for (int bump = 0; bump < 2; ++bump) {
    const int64_t s = std::max<int64_t>(2, static_cast<int64_t>(root) + bump);
    std::vector<int64_t> v(static_cast<size_t>(d), s);
    int adj = d - 1;
    if (skew >= 0) {
      v[static_cast<size_t>(skew)] = 6 * s;
      if (adj == skew) adj = d - 2;
    }
    int64_t rest = 1;
    for (int i = 0; i < d; ++i)
      if (i != adj) rest *= v[static_cast<size_t>(i)];
    v[static_cast<size_t>(adj)] = std::max<int64_t>(
        2, static_cast<int64_t>(std::llround(static_cast<double>(target) / static_cast<double>(rest))));
    const double dev = deviation(v, target);
    if (dev < best_dev) {
      best_dev = dev;
      best = v;
    }
  }
  return best;
}

template <class T>
std::string joined(const std::vector<T>& v, char sep) {
  std::ostringstream os;
  for (size_t i = 0; i < v.size(); ++i) os << (i ? std::string(1, sep) : "") << v[i];
  return os.str();
}

}  // namespace

std::vector<std::string> benchmark_manifest(int64_t volume_bytes, int kind, uint64_t seed) {
  if (volume_bytes < (1 << 20)) throw InvalidArgument{"benchmark: volume must be at least 1 MiB"};
  if (kind < 0 || kind > 3) throw InvalidArgument{"benchmark: bad element kind"};
  const int64_t target = volume_bytes / kind_bytes(kind);
  std::mt19937_64 g(seed);
  std::vector<std::pair<std::vector<int>, const char*>> perms;
  perms.emplace_back(reversed(2), "inverse");
  for (int d = 3; d <= 6; ++d) {
    perms.emplace_back(reversed(d), "inverse");
    const auto keep = candidates_of(d, true);
    perms.emplace_back(keep[below(g, keep.size())], "stride1");
    const auto gen = candidates_of(d, false);
    const int want = d == 3 ? 1 : 3;
    std::vector<std::vector<int>> chosen;
    while (static_cast<int>(chosen.size()) < want) {
      const auto& pick = gen[below(g, gen.size())];
      if (std::find(chosen.begin(), chosen.end(), pick) == chosen.end()) chosen.push_back(pick);
    }
    for (auto& c : chosen) perms.emplace_back(c, "general");
  }
  std::vector<std::string> lines;
  const char kc = kind_letter(kind);
  for (const auto& [perm, category] : perms) {
    const int d = static_cast<int>(perm.size());
    int inv0 = 0;  // the A index that lands on B's first position
    for (int a = 0; a < d; ++a)
      if (perm[static_cast<size_t>(a)] == 1) inv0 = a;
    const std::pair<const char*, int> configs[] = {{"balanced", -1}, {"skewA", 0}, {"skewB", inv0}};
    for (const auto& [cname, skew] : configs) {
      const std::vector<int64_t> sizes = shape(d, target, skew);
      if (deviation(sizes, target) > 0.10)
        throw std::runtime_error("benchmark: volume too small for a ratio-6 shape at dimension " +
                                 std::to_string(d));
      std::string id = "d" + std::to_string(d) + "_";
      for (int v : perm) id += std::to_string(v);
      id += std::string("_") + cname;
      lines.push_back("case=" + id + ";perm=" + joined(perm, ',') + ";size=" + joined(sizes, ',') +
                      ";kinds=" + std::string(2, kc) + ";alpha=1;beta=1;category=" + category +
                      ";config=" + cname);
    }
  }
  return lines;
}

}  // namespace ttb
