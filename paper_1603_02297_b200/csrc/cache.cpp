// cache.cpp -- persistent plan store and the paper's benchmark-suite manifest.
//
// The store keeps the reference's on-disk contract (SolutionCache,
// tuner.cpp:81-205) so files move between the two: one entry per line, five
// tab-separated fields  problem_key, hardware_key, plan, GiB/s ("%.17g"),
// ISO-8601 UTC time; a line that does not split into five non-empty fields
// (the fifth takes the rest of the line) or whose GiB/s is not a whole
// number is skipped and counted in one warning on stderr; the last entry for
// a (problem, hardware) pair wins; appends take an exclusive flock, reads a
// shared one.  A reader may also require that the plan field parses as its
// own plan syntax (ttb_plan_tune_cached asks for a GPU plan): a line that
// fails it counts as malformed too, so it never shadows an earlier valid one.
//
// The suite manifest restates build_benchmark (benchmark.cpp:166-220): the
// same mt19937_64 draw sequence over the same lexicographic permutation
// lists, so it reproduces the reference's manifest line for line.
#include "cache.hpp"

#include <sys/file.h>

#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <random>
#include <stdexcept>
#include <string_view>

#include "problem.hpp"

namespace ttb {

namespace {

// ------------------------------------------------------------- the store --

// An open solution file holding a flock for its lifetime.
class LockedFile {
 public:
  LockedFile(const std::string& path, bool append) {
    fp_ = std::fopen(path.c_str(), append ? "ae" : "re");
    if (!fp_) {
      if (append) throw std::runtime_error("cache: cannot open " + path);
      return;  // no file yet: nothing stored
    }
    if (::flock(fileno(fp_), append ? LOCK_EX : LOCK_SH) != 0) {
      std::fclose(fp_);
      fp_ = nullptr;
      throw std::runtime_error("cache: lock failed");
    }
  }
  ~LockedFile() {
    if (fp_) std::fclose(fp_);  // closing drops the lock
  }
  LockedFile(const LockedFile&) = delete;
  LockedFile& operator=(const LockedFile&) = delete;
  std::FILE* get() const { return fp_; }

 private:
  std::FILE* fp_ = nullptr;
};

// the five fields of one line: the first four end at a tab, the fifth is
// the rest of the line; empty fields make the line malformed
bool split_entry(std::string_view line, std::string_view (&f)[5]) {
  for (int i = 0; i < 4; ++i) {
    const size_t tab = line.find('\t');
    if (tab == std::string_view::npos) return false;
    f[i] = line.substr(0, tab);
    line.remove_prefix(tab + 1);
  }
  f[4] = line;
  for (const std::string_view& x : f)
    if (x.empty()) return false;
  return true;
}

bool whole_number(std::string_view text, double* out) {
  const std::string s(text);
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(s.c_str(), &end);
  if (errno != 0 || end != s.c_str() + s.size()) return false;
  *out = v;
  return true;
}

bool one_line(const std::string& s) { return !s.empty() && s.find_first_of("\t\r\n") == std::string::npos; }

}  // namespace

bool cache_lookup(const std::string& file, const std::string& problem_key, const std::string& hardware_key,
                  CacheEntry* out, const std::function<bool(const std::string&)>& plan_ok) {
  LockedFile lf(file, false);
  if (!lf.get()) return false;
  bool found = false;
  int skipped = 0;
  char* buf = nullptr;
  size_t cap = 0;
  ssize_t n;
  while ((n = ::getline(&buf, &cap, lf.get())) >= 0) {
    std::string_view line(buf, static_cast<size_t>(n));
    if (!line.empty() && line.back() == '\n') line.remove_suffix(1);
    if (line.empty()) continue;
    std::string_view f[5];
    double gibs = 0.0;
    if (!split_entry(line, f) || !whole_number(f[3], &gibs) || (plan_ok && !plan_ok(std::string(f[2])))) {
      ++skipped;
      continue;
    }
    if (f[0] != problem_key || f[1] != hardware_key) continue;
    *out = CacheEntry{std::string(f[0]), std::string(f[1]), std::string(f[2]), gibs, std::string(f[4])};
    found = true;
  }
  const bool read_error = std::ferror(lf.get()) != 0;
  std::free(buf);
  if (read_error) throw std::runtime_error("cache: read failed");
  if (skipped) std::fprintf(stderr, "warning: cache %s: skipped %d malformed line(s)\n", file.c_str(), skipped);
  return found;
}

void cache_store(const std::string& file, const CacheEntry& e) {
  if (!one_line(e.problem_key) || !one_line(e.hardware_key) || !one_line(e.plan) || !one_line(e.timestamp))
    throw InvalidArgument{"cache: entry fields must be non-empty single-line text"};
  char gibs[64];
  std::snprintf(gibs, sizeof gibs, "%.17g", e.bandwidth_gibs);
  const std::string line =
      e.problem_key + '\t' + e.hardware_key + '\t' + e.plan + '\t' + gibs + '\t' + e.timestamp + '\n';
  LockedFile lf(file, true);
  // one write of the whole line under the exclusive lock (O_APPEND)
  if (std::fwrite(line.data(), 1, line.size(), lf.get()) != line.size() || std::fflush(lf.get()) != 0)
    throw std::runtime_error("cache: write failed");
}

std::string iso8601_utc_now() {
  const std::time_t t = std::chrono::system_clock::to_time_t(std::chrono::system_clock::now());
  std::tm u{};
  gmtime_r(&t, &u);
  char buf[32];
  std::snprintf(buf, sizeof buf, "%04d-%02d-%02dT%02d:%02d:%02dZ", u.tm_year + 1900, u.tm_mon + 1, u.tm_mday,
                u.tm_hour, u.tm_min, u.tm_sec);
  return buf;
}

// ------------------------------------------------------------- the suite --

namespace {

// unbiased draw in [0, n): reject the top partial block of the 64-bit range
struct SuiteDraws {
  std::mt19937_64 eng;
  explicit SuiteDraws(uint64_t seed) : eng(seed) {}
  uint64_t below(uint64_t n) {
    const uint64_t cut = UINT64_MAX - UINT64_MAX % n;
    for (;;) {
      const uint64_t v = eng();
      if (v < cut) return v % n;
    }
  }
};

// 1-based maps of rank d in lexicographic order, without an adjacent pair
// (m, m+1) -- nothing index merging could fuse -- pruned while building
void unmergeable_maps(int d, std::vector<int>* cur, std::vector<bool>* used, std::vector<std::vector<int>>* out) {
  if (static_cast<int>(cur->size()) == d) {
    out->push_back(*cur);
    return;
  }
  for (int v = 1; v <= d; ++v) {
    if ((*used)[static_cast<size_t>(v)] || (!cur->empty() && cur->back() + 1 == v)) continue;
    (*used)[static_cast<size_t>(v)] = true;
    cur->push_back(v);
    unmergeable_maps(d, cur, used, out);
    cur->pop_back();
    (*used)[static_cast<size_t>(v)] = false;
  }
}

std::vector<int> descending(int d) {
  std::vector<int> m;
  for (int v = d; v >= 1; --v) m.push_back(v);
  return m;
}

// stride-1 keepers: map[0] == 1 (and not the identity, which is mergeable
// anyway); general: map[0] != 1 and not the full reversal
std::vector<std::vector<int>> suite_maps(int d, bool keeps_stride1) {
  std::vector<std::vector<int>> all, out;
  std::vector<int> cur;
  std::vector<bool> used(static_cast<size_t>(d) + 1, false);
  unmergeable_maps(d, &cur, &used, &all);
  const std::vector<int> rev = descending(d);
  for (const std::vector<int>& m : all) {
    const bool first = m[0] == 1;
    if (keeps_stride1 ? first : (!first && m != rev)) out.push_back(m);
  }
  return out;
}

double off_target(const std::vector<int64_t>& ext, int64_t target) {
  int64_t p = 1;
  for (int64_t e : ext) p *= e;
  return std::fabs(static_cast<double>(p) / static_cast<double>(target) - 1.0);
}

// d extents of about target^(1/d) (the skew axis, if any, 6x its share);
// the last axis (the one before it when that is the skew axis) absorbs the
// rounding; of the floor root and the root + 1 the closer volume wins
std::vector<int64_t> suite_extents(int d, int64_t target, int skew) {
  const double side = std::pow(static_cast<double>(target) / (skew < 0 ? 1.0 : 6.0), 1.0 / d);
  const int fix = (skew == d - 1) ? d - 2 : d - 1;
  std::vector<int64_t> pick;
  double err = 1e300;
  for (int64_t s : {static_cast<int64_t>(side), static_cast<int64_t>(side) + 1}) {
    s = std::max<int64_t>(2, s);
    std::vector<int64_t> ext(static_cast<size_t>(d), s);
    if (skew >= 0) ext[static_cast<size_t>(skew)] = 6 * s;
    int64_t others = 1;
    for (int i = 0; i < d; ++i)
      if (i != fix) others *= ext[static_cast<size_t>(i)];
    ext[static_cast<size_t>(fix)] = std::max<int64_t>(
        2, static_cast<int64_t>(std::llround(static_cast<double>(target) / static_cast<double>(others))));
    const double e = off_target(ext, target);
    if (e < err) {
      err = e;
      pick = ext;
    }
  }
  return pick;
}

template <class T>
std::string comma_list(const std::vector<T>& v) {
  std::string s;
  for (const T& x : v) s += (s.empty() ? "" : ",") + std::to_string(x);
  return s;
}

}  // namespace

std::vector<std::string> benchmark_manifest(int64_t volume_bytes, int kind, uint64_t seed) {
  if (volume_bytes < (int64_t{1} << 20)) throw InvalidArgument{"benchmark: volume must be at least 1 MiB"};
  if (kind < 0 || kind > 3) throw InvalidArgument{"benchmark: bad element kind"};
  const int64_t target = volume_bytes / kind_bytes(kind);
  SuiteDraws draws(seed);
  struct Pick {
    std::vector<int> map;
    const char* category;
  };
  std::vector<Pick> picks{{descending(2), "inverse"}};
  for (int d = 3; d <= 6; ++d) {
    picks.push_back({descending(d), "inverse"});
    const std::vector<std::vector<int>> keep = suite_maps(d, true);
    picks.push_back({keep[draws.below(keep.size())], "stride1"});
    const std::vector<std::vector<int>> gen = suite_maps(d, false);
    std::vector<std::vector<int>> mine;
    while (static_cast<int>(mine.size()) < (d == 3 ? 1 : 3)) {
      const std::vector<int>& m = gen[draws.below(gen.size())];
      bool seen = false;
      for (const auto& q : mine) seen = seen || q == m;
      if (!seen) mine.push_back(m);
    }
    for (const auto& m : mine) picks.push_back({m, "general"});
  }
  std::vector<std::string> out;
  const std::string kinds(2, kind_letter(kind));
  for (const Pick& pk : picks) {
    const int d = static_cast<int>(pk.map.size());
    int b0 = 0;  // the A axis at B's first position (skewB widens it)
    while (pk.map[static_cast<size_t>(b0)] != 1) ++b0;
    for (const auto& [name, skew] : {std::pair<const char*, int>{"balanced", -1}, {"skewA", 0}, {"skewB", b0}}) {
      const std::vector<int64_t> ext = suite_extents(d, target, skew);
      if (off_target(ext, target) > 0.10)
        throw std::runtime_error("benchmark: volume too small for a ratio-6 shape at dimension " + std::to_string(d));
      std::string id = "d" + std::to_string(d) + "_";
      for (int v : pk.map) id += std::to_string(v);
      out.push_back("case=" + id + "_" + name + ";perm=" + comma_list(pk.map) + ";size=" + comma_list(ext) +
                    ";kinds=" + kinds + ";alpha=1;beta=1;category=" + pk.category + ";config=" + name);
    }
  }
  return out;
}

}  // namespace ttb
