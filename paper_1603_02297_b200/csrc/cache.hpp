// cache.hpp -- persistent solution cache and the benchmark-suite generator
// (host side of the engine; no device code).
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace ttb {

// one line of the solution file (tuner.hpp:45-51 SolutionEntry)
struct CacheEntry {
  std::string problem_key, hardware_key, plan;
  double bandwidth_gibs = 0.0;
  std::string timestamp;
};

// last well-formed entry matching both keys; false when none (or no file).
// plan_ok, if given, must accept the plan field or the line is malformed.
bool cache_lookup(const std::string& file, const std::string& problem_key,
                  const std::string& hardware_key, CacheEntry* out,
                  const std::function<bool(const std::string&)>& plan_ok = nullptr);
// append under an exclusive lock; InvalidArgument for empty / multi-line fields
void cache_store(const std::string& file, const CacheEntry& e);
std::string iso8601_utc_now();

// benchmark.cpp:166-220 build_benchmark, as manifest lines
std::vector<std::string> benchmark_manifest(int64_t volume_bytes, int kind, uint64_t seed);

}  // namespace ttb
