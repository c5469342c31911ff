// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" veneer over the UNMODIFIED reference sources
// (/root/reference/proj/core/src/{problem,executor,search,tuner}.cpp), compiled
// where they lie by oracle/Makefile into oracle/_ref/libttune_ref.so.  It lets
// Python tests and bench.py's CPU arm call the reference's own entry points:
//   reference_transpose / execute_plan   (executor.hpp:80-88)
//   validate / merge_indices / canonical_key (problem.hpp:60-102)
//   tune + build_candidates               (tuner.hpp:75-80, search.hpp:61-63)
//   tsup::oracle_transpose                (proj/tests/support.hpp:18-73)
// Nothing here is product code and nothing from the reference is copied: the
// reference headers are included from /root/reference at build time.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "support.hpp"
#include "ttune/benchmark.hpp"
#include "ttune/executor.hpp"
#include "ttune/problem.hpp"
#include "ttune/search.hpp"
#include "ttune/tuner.hpp"

using namespace ttune;

namespace {

ElementKind kind_of(int k) {
  switch (k) {
    case 0: return ElementKind::real32;
    case 1: return ElementKind::real64;
    case 2: return ElementKind::complex64;
    default: return ElementKind::complex128;
  }
}

int kind_id(ElementKind k) {
  switch (k) {
    case ElementKind::real32: return 0;
    case ElementKind::real64: return 1;
    case ElementKind::complex64: return 2;
    case ElementKind::complex128: return 3;
  }
  return -1;
}

void put(char* dst, std::size_t len, const std::string& s) {
  if (!dst || !len) return;
  std::size_t n = std::min(len - 1, s.size());
  std::memcpy(dst, s.data(), n);
  dst[n] = 0;
}

// raw arrays -> make_problem arguments; n < 0 means "not given" (empty vector)
TransposeProblem build(int n_perm, const int* perm, int n_sizes, const std::int64_t* sizes,
                       int n_lda, const std::int64_t* lda, int n_ldb, const std::int64_t* ldb,
                       int ka, int kb, double alpha, double beta) {
  std::vector<int> pm(perm, perm + std::max(n_perm, 0));
  std::vector<std::int64_t> sz(sizes, sizes + std::max(n_sizes, 0));
  std::vector<std::int64_t> la, lb;
  if (n_lda >= 0 && lda) la.assign(lda, lda + n_lda);
  if (n_ldb >= 0 && ldb) lb.assign(ldb, ldb + n_ldb);
  return make_problem(pm, sz, kind_of(ka), kind_of(kb), alpha, beta, la, lb);
}

// run fn, map exceptions to the reference CLI's exit codes (pipeline.cpp:189-200)
template <class Fn>
int guarded(char* msg, std::size_t len, Fn&& fn) {
  try {
    fn();
    put(msg, len, "");
    return 0;
  } catch (const std::invalid_argument& e) {
    put(msg, len, e.what());
    return 1;
  } catch (const std::exception& e) {
    put(msg, len, e.what());
    return 2;
  }
}

struct Session {
  TransposeProblem p;
  TensorBuffer a, b;
};

}  // namespace

extern "C" {

int ref_validate(int n_perm, const int* perm, int n_sizes, const std::int64_t* sizes, int n_lda,
                 const std::int64_t* lda, int n_ldb, const std::int64_t* ldb, int ka, int kb,
                 char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    (void)validate(build(n_perm, perm, n_sizes, sizes, n_lda, lda, n_ldb, ldb, ka, kb, 1.0, 0.0));
  });
}

int ref_merge(int rank, const int* perm, const std::int64_t* sizes, const std::int64_t* lda,
              const std::int64_t* ldb, int* out_rank, int* out_perm, std::int64_t* out_sizes,
              std::int64_t* out_lda, std::int64_t* out_ldb, int* trace_lo, int* trace_hi,
              char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const NormalizedProblem n = merge_indices(
        build(rank, perm, rank, sizes, lda ? rank : -1, lda, ldb ? rank : -1, ldb, 0, 0, 1.0, 0.0));
    *out_rank = n.problem.rank();
    for (int a = 0; a < n.problem.rank(); ++a) {
      out_perm[a] = n.problem.perm.map[a];
      out_sizes[a] = n.problem.sizes[a];
      out_lda[a] = n.problem.lda[a];
      out_ldb[a] = n.problem.ldb[a];
      trace_lo[a] = n.merge_trace[a].from_first;
      trace_hi[a] = n.merge_trace[a].from_last;
    }
  });
}

int ref_canonical_key(int rank, const int* perm, const std::int64_t* sizes,
                      const std::int64_t* lda, const std::int64_t* ldb, int ka, int kb,
                      double alpha, double beta, char* out, std::size_t len) {
  return guarded(nullptr, 0, [&] {
    put(out, len,
        canonical_key(build(rank, perm, rank, sizes, lda ? rank : -1, lda, ldb ? rank : -1, ldb,
                            ka, kb, alpha, beta)));
  });
}

double ref_bandwidth_gibs(int rank, const int* perm, const std::int64_t* sizes, int ka, int kb,
                          double beta, double seconds) {
  try {
    return bandwidth_gibs(build(rank, perm, rank, sizes, -1, nullptr, -1, nullptr, ka, kb, 1.0,
                                beta),
                          seconds);
  } catch (...) {
    return -1.0;
  }
}

// One-shot execution on caller host buffers (copied in and out of the
// reference's TensorBuffers).  which: 0 reference_transpose, 1 the test
// oracle tsup::oracle_transpose, 2 execute_plan(plan_text).
int ref_run(int ka, int kb, int rank, const int* perm, const std::int64_t* sizes,
            const std::int64_t* lda, const std::int64_t* ldb, double alpha, const void* A,
            std::int64_t a_elems, double beta, void* B, std::int64_t b_elems, int threads,
            int which, const char* plan_text, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const TransposeProblem p = build(rank, perm, rank, sizes, lda ? rank : -1, lda,
                                     ldb ? rank : -1, ldb, ka, kb, alpha, beta);
    TensorBuffer a(kind_of(ka), a_elems), b(kind_of(kb), b_elems);
    std::memcpy(a.data(), A, a.bytes());
    std::memcpy(b.data(), B, b.bytes());
    if (which == 0)
      reference_transpose(p, a, b, threads);
    else if (which == 1)
      tsup::oracle_transpose(validate(p), a, b);
    else
      execute_plan(p, CandidatePlan::parse(plan_text), a, b, threads);
    std::memcpy(B, b.data(), b.bytes());
  });
}

// ---- timing sessions: buffers owned by the reference's TensorBuffer ----

void* ref_session_create(int ka, int kb, int rank, const int* perm, const std::int64_t* sizes,
                         const std::int64_t* lda, const std::int64_t* ldb, double alpha,
                         double beta, int merge, char* msg, std::size_t len) {
  Session* s = nullptr;
  int rc = guarded(msg, len, [&] {
    TransposeProblem p = build(rank, perm, rank, sizes, lda ? rank : -1, lda, ldb ? rank : -1,
                               ldb, ka, kb, alpha, beta);
    if (merge) p = merge_indices(p).problem;  // the pipeline's normalization (pipeline.cpp:111)
    s = new Session{p, make_buffer_a(p), make_buffer_b(p)};
  });
  return rc == 0 ? s : nullptr;
}

void ref_session_destroy(void* h) { delete static_cast<Session*>(h); }
void* ref_session_a(void* h) { return static_cast<Session*>(h)->a.data(); }
void* ref_session_b(void* h) { return static_cast<Session*>(h)->b.data(); }
std::int64_t ref_session_a_elems(void* h) { return static_cast<Session*>(h)->a.elements(); }
std::int64_t ref_session_b_elems(void* h) { return static_cast<Session*>(h)->b.elements(); }

// wall seconds of one reference_transpose (plan_text NULL) or execute_plan call
double ref_session_run(void* h, const char* plan_text, int threads) {
  Session* s = static_cast<Session*>(h);
  try {
    const auto t0 = std::chrono::steady_clock::now();
    if (plan_text && plan_text[0])
      execute_plan(s->p, CandidatePlan::parse(plan_text), s->a, s->b, threads);
    else
      reference_transpose(s->p, s->a, s->b, threads);
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (...) {
    return -1.0;
  }
}

// the reference's own autotuner over a capped queue; writes the winning plan
int ref_session_tune(void* h, int threads, int max_impl, int warmups, int reps, char* plan_out,
                     std::size_t len, double* gibs) {
  Session* s = static_cast<Session*>(h);
  return guarded(nullptr, 0, [&] {
    NormalizedProblem n;
    n.problem = s->p;
    SearchConfig cfg;
    cfg.max_implementations = max_impl;
    cfg.prefetch_distances = std::vector<int>{0, 5};
    const CandidateQueue q = build_candidates(n, cfg);
    const TuneResult r = tune(n, q, TimingProtocol{warmups, reps, threads});
    put(plan_out, len, r.records[r.best].plan.serialize());
    if (gibs) *gibs = r.records[r.best].bandwidth_gibs;
  });
}

// the reference's benchmark suite manifest (benchmark.cpp:166-220, 258-270)
int ref_benchmark_manifest(std::int64_t volume_bytes, int kind, std::uint64_t seed, char* out,
                           std::size_t len) {
  return guarded(nullptr, 0, [&] {
    const ElementKind k[] = {ElementKind::real32, ElementKind::real64, ElementKind::complex64,
                             ElementKind::complex128};
    std::ostringstream os;
    write_benchmark_manifest(os, build_benchmark(volume_bytes, k[kind], seed));
    put(out, len, os.str());
  });
}

// the reference's SolutionCache: store one entry / look one up (tuner.cpp:81-205)
int ref_cache_store(const char* file, const char* pkey, const char* hkey, const char* plan,
                    double gibs, const char* ts) {
  return guarded(nullptr, 0, [&] {
    SolutionCache c(file);
    c.store(SolutionEntry{pkey, hkey, CandidatePlan::parse(plan), gibs, ts});
  });
}

int ref_cache_lookup(const char* file, const char* pkey, const char* hkey, char* plan_out,
                     std::size_t len, double* gibs, int* found) {
  return guarded(nullptr, 0, [&] {
    SolutionCache c(file);
    const auto e = c.lookup(pkey, hkey);
    *found = e ? 1 : 0;
    if (e) {
      put(plan_out, len, e->plan.serialize());
      *gibs = e->bandwidth_gibs;
    }
  });
}

int ref_kind_id_of_code(char c) {
  auto k = kind_from_code(c);
  return k ? kind_id(*k) : -1;
}

}  // extern "C"
