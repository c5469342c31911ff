// adapter_check.cpp -- TEST PROGRAM for the ttune adapter (not product code).
//
// Links the reference's own library (oracle/_ref/libttune_ref.so, the
// unmodified ttune sources) and libttb.so through integration/
// ttune_gpu_executor.cpp, i.e. exactly what a ttune build with the adapter
// would contain, and checks that the adapter is a drop-in:
//
//   adapter_check errors   (no GPU) every user error raises the same exception
//                          type and message as ttune::reference_transpose /
//                          execute_plan on the same arguments
//   adapter_check gpu      ttune::gpu::{reference_transpose, execute_plan,
//                          transpose_device} produce the same bytes as
//                          ttune::reference_transpose on ttune TensorBuffers
//                          (whole B buffer, padding included) for problems
//                          shaped like BASELINE's configs
//
// Exit 0 when every check passes; one line per failure otherwise.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ttune/executor.hpp"
#include "ttune/problem.hpp"
#include "ttune_gpu_executor.hpp"

using namespace ttune;

namespace {

int failures = 0;

void fail(const std::string& what) {
  ++failures;
  std::printf("FAIL %s\n", what.c_str());
}

// deterministic values in [-1, 1) per scalar (splitmix64)
void fill(TensorBuffer& t, std::uint64_t seed) {
  const bool dbl = t.kind() == ElementKind::real64 || t.kind() == ElementKind::complex128;
  const std::int64_t n = t.scalars();
  std::uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  for (std::int64_t i = 0; i < n; ++i) {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    if (dbl)
      t.as<double>()[i] = u;
    else
      t.as<float>()[i] = static_cast<float>(u);
  }
}

// outcome of a call: "" on success, else "<type>: <message>"
std::string outcome(const std::function<void()>& f) {
  try {
    f();
    return "";
  } catch (const std::invalid_argument& e) {
    return std::string("invalid_argument: ") + e.what();
  } catch (const std::exception& e) {
    return std::string("other: ") + e.what();
  }
}

CandidatePlan plan_for(const TransposeProblem& p) {
  CandidatePlan c;
  for (int i = 1; i <= p.rank(); ++i) c.loop_order.push_back(i);
  c.block_a = c.block_b = 16;
  c.micro_width = 4;
  return c;
}

void check_errors() {
  struct Case {
    const char* name;
    std::function<TransposeProblem()> make;
    bool small_a = false, small_b = false, wrong_kind = false, bad_plan = false;
    int threads = 1;
  };
  auto base = [] { return make_problem({2, 1}, {5, 7}); };
  std::vector<Case> cases = {
      {"not a permutation", [] { TransposeProblem p = make_problem({2, 1}, {5, 7});
                                  p.perm.map = {1, 1}; return p; }},
      {"rank mismatch", [] { TransposeProblem p = make_problem({2, 1}, {5, 7});
                              p.sizes = {5, 7, 2}; return p; }},
      {"lda length", [] { TransposeProblem p = make_problem({2, 1}, {5, 7});
                           p.lda = {5}; return p; }},
      {"lda below size", [] { return make_problem({2, 1}, {5, 7}, ElementKind::real32,
                                                  ElementKind::real32, 1.0, 0.0, {4, 7}); }},
      {"ldb below size", [] { return make_problem({2, 1}, {5, 7}, ElementKind::real32,
                                                  ElementKind::real32, 1.0, 0.0, {}, {7, 4}); }},
      {"zero extent", [] { return make_problem({2, 1}, {0, 7}); }},
      {"kind pair", [] { return make_problem({2, 1}, {5, 7}, ElementKind::real32,
                                             ElementKind::complex64); }},
      {"A too small", base, true},
      {"B too small", base, false, true},
      {"buffer kind", base, false, false, true},
      {"bad plan", base, false, false, false, true},
      {"threads", base, false, false, false, false, 0},
  };
  for (const Case& c : cases) {
    TransposeProblem p = c.make();
    // buffers sized by the valid part of the problem, as a caller would
    TransposeProblem q = base();
    TensorBuffer a(c.wrong_kind ? ElementKind::real64 : ElementKind::real32,
                   required_elements_a(q) - (c.small_a ? 1 : 0));
    TensorBuffer b(ElementKind::real32, required_elements_b(q) - (c.small_b ? 1 : 0));
    CandidatePlan plan = plan_for(q);
    if (c.bad_plan) plan.micro_width = 0;
    std::string want_ref, got_ref;
    if (!c.bad_plan) {
      want_ref = outcome([&] { ttune::reference_transpose(p, a, b, c.threads); });
      got_ref = outcome([&] { ttune::gpu::reference_transpose(p, a, b, c.threads); });
    }
    const std::string want_plan = outcome([&] { ttune::execute_plan(p, plan, a, b, c.threads); });
    const std::string got_plan =
        outcome([&] { ttune::gpu::execute_plan(p, plan, a, b, c.threads); });
    // a bad CPU plan only concerns execute_plan (reference_transpose takes none)
    if (!c.bad_plan && (want_ref.empty() || want_ref != got_ref))
      fail(std::string(c.name) + ": reference_transpose '" + want_ref + "' vs adapter '" +
           got_ref + "'");
    if (want_plan.empty() || want_plan != got_plan)
      fail(std::string(c.name) + ": execute_plan '" + want_plan + "' vs adapter '" + got_plan +
           "'");
  }
  std::printf("errors: %zu cases checked\n", cases.size());
}

struct Shape {
  const char* name;
  std::vector<int> perm;  // 1-based scatter map, ttune convention
  std::vector<std::int64_t> sizes, lda, ldb;
  ElementKind ka, kb;
  double alpha, beta;
};

void check_gpu() {
  const ElementKind s = ElementKind::real32, d = ElementKind::real64,
                    c = ElementKind::complex64, z = ElementKind::complex128;
  const std::vector<Shape> shapes = {
      {"c1-like 2D", {2, 1}, {727, 519}, {}, {}, s, s, 1.0, 0.0},
      {"c2a-like", {2, 4, 1, 3}, {96, 32, 72, 16}, {}, {}, s, s, 1.3, 0.0},
      {"c2b-like copy", {1, 4, 3, 2}, {96, 32, 72, 16}, {}, {}, s, s, 1.3, 0.0},
      {"c3-like 6D beta", {3, 5, 2, 6, 4, 1}, {24, 20, 22, 18, 6, 4}, {}, {}, d, d, 0.7, 1.1},
      {"c4-like complex", {3, 2, 1}, {4, 512, 384}, {}, {}, c, c, 1.0, 0.0},
      {"c4s-like outer sizes", {3, 2, 1}, {4, 512, 384}, {8, 512, 384}, {384, 512, 8}, c, c,
       1.0, 0.0},
      {"z beta", {2, 3, 1}, {33, 17, 9}, {}, {}, z, z, 2.0, 3.0},
      {"mixed s->d", {2, 1}, {301, 129}, {}, {}, s, d, 1.5, 0.5},
      {"mixed z->c", {2, 1}, {65, 47}, {}, {}, z, c, 1.0, 0.0},
      {"identity", {1, 2, 3}, {64, 33, 7}, {}, {}, s, s, 1.0, 0.0},
      {"rank 1", {1}, {100003}, {}, {}, d, d, 0.5, 0.25},
  };
  for (const Shape& sh : shapes) {
    const TransposeProblem p =
        make_problem(sh.perm, sh.sizes, sh.ka, sh.kb, sh.alpha, sh.beta, sh.lda, sh.ldb);
    TensorBuffer a = make_buffer_a(p);
    TensorBuffer b0 = make_buffer_b(p);
    fill(a, 11);
    fill(b0, 12);  // padding and (beta != 0) the update operand
    TensorBuffer want = b0;
    ttune::reference_transpose(p, a, want, 4);
    auto same = [&](const TensorBuffer& got, const char* path) {
      if (std::memcmp(got.data(), want.data(), want.bytes()) != 0)
        fail(std::string(sh.name) + ": " + path + " differs from ttune::reference_transpose");
    };
    TensorBuffer got = b0;
    ttune::gpu::reference_transpose(p, a, got);
    same(got, "gpu::reference_transpose");
    got = b0;
    ttune::gpu::execute_plan(p, plan_for(p), a, got);
    same(got, "gpu::execute_plan");
    // device buffers through the device entry point
    void *da = nullptr, *db = nullptr;
    if (cudaMalloc(&da, a.bytes()) != cudaSuccess || cudaMalloc(&db, b0.bytes()) != cudaSuccess) {
      fail(std::string(sh.name) + ": cudaMalloc");
      continue;
    }
    cudaMemcpy(da, a.data(), a.bytes(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, b0.data(), b0.bytes(), cudaMemcpyHostToDevice);
    ttune::gpu::transpose_device(p, da, a.elements(), db, b0.elements(), nullptr);
    got = b0;
    if (cudaMemcpy(got.data(), db, got.bytes(), cudaMemcpyDeviceToHost) != cudaSuccess)
      fail(std::string(sh.name) + ": device copy back");
    same(got, "gpu::transpose_device");
    cudaFree(da);
    cudaFree(db);
  }
  std::printf("gpu: %zu problems checked (3 entry points each)\n", shapes.size());
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "errors";
  try {
    if (mode == "errors" || mode == "all") check_errors();
    if (mode == "gpu" || mode == "all") check_gpu();
  } catch (const std::exception& e) {
    fail(std::string("uncaught: ") + e.what());
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
