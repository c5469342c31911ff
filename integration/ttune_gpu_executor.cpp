// ttune_gpu_executor.cpp -- see ttune_gpu_executor.hpp.
//
// The adapter only translates: ttune's TransposeProblem (problem.hpp:37-49)
// becomes the C ABI's argument set (include/ttb.h), ttb status codes become
// the reference's exception types (pipeline.cpp:189-200), and the order of the
// checks follows run_any (executor.cpp:371-385).
#include "ttune_gpu_executor.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "ttb.h"

namespace ttune::gpu {
namespace {

int kind_id(ElementKind k) {
  switch (k) {
    case ElementKind::real32: return TTB_REAL32;
    case ElementKind::real64: return TTB_REAL64;
    case ElementKind::complex64: return TTB_COMPLEX64;
    case ElementKind::complex128: return TTB_COMPLEX128;
  }
  return -1;
}

void raise(int rc) {
  if (rc == TTB_OK) return;
  if (rc == TTB_EINVAL) throw std::invalid_argument(ttb_last_error());
  throw std::runtime_error(std::string("ttb: ") + ttb_last_error());
}

// validate(p) through the ABI: every vector passes its own length, so a
// mismatched lda/ldb gets the reference's message (problem.cpp:107-159)
void validate_abi(const TransposeProblem& p) {
  raise(ttb_validate(static_cast<int>(p.perm.map.size()), p.perm.map.data(),
                     static_cast<int>(p.sizes.size()), p.sizes.data(),
                     static_cast<int>(p.lda.size()), p.lda.data(),
                     static_cast<int>(p.ldb.size()), p.ldb.data(), kind_id(p.kind_a),
                     kind_id(p.kind_b)));
}

// check_buffers (executor.cpp:315-322)
void check_buffers(const TransposeProblem& p, const TensorBuffer& a, const TensorBuffer& b) {
  if (a.kind() != p.kind_a) throw std::invalid_argument("A buffer: element kind mismatch");
  if (b.kind() != p.kind_b) throw std::invalid_argument("B buffer: element kind mismatch");
  if (a.elements() < ttb_required_elements_a(p.rank(), p.sizes.data(), p.lda.data()))
    throw std::invalid_argument("A buffer: too small for problem");
  if (b.elements() <
      ttb_required_elements_b(p.rank(), p.perm.map.data(), p.sizes.data(), p.ldb.data()))
    throw std::invalid_argument("B buffer: too small for problem");
}

// check_plan (executor.cpp:324-339): the CPU plan's own consistency rules
void check_plan(const TransposeProblem& p, const CandidatePlan& plan) {
  std::vector<int> order = plan.loop_order;
  std::sort(order.begin(), order.end());
  bool ok = static_cast<int>(order.size()) == p.rank();
  for (int i = 0; ok && i < p.rank(); ++i) ok = order[static_cast<std::size_t>(i)] == i + 1;
  if (!ok) throw std::invalid_argument("plan: loop order does not cover the problem's indices");
  if (plan.micro_width < 1) throw std::invalid_argument("plan: micro width must be >= 1");
  if (plan.block_a < 1 || plan.block_b < 1)
    throw std::invalid_argument("plan: block extents must be >= 1");
  if (plan.prefetch_distance < 0) throw std::invalid_argument("plan: negative prefetch distance");
  if (plan.prefetch_distance > 0 && p.perm.preserves_stride1())
    throw std::invalid_argument("plan: prefetch distance requires a transposed stride-1 index");
  if (plan.streaming_stores && p.beta != 0.0)
    throw std::invalid_argument("plan: streaming stores require beta == 0");
}

struct Plan {
  ttb_plan h = nullptr;
  explicit Plan(const TransposeProblem& p) {
    raise(ttb_plan_create(&h, kind_id(p.kind_a), kind_id(p.kind_b), p.rank(), p.perm.map.data(),
                          p.sizes.data(), p.lda.data(), p.ldb.data(), p.alpha, p.beta,
                          TTB_PLAN_DEFAULT));
  }
  ~Plan() { ttb_plan_destroy(h); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
};

void run_host(const TransposeProblem& p, const CandidatePlan* plan, const TensorBuffer& a,
              TensorBuffer& b, int threads) {
  validate_abi(p);
  check_buffers(p, a, b);
  if (plan) check_plan(p, *plan);
  if (threads < 1) throw std::invalid_argument("threads: must be >= 1");
  Plan gp(p);
  raise(ttb_plan_execute_host(gp.h, a.data(), b.data()));
}

}  // namespace

void reference_transpose(const TransposeProblem& p, const TensorBuffer& a, TensorBuffer& b,
                         int threads) {
  run_host(p, nullptr, a, b, threads);
}

void execute_plan(const TransposeProblem& p, const CandidatePlan& plan, const TensorBuffer& a,
                  TensorBuffer& b, int threads) {
  run_host(p, &plan, a, b, threads);
}

void transpose_device(const TransposeProblem& p, const void* A, std::int64_t a_elements, void* B,
                      std::int64_t b_elements, void* stream) {
  validate_abi(p);
  raise(ttb_transpose(kind_id(p.kind_a), kind_id(p.kind_b), p.rank(), p.perm.map.data(),
                      p.sizes.data(), p.lda.data(), p.ldb.data(), p.alpha, A, a_elements, p.beta,
                      B, b_elements, static_cast<ttb_stream>(stream)));
}

}  // namespace ttune::gpu
