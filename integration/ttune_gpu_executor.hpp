// ttune_gpu_executor.hpp -- the adapter a ttune maintainer adds to route the
// reference's executor entry points (executor.hpp:80-88) to libttb.so.
//
// Same signatures and error behaviour as ttune::reference_transpose /
// ttune::execute_plan (executor.cpp:315-398): validate(p) first, then the
// buffer checks with the reference's messages, std::invalid_argument for
// every user error, std::runtime_error for CUDA failures.  The plan argument
// of execute_plan is the CPU search's CandidatePlan; on the GPU the engine
// plans for itself, so it is checked (check_plan's rules) and otherwise unused.
//
// Compiled against the reference's headers (include path of ttune_core) and
// this repository's include/ttb.h; oracle/Makefile builds it that way
// (target `adapter`) and tests/test_adapter.py + tests/test_gpu_adapter.py run it.
#pragma once

#include "ttune/executor.hpp"
#include "ttune/plan.hpp"
#include "ttune/problem.hpp"

namespace ttune::gpu {

// reference_transpose on host TensorBuffers: H2D, kernel, D2H (synchronous)
void reference_transpose(const TransposeProblem& p, const TensorBuffer& a, TensorBuffer& b,
                         int threads = 1);

// execute_plan on host TensorBuffers; `plan` is validated like the reference does
void execute_plan(const TransposeProblem& p, const CandidatePlan& plan, const TensorBuffer& a,
                  TensorBuffer& b, int threads = 1);

// device-resident variant: A and B already in HBM, asynchronous on `stream`
// (a cudaStream_t; nullptr = legacy default stream).  a_elements / b_elements
// are the buffers' capacities (-1 skips the check).
void transpose_device(const TransposeProblem& p, const void* A, std::int64_t a_elements, void* B,
                      std::int64_t b_elements, void* stream = nullptr);

}  // namespace ttune::gpu
