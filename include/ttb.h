/*
 * ttb.h -- C ABI of the B200 tensor-transposition engine (libttb.so).
 *
 * Computes Eq. 1 of arXiv:1603.02297 on column-major tensors held in device
 * (HBM) memory of an sm_100a GPU:
 *
 *     B_perm(i1..iN) <- alpha * A(i1..iN) + beta * B_perm(i1..iN)
 *
 * It is a drop-in for the reference's hot path, ttune's executor
 * (/root/reference/proj/core/include/ttune/executor.hpp:80-88):
 *
 *     void reference_transpose(const TransposeProblem&, const TensorBuffer& a,
 *                              TensorBuffer& b, int threads = 1);
 *     void execute_plan(const TransposeProblem&, const CandidatePlan&,
 *                       const TensorBuffer& a, TensorBuffer& b, int threads = 1);
 *
 * with the problem built by ttune::make_problem(perm_map, sizes, kind_a,
 * kind_b, alpha, beta, lda, ldb) (problem.hpp:51-58).  The argument set and its
 * meaning are kept; C++ types become plain pointers and sizes, `threads`
 * becomes a CUDA stream, and exceptions become status codes plus a
 * thread-local message that reuses the reference's exact text.
 *
 * Conventions (identical to the reference):
 *   perm   1-based SCATTER map, perm[a] = B position of A index a+1
 *          (Permutation::map, problem.hpp:22-35)
 *   sizes  extents in A index order
 *   lda    leading dimensions in A index order; NULL = dense (= sizes)
 *   ldb    leading dimensions in B index order; NULL = dense (= sizes_b)
 *   kinds  TTB_REAL32 'S', TTB_REAL64 'D', TTB_COMPLEX64 'C', TTB_COMPLEX128
 *          'Z' (ElementKind, problem.hpp:11); complex data is interleaved
 *          (re, im) and alpha/beta are real, applied to both components.
 *          Mixed pairs S<->D and C<->Z are accepted (problem.cpp:45-52).
 *
 * Arithmetic contract (executor.hpp:18-40): W = double if either side is
 * double, else float; beta == 0 never reads B; otherwise
 * B = SB(alpha_W*W(A) + beta_W*W(B)) with two separately rounded products and
 * one rounded sum (no FMA), so results are bit-identical to the reference.
 * Padding of B (outside the logical box) is never written, padding of A is
 * never read.  Calls are asynchronous on the given stream.
 */
#ifndef TTB_H
#define TTB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTB_VERSION "0.1.0"
#define TTB_MAX_RANK 16 /* rank after merging (the reference's limit is
                           search.cpp:200-202 / plan text 64); larger -> EINVAL */

typedef enum {
  TTB_REAL32 = 0,
  TTB_REAL64 = 1,
  TTB_COMPLEX64 = 2,
  TTB_COMPLEX128 = 3
} ttb_kind;

typedef enum {
  TTB_OK = 0,
  TTB_EINVAL = 1,    /* std::invalid_argument in the reference (CLI exit 1) */
  TTB_ECUDA = 2,     /* CUDA runtime failure */
  TTB_ENOMEM = 3,    /* device/host allocation failure */
  TTB_EINTERNAL = 4  /* anything else (CLI exit 2 in the reference) */
} ttb_status;

/* ABI-compatible with cudaStream_t / CUstream; NULL = legacy default stream */
typedef struct CUstream_st* ttb_stream;

/* opaque execution plan (the GPU counterpart of ttune::CandidatePlan) */
typedef struct ttb_plan_s* ttb_plan;

/* ------------------------------------------------------------ errors -- */

/* message of the last failing call on this host thread ("" after success);
 * the reference's std::invalid_argument text where one exists */
const char* ttb_last_error(void);
const char* ttb_version(void);

/* ---------------------------------------------- problem model (host) -- */

/* ttune::validate (problem.cpp:107-159).  Each array carries its own length,
 * as the reference's std::vectors do; n_lda / n_ldb < 0 select make_problem's
 * dense defaults (problem.cpp:85-105).  TTB_OK or TTB_EINVAL + message. */
int ttb_validate(int n_perm, const int* perm, int n_sizes, const int64_t* sizes, int n_lda,
                 const int64_t* lda, int n_ldb, const int64_t* ldb, int kind_a, int kind_b);

/* required_elements_a / _b (problem.cpp:201-218); -1 on an invalid problem */
int64_t ttb_required_elements_a(int rank, const int64_t* sizes, const int64_t* lda);
int64_t ttb_required_elements_b(int rank, const int* perm, const int64_t* sizes,
                                const int64_t* ldb);

/* merge_indices (problem.cpp:270-340): all output arrays hold `rank` entries;
 * *out_rank receives the merged rank; trace_lo/hi the 1-based original index
 * range folded into each merged index (MergeRecord, problem.hpp:84-92). */
int ttb_merge_indices(int rank, const int* perm, const int64_t* sizes, const int64_t* lda,
                      const int64_t* ldb, int* out_rank, int* out_perm, int64_t* out_sizes,
                      int64_t* out_lda, int64_t* out_ldb, int* trace_lo, int* trace_hi);

/* canonical_key (problem.cpp:228-241), e.g.
 * "perm=2,1;size=4,4;lda=4,4;ldb=4,4;kinds=ss;beta=z" */
int ttb_canonical_key(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                      const int64_t* lda, const int64_t* ldb, double alpha, double beta,
                      char* buf, size_t len);

/* effective bandwidth in decimal GB/s: (N*bytes(A) + N*bytes(B)
 * [+ N*bytes(B) if beta != 0]) / 1e9 / seconds  (tuner.cpp:18-25 with 1e9
 * instead of 2^30).  Negative on invalid input. */
double ttb_bandwidth_gbs(int kind_a, int kind_b, int64_t elements, double beta,
                         double seconds);

/* ------------------------------------------------------- execution -- */

/* One-shot transposition on DEVICE buffers: plan from the in-memory plan
 * cache (keyed by canonical_key + device), created by heuristic on a miss.
 * a_elements / b_elements are the buffer capacities in elements
 * (TensorBuffer::elements(), executor.hpp:50-55) checked against
 * required_elements_*; pass -1 to skip the check.  Replaces
 * reference_transpose / execute_plan (executor.hpp:80-88, executor.cpp:371-398). */
int ttb_transpose(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                  const int64_t* lda, const int64_t* ldb, double alpha, const void* A,
                  int64_t a_elements, double beta, void* B, int64_t b_elements,
                  ttb_stream stream);

/* plan flags */
#define TTB_PLAN_DEFAULT 0
#define TTB_PLAN_NO_CACHE 1 /* do not consult / fill the in-memory plan cache */

/* Plan a problem for the current device (validate -> merge_indices -> choose
 * kernel variant, tile, vector widths, launch shape).  The plan keeps a copy
 * of the problem; its buffers are supplied at execution. */
int ttb_plan_create(ttb_plan* out, int kind_a, int kind_b, int rank, const int* perm,
                    const int64_t* sizes, const int64_t* lda, const int64_t* ldb, double alpha,
                    double beta, int flags);
int ttb_plan_destroy(ttb_plan plan);

/* Run the plan on device buffers (stream-ordered, asynchronous). */
int ttb_plan_execute(ttb_plan plan, const void* A, void* B, ttb_stream stream);

/* End-to-end call on HOST buffers: host->device copy of A (and of B when
 * beta != 0 or padded), the kernel, device->host copy of B, on plan-owned
 * device buffers.  Synchronous; returns when B_host is written.  With both
 * buffers pinned (cudaHostAlloc / cudaHostRegister) the problem is cut into
 * slabs along one merged axis and the slabs are pipelined: slab i+1 streams in
 * while slab i's kernel runs and its B part streams out (PCIe is full duplex);
 * pageable buffers take the sequential path.  Env overrides (tuning/tests):
 * TTB_HOST_SLABS (max slabs, 32), TTB_HOST_MIN_ROW (bytes per 2D-copy row,
 * 4096), TTB_HOST_MIN_SLAB_KB (4096), TTB_HOST_PATH=staged. */
int ttb_plan_execute_host(ttb_plan plan, const void* A_host, void* B_host);

/* The same call without the final wait: returns once the copies and kernels
 * are queued (pinned buffers; pageable ones make the copies themselves
 * blocking).  B_host is written, and A_host / B_host may be reused, only after
 * ttb_plan_host_sync(plan).  Calls on different plans overlap -- the next
 * transposition's host->device copies run while this one's last slabs compute
 * and stream out; a second call on the same plan first waits for the one in
 * flight (one set of staging buffers per plan). */
int ttb_plan_execute_host_async(ttb_plan plan, const void* A_host, void* B_host);
int ttb_plan_host_sync(ttb_plan plan);

/* Measured autotune: time every candidate variant of the plan on the given
 * device buffers with CUDA events (warmups + reps, best-of, as
 * measure_candidate, tuner.cpp:27-46) and keep the fastest; the choice is
 * written back to the plan cache.  When beta != 0 the candidates run on a
 * scratch copy of B.  On return B holds exactly one application of the tuned
 * plan, as after ttb_plan_execute. */
int ttb_plan_autotune(ttb_plan plan, const void* A, void* B, int warmups, int reps,
                      ttb_stream stream);

/* serialized plan, e.g. "kern=rt;x=0;y=1;mx=4;my=4;lx=4;order=x;ctas=1184",
 * and the candidate list (one plan per line) */
int ttb_plan_describe(ttb_plan plan, char* buf, size_t len);
int ttb_plan_candidates(ttb_plan plan, char* buf, size_t len);
/* force a candidate by its serialized text (TTB_EINVAL if not applicable) */
int ttb_plan_select(ttb_plan plan, const char* plan_text);
/* kernel launches of one ttb_plan_execute: 1, or the number of < 2^31-element
   boxes an oversized problem runs as */
int ttb_plan_launches(ttb_plan plan, int* launches_per_execute);

/* Standalone CUDA source for one plan on one problem (replaces ttune's
 * emit_source, emit.cpp:622-715, which writes C/OpenMP): the header and .cu
 * text of a kernel whose extents, strides and tile are compile-time
 * constants, entry `transpose_<perm>_<sizes>_<kinds>(const TA* A, TB* B,
 * TW alpha, TW beta)` (device pointers, default stream) plus `<entry>_async`
 * with a stream.  plan_text: a serialized plan (ttb_plan_describe) or NULL;
 * basename: file stem the source includes its header by (NULL: the entry
 * symbol).  Any output buffer may be NULL; no device is needed. */
int ttb_emit_source(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                    const int64_t* lda, const int64_t* ldb, double alpha, double beta,
                    const char* plan_text, const char* basename, char* entry, size_t entry_len,
                    char* header, size_t header_len, char* source, size_t source_len);

/* ------------------------------------------ persistent solution cache -- */

/* The reference's SolutionCache (tuner.cpp:81-205) as a native file store:
 * one tab-separated line per entry, "problem_key \t hardware_key \t plan \t
 * bandwidth_gibs \t ISO-8601 UTC timestamp", appended under an exclusive
 * flock; lookup reads under a shared flock, skips malformed lines (warning on
 * stderr) and returns the LAST entry matching both keys.  Bandwidth is GiB/s
 * (2^30), as the reference stores it. */
int ttb_cache_store(const char* file, const char* problem_key, const char* hardware_key,
                    const char* plan_text, double bandwidth_gibs);
/* *found = 0/1; plan text into plan_buf; bandwidth / timestamp optional (NULL) */
int ttb_cache_lookup(const char* file, const char* problem_key, const char* hardware_key,
                     char* plan_buf, size_t plan_len, double* bandwidth_gibs, char* ts_buf,
                     size_t ts_len, int* found);
/* this GPU: "<device name>:sm<major><minor>:<SMs>sms:ttb<version>" (the
 * reference keys hardware by host/threads/micro-width, default_hardware_key) */
int ttb_hardware_key(char* buf, size_t len);
/* pipeline.cpp:102-185 for one plan: look the plan up by (canonical_key of
 * the original problem, hardware key); on a hit select it, on a miss (or a
 * stale entry that no longer applies) autotune on A/B and store the winner.
 * *hit = 1 on a cache hit.  B ends holding one application, as autotune. */
int ttb_plan_tune_cached(ttb_plan plan, const char* cache_file, const void* A, void* B,
                         int warmups, int reps, ttb_stream stream, int* hit);

/* ------------------------------------------ the paper's benchmark suite -- */

/* build_benchmark (benchmark.cpp:166-220): the 57 synthetic cases (19
 * non-mergeable perms over d = 2..6 times balanced / skewA / skewB extents of
 * ~volume_bytes, alpha = beta = 1), drawn with mt19937_64(seed).  Writes the
 * manifest, one benchmark_case_line per case ("case=...;perm=...;size=...;
 * kinds=..;alpha=..;beta=..;category=..;config=.."), '\n'-separated. */
int ttb_benchmark_manifest(int64_t volume_bytes, int kind, uint64_t seed, char* buf, size_t len);

/* ------------------------------------------- multi-GPU partitioning -- */

/* Split B's index space for rank r of `world`: the flattened
 * range over the k slowest split axes -- B's indices from the outermost, with
 * A's and B's stride-1 indices moved last (cutting them cuts the tiles' runs)
 * -- k the smallest with a max/mean imbalance <= 1.05; an axis of that order
 * that splits within 1.07 on its own is taken alone (one box per rank).
 * Writes *n_boxes <= 2*rank-1 boxes (origin +
 * extent, `rank` entries each in A index order, over the problem's index
 * space; pass NULL arrays to query the count); each box is an independent
 * sub-problem (same perm/lda/ldb, sizes = extent, buffers offset by origin). */
int ttb_shard_boxes(int rank, const int* perm, const int64_t* sizes, int world, int r,
                    int64_t* origins, int64_t* extents, int* n_boxes);

/* --------------------------------------------- device data utilities -- */

/* Seeded counter-based generator (the bench's synthetic inputs): for logical
 * element i of the box (column-major over global_sizes after adding origin)
 * and component q, u = splitmix64(seed*0x9E3779B97F4A7C15 + i*C + q);
 * fp32 ((u>>40)*2^-24)*2-1, fp64 ((u>>11)*2^-53)*2-1.  origin/global_sizes
 * may be NULL (box = whole tensor). ld = leading dims (NULL = dense). */
int ttb_fill_uniform(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                     const int64_t* origin, const int64_t* global_sizes, uint64_t seed, void* buf,
                     ttb_stream stream);
/* every scalar of buf <- NaN sentinel (0x7FC0FFEE / 0x7FF8DEADBEEF0001) */
int ttb_fill_sentinel(int kind, int64_t elements, void* buf, ttb_stream stream);
/* order-independent u64 checksum over a box (same definition as above for
 * the global index): sum of splitmix64((i*C+q)*0xD1B54A32D192ED03 ^ bits).
 * Synchronous; result in *out. */
int ttb_checksum(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                 const int64_t* origin, const int64_t* global_sizes, const void* buf,
                 uint64_t* out, ttb_stream stream);

/* total kernels this library has launched in the process (evidence counter) */
uint64_t ttb_launch_count(void);

/* ------------------------------------------------------- diagnostics -- */

/* the planner's ranked candidate list for a problem, one serialized plan per
 * line, computed on the host only (no device needed) */
int ttb_debug_candidates(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                         const int64_t* lda, const int64_t* ldb, double alpha, double beta,
                         char* buf, size_t len);

#ifdef __cplusplus
}
#endif

#endif /* TTB_H */
