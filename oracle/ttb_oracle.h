/*
 * ttb_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference's algorithm for the hot path
 * (ttune, /root/reference/proj).  It is the checker the GPU engine is compared
 * against; it is never linked into, called by or shipped with the product
 * library (paper_1603_02297_b200/_lib/libttb.so).  Only tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load it.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * reference sources are compiled in place by oracle/Makefile into
 * oracle/_ref/libttune_ref.so and tests/test_oracle_pin.py compares the two on
 * random problems; tests/golden/ holds fixtures produced by the reference.
 *
 * Conventions follow the reference exactly:
 *   - perm is ttune's 1-based SCATTER map: perm[a] = B position of A index a+1
 *     (proj/core/include/ttune/problem.hpp:22-35);
 *   - sizes and lda are in A index order, ldb in B index order
 *     (problem.hpp:37-49);
 *   - kinds: 0 = s (real32), 1 = d (real64), 2 = c (complex64),
 *     3 = z (complex128) (problem.hpp:11).
 */
#ifndef TTB_ORACLE_H
#define TTB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_RANK 64

/* element_bytes / element_components (problem.cpp:9-23) */
int orc_element_bytes(int kind);
int orc_components(int kind);

/* validate (problem.cpp:107-159): 0 when valid, else 1 and the reference's
 * exact std::invalid_argument message in msg.  Each array carries its own
 * length like the reference's std::vectors; n_lda/n_ldb < 0 = dense default
 * (make_problem, problem.cpp:85-105). */
int orc_validate(int n_perm, const int* perm, int n_sizes, const int64_t* sizes, int n_lda,
                 const int64_t* lda, int n_ldb, const int64_t* ldb, int kind_a, int kind_b,
                 char* msg, size_t msglen);

/* required_elements_a / required_elements_b (problem.cpp:201-218) */
int64_t orc_required_elements_a(int rank, const int64_t* sizes, const int64_t* lda);
int64_t orc_required_elements_b(int rank, const int* perm, const int64_t* sizes,
                                const int64_t* ldb);

/* merge_indices (problem.cpp:270-340).  Outputs have room for `rank` entries;
 * trace_lo/trace_hi are the 1-based original index ranges per merged index.
 * Returns the merged rank (>=1) or -1 if the problem is invalid. */
int orc_merge(int rank, const int* perm, const int64_t* sizes, const int64_t* lda,
              const int64_t* ldb, int* out_perm, int64_t* out_sizes, int64_t* out_lda,
              int64_t* out_ldb, int* trace_lo, int* trace_hi);

/* Element walk straight from Eq. 1 (support.hpp:18-60 index walk,
 * executor.hpp:18-40 arithmetic).  B is updated in place; padding untouched. */
void orc_transpose(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                   const int64_t* lda, const int64_t* ldb, double alpha, const void* A,
                   double beta, void* B);

/* The paper's "reference routine": B-linear loop nest, inner loop along B's
 * stride-1 index (executor.cpp:283-313), split over `threads` pthreads with
 * the reference's static contiguous ranges (executor.cpp:91-105). */
void orc_reference_nest(int kind_a, int kind_b, int rank, const int* perm,
                        const int64_t* sizes, const int64_t* lda, const int64_t* ldb,
                        double alpha, const void* A, double beta, void* B, int threads);

/* Seeded counter-based generator: for logical element i
 * (column-major over `sizes`, offsets through `ld`) and component q, scalar
 * index j = (i + index_offset)*C + q, u = splitmix64(seed*0x9E3779B97F4A7C15 + j);
 * fp32 value ((u>>40)*2^-24)*2-1, fp64 value ((u>>11)*2^-53)*2-1.
 * `origin`/`global_sizes` (may be NULL) place the box inside a larger tensor
 * so that shards generate the same values as the global tensor. */
void orc_fill_uniform(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                      const int64_t* origin, const int64_t* global_sizes, uint64_t seed,
                      void* buf);

/* Fill every scalar of a buffer with a sentinel bit pattern (NaN payload). */
void orc_fill_sentinel(int kind, int64_t elements, void* buf);

/* Order-independent u64 checksum over the logical box of a tensor:
 * sum over elements i (global column-major index over global_sizes) and
 * components q of h(i*C+q, raw bits), wrapping mod 2^64. */
uint64_t orc_checksum(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                      const int64_t* origin, const int64_t* global_sizes, const void* buf);

uint64_t orc_splitmix64(uint64_t x);

/* bandwidth in decimal GB/s with the reference's byte count
 * (tuner.cpp:18-25, divided by 1e9 instead of 2^30). */
double orc_bandwidth_gbs(int64_t elements, int kind_a, int kind_b, double beta,
                         double seconds);

#ifdef __cplusplus
}
#endif

#endif
