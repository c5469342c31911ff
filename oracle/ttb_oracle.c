/*
 * ttb_oracle.c -- TEST INFRASTRUCTURE ONLY (see ttb_oracle.h).
 *
 * Plain-C restatement of the reference's hot-path algorithm.  Every function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Build flags mirror the reference's Release build:
 * -O3 -ffp-contract=off (proj/CMakeLists.txt:17-21), no fast-math, so float
 * arithmetic is single-rounded IEEE with subnormals kept.
 */
#include "ttb_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- kinds -- */

/* problem.cpp:9-17 */
int orc_element_bytes(int kind) {
  static const int bytes[4] = {4, 8, 8, 16};
  return (kind >= 0 && kind < 4) ? bytes[kind] : 0;
}

/* problem.cpp:19-23 */
int orc_components(int kind) { return (kind == 2 || kind == 3) ? 2 : 1; }

static int scalar_is_double(int kind) { return kind == 1 || kind == 3; }

static char kind_char(int kind) {
  static const char c[4] = {'s', 'd', 'c', 'z'};
  return (kind >= 0 && kind < 4) ? c[kind] : '?';
}

/* kind_pair_supported (problem.cpp:45-52): equal kinds, or s<->d, or c<->z */
static int kinds_compatible(int a, int b) {
  if (a < 0 || a > 3 || b < 0 || b > 3) return 0;
  if (a == b) return 1;
  return (orc_components(a) == orc_components(b));
}

/* ----------------------------------------------------------- geometry -- */

/* Permutation::is_valid (problem.cpp:54-63) */
static int perm_ok(int n, const int* perm) {
  unsigned char seen[ORC_MAX_RANK];
  if (n < 1 || n > ORC_MAX_RANK) return 0;
  memset(seen, 0, sizeof seen);
  for (int a = 0; a < n; ++a) {
    int v = perm[a];
    if (v < 1 || v > n || seen[v - 1]) return 0;
    seen[v - 1] = 1;
  }
  return 1;
}

/* sizes_b (problem.cpp:161-168): B's k-th extent is the size of the A index
 * scattered to position k+1 */
static void b_extents(int n, const int* perm, const int64_t* sizes, int64_t* sb) {
  for (int a = 0; a < n; ++a) sb[perm[a] - 1] = sizes[a];
}

/* element_strides_a / element_strides_b (problem.cpp:170-188): column-major
 * prefix products of the leading dimensions */
static void prefix_strides(int n, const int64_t* ld, int64_t* st) {
  int64_t acc = 1;
  for (int i = 0; i < n; ++i) {
    st[i] = acc;
    acc *= ld[i];
  }
}

/* A-order strides in A and in B (element_strides_b_for_a, problem.cpp:190-197) */
static void axis_strides(int n, const int* perm, const int64_t* sizes, const int64_t* lda,
                         const int64_t* ldb, int64_t* sa, int64_t* sb_for_a) {
  int64_t dense_b[ORC_MAX_RANK], sbpos[ORC_MAX_RANK];
  if (!ldb) {
    b_extents(n, perm, sizes, dense_b);
    ldb = dense_b;
  }
  prefix_strides(n, lda ? lda : sizes, sa);
  prefix_strides(n, ldb, sbpos);
  for (int a = 0; a < n; ++a) sb_for_a[a] = sbpos[perm[a] - 1];
}

/* required_elements (problem.cpp:206-211): 1 + sum (size-1)*stride */
static int64_t footprint(int n, const int64_t* ext, const int64_t* st) {
  int64_t r = 1;
  for (int i = 0; i < n; ++i) r += (ext[i] - 1) * st[i];
  return r;
}

int64_t orc_required_elements_a(int rank, const int64_t* sizes, const int64_t* lda) {
  int64_t st[ORC_MAX_RANK];
  prefix_strides(rank, lda ? lda : sizes, st);
  return footprint(rank, sizes, st);
}

int64_t orc_required_elements_b(int rank, const int* perm, const int64_t* sizes,
                                const int64_t* ldb) {
  int64_t sb[ORC_MAX_RANK], st[ORC_MAX_RANK];
  b_extents(rank, perm, sizes, sb);
  prefix_strides(rank, ldb ? ldb : sb, st);
  return footprint(rank, sb, st);
}

/* ----------------------------------------------------------- validate -- */

/* validate (problem.cpp:107-159).  Same checks, same order, same text. */
int orc_validate(int n_perm, const int* perm, int n_sizes, const int64_t* sizes, int n_lda,
                 const int64_t* lda, int n_ldb, const int64_t* ldb, int kind_a, int kind_b,
                 char* msg, size_t msglen) {
  const int n = n_perm;
  int64_t sb[ORC_MAX_RANK];
  if (n < 1) {
    snprintf(msg, msglen, "perm: empty permutation");
    return 1;
  }
  if (!perm_ok(n, perm)) {
    snprintf(msg, msglen, "perm: not a permutation of 1..%d", n);
    return 1;
  }
  /* make_problem defaults (problem.cpp:95-102): lda <- sizes; ldb <- sizes_b
   * only when the sizes vector matches the permutation */
  if (n_lda < 0) {
    n_lda = n_sizes;
    lda = sizes;
  }
  if (n_ldb < 0) {
    if (n_sizes == n) {
      b_extents(n, perm, sizes, sb);
      n_ldb = n;
      ldb = sb;
    } else {
      n_ldb = 0;
    }
  }
  if (n_sizes != n) {
    snprintf(msg, msglen, "sizes: expected %d entries, got %d", n, n_sizes);
    return 1;
  }
  if (n_lda != n) {
    snprintf(msg, msglen, "lda: expected %d entries, got %d", n, n_lda);
    return 1;
  }
  if (n_ldb != n) {
    snprintf(msg, msglen, "ldb: expected %d entries, got %d", n, n_ldb);
    return 1;
  }
  for (int m = 0; m < n; ++m) {
    if (sizes[m] < 1) {
      snprintf(msg, msglen, "sizes[%d] = %lld < 1", m + 1, (long long)sizes[m]);
      return 1;
    }
    if (lda[m] < sizes[m]) {
      snprintf(msg, msglen, "lda[%d] = %lld < size %lld", m + 1, (long long)lda[m],
               (long long)sizes[m]);
      return 1;
    }
  }
  {
    int64_t ext[ORC_MAX_RANK];
    b_extents(n, perm, sizes, ext);
    for (int k = 0; k < n; ++k) {
      if (ldb[k] < ext[k]) {
        snprintf(msg, msglen, "ldb[%d] = %lld < size %lld", k + 1, (long long)ldb[k],
                 (long long)ext[k]);
        return 1;
      }
    }
  }
  if (!kinds_compatible(kind_a, kind_b)) {
    snprintf(msg, msglen, "dataType: unsupported kind pair %c%c", kind_char(kind_a),
             kind_char(kind_b));
    return 1;
  }
  {
    const int64_t cap = (int64_t)1 << 62;
    int64_t vol = 1;
    for (int m = 0; m < n; ++m) {
      if (lda[m] > cap / (vol > 1 ? vol : 1)) {
        snprintf(msg, msglen, "sizes: volume overflow");
        return 1;
      }
      vol *= lda[m];
    }
  }
  if (msglen) msg[0] = 0;
  return 0;
}

/* -------------------------------------------------------------- merge -- */

/* State of the index-merging fixpoint (problem.cpp:245-268).  A-order arrays
 * (pos = 1-based B position, ext, lda, lo/hi trace) and the B-order ldb. */
typedef struct {
  int n;
  int pos[ORC_MAX_RANK];
  int64_t ext[ORC_MAX_RANK], lda[ORC_MAX_RANK], ldb[ORC_MAX_RANK];
  int lo[ORC_MAX_RANK], hi[ORC_MAX_RANK];
} merge_state;

static void drop_a(merge_state* s, int a) {
  for (int i = a; i + 1 < s->n; ++i) {
    s->pos[i] = s->pos[i + 1];
    s->ext[i] = s->ext[i + 1];
    s->lda[i] = s->lda[i + 1];
    s->lo[i] = s->lo[i + 1];
    s->hi[i] = s->hi[i + 1];
  }
}

/* remove B position k (1-based); positions above it shift down.  Must run
 * after drop_a, with s->n still counting the old rank. */
static void drop_b(merge_state* s, int k) {
  for (int i = k - 1; i + 1 < s->n; ++i) s->ldb[i] = s->ldb[i + 1];
  s->n -= 1;
  for (int a = 0; a < s->n; ++a)
    if (s->pos[a] > k) s->pos[a] -= 1;
}

/* merge_indices (problem.cpp:270-340) */
int orc_merge(int rank, const int* perm, const int64_t* sizes, const int64_t* lda,
              const int64_t* ldb, int* out_perm, int64_t* out_sizes, int64_t* out_lda,
              int64_t* out_ldb, int* trace_lo, int* trace_hi) {
  char msg[256];
  merge_state s;
  if (orc_validate(rank, perm, rank, sizes, lda ? rank : -1, lda, ldb ? rank : -1, ldb, 0, 0,
                   msg, sizeof msg))
    return -1;
  s.n = rank;
  for (int a = 0; a < rank; ++a) {
    s.pos[a] = perm[a];
    s.ext[a] = sizes[a];
    s.lda[a] = lda ? lda[a] : sizes[a];
    s.lo[a] = s.hi[a] = a + 1;
  }
  if (ldb)
    memcpy(s.ldb, ldb, sizeof(int64_t) * (size_t)rank);
  else
    b_extents(rank, perm, sizes, s.ldb);

  /* stage 1 (problem.cpp:282-304): an extent-1 index disappears unless it is
   * a padded stride-1 index of A or of B (its padding would be lost); the
   * padding of an interior index folds into the next-inner index */
  for (int removed = 1; removed && s.n > 1;) {
    removed = 0;
    for (int a = 0; a < s.n && s.n > 1; ++a) {
      const int k = s.pos[a];
      if (s.ext[a] != 1) continue;
      if (a == 0 && s.lda[0] != 1) continue;
      if (k == 1 && s.ldb[0] != 1) continue;
      if (a > 0 && a < s.n - 1) s.lda[a - 1] *= s.lda[a];
      if (k > 1 && k < s.n) s.ldb[k - 2] *= s.ldb[k - 1];
      if (a > 0)
        s.hi[a - 1] = s.hi[a];
      else
        s.lo[1] = s.lo[0];
      drop_a(&s, a);
      drop_b(&s, k);
      removed = 1;
      break;
    }
  }

  /* stage 2 (problem.cpp:306-327): index a absorbs a+1 when they are
   * neighbours in B too and a is unpadded in both tensors; repeat until no
   * pair qualifies */
  for (int fused = 1; fused;) {
    fused = 0;
    int a = 0;
    while (a + 1 < s.n) {
      const int k = s.pos[a];
      const int64_t e = s.ext[a];
      if (s.pos[a + 1] == k + 1 && s.lda[a] == e && s.ldb[k - 1] == e) {
        s.ext[a] *= s.ext[a + 1];
        s.lda[a] *= s.lda[a + 1];
        s.ldb[k - 1] *= s.ldb[k];
        s.hi[a] = s.hi[a + 1];
        drop_a(&s, a + 1);
        drop_b(&s, k + 1);
        fused = 1;
      } else {
        ++a;
      }
    }
  }

  for (int a = 0; a < s.n; ++a) {
    out_perm[a] = s.pos[a];
    out_sizes[a] = s.ext[a];
    out_lda[a] = s.lda[a];
    out_ldb[a] = s.ldb[a];
    if (trace_lo) trace_lo[a] = s.lo[a];
    if (trace_hi) trace_hi[a] = s.hi[a];
  }
  return s.n;
}

/* --------------------------------------------------------- arithmetic -- */

/* executor.hpp:18-40: W = double if either side is double; beta == 0 never
 * reads B; otherwise alpha*W(a) + beta*W(b), two roundings, no FMA. */
#define ORC_UPDATE(W, SB, out_ptr, av, al, be, beta_zero)                   \
  do {                                                                      \
    if (beta_zero)                                                          \
      *(out_ptr) = (SB)((al) * (W)(av));                                    \
    else                                                                    \
      *(out_ptr) = (SB)((al) * (W)(av) + (be) * (W)(*(out_ptr)));           \
  } while (0)

/* --------------------------------------------------- odometer element walk */

/* support.hpp:18-60: one multi-index odometer in A order, offsets recomputed
 * from the strides for every element. */
#define ORC_WALK(SA, SB, W)                                                          \
  do {                                                                               \
    const SA* a_ = (const SA*)A;                                                     \
    SB* b_ = (SB*)B;                                                                 \
    const W al = (W)alpha, be = (W)beta;                                             \
    const int bz = (beta == 0.0);                                                    \
    int64_t idx[ORC_MAX_RANK];                                                       \
    memset(idx, 0, sizeof idx);                                                      \
    for (;;) {                                                                       \
      int64_t oa = 0, ob = 0;                                                        \
      for (int d = 0; d < rank; ++d) {                                               \
        oa += idx[d] * sa[d];                                                        \
        ob += idx[d] * sb[d];                                                        \
      }                                                                              \
      for (int q = 0; q < C; ++q) ORC_UPDATE(W, SB, &b_[ob * C + q], a_[oa * C + q], al, be, bz); \
      int d = 0;                                                                     \
      while (d < rank && ++idx[d] == sizes[d]) idx[d++] = 0;                         \
      if (d == rank) break;                                                          \
    }                                                                                \
  } while (0)

void orc_transpose(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                   const int64_t* lda, const int64_t* ldb, double alpha, const void* A,
                   double beta, void* B) {
  int64_t sa[ORC_MAX_RANK], sb[ORC_MAX_RANK];
  const int C = orc_components(kind_a);
  axis_strides(rank, perm, sizes, lda, ldb, sa, sb);
  const int da = scalar_is_double(kind_a), db = scalar_is_double(kind_b);
  if (!da && !db)
    ORC_WALK(float, float, float);
  else if (!da && db)
    ORC_WALK(float, double, double);
  else if (da && !db)
    ORC_WALK(double, float, double);
  else
    ORC_WALK(double, double, double);
}

/* ------------------------------------------------------ B-linear nest -- */

typedef struct {
  int kind_a, kind_b, C;
  int nouter;                       /* B positions 2..N, outermost last */
  int64_t ext[ORC_MAX_RANK];        /* extents of the outer B positions */
  int64_t osa[ORC_MAX_RANK], osb[ORC_MAX_RANK];
  int64_t n1, sa_in;                /* inner loop: B's stride-1 index */
  double alpha, beta;
  const void* A;
  void* B;
  int64_t lo, hi;
} nest_job;

#define ORC_NEST_BODY(SA, SB, W)                                                       \
  do {                                                                                 \
    const SA* a_ = (const SA*)j->A;                                                    \
    SB* b_ = (SB*)j->B;                                                                \
    const W al = (W)j->alpha, be = (W)j->beta;                                         \
    const int bz = (j->beta == 0.0);                                                   \
    int64_t idx[ORC_MAX_RANK];                                                         \
    int64_t rem = j->lo, oa = 0, ob = 0;                                               \
    for (int d = 0; d < j->nouter; ++d) {                                              \
      idx[d] = rem % j->ext[d];                                                        \
      rem /= j->ext[d];                                                                \
      oa += idx[d] * j->osa[d];                                                        \
      ob += idx[d] * j->osb[d];                                                        \
    }                                                                                  \
    for (int64_t t = j->lo; t < j->hi; ++t) {                                          \
      const SA* ab = a_ + oa * C;                                                      \
      SB* bb = b_ + ob * C;                                                            \
      for (int64_t i = 0; i < j->n1; ++i)                                              \
        for (int q = 0; q < C; ++q)                                                    \
          ORC_UPDATE(W, SB, &bb[i * C + q], ab[i * j->sa_in * C + q], al, be, bz);      \
      for (int d = 0; d < j->nouter; ++d) {                                            \
        oa += j->osa[d];                                                               \
        ob += j->osb[d];                                                               \
        if (++idx[d] < j->ext[d]) break;                                               \
        oa -= j->ext[d] * j->osa[d];                                                   \
        ob -= j->ext[d] * j->osb[d];                                                   \
        idx[d] = 0;                                                                    \
      }                                                                                \
    }                                                                                  \
  } while (0)

static void* nest_worker(void* arg) {
  const nest_job* j = (const nest_job*)arg;
  const int C = j->C;
  const int da = scalar_is_double(j->kind_a), db = scalar_is_double(j->kind_b);
  if (!da && !db)
    ORC_NEST_BODY(float, float, float);
  else if (!da && db)
    ORC_NEST_BODY(float, double, double);
  else if (da && !db)
    ORC_NEST_BODY(double, float, double);
  else
    ORC_NEST_BODY(double, double, double);
  return NULL;
}

/* run_reference (executor.cpp:283-313) + parallel_ranges (executor.cpp:91-105):
 * outer loops walk B positions N..2, the innermost runs along B's stride-1
 * index; the flattened outer space is cut into `threads` contiguous ranges. */
void orc_reference_nest(int kind_a, int kind_b, int rank, const int* perm,
                        const int64_t* sizes, const int64_t* lda, const int64_t* ldb,
                        double alpha, const void* A, double beta, void* B, int threads) {
  int64_t sa[ORC_MAX_RANK], sb[ORC_MAX_RANK];
  int inv[ORC_MAX_RANK] = {0};
  nest_job base;
  memset(&base, 0, sizeof base);
  axis_strides(rank, perm, sizes, lda, ldb, sa, sb);
  for (int a = 0; a < rank; ++a) inv[perm[a] - 1] = a;
  base.kind_a = kind_a;
  base.kind_b = kind_b;
  base.C = orc_components(kind_a);
  base.alpha = alpha;
  base.beta = beta;
  base.A = A;
  base.B = B;
  base.n1 = sizes[inv[0]];
  base.sa_in = sa[inv[0]];
  int64_t total = 1;
  /* odometer digit 0 = B position 2 (fastest), last digit = B position N */
  for (int k = 1; k < rank; ++k) {
    const int axis = inv[k];
    base.ext[base.nouter] = sizes[axis];
    base.osa[base.nouter] = sa[axis];
    base.osb[base.nouter] = sb[axis];
    base.nouter++;
    total *= sizes[axis];
  }
  int64_t n = threads < 1 ? 1 : threads;
  if (n > total) n = total;
  if (n <= 1) {
    base.lo = 0;
    base.hi = total;
    nest_worker(&base);
    return;
  }
  nest_job* jobs = (nest_job*)malloc(sizeof(nest_job) * (size_t)n);
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n);
  for (int64_t t = 0; t < n; ++t) {
    jobs[t] = base;
    jobs[t].lo = total * t / n;
    jobs[t].hi = total * (t + 1) / n;
    if (t) pthread_create(&tid[t], NULL, nest_worker, &jobs[t]);
  }
  nest_worker(&jobs[0]);
  for (int64_t t = 1; t < n; ++t) pthread_join(tid[t], NULL);
  free(jobs);
  free(tid);
}

/* -------------------------------------------------- generator/checksum -- */

uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* walk the logical box; callback gets memory offset (elements) and the global
 * column-major logical index */
#define ORC_BOX_WALK(BODY)                                                          \
  do {                                                                              \
    int64_t st_[ORC_MAX_RANK], gst_[ORC_MAX_RANK], idx_[ORC_MAX_RANK];              \
    int64_t acc_ = 1;                                                               \
    prefix_strides(rank, ld ? ld : sizes, st_);                                     \
    for (int d_ = 0; d_ < rank; ++d_) {                                             \
      gst_[d_] = acc_;                                                              \
      acc_ *= global_sizes ? global_sizes[d_] : sizes[d_];                          \
      idx_[d_] = 0;                                                                 \
    }                                                                               \
    int64_t gbase_ = 0;                                                             \
    if (origin)                                                                     \
      for (int d_ = 0; d_ < rank; ++d_) gbase_ += origin[d_] * gst_[d_];            \
    for (;;) {                                                                      \
      int64_t off = 0, gidx = gbase_;                                               \
      for (int d_ = 0; d_ < rank; ++d_) {                                           \
        off += idx_[d_] * st_[d_];                                                  \
        gidx += idx_[d_] * gst_[d_];                                                \
      }                                                                             \
      BODY;                                                                         \
      int d_ = 0;                                                                   \
      while (d_ < rank && ++idx_[d_] == sizes[d_]) idx_[d_++] = 0;                  \
      if (d_ == rank) break;                                                        \
    }                                                                               \
  } while (0)

void orc_fill_uniform(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                      const int64_t* origin, const int64_t* global_sizes, uint64_t seed,
                      void* buf) {
  const int C = orc_components(kind);
  const uint64_t key = seed * 0x9E3779B97F4A7C15ull;
  if (scalar_is_double(kind)) {
    double* p = (double*)buf;
    ORC_BOX_WALK({
      for (int q = 0; q < C; ++q) {
        const uint64_t u = orc_splitmix64(key + (uint64_t)(gidx * C + q));
        p[off * C + q] = (double)(u >> 11) * 0x1.0p-53 * 2.0 - 1.0;
      }
    });
  } else {
    float* p = (float*)buf;
    ORC_BOX_WALK({
      for (int q = 0; q < C; ++q) {
        const uint64_t u = orc_splitmix64(key + (uint64_t)(gidx * C + q));
        p[off * C + q] = (float)(u >> 40) * 0x1.0p-24f * 2.0f - 1.0f;
      }
    });
  }
}

void orc_fill_sentinel(int kind, int64_t elements, void* buf) {
  const int64_t n = elements * orc_components(kind);
  if (scalar_is_double(kind)) {
    const uint64_t bits = 0x7FF8DEADBEEF0001ull;
    uint64_t* p = (uint64_t*)buf;
    for (int64_t i = 0; i < n; ++i) p[i] = bits;
  } else {
    const uint32_t bits = 0x7FC0FFEEu;
    uint32_t* p = (uint32_t*)buf;
    for (int64_t i = 0; i < n; ++i) p[i] = bits;
  }
}

uint64_t orc_checksum(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                      const int64_t* origin, const int64_t* global_sizes, const void* buf) {
  const int C = orc_components(kind);
  uint64_t sum = 0;
  if (scalar_is_double(kind)) {
    const uint64_t* p = (const uint64_t*)buf;
    ORC_BOX_WALK({
      for (int q = 0; q < C; ++q) {
        const uint64_t j = (uint64_t)(gidx * C + q);
        sum += orc_splitmix64((j * 0xD1B54A32D192ED03ull) ^ p[off * C + q]);
      }
    });
  } else {
    const uint32_t* p = (const uint32_t*)buf;
    ORC_BOX_WALK({
      for (int q = 0; q < C; ++q) {
        const uint64_t j = (uint64_t)(gidx * C + q);
        sum += orc_splitmix64((j * 0xD1B54A32D192ED03ull) ^ (uint64_t)p[off * C + q]);
      }
    });
  }
  return sum;
}

/* bandwidth_gibs (tuner.cpp:18-25) in decimal GB/s */
double orc_bandwidth_gbs(int64_t elements, int kind_a, int kind_b, double beta,
                         double seconds) {
  const double n = (double)elements;
  double bytes = n * orc_element_bytes(kind_a) + n * orc_element_bytes(kind_b);
  if (beta != 0.0) bytes += n * orc_element_bytes(kind_b);
  return bytes / 1e9 / seconds;
}
