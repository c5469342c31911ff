// api.cpp -- the extern "C" boundary (include/ttb.h).
//
// Mirrors the reference's entry points (executor.hpp:80-88, problem.hpp:51-102,
// tuner.hpp:53-62): problem checks with the reference's messages, an
// in-memory plan cache keyed by canonical_key (problem.cpp:228-241) plus the
// device, CUDA-event autotuning, and the stream-ordered launch.  No exception
// crosses the ABI; failures become status codes plus ttb_last_error().
#include "../../include/ttb.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "cache.hpp"
#include "launch.hpp"
#include "plan.hpp"
#include "problem.hpp"

namespace ttb {
unsigned long long launch_total();
std::string emit_entry_symbol(const Problem& p);
void emit_cuda(const Problem& m, const Geo& g, const Spec& spec, const std::string& base,
               const std::string& plan_text, const std::string& key, std::string* header,
               std::string* source);
}

using namespace ttb;

namespace {

thread_local std::string t_err;

int ok() {
  t_err.clear();
  return TTB_OK;
}

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? TTB_ENOMEM : TTB_ECUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

std::vector<int64_t> vec64(const int64_t* p, int n) {
  return p ? std::vector<int64_t>(p, p + n) : std::vector<int64_t>{};
}

Problem from_args(int ka, int kb, int rank, const int* perm, const int64_t* sizes,
                  const int64_t* lda, const int64_t* ldb, double alpha, double beta) {
  std::vector<int> pm = perm && rank > 0 ? std::vector<int>(perm, perm + rank) : std::vector<int>{};
  return make(std::move(pm), vec64(sizes, std::max(rank, 0)), ka, kb, alpha, beta,
              vec64(lda, std::max(rank, 0)), vec64(ldb, std::max(rank, 0)));
}

int current_device(int* dev, int* sms) {
  cudaError_t e = cudaGetDevice(dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, *dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  return TTB_OK;
}

}  // namespace

struct ttb_plan_s;

// A box of an oversized problem: its element offsets in A and B and the plan
// of its extents (same strides as the whole problem)
struct SubBox {
  int64_t off_a = 0, off_b = 0;
  std::shared_ptr<ttb_plan_s> plan;
};

struct ttb_plan_s {
  Problem orig;
  Merged merged;
  Geo geo;
  std::vector<Spec> cands;
  Prepared prep;      // chosen variant
  Prepared fallback;  // element-aligned variant for misaligned buffers
  int device = 0, sms = 148;
  std::string key;    // canonical_key + device
  bool cached = true;
  float tuned_ms = 0.0f;  // best time of the last autotune
  // end-to-end staging (ttb_plan_execute_host)
  void* dA = nullptr;
  void* dB = nullptr;
  cudaStream_t hs = nullptr;  // host->device copies
  cudaStream_t ks = nullptr;  // slab kernels (pipelined path)
  cudaStream_t ds = nullptr;  // device->host copies (pipelined path)
  cudaStream_t host_tail = nullptr;  // stream that ends the last host call (hs or ds), null before the first
  std::vector<cudaEvent_t> evs;
  std::unordered_map<int64_t, std::unique_ptr<ttb_plan_s>> chunk_plans;  // by slab extent
  // problems whose A or B footprint reaches 2^31 elements run as boxes below
  // that size (every kernel keeps 32-bit index spaces); empty otherwise
  std::vector<SubBox> boxes;
  ~ttb_plan_s() {
    if (dA) cudaFree(dA);
    if (dB) cudaFree(dB);
    if (hs) cudaStreamDestroy(hs);
    if (ks) cudaStreamDestroy(ks);
    if (ds) cudaStreamDestroy(ds);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
  }
  size_t bytes_a() const { return static_cast<size_t>(orig.footprint_a()) * kind_bytes(orig.kind_a); }
  size_t bytes_b() const { return static_cast<size_t>(orig.footprint_b()) * kind_bytes(orig.kind_b); }
};

namespace {

std::mutex g_mu;
std::unordered_map<std::string, std::string> g_choice;                 // key -> spec text
// one-shot API plans, shared: a caller keeps its plan alive while executing
// even if an autotune elsewhere drops the cache (re-entrant)
std::unordered_map<std::string, std::shared_ptr<ttb_plan_s>> g_plans;

constexpr int64_t kBoxLimit = int64_t{1} << 31;

// Halve the box along its largest-stride axis (of the side that is too big)
// until both footprints are below 2^31 elements.
void split_boxes(const Problem& m, std::vector<std::pair<std::vector<int64_t>, std::vector<int64_t>>>* out) {
  const std::vector<int64_t> sa = m.a_strides(), sb = m.b_strides_of_a();
  const int r = m.rank();
  std::vector<std::pair<std::vector<int64_t>, std::vector<int64_t>>> work{
      {std::vector<int64_t>(static_cast<size_t>(r), 0), m.sizes}};
  while (!work.empty()) {
    auto b = work.back();
    work.pop_back();
    int64_t fa = 1, fb = 1;
    for (int a = 0; a < r; ++a) {
      fa += (b.second[a] - 1) * sa[a];
      fb += (b.second[a] - 1) * sb[a];
    }
    if (fa < kBoxLimit && fb < kBoxLimit) {
      out->push_back(b);
      continue;
    }
    const std::vector<int64_t>& st = fa >= kBoxLimit ? sa : sb;
    int ax = -1;
    for (int a = 0; a < r; ++a)
      if (b.second[a] > 1 && (ax < 0 || st[a] > st[ax])) ax = a;
    auto lo = b, hi = b;
    lo.second[ax] = b.second[ax] / 2;
    hi.first[ax] += lo.second[ax];
    hi.second[ax] = b.second[ax] - lo.second[ax];
    work.push_back(hi);
    work.push_back(lo);
  }
}

int build_plan(const Problem& p, int flags, std::unique_ptr<ttb_plan_s>* out) {
  auto pl = std::make_unique<ttb_plan_s>();
  pl->orig = p;
  pl->merged = fuse_indices(p);
  if (pl->merged.p.rank() > kMaxRank)
    return fail(TTB_EINVAL, "perm: rank " + std::to_string(pl->merged.p.rank()) +
                                " after merging exceeds TTB_MAX_RANK");
  pl->geo = make_geo(pl->merged.p);
  int rc = current_device(&pl->device, &pl->sms);
  if (rc) return rc;
  pl->key = cache_key(p) + "@dev" + std::to_string(pl->device);
  pl->cached = !(flags & TTB_PLAN_NO_CACHE);
  if (pl->geo.foot_a >= kBoxLimit || pl->geo.foot_b >= kBoxLimit) {
    // oversized: boxes of the merged problem, one plan per distinct extent
    const Problem& m = pl->merged.p;
    const std::vector<int64_t> sa = m.a_strides(), sb = m.b_strides_of_a();
    std::vector<std::pair<std::vector<int64_t>, std::vector<int64_t>>> boxes;
    split_boxes(m, &boxes);
    std::map<std::vector<int64_t>, std::shared_ptr<ttb_plan_s>> by_ext;
    for (const auto& b : boxes) {
      std::shared_ptr<ttb_plan_s>& sub = by_ext[b.second];
      if (!sub) {
        Problem q = m;
        q.sizes = b.second;
        std::unique_ptr<ttb_plan_s> fresh;
        rc = build_plan(q, flags | TTB_PLAN_NO_CACHE, &fresh);
        if (rc) return rc;
        sub = std::shared_ptr<ttb_plan_s>(std::move(fresh));
      }
      SubBox x;
      for (int a = 0; a < m.rank(); ++a) {
        x.off_a += b.first[a] * sa[a];
        x.off_b += b.first[a] * sb[a];
      }
      x.plan = sub;
      pl->boxes.push_back(x);
    }
    const ttb_plan_s& first = *pl->boxes.front().plan;
    pl->cands = first.cands;
    pl->prep = first.prep;
    pl->fallback = first.fallback;
    *out = std::move(pl);
    return TTB_OK;
  }
  pl->cands = candidates(pl->geo);
  std::string why;
  bool have = false;
  if (pl->cached) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_choice.find(pl->key);
    Spec s;
    if (it != g_choice.end() && Spec::parse(it->second, &s))
      have = prepare(pl->geo, s, pl->sms, &pl->prep, &why);
  }
  for (size_t i = 0; !have && i < pl->cands.size(); ++i)
    have = prepare(pl->geo, pl->cands[i], pl->sms, &pl->prep, &why);
  if (!have) return fail(TTB_EINTERNAL, "plan: no applicable kernel variant (" + why + ")");
  if (!prepare(pl->geo, pl->cands.back(), pl->sms, &pl->fallback, &why)) pl->fallback = pl->prep;
  cudaError_t e = cudaGetLastError();  // occupancy queries surface context errors here
  if (e != cudaSuccess) return cuda_fail(e, "plan");
  *out = std::move(pl);
  return TTB_OK;
}

cudaError_t launch(const Geo& g, Prepared pr, const void* A, void* B, cudaStream_t s) {
  switch (pr.spec.v) {
    case kCopy:
      pr.cp.A = A;
      pr.cp.B = B;
      return launch_copy(g.ka, g.kb, pr.spec.w1, pr.mode, pr.cp, pr.l, s);
    case kRt:
      pr.rp.A = A;
      pr.rp.B = B;
      return launch_rt(g.ka, g.kb, pr.spec.w1, pr.spec.w2, pr.mode, pr.rp, pr.l, s);
    case kTma:
      return launch_tma(g.ka, g.kb, pr.mode, pr.tp, A, B, pr.l, s);
    default:
      pr.sp.A = A;
      pr.sp.B = B;
      if (pr.sp.dense == 5) return launch_btile(g.ka, g.kb, pr.mode, pr.sp, pr.bt, pr.l, s);
      return launch_smem(g.ka, g.kb, pr.mode, pr.sp, pr.l, s);
  }
}

bool aligned(const void* p, int a) { return reinterpret_cast<uintptr_t>(p) % static_cast<uintptr_t>(a) == 0; }

// alpha/beta come from the call: one-shot plans are shared by every problem
// with the same canonical key and update mode (move / scale / update)
int execute(ttb_plan_s* pl, const Prepared& pr0, const void* A, void* B, cudaStream_t s,
            double alpha, double beta) {
  if (!A) return fail(TTB_EINVAL, "A buffer: null pointer");
  if (!B) return fail(TTB_EINVAL, "B buffer: null pointer");
  if (!pl->boxes.empty()) {
    const size_t ea = static_cast<size_t>(kind_bytes(pl->orig.kind_a));
    const size_t eb = static_cast<size_t>(kind_bytes(pl->orig.kind_b));
    for (const SubBox& x : pl->boxes) {
      const int rc = execute(x.plan.get(), x.plan->prep,
                             static_cast<const char*>(A) + static_cast<size_t>(x.off_a) * ea,
                             static_cast<char*>(B) + static_cast<size_t>(x.off_b) * eb, s, alpha, beta);
      if (rc) return rc;
    }
    return ok();
  }
  const Prepared* pr = &pr0;
  if (!aligned(A, pr->a_align) || !aligned(B, pr->b_align)) pr = &pl->fallback;
  if (!aligned(A, pr->a_align)) return fail(TTB_EINVAL, "A buffer: misaligned for its element kind");
  if (!aligned(B, pr->b_align)) return fail(TTB_EINVAL, "B buffer: misaligned for its element kind");
  Prepared run = *pr;
  run.cp.sc = run.rp.sc = run.sp.sc = run.tp.sc = Scale{alpha, beta};
  // an error left behind by an unrelated earlier runtime call must not be
  // reported as this launch's (cudaGetLastError after the launch reads it)
  const cudaError_t stale = cudaGetLastError();
  if (stale != cudaSuccess && cudaPeekAtLastError() != cudaSuccess)
    return cuda_fail(stale, "before the kernel launch (sticky)");
  const cudaError_t e = launch(pl->geo, run, A, B, s);
  if (e != cudaSuccess)
    return cuda_fail(e, ("kernel launch (" + run.spec.text() + ", grid " + std::to_string(run.l.grid) + ", block " +
                            std::to_string(run.l.block) + ", smem " + std::to_string(run.l.smem) + ")").c_str());
  return ok();
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const InvalidArgument& e) {
    return fail(TTB_EINVAL, e.what);
  } catch (const std::bad_alloc&) {
    return fail(TTB_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(TTB_EINTERNAL, e.what());
  } catch (...) {
    return fail(TTB_EINTERNAL, "unknown error");
  }
}

int box_params(int kind, int rank, const int64_t* sizes, const int64_t* ld, const int64_t* origin,
               const int64_t* gsizes, BoxParams* bp) {
  if (rank < 1 || rank > 16 || !sizes) return fail(TTB_EINVAL, "box: bad rank");
  if (kind < 0 || kind > 3) return fail(TTB_EINVAL, "box: bad kind");
  bp->rank = rank;
  bp->C = kind_components(kind);
  int64_t acc = 1, gacc = 1;
  bp->gbase = 0;
  bp->total = 1;
  for (int d = 0; d < rank; ++d) {
    if (sizes[d] < 1) return fail(TTB_EINVAL, "box: extent < 1");
    bp->ext[d] = sizes[d];
    bp->st[d] = acc;
    acc *= ld ? ld[d] : sizes[d];
    bp->gst[d] = gacc;
    if (origin) bp->gbase += origin[d] * gacc;
    gacc *= gsizes ? gsizes[d] : sizes[d];
    bp->total *= sizes[d];
  }
  return TTB_OK;
}

// ---------------------------------------------------------------------------
// Pipelined host path.  PCIe is full duplex (both directions at once measure
// ~2x one direction), so ttb_plan_execute_host cuts the problem into K slabs
// along one (merged) axis `a`: slab i's A part streams in on one copy engine,
// its kernel runs, and its B part streams out on the other while slab i+1
// streams in.  A slab is, on each side, `height` rows of `width` bytes at a
// fixed pitch: the axis is chosen so that every axis above it on that side is
// unpadded (a 2D copy) and the rows are long enough for the copy engines.

bool pinned(const void* p) {
  cudaPointerAttributes at{};
  const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();  // a pageable pointer can leave "invalid value" behind
  return ok;
}

struct SlabSide {
  int64_t stride = 0;  // elements between consecutive indices of the slab axis
  int64_t pitch = 0;   // elements between rows
  int64_t height = 1;  // rows
  int64_t foot = 0;    // required elements of the whole buffer
  int eb = 4;          // element bytes
};

struct HostPipe {
  int axis = 0;        // merged A axis the slabs cut
  int64_t n = 0, ext = 0;
  SlabSide a, b;
  bool b_in = false;   // B slabs travel to the device too (beta != 0 or padded below the axis)
};

// rows of one side for slab axis extent at position `q` of the side's order
bool slab_side(const std::vector<int64_t>& n, const std::vector<int64_t>& ld, int q, int eb,
               int64_t foot, SlabSide* out) {
  const int r = static_cast<int>(n.size());
  int64_t st = 1;
  for (int k = 0; k < q; ++k) st *= ld[static_cast<size_t>(k)];
  out->stride = st;
  out->pitch = st * ld[static_cast<size_t>(q)];
  out->height = 1;
  for (int k = q + 1; k < r; ++k) {
    if (k < r - 1 && ld[static_cast<size_t>(k)] != n[static_cast<size_t>(k)]) return false;
    out->height *= n[static_cast<size_t>(k)];
  }
  out->foot = foot;
  out->eb = eb;
  return true;
}

int64_t env_i64(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  return v && std::atoll(v) > 0 ? std::atoll(v) : dflt;
}

bool pick_pipe(const Problem& p, HostPipe* out) {
  const int r = p.rank();
  const int64_t kmax = env_i64("TTB_HOST_SLABS", 32);
  const int64_t min_row = env_i64("TTB_HOST_MIN_ROW", 4096);       // bytes
  const int64_t min_slab = env_i64("TTB_HOST_MIN_SLAB_KB", 4096) << 10;
  const int ea = kind_bytes(p.kind_a), eb = kind_bytes(p.kind_b);
  const int64_t bytes = p.footprint_a() * ea + p.footprint_b() * eb;
  const int64_t kwant = std::min(kmax, bytes / std::max<int64_t>(1, min_slab));
  if (kwant < 2) return false;
  const std::vector<int64_t> nb = p.b_extents();
  bool found = false;
  int64_t best_k = 0, best_w = 0;
  int best_cb = 0;
  for (int a = 0; a < r; ++a) {
    const int64_t n = p.sizes[static_cast<size_t>(a)];
    HostPipe h;
    const int q = p.perm[static_cast<size_t>(a)] - 1;
    if (!slab_side(p.sizes, p.lda, a, ea, p.footprint_a(), &h.a) ||
        !slab_side(nb, p.ldb, q, eb, p.footprint_b(), &h.b))
      continue;
    // as many slabs as the axis allows while both sides keep rows >= min_row
    // (fewer, wider slabs rather than no pipeline at all)
    int64_t k = std::min(n, kwant), ext = 0, w = 0, wa = 0, wb = 0;
    for (; k >= 2; k = k > 8 ? k * 3 / 4 : k - 1) {
      ext = (n + k - 1) / k;
      wa = h.a.height == 1 ? INT64_MAX : ext * h.a.stride * ea;
      wb = h.b.height == 1 ? INT64_MAX : ext * h.b.stride * eb;
      w = std::min(wa, wb);
      if (w >= min_row) break;
    }
    if (k < 2) continue;
    k = (n + ext - 1) / ext;
    // 2D copies with narrow rows at a wide pitch lose up to a quarter of the
    // link (device->host, 5 KB rows: 43.8 of 57 GB/s, scripts/copy2d_probe.py),
    // so the axis with more sides whose rows stay >= 32 KB wins (c5_t17: both
    // sides contiguous along its outermost axis, 61 -> 83 GB/s end to end)
    const int cb = (wa >= 32768 ? 1 : 0) + (wb >= 32768 ? 1 : 0);
    if (found && (cb < best_cb || (cb == best_cb && (k < best_k || (k == best_k && w <= best_w))))) continue;
    found = true;
    best_cb = cb;
    best_k = k;
    best_w = w;
    h.axis = a;
    h.n = n;
    h.ext = ext;
    h.b_in = p.beta != 0.0;
    for (int j = 0; j < q; ++j)
      if (p.ldb[static_cast<size_t>(j)] != nb[static_cast<size_t>(j)]) h.b_in = true;
    *out = h;
  }
  if (found && std::getenv("TTB_HOST_DEBUG"))
    std::fprintf(stderr, "[ttb host pipe] axis %d of %d, extent %lld, %lld slabs of %lld; A rows %lld x %lld B (pitch %lld), B rows %lld x %lld B (pitch %lld)\n",
                 out->axis, r, static_cast<long long>(out->n), static_cast<long long>(best_k),
                 static_cast<long long>(out->ext), static_cast<long long>(out->a.height),
                 static_cast<long long>(out->ext * out->a.stride * ea), static_cast<long long>(out->a.pitch * ea),
                 static_cast<long long>(out->b.height), static_cast<long long>(out->ext * out->b.stride * eb),
                 static_cast<long long>(out->b.pitch * eb));
  return found;
}

// rows [j0, j1) of the slab axis on one side, host <-> device, same layout
cudaError_t copy_slab(const SlabSide& sd, int64_t j0, int64_t j1, char* dst, const char* src,
                      cudaMemcpyKind kind, cudaStream_t s) {
  const int64_t w = (j1 - j0) * sd.stride;  // elements per row
  const int64_t base = j0 * sd.stride;
  int64_t h = sd.height;
  // the last row may run past the buffer's end (padding of the lower axes)
  const int64_t last = base + (h - 1) * sd.pitch;
  const int64_t tail = std::min(w, sd.foot - last);
  if (tail < w) --h;
  const size_t e = static_cast<size_t>(sd.eb);
  cudaError_t err = cudaSuccess;
  for (int64_t h0 = 0; h0 < h && err == cudaSuccess; h0 += 32768) {
    const int64_t hh = std::min<int64_t>(32768, h - h0);
    const size_t off = static_cast<size_t>(base + h0 * sd.pitch) * e;
    err = hh == 1 ? cudaMemcpyAsync(dst + off, src + off, static_cast<size_t>(w) * e, kind, s)
                  : cudaMemcpy2DAsync(dst + off, static_cast<size_t>(sd.pitch) * e, src + off,
                                      static_cast<size_t>(sd.pitch) * e, static_cast<size_t>(w) * e,
                                      static_cast<size_t>(hh), kind, s);
  }
  if (err == cudaSuccess && tail < w) {
    const size_t off = static_cast<size_t>(last) * e;
    err = cudaMemcpyAsync(dst + off, src + off, static_cast<size_t>(tail) * e, kind, s);
  }
  return err;
}

int run_pipe(ttb_plan_s* plan, const HostPipe& hp, const void* A_host, void* B_host, bool wait) {
  cudaError_t e;
  for (cudaStream_t* st : {&plan->ks, &plan->ds})
    if (!*st && (e = cudaStreamCreateWithFlags(st, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
  const int64_t k = (hp.n + hp.ext - 1) / hp.ext;
  while (static_cast<int64_t>(plan->evs.size()) < 2 * k) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "cudaEventCreate");
    plan->evs.push_back(ev);
  }
  const Problem& mp = plan->merged.p;
  char* dA = static_cast<char*>(plan->dA);
  char* dB = static_cast<char*>(plan->dB);
  const char* hA = static_cast<const char*>(A_host);
  char* hB = static_cast<char*>(B_host);
  for (int64_t i = 0; i < k; ++i) {
    const int64_t j0 = i * hp.ext, j1 = std::min(hp.n, j0 + hp.ext), ext = j1 - j0;
    cudaEvent_t ev_in = plan->evs[static_cast<size_t>(2 * i)];
    cudaEvent_t ev_k = plan->evs[static_cast<size_t>(2 * i + 1)];
    if ((e = copy_slab(hp.a, j0, j1, dA, hA, cudaMemcpyHostToDevice, plan->hs)) != cudaSuccess)
      return cuda_fail(e, "H2D A slab");
    if (hp.b_in && (e = copy_slab(hp.b, j0, j1, dB, hB, cudaMemcpyHostToDevice, plan->hs)) != cudaSuccess)
      return cuda_fail(e, "H2D B slab");
    cudaEventRecord(ev_in, plan->hs);
    cudaStreamWaitEvent(plan->ks, ev_in, 0);
    std::unique_ptr<ttb_plan_s>& sub = plan->chunk_plans[ext];
    if (!sub) {  // the slab's problem: same perm/lda/ldb, slab axis extent = ext
      Problem q = mp;
      q.sizes[static_cast<size_t>(hp.axis)] = ext;
      const int rc = build_plan(q, TTB_PLAN_NO_CACHE, &sub);
      if (rc) return rc;
      std::string why;
      Prepared pr;  // keep the parent's (possibly autotuned) variant where it applies
      if (prepare(sub->geo, plan->prep.spec, sub->sms, &pr, &why)) sub->prep = pr;
    }
    const int rc = execute(sub.get(), sub->prep, dA + static_cast<size_t>(j0 * hp.a.stride) * hp.a.eb,
                           dB + static_cast<size_t>(j0 * hp.b.stride) * hp.b.eb, plan->ks, mp.alpha,
                           mp.beta);
    if (rc) return rc;
    cudaEventRecord(ev_k, plan->ks);
    cudaStreamWaitEvent(plan->ds, ev_k, 0);
    if ((e = copy_slab(hp.b, j0, j1, hB, dB, cudaMemcpyDeviceToHost, plan->ds)) != cudaSuccess)
      return cuda_fail(e, "D2H B slab");
  }
  plan->host_tail = plan->ds;  // the stream whose end is the call's end
  if (wait && (e = cudaStreamSynchronize(plan->ds)) != cudaSuccess) return cuda_fail(e, "sync");
  return ok();
}

int host_call(ttb_plan plan, const void* A_host, void* B_host, bool wait) {
  if (!A_host || !B_host) return fail(TTB_EINVAL, "host buffers: null pointer");
  cudaError_t e;
  const size_t na = plan->bytes_a(), nb = plan->bytes_b();
  if (!plan->hs && (e = cudaStreamCreateWithFlags(&plan->hs, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_fail(e, "cudaStreamCreate");
  if (!plan->dA && (e = cudaMalloc(&plan->dA, na)) != cudaSuccess) return cuda_fail(e, "cudaMalloc A");
  if (!plan->dB && (e = cudaMalloc(&plan->dB, nb)) != cudaSuccess) return cuda_fail(e, "cudaMalloc B");
  // a call still in flight on this plan (execute_host_async without host_sync)
  // owns the staging buffers and the slab events: finish it first
  if (plan->host_tail && (e = cudaStreamSynchronize(plan->host_tail)) != cudaSuccess)
    return cuda_fail(e, "sync of the previous host call");
  const char* hp = std::getenv("TTB_HOST_PATH");  // "staged": force the sequential path
  if (!(hp && std::strcmp(hp, "staged") == 0) && pinned(A_host) && pinned(B_host)) {
    HostPipe hpipe;
    if (pick_pipe(plan->merged.p, &hpipe)) return run_pipe(plan, hpipe, A_host, B_host, wait);
  }
  cudaStream_t s = plan->hs;
  // B's padding must come back unchanged, so B travels to the device when
  // it is read (beta != 0) or padded
  const bool b_in = plan->orig.beta != 0.0 || plan->orig.footprint_b() != plan->orig.elements();
  if ((e = cudaMemcpyAsync(plan->dA, A_host, na, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "H2D A");
  if (b_in && (e = cudaMemcpyAsync(plan->dB, B_host, nb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "H2D B");
  const int rc = execute(plan, plan->prep, plan->dA, plan->dB, s, plan->orig.alpha, plan->orig.beta);
  if (rc) return rc;
  if ((e = cudaMemcpyAsync(B_host, plan->dB, nb, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "D2H B");
  plan->host_tail = s;
  if (wait && (e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "sync");
  return ok();
}

}  // namespace

extern "C" {

const char* ttb_last_error(void) { return t_err.c_str(); }
const char* ttb_version(void) { return TTB_VERSION; }

int ttb_validate(int n_perm, const int* perm, int n_sizes, const int64_t* sizes, int n_lda,
                 const int64_t* lda, int n_ldb, const int64_t* ldb, int kind_a, int kind_b) {
  return guarded([&] {
    Problem p = make(perm ? std::vector<int>(perm, perm + std::max(n_perm, 0)) : std::vector<int>{},
                     vec64(sizes, std::max(n_sizes, 0)), kind_a, kind_b, 1.0, 0.0,
                     n_lda >= 0 ? vec64(lda, n_lda) : std::vector<int64_t>{},
                     n_ldb >= 0 ? vec64(ldb, n_ldb) : std::vector<int64_t>{});
    // an explicitly empty lda/ldb (n = 0) must still be reported as such
    if (n_lda == 0) p.lda.clear();
    if (n_ldb == 0) p.ldb.clear();
    check(p);
    return ok();
  });
}

int64_t ttb_required_elements_a(int rank, const int64_t* sizes, const int64_t* lda) {
  if (rank < 1 || !sizes) return -1;
  Problem p;
  p.sizes = vec64(sizes, rank);
  p.lda = lda ? vec64(lda, rank) : p.sizes;
  return p.footprint_a();
}

int64_t ttb_required_elements_b(int rank, const int* perm, const int64_t* sizes,
                                const int64_t* ldb) {
  if (rank < 1 || !sizes || !perm) return -1;
  Problem p = make(std::vector<int>(perm, perm + rank), vec64(sizes, rank), 0, 0, 1.0, 0.0, {},
                   ldb ? vec64(ldb, rank) : std::vector<int64_t>{});
  if (p.ldb.size() != static_cast<size_t>(rank)) return -1;
  return p.footprint_b();
}

int ttb_merge_indices(int rank, const int* perm, const int64_t* sizes, const int64_t* lda,
                      const int64_t* ldb, int* out_rank, int* out_perm, int64_t* out_sizes,
                      int64_t* out_lda, int64_t* out_ldb, int* trace_lo, int* trace_hi) {
  return guarded([&] {
    const Merged m = fuse_indices(from_args(0, 0, rank, perm, sizes, lda, ldb, 1.0, 0.0));
    const int r = m.p.rank();
    if (out_rank) *out_rank = r;
    for (int a = 0; a < r; ++a) {
      if (out_perm) out_perm[a] = m.p.perm[a];
      if (out_sizes) out_sizes[a] = m.p.sizes[a];
      if (out_lda) out_lda[a] = m.p.lda[a];
      if (out_ldb) out_ldb[a] = m.p.ldb[a];
      if (trace_lo) trace_lo[a] = m.runs[a].first;
      if (trace_hi) trace_hi[a] = m.runs[a].second;
    }
    return ok();
  });
}

int ttb_canonical_key(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                      const int64_t* lda, const int64_t* ldb, double alpha, double beta,
                      char* buf, size_t len) {
  return guarded([&] {
    const std::string k =
        cache_key(from_args(kind_a, kind_b, rank, perm, sizes, lda, ldb, alpha, beta));
    if (!buf || len <= k.size()) return fail(TTB_EINVAL, "canonical_key: buffer too small");
    std::memcpy(buf, k.c_str(), k.size() + 1);
    return ok();
  });
}

double ttb_bandwidth_gbs(int kind_a, int kind_b, int64_t elements, double beta, double seconds) {
  if (!(seconds > 0.0) || kind_a < 0 || kind_a > 3 || kind_b < 0 || kind_b > 3) return -1.0;
  const double n = static_cast<double>(elements);
  double bytes = n * kind_bytes(kind_a) + n * kind_bytes(kind_b);
  if (beta != 0.0) bytes += n * kind_bytes(kind_b);
  return bytes / 1e9 / seconds;
}

int ttb_plan_create(ttb_plan* out, int kind_a, int kind_b, int rank, const int* perm,
                    const int64_t* sizes, const int64_t* lda, const int64_t* ldb, double alpha,
                    double beta, int flags) {
  return guarded([&] {
    if (!out) return fail(TTB_EINVAL, "plan: null output handle");
    *out = nullptr;
    const Problem p = from_args(kind_a, kind_b, rank, perm, sizes, lda, ldb, alpha, beta);
    check(p);
    std::unique_ptr<ttb_plan_s> pl;
    const int rc = build_plan(p, flags, &pl);
    if (rc) return rc;
    *out = pl.release();
    return ok();
  });
}

int ttb_plan_destroy(ttb_plan plan) {
  delete plan;
  return ok();
}

int ttb_plan_execute(ttb_plan plan, const void* A, void* B, ttb_stream stream) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  return guarded([&] {
    return execute(plan, plan->prep, A, B, reinterpret_cast<cudaStream_t>(stream), plan->orig.alpha,
                   plan->orig.beta);
  });
}

int ttb_transpose(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                  const int64_t* lda, const int64_t* ldb, double alpha, const void* A,
                  int64_t a_elements, double beta, void* B, int64_t b_elements,
                  ttb_stream stream) {
  return guarded([&] {
    const Problem p = from_args(kind_a, kind_b, rank, perm, sizes, lda, ldb, alpha, beta);
    check(p);  // validate first, then buffers (executor.cpp:373-374, 315-322)
    if (a_elements >= 0 && a_elements < p.footprint_a())
      return fail(TTB_EINVAL, "A buffer: too small for problem");
    if (b_elements >= 0 && b_elements < p.footprint_b())
      return fail(TTB_EINVAL, "B buffer: too small for problem");
    int dev = 0, sms = 0;
    int rc = current_device(&dev, &sms);
    if (rc) return rc;
    const int mode = p.beta != 0.0 ? 2 : (p.alpha == 1.0 ? 0 : 1);
    const std::string key = cache_key(p) + "@dev" + std::to_string(dev) + "|m" + std::to_string(mode);
    std::shared_ptr<ttb_plan_s> pl;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_plans.find(key);
      if (it != g_plans.end()) pl = it->second;
    }
    if (!pl) {
      std::unique_ptr<ttb_plan_s> fresh;
      rc = build_plan(p, TTB_PLAN_DEFAULT, &fresh);
      if (rc) return rc;
      std::lock_guard<std::mutex> lk(g_mu);
      auto& slot = g_plans[key];
      if (!slot) slot = std::shared_ptr<ttb_plan_s>(std::move(fresh));
      pl = slot;
    }
    return execute(pl.get(), pl->prep, A, B, reinterpret_cast<cudaStream_t>(stream), alpha, beta);
  });
}

int ttb_plan_execute_host(ttb_plan plan, const void* A_host, void* B_host) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  return guarded([&] { return host_call(plan, A_host, B_host, true); });
}

int ttb_plan_execute_host_async(ttb_plan plan, const void* A_host, void* B_host) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  return guarded([&] { return host_call(plan, A_host, B_host, false); });
}

int ttb_plan_host_sync(ttb_plan plan) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  return guarded([&] {
    if (plan->host_tail) {
      const cudaError_t e = cudaStreamSynchronize(plan->host_tail);
      if (e != cudaSuccess) return cuda_fail(e, "host sync");
    }
    return ok();
  });
}

int ttb_plan_autotune(ttb_plan plan, const void* A, void* B, int warmups, int reps,
                      ttb_stream stream) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  return guarded([&] {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (warmups < 0 || reps < 1)
      return fail(TTB_EINVAL, "protocol: need warmups >= 0 and repetitions >= 1");
    if (!plan->boxes.empty()) {
      // oversized problem: tune the first box (one application on return),
      // give its variant to every other box plan it applies to, and run the
      // remaining boxes once so that B holds exactly one application
      const size_t ea = static_cast<size_t>(kind_bytes(plan->orig.kind_a));
      const size_t eb = static_cast<size_t>(kind_bytes(plan->orig.kind_b));
      const SubBox& x0 = plan->boxes.front();
      int rc = ttb_plan_autotune(x0.plan.get(), static_cast<const char*>(A) + static_cast<size_t>(x0.off_a) * ea,
                                 static_cast<char*>(B) + static_cast<size_t>(x0.off_b) * eb, warmups, reps,
                                 stream);
      if (rc) return rc;
      const Spec spec = x0.plan->prep.spec;
      for (size_t i = 1; i < plan->boxes.size(); ++i) {
        ttb_plan_s* sub = plan->boxes[i].plan.get();
        Prepared pr;
        if (sub != x0.plan.get() && prepare(sub->geo, spec, sub->sms, &pr, nullptr)) sub->prep = pr;
      }
      for (size_t i = 1; i < plan->boxes.size(); ++i) {
        const SubBox& x = plan->boxes[i];
        rc = execute(x.plan.get(), x.plan->prep, static_cast<const char*>(A) + static_cast<size_t>(x.off_a) * ea,
                     static_cast<char*>(B) + static_cast<size_t>(x.off_b) * eb, s, plan->orig.alpha,
                     plan->orig.beta);
        if (rc) return rc;
      }
      plan->prep = x0.plan->prep;
      plan->tuned_ms = x0.plan->tuned_ms * static_cast<float>(plan->boxes.size());
      return ok();
    }
    void* target = B;
    void* scratch = nullptr;
    cudaError_t e;
    if (plan->orig.beta != 0.0) {  // candidates must not keep updating the caller's B
      if ((e = cudaMalloc(&scratch, plan->bytes_b())) != cudaSuccess) return cuda_fail(e, "scratch");
      if ((e = cudaMemcpyAsync(scratch, B, plan->bytes_b(), cudaMemcpyDeviceToDevice, s)) != cudaSuccess) {
        cudaFree(scratch);
        return cuda_fail(e, "scratch copy");
      }
      target = scratch;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int rc = TTB_OK;
    // best-of-reps time of one prepared candidate (measure_candidate)
    auto measure = [&](const Prepared& pr, int w, int n) {
      float b = 1e30f;
      for (int i = 0; i < w && rc == TTB_OK; ++i)
        if (launch(plan->geo, pr, A, target, s) != cudaSuccess) rc = TTB_ECUDA;
      for (int i = 0; i < n && rc == TTB_OK; ++i) {
        cudaEventRecord(e0, s);
        if (launch(plan->geo, pr, A, target, s) != cudaSuccess) rc = TTB_ECUDA;
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        b = std::min(b, ms);
      }
      return b;
    };
    std::vector<std::pair<float, Prepared>> timed;
    for (const Spec& sp : plan->cands) {
      Prepared pr;
      if (!prepare(plan->geo, sp, plan->sms, &pr, nullptr)) continue;
      if (!aligned(A, pr.a_align) || !aligned(target, pr.b_align)) continue;
      timed.emplace_back(measure(pr, warmups, reps), pr);
      if (rc) break;
    }
    // second round: the four fastest again (three times), interleaved, so one noisy sample
    // cannot decide; ties keep the earlier (heuristically better) candidate,
    // like select_solution's cost tie-break (tuner.cpp:48-64)
    std::vector<size_t> order(timed.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return timed[a].first < timed[b].first; });
    if (order.size() > 4) order.resize(4);
    // the finalists are judged on the interleaved rounds alone: the first
    // round times the list in order on a device that warms up and reaches its
    // power cap on the way, which favours whoever ran early
    if (order.size() > 1) {
      std::vector<float> again(order.size(), 1e30f);
      for (int round = 0; round < 3 && rc == TTB_OK; ++round)
        for (size_t k = 0; k < order.size(); ++k)
          again[k] = std::min(again[k], measure(timed[order[k]].second, 1, reps));
      for (size_t k = 0; k < order.size(); ++k) timed[order[k]].first = again[k];
    }
    float best = 1e30f;
    Prepared winner = plan->prep;
    for (size_t i : order)
      if (timed[i].first < best) {
        best = timed[i].first;
        winner = timed[i].second;
      }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (scratch) cudaFree(scratch);
    if (rc) return cuda_fail(cudaGetLastError(), "autotune");
    plan->prep = winner;
    plan->tuned_ms = best;
    if (plan->cached) {
      std::lock_guard<std::mutex> lk(g_mu);
      g_choice[plan->key] = winner.spec.text();
      g_plans.clear();  // one-shot plans re-plan and pick the tuned choice up
    }
    // like a plain execute, leave B holding exactly one application (with
    // beta == 0 every candidate overwrote it; with beta != 0 it is untouched)
    const int r2 = execute(plan, plan->prep, A, B, s, plan->orig.alpha, plan->orig.beta);
    if (r2) return r2;
    return ok();
  });
}

int ttb_cache_store(const char* file, const char* problem_key, const char* hardware_key,
                    const char* plan_text, double bandwidth_gibs) {
  return guarded([&] {
    if (!file || !*file) return fail(TTB_EINVAL, "cache: no file");
    cache_store(file, CacheEntry{problem_key ? problem_key : "", hardware_key ? hardware_key : "",
                                 plan_text ? plan_text : "", bandwidth_gibs, iso8601_utc_now()});
    return ok();
  });
}

int ttb_cache_lookup(const char* file, const char* problem_key, const char* hardware_key,
                     char* plan_buf, size_t plan_len, double* bandwidth_gibs, char* ts_buf,
                     size_t ts_len, int* found) {
  return guarded([&] {
    if (!file || !problem_key || !hardware_key || !found)
      return fail(TTB_EINVAL, "cache: null argument");
    CacheEntry e;
    *found = cache_lookup(file, problem_key, hardware_key, &e) ? 1 : 0;
    if (!*found) return ok();
    if (plan_buf) {
      if (plan_len <= e.plan.size()) return fail(TTB_EINVAL, "cache: plan buffer too small");
      std::memcpy(plan_buf, e.plan.c_str(), e.plan.size() + 1);
    }
    if (ts_buf) {
      if (ts_len <= e.timestamp.size()) return fail(TTB_EINVAL, "cache: timestamp buffer too small");
      std::memcpy(ts_buf, e.timestamp.c_str(), e.timestamp.size() + 1);
    }
    if (bandwidth_gibs) *bandwidth_gibs = e.bandwidth_gibs;
    return ok();
  });
}

int ttb_hardware_key(char* buf, size_t len) {
  return guarded([&] {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    cudaDeviceProp prop{};
    if ((e = cudaGetDeviceProperties(&prop, dev)) != cudaSuccess)
      return cuda_fail(e, "cudaGetDeviceProperties");
    const std::string k = std::string(prop.name) + ":sm" + std::to_string(prop.major) +
                          std::to_string(prop.minor) + ":" + std::to_string(prop.multiProcessorCount) +
                          "sms:ttb" + TTB_VERSION;
    if (!buf || len <= k.size()) return fail(TTB_EINVAL, "hardware key: buffer too small");
    std::memcpy(buf, k.c_str(), k.size() + 1);
    return ok();
  });
}

int ttb_plan_tune_cached(ttb_plan plan, const char* cache_file, const void* A, void* B,
                         int warmups, int reps, ttb_stream stream, int* hit) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  return guarded([&] {
    if (!cache_file || !*cache_file) return fail(TTB_EINVAL, "cache: no file");
    char hk[512];
    int rc = ttb_hardware_key(hk, sizeof hk);
    if (rc) return rc;
    const std::string pkey = cache_key(plan->orig);  // canonical_key of the original problem
    CacheEntry e;
    if (hit) *hit = 0;
    // a line whose plan is not a GPU plan is malformed here: it can neither
    // be selected nor shadow an earlier entry that can
    const auto gpu_plan = [](const std::string& t) {
      Spec sp;
      return Spec::parse(t, &sp);
    };
    if (cache_lookup(cache_file, pkey, hk, &e, gpu_plan)) {
      Spec sp;
      Prepared pr;
      if (Spec::parse(e.plan, &sp) && prepare(plan->geo, sp, plan->sms, &pr, nullptr)) {
        plan->prep = pr;
        if (hit) *hit = 1;
        return execute(plan, plan->prep, A, B, reinterpret_cast<cudaStream_t>(stream),
                       plan->orig.alpha, plan->orig.beta);
      }
    }
    rc = ttb_plan_autotune(plan, A, B, warmups, reps, stream);
    if (rc) return rc;
    const Problem& p = plan->orig;
    const double bytes = static_cast<double>(p.elements()) *
                         (kind_bytes(p.kind_a) + kind_bytes(p.kind_b) * (p.beta != 0.0 ? 2 : 1));
    const double gibs = bytes / 1073741824.0 / (std::max(plan->tuned_ms, 1e-6f) * 1e-3);
    cache_store(cache_file, CacheEntry{pkey, hk, plan->prep.spec.text(), gibs, iso8601_utc_now()});
    return ok();
  });
}

int ttb_benchmark_manifest(int64_t volume_bytes, int kind, uint64_t seed, char* buf, size_t len) {
  return guarded([&] {
    std::string t;
    for (const std::string& l : benchmark_manifest(volume_bytes, kind, seed)) t += l + "\n";
    if (!buf || len <= t.size()) return fail(TTB_EINVAL, "benchmark: buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return ok();
  });
}

int ttb_plan_describe(ttb_plan plan, char* buf, size_t len) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  // the plan text plus the kernel that runs it (informational "fn" key)
  const Prepared& p = plan->prep;
  const char* fn = p.spec.v == kTma ? "tma" : p.spec.v == kRt ? "rt" : p.spec.v == kCopy ? (p.cp.bulk ? "rowcopy" : p.cp.long_rows ? "copy_rows" : "copy")
                   : p.sp.dense == 5 ? (p.sp.ly ? "btile" : "btile_lin") : p.sp.dense == 4 ? "vtile" : p.sp.dense >= 2 ? "dense" : p.sp.dense == 1 ? "tile" : "smem";
  std::string t = p.spec.text() + ";fn=" + fn;
  if (!plan->boxes.empty()) t += ";boxes=" + std::to_string(plan->boxes.size());
  if (!buf || len <= t.size()) return fail(TTB_EINVAL, "describe: buffer too small");
  std::memcpy(buf, t.c_str(), t.size() + 1);
  return ok();
}

int ttb_plan_candidates(ttb_plan plan, char* buf, size_t len) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  std::string t;
  for (const Spec& s : plan->cands) t += s.text() + "\n";
  if (!buf || len <= t.size()) return fail(TTB_EINVAL, "candidates: buffer too small");
  std::memcpy(buf, t.c_str(), t.size() + 1);
  return ok();
}

int ttb_plan_select(ttb_plan plan, const char* plan_text) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  return guarded([&] {
    Spec s;
    if (!plan_text || !Spec::parse(plan_text, &s)) return fail(TTB_EINVAL, "plan: cannot parse plan text");
    std::string why;
    Prepared pr;
    if (!plan->boxes.empty()) {  // every box plan it applies to (the first one must)
      for (size_t i = 0; i < plan->boxes.size(); ++i) {
        ttb_plan_s* sub = plan->boxes[i].plan.get();
        if (prepare(sub->geo, s, sub->sms, &pr, &why))
          sub->prep = pr;
        else if (i == 0)
          return fail(TTB_EINVAL, "plan: " + why);
      }
      plan->prep = plan->boxes.front().plan->prep;
      return ok();
    }
    if (!prepare(plan->geo, s, plan->sms, &pr, &why)) return fail(TTB_EINVAL, "plan: " + why);
    plan->prep = pr;
    return ok();
  });
}

int ttb_plan_launches(ttb_plan plan, int* launches_per_execute) {
  if (!plan) return fail(TTB_EINVAL, "plan: null handle");
  // one kernel per execute, one per box for oversized problems
  if (launches_per_execute) *launches_per_execute = plan->boxes.empty() ? 1 : static_cast<int>(plan->boxes.size());
  return ok();
}

int ttb_emit_source(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                    const int64_t* lda, const int64_t* ldb, double alpha, double beta, const char* plan_text,
                    const char* basename, char* entry, size_t entry_len, char* header, size_t header_len,
                    char* source, size_t source_len) {
  return guarded([&] {
    const Problem p = from_args(kind_a, kind_b, rank, perm, sizes, lda, ldb, alpha, beta);
    check(p);
    const Merged mg = fuse_indices(p);  // the reference emits for the normalized problem
    const Problem& m = mg.p;
    if (m.rank() > kMaxRank) return fail(TTB_EINVAL, "perm: rank after merging exceeds TTB_MAX_RANK");
    Spec spec;
    if (plan_text && *plan_text && !Spec::parse(plan_text, &spec))
      return fail(TTB_EINVAL, "emit: cannot parse plan text");
    if (!(plan_text && *plan_text)) spec.tx = spec.ty = 32;
    const std::string sym = emit_entry_symbol(m);
    const std::string base = basename && *basename ? basename : sym;
    for (char ch : base)
      if (!(std::isalnum(static_cast<unsigned char>(ch)) || ch == '_' || ch == '-' || ch == '.'))
        return fail(TTB_EINVAL, "emit: basename must be a plain file name");
    std::string h, s;
    emit_cuda(m, make_geo(m), spec, base, spec.text(), cache_key(m), &h, &s);
    const std::pair<const std::string*, std::pair<char*, size_t>> outs[] = {
        {&sym, {entry, entry_len}}, {&h, {header, header_len}}, {&s, {source, source_len}}};
    for (const auto& o : outs) {
      if (!o.second.first) continue;
      if (o.second.second <= o.first->size()) return fail(TTB_EINVAL, "emit: buffer too small");
      std::memcpy(o.second.first, o.first->c_str(), o.first->size() + 1);
    }
    return ok();
  });
}

int ttb_fill_uniform(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                     const int64_t* origin, const int64_t* global_sizes, uint64_t seed, void* buf,
                     ttb_stream stream) {
  BoxParams bp;
  int rc = box_params(kind, rank, sizes, ld, origin, global_sizes, &bp);
  if (rc) return rc;
  const cudaError_t e = launch_fill_uniform(kind_double(kind), bp, seed, buf,
                                            reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? ok() : cuda_fail(e, "fill_uniform");
}

int ttb_fill_sentinel(int kind, int64_t elements, void* buf, ttb_stream stream) {
  if (kind < 0 || kind > 3 || elements < 0) return fail(TTB_EINVAL, "sentinel: bad arguments");
  const cudaError_t e = launch_fill_sentinel(kind_double(kind), elements * kind_components(kind), buf,
                                             reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? ok() : cuda_fail(e, "fill_sentinel");
}

int ttb_checksum(int kind, int rank, const int64_t* sizes, const int64_t* ld,
                 const int64_t* origin, const int64_t* global_sizes, const void* buf,
                 uint64_t* out, ttb_stream stream) {
  BoxParams bp;
  int rc = box_params(kind, rank, sizes, ld, origin, global_sizes, &bp);
  if (rc) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(*d), s);
  if (e != cudaSuccess) return cuda_fail(e, "checksum alloc");
  cudaMemsetAsync(d, 0, sizeof(*d), s);
  e = launch_checksum(kind_double(kind), bp, buf, d, s);
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "checksum");
  if (out) *out = h;
  return ok();
}

uint64_t ttb_launch_count(void) { return ttb::launch_total(); }

int ttb_debug_candidates(int kind_a, int kind_b, int rank, const int* perm, const int64_t* sizes,
                         const int64_t* lda, const int64_t* ldb, double alpha, double beta,
                         char* buf, size_t len) {
  return guarded([&] {
    const Problem p = from_args(kind_a, kind_b, rank, perm, sizes, lda, ldb, alpha, beta);
    check(p);
    const Merged m = fuse_indices(p);
    std::string t;
    for (const Spec& s : candidates(make_geo(m.p))) t += s.text() + "\n";
    if (!buf || len <= t.size()) return fail(TTB_EINVAL, "candidates: buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return ok();
  });
}

}  // extern "C"
