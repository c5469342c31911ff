// ttb_cli.cpp -- command-line front end of the engine, the GPU counterpart of
// the reference's `ttune` CLI (cli.cpp:14-71 flags, pipeline.cpp:102-200
// run_single / run_benchmark_mode).  It is a client of the C ABI only
// (include/ttb.h): a maintainer can read it as the reference-side integration.
//
//   ttb --perm=2,1 --size=7264,7264 [--dataType=s] [--alpha=1] [--beta=0]
//       [--lda=..] [--ldb=..] [--cacheFile=F | $TTUNE_CACHE] [--hardwareKey=K]
//       [--warmups=2] [--reps=3] [--seed=42] [--emit=BASE] [--json]
//   ttb --benchmark [--volume=200] [--dataType=s] [--seed=42] [--manifest=F] [--json]
//
// Single mode: validate, look the problem up in the solution cache by
// (canonical_key, hardware key); on a miss autotune every candidate on device
// buffers filled by the counter generator and append the winner.  Prints the
// reference's text report or JSON.  Benchmark mode: the 57 cases; per case the
// heuristic first-choice plan ("refGiBs": the untuned engine, since the
// reference's CPU nest is not part of this product) and the autotuned plan
// ("tunedGiBs"), CSV in the reference's columns or JSON.  CPU-search flags of
// the reference (--prefetchDistances, --no-streaming-stores, --blockings,
// --threads) are accepted and ignored; --maxImplementations caps the
// candidates measured; --emit=BASE writes the solution's standalone sm_100a
// kernel as BASE.cu plus its header next to it (pipeline.cpp:142-146, 182).
// Exit codes as pipeline.cpp:189-200: 0 ok, 1 invalid argument, 2 other error.
#include <cuda_runtime.h>

#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ttb.h"

namespace {

struct Invalid : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Config {
  std::vector<int> perm;
  std::vector<int64_t> size, lda, ldb;
  std::string data_type = "s";
  double alpha = 1.0, beta = 0.0;
  int max_impl = -1;
  std::string cache_file = "ttune_cache.tsv";
  std::string hardware_key;
  bool benchmark = false;
  int64_t volume_mib = 200;
  std::string manifest;
  uint64_t seed = 42;
  int warmups = 2, reps = 3;
  bool json = false;
  std::string emit_base;
};

const char* kUsage =
    "usage: ttb --perm=<p1,p2,...> --size=<n1,n2,...> [options], or ttb --benchmark\n";

template <class T>
std::vector<T> parse_list(const std::string& flag, const std::string& v) {
  std::vector<T> out;
  std::stringstream ss(v);
  std::string item;
  while (std::getline(ss, item, ',')) {
    char* end = nullptr;
    const long long x = std::strtoll(item.c_str(), &end, 10);
    if (item.empty() || *end) throw Invalid(flag + ": '" + v + "' is not a comma-separated integer list");
    out.push_back(static_cast<T>(x));
  }
  return out;
}

double parse_double(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end) throw Invalid(flag + ": '" + v + "' is not a number");
  return x;
}

long long parse_int(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (v.empty() || *end) throw Invalid(flag + ": '" + v + "' is not an integer");
  return x;
}

// --flag=value or --flag value; returns the exit code to use, -1 to continue
int parse_args(int argc, char** argv, Config* c) {
  if (const char* e = std::getenv("TTUNE_CACHE")) c->cache_file = e;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i], v;
    if (a == "-h" || a == "--help") {
      std::cout << kUsage;
      return 0;
    }
    const auto eq = a.find('=');
    const bool is_flag = a == "--benchmark" || a == "--json" || a == "--no-streaming-stores";
    if (eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    } else if (!is_flag) {
      if (i + 1 >= argc) throw Invalid(a + ": missing value");
      v = argv[++i];
    }
    if (a == "--perm") c->perm = parse_list<int>(a, v);
    else if (a == "--size") c->size = parse_list<int64_t>(a, v);
    else if (a == "--lda") c->lda = parse_list<int64_t>(a, v);
    else if (a == "--ldb") c->ldb = parse_list<int64_t>(a, v);
    else if (a == "--dataType") {
      static const char* ok[] = {"s", "d", "c", "z", "sd", "ds", "cz", "zc"};
      bool found = false;
      for (const char* k : ok) found = found || v == k;
      if (!found) throw Invalid("--dataType: " + v + " not in {s,d,c,z,sd,ds,cz,zc}");
      c->data_type = v;
    } else if (a == "--alpha") c->alpha = parse_double(a, v);
    else if (a == "--beta") c->beta = parse_double(a, v);
    else if (a == "--maxImplementations") c->max_impl = static_cast<int>(parse_int(a, v));
    else if (a == "--cacheFile") c->cache_file = v;
    else if (a == "--hardwareKey") c->hardware_key = v;
    else if (a == "--benchmark") c->benchmark = true;
    else if (a == "--volume") c->volume_mib = parse_int(a, v);
    else if (a == "--manifest") c->manifest = v;
    else if (a == "--seed") c->seed = static_cast<uint64_t>(parse_int(a, v));
    else if (a == "--warmups") c->warmups = static_cast<int>(parse_int(a, v));
    else if (a == "--reps") c->reps = static_cast<int>(parse_int(a, v));
    else if (a == "--json") c->json = true;
    else if (a == "--emit") c->emit_base = v;
    else if (a == "--prefetchDistances" || a == "--blockings" || a == "--threads" ||
             a == "--no-streaming-stores") {
      // the reference's CPU search space; the GPU plan space replaces it
    } else {
      throw Invalid("unknown option " + a);
    }
  }
  if (!c->benchmark && (c->perm.empty() || c->size.empty())) {
    std::cerr << "ttb: --perm and --size are required\n" << kUsage;
    return 1;
  }
  return -1;
}

int kind_of(char ch) { return ch == 's' ? 0 : ch == 'd' ? 1 : ch == 'c' ? 2 : 3; }
int kind_bytes(int k) { return k == 0 ? 4 : k == 3 ? 16 : 8; }

void check(int rc) {
  if (rc == TTB_OK) return;
  if (rc == TTB_EINVAL) throw std::invalid_argument(ttb_last_error());
  throw std::runtime_error(ttb_last_error());
}

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}

template <class T>
std::string json_arr(const std::vector<T>& v) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < v.size(); ++i) os << (i ? ", " : "") << v[i];
  os << "]";
  return os.str();
}

std::string fmt(double x, const char* f = "%.6g") {
  char b[64];
  std::snprintf(b, sizeof b, f, x);
  return b;
}

// one problem on the device: buffers, generator fill, plan
struct Run {
  ttb_plan plan = nullptr;
  void *A = nullptr, *B = nullptr;
  int ka = 0, kb = 0, rank = 0;
  std::vector<int> perm;
  std::vector<int64_t> sizes, lda, ldb;
  double alpha = 1, beta = 0;
  int64_t elements = 1;

  Run(const std::vector<int>& p, const std::vector<int64_t>& s, const std::vector<int64_t>& la,
      const std::vector<int64_t>& lb, int ka_, int kb_, double al, double be, uint64_t seed)
      : ka(ka_), kb(kb_), rank(static_cast<int>(p.size())), perm(p), sizes(s), lda(la), ldb(lb),
        alpha(al), beta(be) {
    const int64_t* pla = lda.empty() ? nullptr : lda.data();
    const int64_t* plb = ldb.empty() ? nullptr : ldb.data();
    check(ttb_validate(static_cast<int>(perm.size()), perm.data(), static_cast<int>(sizes.size()),
                       sizes.data(), lda.empty() ? -1 : static_cast<int>(lda.size()), pla,
                       ldb.empty() ? -1 : static_cast<int>(ldb.size()), plb, ka, kb));
    check(ttb_plan_create(&plan, ka, kb, rank, perm.data(), sizes.data(), pla, plb, alpha, beta,
                          TTB_PLAN_NO_CACHE));
    for (int64_t e : sizes) elements *= e;
    const int64_t na = ttb_required_elements_a(rank, sizes.data(), pla);
    const int64_t nb = ttb_required_elements_b(rank, perm.data(), sizes.data(), plb);
    cuda(cudaMalloc(&A, static_cast<size_t>(na) * kind_bytes(ka)), "cudaMalloc A");
    cuda(cudaMalloc(&B, static_cast<size_t>(nb) * kind_bytes(kb)), "cudaMalloc B");
    check(ttb_fill_sentinel(ka, na, A, nullptr));
    check(ttb_fill_sentinel(kb, nb, B, nullptr));
    check(ttb_fill_uniform(ka, rank, sizes.data(), pla, nullptr, nullptr, seed, A, nullptr));
    std::vector<int64_t> sb(static_cast<size_t>(rank));
    for (int a = 0; a < rank; ++a) sb[static_cast<size_t>(perm[static_cast<size_t>(a)] - 1)] = sizes[static_cast<size_t>(a)];
    if (beta != 0.0)
      check(ttb_fill_uniform(kb, rank, sb.data(), plb, nullptr, nullptr, seed ^ 0x9e3779b97f4a7c15ull, B,
                             nullptr));
    cuda(cudaDeviceSynchronize(), "fill");
  }
  ~Run() {
    if (plan) ttb_plan_destroy(plan);
    if (A) cudaFree(A);
    if (B) cudaFree(B);
  }
  // reference bytes formula (tuner.cpp:18-25) in GiB
  double gib() const {
    return static_cast<double>(elements) *
           (kind_bytes(ka) + kind_bytes(kb) * (beta != 0.0 ? 2 : 1)) / 1073741824.0;
  }
  // best-of-reps device seconds of the current plan (and every trial)
  double time(int warmups, int reps, std::vector<double>* trials) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < warmups; ++i) check(ttb_plan_execute(plan, A, B, nullptr));
    double best = 1e30;
    for (int i = 0; i < reps; ++i) {
      cudaEventRecord(e0);
      check(ttb_plan_execute(plan, A, B, nullptr));
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (trials) trials->push_back(ms * 1e-3);
      best = std::min(best, ms * 1e-3);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
  }
  std::string describe() {
    char b[512];
    check(ttb_plan_describe(plan, b, sizeof b));
    return b;
  }
  int candidates() {
    std::vector<char> b(1 << 16);
    check(ttb_plan_candidates(plan, b.data(), b.size()));
    int n = 0;
    for (char ch : b) {
      if (!ch) break;
      n += ch == '\n';
    }
    return n;
  }
};

int run_single(const Config& c) {
  const int ka = kind_of(c.data_type[0]);
  const int kb = kind_of(c.data_type.size() > 1 ? c.data_type[1] : c.data_type[0]);
  Run r(c.perm, c.size, c.lda, c.ldb, ka, kb, c.alpha, c.beta, c.seed);
  const int64_t* pla = c.lda.empty() ? nullptr : c.lda.data();
  const int64_t* plb = c.ldb.empty() ? nullptr : c.ldb.data();
  char key[1024], mkey[1024], hw[512];
  check(ttb_canonical_key(ka, kb, r.rank, c.perm.data(), c.size.data(), pla, plb, c.alpha, c.beta,
                          key, sizeof key));
  if (c.hardware_key.empty())
    check(ttb_hardware_key(hw, sizeof hw));
  else
    std::snprintf(hw, sizeof hw, "%s", c.hardware_key.c_str());
  // merged problem (reported like the reference's "merged:" line)
  const int n = r.rank;
  std::vector<int> mp(static_cast<size_t>(n)), lo(static_cast<size_t>(n)), hi(static_cast<size_t>(n));
  std::vector<int64_t> ms(static_cast<size_t>(n)), mla(static_cast<size_t>(n)), mlb(static_cast<size_t>(n));
  int mr = 0;
  check(ttb_merge_indices(n, c.perm.data(), c.size.data(), pla, plb, &mr, mp.data(), ms.data(),
                          mla.data(), mlb.data(), lo.data(), hi.data()));
  mp.resize(static_cast<size_t>(mr));
  ms.resize(static_cast<size_t>(mr));
  mla.resize(static_cast<size_t>(mr));
  mlb.resize(static_cast<size_t>(mr));
  check(ttb_canonical_key(ka, kb, mr, mp.data(), ms.data(), mla.data(), mlb.data(), c.alpha, c.beta,
                          mkey, sizeof mkey));

  char plan_text[512] = {0}, ts[64];
  double gibs = 0.0;
  int found = 0;
  check(ttb_cache_lookup(c.cache_file.c_str(), key, hw, plan_text, sizeof plan_text, &gibs, ts,
                         sizeof ts, &found));
  bool hit = false;
  int measured = 0;
  double best = 0.0;
  std::vector<double> trials;
  if (found && ttb_plan_select(r.plan, plan_text) == TTB_OK) {
    hit = true;
  } else {
    measured = r.candidates();
    if (c.max_impl > 0 && c.max_impl < measured) {
      // measure only the first max_impl candidates: select the best by timing
      std::vector<char> b(1 << 16);
      check(ttb_plan_candidates(r.plan, b.data(), b.size()));
      std::stringstream ss(b.data());
      std::string line, win;
      double wbest = 1e30;
      for (int i = 0; i < c.max_impl && std::getline(ss, line); ++i) {
        if (ttb_plan_select(r.plan, line.c_str()) != TTB_OK) continue;
        const double t = r.time(c.warmups, c.reps, nullptr);
        if (t < wbest) {
          wbest = t;
          win = line;
        }
      }
      check(ttb_plan_select(r.plan, win.c_str()));
      measured = c.max_impl;
      gibs = r.gib() / wbest;
      check(ttb_cache_store(c.cache_file.c_str(), key, hw, win.c_str(), gibs));
    } else {
      int h = 0;
      check(ttb_plan_tune_cached(r.plan, c.cache_file.c_str(), r.A, r.B, c.warmups, c.reps, nullptr,
                                 &h));
      check(ttb_cache_lookup(c.cache_file.c_str(), key, hw, plan_text, sizeof plan_text, &gibs, ts,
                             sizeof ts, &found));
    }
    best = r.time(c.warmups, c.reps, &trials);
  }
  const std::string solution = r.describe();
  std::string emitted_src, emitted_hdr;
  if (!c.emit_base.empty()) {
    // the solution's kernel as standalone source (emit_source + write_kernel_files)
    const size_t slash = c.emit_base.find_last_of('/');
    const std::string dir = slash == std::string::npos ? "" : c.emit_base.substr(0, slash + 1);
    const std::string stem = slash == std::string::npos ? c.emit_base : c.emit_base.substr(slash + 1);
    std::vector<char> hdr(1 << 14), src(1 << 17);
    check(ttb_emit_source(ka, kb, r.rank, c.perm.data(), c.size.data(), pla, plb, c.alpha, c.beta,
                          solution.c_str(), stem.c_str(), nullptr, 0, hdr.data(), hdr.size(), src.data(),
                          src.size()));
    emitted_src = c.emit_base + ".cu";
    emitted_hdr = dir + stem + ".h";
    for (const auto& f : {std::make_pair(emitted_src, src.data()), std::make_pair(emitted_hdr, hdr.data())}) {
      std::ofstream out(f.first, std::ios::binary);
      if (!out) throw std::runtime_error("emit: cannot write " + f.first);
      out << f.second;
    }
  }
  if (c.json) {
    std::cout << "{\n  \"problemKey\": " << json_str(key) << ",\n  \"hardwareKey\": " << json_str(hw)
              << ",\n  \"cacheHit\": " << (hit ? "true" : "false")
              << ",\n  \"cacheFile\": " << json_str(c.cache_file) << ",\n  \"mergedPerm\": "
              << json_arr(mp) << ",\n  \"mergedSize\": " << json_arr(ms)
              << ",\n  \"measuredCandidates\": " << measured << ",\n  \"plan\": {\"serialized\": "
              << json_str(solution) << "},\n  \"bandwidthGiBs\": " << fmt(gibs, "%.17g")
              << ",\n  \"bestSeconds\": " << fmt(best, "%.17g") << ",\n  \"trialSeconds\": [";
    for (size_t i = 0; i < trials.size(); ++i) std::cout << (i ? ", " : "") << fmt(trials[i], "%.17g");
    std::cout << "]";
    if (!emitted_src.empty())
      std::cout << ",\n  \"emitted\": {\"source\": " << json_str(emitted_src) << ", \"header\": "
                << json_str(emitted_hdr) << "}";
    std::cout << "\n}\n";
  } else {
    std::cout << "problem: " << key << "\n"
              << "merged: " << mkey << "\n"
              << "hardware: " << hw << "\n"
              << "cache: " << (hit ? "hit" : "miss") << " (" << c.cache_file << ")\n"
              << "candidates measured: " << measured << "\n"
              << "solution: " << solution << "\n"
              << "bandwidth: " << fmt(gibs) << " GiB/s\n";
    if (!emitted_src.empty()) std::cout << "emitted: " << emitted_src << " " << emitted_hdr << "\n";
  }
  return 0;
}

int run_benchmark(const Config& c) {
  const int kind = kind_of(c.data_type[0]);
  std::vector<char> buf(1 << 16);
  check(ttb_benchmark_manifest(c.volume_mib << 20, kind, c.seed, buf.data(), buf.size()));
  const std::string text(buf.data());
  if (!c.manifest.empty()) {
    std::ofstream mf(c.manifest);
    if (!mf) throw std::runtime_error("cannot write " + c.manifest);
    mf << text;
  }
  std::stringstream ss(text);
  std::string line;
  if (c.json)
    std::cout << "[\n";
  else
    std::cout << "caseId,dim,perm,sizes,category,config,refGiBs,tunedGiBs,speedup,plan\n";
  bool first = true;
  uint64_t seed = c.seed;
  while (std::getline(ss, line)) {
    if (line.empty()) continue;
    std::string id, perm_s, size_s, cat, conf;
    std::stringstream ls(line);
    std::string kv;
    while (std::getline(ls, kv, ';')) {
      const auto eq = kv.find('=');
      const std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
      if (k == "case") id = v;
      else if (k == "perm") perm_s = v;
      else if (k == "size") size_s = v;
      else if (k == "category") cat = v;
      else if (k == "config") conf = v;
    }
    const auto perm = parse_list<int>("perm", perm_s);
    const auto sizes = parse_list<int64_t>("size", size_s);
    Run r(perm, sizes, {}, {}, kind, kind, 1.0, 1.0, seed++);
    const double t_ref = r.time(c.warmups, c.reps, nullptr);  // heuristic first choice
    check(ttb_plan_autotune(r.plan, r.A, r.B, c.warmups, c.reps, nullptr));
    const double t_tuned = r.time(c.warmups, c.reps, nullptr);
    const double ref = r.gib() / t_ref, tuned = r.gib() / t_tuned;
    std::string perm_dash = perm_s, size_x = size_s;
    for (char& ch : perm_dash) ch = ch == ',' ? '-' : ch;
    for (char& ch : size_x) ch = ch == ',' ? 'x' : ch;
    const std::string plan = r.describe();
    if (c.json) {
      std::cout << (first ? "" : ",\n") << "  {\"caseId\": " << json_str(id)
                << ", \"dim\": " << perm.size() << ", \"perm\": " << json_arr(perm)
                << ", \"sizes\": " << json_arr(sizes) << ", \"category\": " << json_str(cat)
                << ", \"config\": " << json_str(conf) << ", \"refGiBs\": " << fmt(ref)
                << ", \"tunedGiBs\": " << fmt(tuned) << ", \"speedup\": " << fmt(tuned / ref)
                << ", \"plan\": " << json_str(plan) << "}";
    } else {
      std::cout << id << ',' << perm.size() << ',' << perm_dash << ',' << size_x << ',' << cat << ','
                << conf << ',' << fmt(ref) << ',' << fmt(tuned) << ',' << fmt(tuned / ref) << ",\""
                << plan << "\"\n";
    }
    std::cout.flush();
    first = false;
  }
  if (c.json) std::cout << "\n]\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Config c;
  try {
    const int rc = parse_args(argc, argv, &c);
    if (rc >= 0) return rc;
    return c.benchmark ? run_benchmark(c) : run_single(c);
  } catch (const Invalid& e) {
    std::cerr << "ttb: " << e.what() << "\n" << kUsage;
    return 1;
  } catch (const std::invalid_argument& e) {
    std::cerr << "ttb: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "ttb: error: " << e.what() << "\n";
    return 2;
  }
}
