// api.cu -- the C ABI (include/helrm.h): context and device tables, client
// keys and ciphertexts, server setup (plan), and the lookup engine.
//
// The lookup (helrm_lookup) follows SURVEY.md D20 (double-hoisted BSGS,
// PAPER.md:289, :584) step by step:
//   L1 ModUp of each input c1 (hoist #1)        -> modup()
//   L2 lazy baby steps (a_j, b_j) over Q_l P     -> launch_kip (fused phi + KIP)
//   L3 inner sums with the pre-rotated diagonals  -> launch_diag_mac
//   L4 giant steps: ModDown(B), ModUp, KIP, +phi(A) (hoist #2)
//   L6 ModDown, L7 rescale, L8 RotSum
// Every arithmetic step runs in the kernels of kernels_ntt.cu / kernels_rns.cu;
// the host only schedules launches on the context stream.
#include <omp.h>

#include <chrono>

#include <atomic>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>
#include <tuple>
#include <unordered_map>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

using namespace helrm;

namespace helrm {
NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }
}  // namespace helrm

namespace {
thread_local std::string g_last_error;

template <typename F>
helrm_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return HELRM_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return HELRM_ERR_ALLOC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HELRM_ERR_ARG;
  }
}

void need(bool ok, helrm_status code, const char* msg) {
  if (!ok) throw Error(code, msg);
}
}  // namespace

// Every entry point that enqueues work for a context first makes the
// context's device current (a process may hold contexts on several devices).
struct DevGuard {
  explicit DevGuard(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) HCUDA(cudaSetDevice(dev));
  }
};

// ============================================================================
// handles
// ============================================================================
struct helrm_params {
  Params P;
};

struct LevelConst {
  uint64_t* pmod = nullptr;       // [l+1] P mod q_i, shoup companions
  uint64_t* pmods = nullptr;
  uint64_t* pinv = nullptr;       // [l+1] P^-1 mod q_i
  uint64_t* pinvs = nullptr;
  uint64_t* qlinv = nullptr;      // [l] q_l^-1 mod q_i
  uint64_t* qlinvs = nullptr;
  // fused base conversions (D14 inside the NTT): INTT post-factors
  // N^-1 [(B/b)^-1]_b (y-form) and per-output-row coefficient tables
  double2* modup_post = nullptr;   // [l+1]
  ConvRowDev* modup_tab = nullptr; // [dnum(l)][modup_rows]: the rows outside digit k
  int modup_rows = 0;
  double2* moddown_post = nullptr; // [K]
  ConvRowDev* moddown_tab = nullptr; // [l+1]
};

struct helrm_ctx {
  Params P;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<PrimeDev> hprimes;
  PrimeDev* dprimes = nullptr;
  uint64_t* dtw = nullptr;
  uint32_t* dslotpos = nullptr;
  uint32_t* dgrp = nullptr;
  const double* dtwb = nullptr;
  uint8_t* dtpos = nullptr;
  uint64_t* dcdt = nullptr;
  uint64_t* scratch = nullptr;
  std::map<int, LevelConst> lconst;
  std::map<std::pair<int, int>, uint32_t*> modup_lidx;   // (level, G) -> NTT limb table of modup_batch
  std::map<std::pair<int, int>, uint32_t*> pm_lidx;      // (G, n) -> prime-major limb table
  // row-slice tables of the RNS-limb partition, keyed by (level, first row, end row, G)
  struct SliceTabs {
    ConvRowDev* up_tab = nullptr;   // [dnum][up_rows]: ModUp conversion rows of digit k inside the slice
    int up_rows = 0;
    uint32_t* up_lidx = nullptr;    // ModUp NTT limbs (g dnum + k) nl + r, r in the slice, outside digit k
    size_t n_up = 0;
    ConvRowDev* dn_tab = nullptr;   // ModDown conversion rows: Q rows of the slice
    int dn_rows = 0;
    uint32_t* q_lidx = nullptr;     // the slice's Q rows g nq + r (INTT / ModDown NTT)
    size_t n_q = 0;
  };
  std::map<std::tuple<int, int, int, int>, SliceTabs> slices;
  // CUDA-graph replay of the double-hoisted lookup (one graph per plan, key
  // set and query-chunk size): the ~400 launches, allocations and copies of a
  // lookup are enqueued once at capture; a replay costs one graph launch.
  struct LookupGraph {
    cudaGraphExec_t exec = nullptr;
    uint64_t* X = nullptr;        // staged inputs [Qc][C][2][l+1][N]
    uint64_t* S = nullptr;        // outputs [O][Qc][2][l][N]
    void* pinned = nullptr;       // host copy of the MAC work list the graph re-uploads
    uint64_t* scratch = nullptr;  // own NTT scratch (second serving slot)
    size_t uses = 0;
    uint64_t launches = 0;        // kernel launches inside the graph (added to the counter per replay)
    bool failed = false;
  };
  std::map<std::tuple<uint64_t, uint64_t, int>, LookupGraph> graphs;   // (plan id, key-set id, Qc)
  void drop_graphs(uint64_t id) {
    for (auto it = graphs.begin(); it != graphs.end();) {
      if (std::get<0>(it->first) == id || std::get<1>(it->first) == id) {
        cudaStreamSynchronize(stream);
        if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
        if (it->second.pinned) cudaFreeHost(it->second.pinned);
        dfree(it->second.X);
        dfree(it->second.S);
        dfree(it->second.scratch);
        it = graphs.erase(it);
      } else {
        ++it;
      }
    }
  }
  std::vector<void*> owned;       // device allocations freed at destroy
  uint64_t launches = 0;
  std::vector<uint32_t> dlog5;    // dlog5[g] for odd g < 2N (0xffffffff if not a power of 5)

  Profiler prof;
  std::string prof_json;
  ncclComm_t comm = nullptr;      // helrm_comm_init
  int rank = 0, world = 1;

  // side streams of the pipelined giant steps (lookup_double_part): NTT work
  // (FP64-bound) on s_ntt at the highest priority, key switches (HBM-bound)
  // on s_kip, so they overlap the diagonal MACs on the context stream
  cudaStream_t s_ntt = nullptr, s_kip = nullptr, s_mac = nullptr;
  cudaStream_t s_cap = nullptr;   // private stream the lookup graphs are captured on
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;   // copy streams of helrm_lookup_host
  cudaEvent_t hev[12] = {};                         // its events (outside the pool the lookup recycles)
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  cudaEvent_t ev() {
    if (evnext == evpool.size()) {
      cudaEvent_t e;
      HCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evpool.push_back(e);
    }
    return evpool[evnext++];
  }
  // s waits for everything enqueued on `on` so far
  void join(cudaStream_t s, cudaStream_t on) {
    HostTimer ht_("join");
    cudaEvent_t e = ev();
    HCUDA(cudaEventRecord(e, on));
    HCUDA(cudaStreamWaitEvent(s, e, 0));
  }

  int persist = 0;                // persistent CTAs per SM for the HBM-bound kernels (0 = full grids)
  int n_sm = 148;                 // multiprocessor count of `device`
  cudaMemPool_t pool = nullptr;   // private stream-ordered pool (the device's default pool is left alone)
  DevCtx dc(cudaStream_t s = nullptr, int pers = 0) {
    return DevCtx{dprimes, dslotpos, dgrp, dtwb, dtpos, P.log_n, P.N, s ? s : stream, pers, n_sm, &launches, &prof};
  }

  void* dalloc(size_t bytes, cudaStream_t s = nullptr) {
    HostTimer ht_("cudaMallocAsync");
    void* p = nullptr;
    if (bytes == 0) bytes = 8;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, s ? s : stream);
    if (e != cudaSuccess) throw Error(HELRM_ERR_ALLOC, std::string("device allocation failed: ") + cudaGetErrorString(e));
    return p;
  }
  void dfree(void* p, cudaStream_t s = nullptr) {
    HostTimer ht_("cudaFreeAsync");
    if (p) cudaFreeAsync(p, s ? s : stream);
  }
  // give memory freed by destroyed plans / key sets back to the device
  void trim() {
    cudaStreamSynchronize(stream);
    cudaMemPoolTrimTo(pool, 0);
  }
  uint64_t* upload_u64(const std::vector<uint64_t>& v) {
    uint64_t* d = (uint64_t*)dalloc(v.size() * 8);
    HCUDA(cudaMemcpyAsync(d, v.data(), v.size() * 8, cudaMemcpyHostToDevice, stream));
    HCUDA(cudaStreamSynchronize(stream));
    owned.push_back(d);
    return d;
  }
};

// RAII device buffer, stream-ordered on the context stream (or on s)
struct DBuf {
  helrm_ctx* c;
  cudaStream_t s;
  uint64_t* p;
  DBuf(helrm_ctx* c_, size_t words, cudaStream_t s_ = nullptr)
      : c(c_), s(s_), p((uint64_t*)c_->dalloc(words * 8, s_)) {}
  ~DBuf() { c->dfree(p, s); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

struct helrm_sk {
  helrm_ctx* c;
  uint64_t* sntt;                 // [L+1+K][N]
  std::vector<int64_t> s;         // coefficients (host copy)
};
struct helrm_pk {
  helrm_ctx* c;
  uint64_t* d;                    // [2][L+1][N]: b, a
};
static std::atomic<uint64_t> g_obj_id{1};   // identity of plans / key sets for the graph cache

struct helrm_rotkeys {
  helrm_ctx* c;
  std::map<uint64_t, uint64_t*> keys;   // galois -> [dnum][2][L+1+K][N]
  size_t words_per_key = 0;
  uint64_t id = g_obj_id++;
};
struct helrm_ct {
  helrm_ctx* c;
  uint32_t level;
  double scale;
  uint64_t* d;                    // [2][level+1][N]
};

struct Block {
  int64_t k, d, p, l, w, I, R;
  bool comp;
  int wid;                        // index into weights store
};
struct helrm_tables {
  Params P;
  std::vector<Block> blocks;
  std::vector<std::vector<double>> weights;
  uint32_t n_dense;
  int64_t K, M;
};

struct Entry {
  int c, j, uid;
};
struct helrm_plan {
  helrm_ctx* c;
  uint32_t level, mode;
  int64_t K, M, mbar, O, C, n1;
  std::vector<int64_t> t0, span, n2;
  std::vector<std::vector<std::vector<Entry>>> entries;  // [o][i]
  std::vector<std::vector<int64_t>> giants;               // [o][i]
  std::vector<std::vector<int>> babies;                   // [c] sorted j used
  int64_t n_diag = 0;
  uint64_t* diag = nullptr;                               // [n_unique][nl][N]
  bool compact = false;                                   // HELRM_PLAN_COMPACT: diagonals as coefficients
  int64_t* coef = nullptr;                                // compact: [n_unique][N] encoded int64
  int64_t n_unique = 0;
  uint32_t nl = 0;
  std::vector<int64_t> rotations;
  uint64_t id = g_obj_id++;
};

// ============================================================================
// profiler (per-kernel CUDA events on the context stream)
// ============================================================================
namespace helrm {
cudaEvent_t Profiler::get() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  HCUDA(cudaEventCreate(&e));
  return e;
}
static const bool g_hostprof = getenv("HELRM_HOSTPROF") && atoi(getenv("HELRM_HOSTPROF")) != 0;
static std::map<std::string, std::pair<uint64_t, double>> g_hostt;
bool hostprof_on() { return g_hostprof; }
bool pdl_on() {
  // measured neutral inside the lookup graphs (6.82-6.85 ms either way): off unless HELRM_PDL=1
  static const bool on = getenv("HELRM_PDL") ? atoi(getenv("HELRM_PDL")) != 0 : false;
  return on;
}
void hostprof_add(const char* name, double us) {
  auto& e = g_hostt[name];
  e.first++;
  e.second += us;
}
double hostprof_now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static void hostprof_dump(const char* tag) {
  if (!g_hostprof) return;
  fprintf(stderr, "[helrm hostprof] %s\n", tag);
  for (auto& kv : g_hostt)
    fprintf(stderr, "  %-24s %6llu calls %10.1f us\n", kv.first.c_str(), (unsigned long long)kv.second.first,
            kv.second.second);
  g_hostt.clear();
}

ProfScope::ProfScope(const DevCtx& c_, const char* name, double bytes) : c(c_), ht(name) {
  if (c.prof && c.prof->on) {
    Profiler::Rec r{name, c.prof->get(), c.prof->get(), bytes};
    HCUDA(cudaEventRecord(r.a, c.stream));
    idx = (int)c.prof->recs.size();
    c.prof->recs.push_back(r);
  }
}
ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(c.prof->recs[idx].b, c.stream);
}
}  // namespace helrm

// ============================================================================
// context helpers
// ============================================================================
static uint64_t* ct_c0(const helrm_ct* ct) { return ct->d; }
static uint64_t* ct_c1(const helrm_ct* ct) { return ct->d + (size_t)(ct->level + 1) * ct->c->P.N; }

static helrm_ct* new_ct(helrm_ctx* c, uint32_t level, double scale) {
  helrm_ct* ct = new helrm_ct{c, level, scale, nullptr};
  ct->d = (uint64_t*)c->dalloc((size_t)2 * (level + 1) * c->P.N * 8);
  return ct;
}

static LimbMap sub_map(const LimbMap& m, int first, int count) {
  LimbMap r{};
  r.n = count;
  for (int i = 0; i < count; i++) r.pr[i] = m.pr[first + i];
  return r;
}

static void ntt_fwd(helrm_ctx* c, const uint64_t* src, uint64_t* dst, size_t n, const LimbMap& map, size_t ss = 0,
                    size_t ds = 0) {
  if (n) launch_ntt_fwd(c->dc(), src, dst, c->scratch, n, map, ss, ds);
}
static void ntt_inv(helrm_ctx* c, const uint64_t* src, uint64_t* dst, size_t n, const LimbMap& map, size_t ss = 0,
                    size_t ds = 0) {
  if (n) launch_ntt_inv(c->dc(), src, dst, c->scratch, n, map, ss, ds);
}

static const LevelConst& level_const(helrm_ctx* c, uint32_t l) {
  auto it = c->lconst.find((int)l);
  if (it != c->lconst.end()) return it->second;
  const Params& P = c->P;
  std::vector<uint64_t> pm(l + 1), pms(l + 1), pi(l + 1), pis(l + 1), qi(l + 1, 0), qis(l + 1, 0);
  for (uint32_t i = 0; i <= l; i++) {
    uint64_t q = P.primes[i], pmod = 1;
    for (uint32_t j = 0; j < P.K; j++) pmod = mulm(pmod, P.primes[P.L + 1 + j] % q, q);
    pm[i] = pmod;
    pms[i] = shoup_pre(pmod, q);
    pi[i] = inv_mod(pmod, q);
    pis[i] = shoup_pre(pi[i], q);
    if (i < l) {
      qi[i] = inv_mod(P.primes[l] % q, q);
      qis[i] = shoup_pre(qi[i], q);
    }
  }
  LevelConst lc;
  {
    const uint32_t nl = l + 1 + P.K, dn = P.dnum(l);
    const uint64_t ninv_base = 0;
    (void)ninv_base;
    auto hat_mod = [&](const std::vector<uint32_t>& B, size_t skip, uint64_t t) {
      uint64_t h = 1;
      for (size_t b = 0; b < B.size(); b++)
        if (b != skip) h = mulm(h, P.primes[B[b]] % t, t);
      return h;
    };
    auto pair = [&](uint64_t w, uint64_t q) { return make_double2((double)w, (double)w / (double)q); };
    std::vector<double2> upost(l + 1), dpost(P.K);
    // rows outside digit k (the digit's own limbs are copied, not converted)
    uint32_t min_dig = P.alpha;
    for (uint32_t k = 0; k < dn; k++) min_dig = std::min(min_dig, std::min((k + 1) * P.alpha, l + 1) - k * P.alpha);
    const uint32_t urows = nl - min_dig;
    lc.modup_rows = (int)urows;
    std::vector<ConvRowDev> utab((size_t)dn * urows), dtab(l + 1);
    for (uint32_t k = 0; k < dn; k++) {
      std::vector<uint32_t> B;
      const uint32_t lo = k * P.alpha, hi = std::min((k + 1) * P.alpha, l + 1);
      for (uint32_t i = lo; i < hi; i++) B.push_back(i);
      for (size_t b = 0; b < B.size(); b++) {
        const uint64_t q = P.primes[B[b]];
        const uint64_t binv = inv_mod(hat_mod(B, b, q), q);
        upost[B[b]] = pair(mulm(inv_mod(P.N % q, q), binv, q), q);
      }
      uint32_t j = 0;
      for (uint32_t r = 0; r < nl; r++) {
        if (r >= lo && r < hi) continue;
        ConvRowDev& cr = utab[(size_t)k * urows + j++];
        cr = ConvRowDev{};
        cr.src_row0 = (int)lo;
        cr.nb = (int)B.size();
        cr.out_row = (int)r;
        const uint64_t qr = P.primes[P.qp_chain(l, r)];
        cr.q = (double)qr;
        cr.qinv = 1.0 / (double)qr;
        for (size_t b = 0; b < B.size(); b++) {
          const uint64_t w = hat_mod(B, b, qr);   // (B/b) mod q_r
          cr.cf[b] = make_double2((double)w, (double)w / (double)qr);
        }
      }
      for (; j < urows; j++) {   // padding rows (a digit with fewer primes than alpha has more outside rows)
        ConvRowDev& cr = utab[(size_t)k * urows + j];
        cr = ConvRowDev{};
        cr.src_row0 = (int)lo;
        cr.nb = (int)B.size();
        cr.out_row = -1;
        cr.q = 1.0;
        cr.qinv = 1.0;
      }
    }
    std::vector<uint32_t> PB;
    for (uint32_t j = 0; j < P.K; j++) PB.push_back(P.L + 1 + j);
    for (uint32_t b = 0; b < P.K; b++) {
      const uint64_t q = P.primes[PB[b]];
      dpost[b] = pair(mulm(inv_mod(P.N % q, q), inv_mod(hat_mod(PB, b, q), q), q), q);
    }
    for (uint32_t r = 0; r <= l; r++) {
      ConvRowDev& cr = dtab[r];
      cr = ConvRowDev{};
      cr.src_row0 = 0;
      cr.nb = (int)P.K;
      cr.out_row = (int)r;
      const uint64_t qr = P.primes[r];
      cr.q = (double)qr;
      cr.qinv = 1.0 / (double)qr;
      for (uint32_t b = 0; b < P.K; b++) {
        const uint64_t w = hat_mod(PB, b, qr);
        cr.cf[b] = make_double2((double)w, (double)w / (double)qr);
      }
    }
    auto up = [&](const void* h, size_t bytes) {
      void* d = c->dalloc(bytes);
      HCUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream));
      c->owned.push_back(d);
      return d;
    };
    lc.modup_post = (double2*)up(upost.data(), upost.size() * sizeof(double2));
    lc.modup_tab = (ConvRowDev*)up(utab.data(), utab.size() * sizeof(ConvRowDev));
    lc.moddown_post = (double2*)up(dpost.data(), dpost.size() * sizeof(double2));
    lc.moddown_tab = (ConvRowDev*)up(dtab.data(), dtab.size() * sizeof(ConvRowDev));
    HCUDA(cudaStreamSynchronize(c->stream));
  }
  lc.pmod = c->upload_u64(pm);
  lc.pmods = c->upload_u64(pms);
  lc.pinv = c->upload_u64(pi);
  lc.pinvs = c->upload_u64(pis);
  lc.qlinv = c->upload_u64(qi);
  lc.qlinvs = c->upload_u64(qis);
  return c->lconst.emplace((int)l, lc).first->second;
}

// D15 for G polynomials at once, all digits: in_g = in + g in_stride ([l+1][N],
// NTT form) -> out [G][dnum][l+1+K][N] (NTT form).  One INTT of the G (l+1)
// limbs into y-form, one fused conversion + NTT over every output limb (the
// digit's own limbs go through INTT/NTT unchanged: a bit-exact copy).
// NTT limb table of modup_batch: every (g, k, r) with r outside digit k, as
// layout limb (g dnum + k)(l+1+K) + r of out (cached per (level, G))
static const uint32_t* modup_lidx(helrm_ctx* c, uint32_t l, int G, size_t* count) {
  const Params& P = c->P;
  const uint32_t nl = l + 1 + P.K, dn = P.dnum(l);
  // prime-major: a launch's CTAs run in table order, so the limbs of one prime
  // follow each other and its 1 MiB pass-2 twiddle table stays in L2
  static const bool pm = getenv("HELRM_NTT_PM") ? atoi(getenv("HELRM_NTT_PM")) != 0 : true;
  std::vector<uint32_t> v;
  for (uint32_t r = 0; r < nl; r++)
    for (int g = 0; g < G; g++)
      for (uint32_t k = 0; k < dn; k++) {
        const uint32_t lo = k * P.alpha, hi = std::min((k + 1) * P.alpha, l + 1);
        if (r < lo || r >= hi) v.push_back(((uint32_t)g * dn + k) * nl + r);
      }
  if (!pm) std::sort(v.begin(), v.end());
  *count = v.size();
  auto key = std::make_pair((int)l, G);
  auto it = c->modup_lidx.find(key);
  if (it != c->modup_lidx.end()) return it->second;
  uint32_t* d = (uint32_t*)c->dalloc(v.size() * 4);
  HCUDA(cudaMemcpyAsync(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice, c->stream));
  HCUDA(cudaStreamSynchronize(c->stream));
  c->owned.push_back(d);
  c->modup_lidx.emplace(key, d);
  return d;
}

// Prime-major limb table for a launch over G polynomials of n limbs each
// (launch limb -> layout limb g n + r, r outer): consecutive CTAs share a
// prime and its pass-2 twiddles.  nullptr (identity) when G == 1.
static const uint32_t* pm_lidx(helrm_ctx* c, int G, uint32_t n) {
  static const bool pm = getenv("HELRM_NTT_PM") ? atoi(getenv("HELRM_NTT_PM")) != 0 : true;
  if (!pm || G <= 1) return nullptr;
  auto key = std::make_pair(G, (int)n);
  auto it = c->pm_lidx.find(key);
  if (it != c->pm_lidx.end()) return it->second;
  std::vector<uint32_t> v;
  for (uint32_t r = 0; r < n; r++)
    for (int g = 0; g < G; g++) v.push_back((uint32_t)g * n + r);
  uint32_t* d = (uint32_t*)c->dalloc(v.size() * 4);
  HCUDA(cudaMemcpyAsync(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice, c->stream));
  HCUDA(cudaStreamSynchronize(c->stream));
  c->owned.push_back(d);
  c->pm_lidx.emplace(key, d);
  return d;
}

// Row-slice tables for rows [r0, r1) of the Q_l P limbs and G polynomials
// (the RNS-limb partition): the ModUp conversion rows of each digit that fall
// in the slice (padded per digit), the ModUp NTT limbs of the slice, and the
// slice's Q rows for the ModDown conversion, the INTTs and the ModDown NTT.
static const helrm_ctx::SliceTabs& slice_tabs(helrm_ctx* c, uint32_t l, int r0, int r1, int G) {
  auto key = std::make_tuple((int)l, r0, r1, G);
  auto it = c->slices.find(key);
  if (it != c->slices.end()) return it->second;
  const Params& P = c->P;
  const LevelConst& lc = level_const(c, l);
  const uint32_t nl = l + 1 + P.K, nq = l + 1, dn = P.dnum(l);
  helrm_ctx::SliceTabs t;
  std::vector<ConvRowDev> ut((size_t)dn * lc.modup_rows);
  HCUDA(cudaMemcpy(ut.data(), lc.modup_tab, ut.size() * sizeof(ConvRowDev), cudaMemcpyDeviceToHost));
  std::vector<std::vector<ConvRowDev>> per(dn);
  for (uint32_t k = 0; k < dn; k++)
    for (int j = 0; j < lc.modup_rows; j++) {
      const ConvRowDev& e = ut[(size_t)k * lc.modup_rows + j];
      if (e.out_row >= r0 && e.out_row < r1) per[k].push_back(e);
    }
  size_t mx = 1;
  for (auto& v : per) mx = std::max(mx, v.size());
  std::vector<ConvRowDev> st(dn * mx);
  for (uint32_t k = 0; k < dn; k++)
    for (size_t j = 0; j < mx; j++) {
      if (j < per[k].size()) {
        st[k * mx + j] = per[k][j];
      } else {   // padding: nothing written
        st[k * mx + j] = ut[(size_t)k * lc.modup_rows];
        st[k * mx + j].out_row = -1;
      }
    }
  t.up_rows = (int)mx;
  std::vector<uint32_t> up, ql;
  for (int r = r0; r < r1; r++)
    for (int g = 0; g < G; g++) {
      for (uint32_t k = 0; k < dn; k++) {
        const uint32_t lo = k * P.alpha, hi = std::min((k + 1) * P.alpha, nq);
        if ((uint32_t)r < lo || (uint32_t)r >= hi) up.push_back(((uint32_t)g * dn + k) * nl + (uint32_t)r);
      }
      if ((uint32_t)r < nq) ql.push_back((uint32_t)g * nq + (uint32_t)r);
    }
  std::vector<ConvRowDev> dt;
  const int q1 = std::min<int>(r1, (int)nq);
  if (q1 > r0) {
    dt.resize(q1 - r0);
    HCUDA(cudaMemcpy(dt.data(), lc.moddown_tab + r0, dt.size() * sizeof(ConvRowDev), cudaMemcpyDeviceToHost));
  }
  auto up_dev = [&](const void* h, size_t bytes) {
    void* d = c->dalloc(std::max<size_t>(bytes, 16));
    if (bytes) HCUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream));
    c->owned.push_back(d);
    return d;
  };
  t.up_tab = (ConvRowDev*)up_dev(st.data(), st.size() * sizeof(ConvRowDev));
  t.up_lidx = (uint32_t*)up_dev(up.data(), up.size() * 4);
  t.n_up = up.size();
  t.dn_tab = (ConvRowDev*)up_dev(dt.data(), dt.size() * sizeof(ConvRowDev));
  t.dn_rows = (int)dt.size();
  t.q_lidx = (uint32_t*)up_dev(ql.data(), ql.size() * 4);
  t.n_q = ql.size();
  HCUDA(cudaStreamSynchronize(c->stream));
  return c->slices.emplace(key, t).first->second;
}

// copy_own = false: the digit's own limbs of out are left unwritten; the key
// switch reads them from `in` (KipArgs::own)
static void modup_batch(helrm_ctx* c, const uint64_t* in, size_t in_stride, int G, uint32_t l, uint64_t* out,
                        cudaStream_t st = nullptr, bool copy_own = true) {
  const Params& P = c->P;
  const size_t N = P.N, nq = l + 1, nl = l + 1 + P.K, dn = P.dnum(l);
  const LevelConst& lc = level_const(c, l);
  if (in_stride == 0) in_stride = nq * N;
  size_t n_conv = 0;
  const uint32_t* lidx = modup_lidx(c, l, G, &n_conv);
  if (!st) st = c->stream;
  DBuf y(c, G * nq * N, st);
  // D15 step 1: INTT straight into y-form (times [(Q_k/q_i)^-1]_{q_i});
  // step 2: one conversion launch over (g, digit) writing the rows outside
  // the digit; step 3: one NTT over exactly those limbs.  The digit's own
  // limbs are copied unchanged (NTT form).
  launch_ntt_inv(c->dc(st), in, y.p, c->scratch, G * nq, P.map_q(l), in_stride, nq * N, lc.modup_post,
                 pm_lidx(c, G, (uint32_t)nq));
  launch_conv_rows(c->dc(st), lc.modup_tab, (int)dn, lc.modup_rows, (int)P.alpha, y.p, nq * N, out, dn * nl * N,
                   nl * N, G, P.map_qp(l));
  launch_ntt_fwd(c->dc(st), out, out, c->scratch, n_conv, P.map_qp(l), 0, 0, true, lidx);
  HostTimer ht_("modup own-limb copies");
  for (size_t k = 0; copy_own && k < dn; k++) {
    const size_t lo = k * P.alpha, hi = std::min<size_t>((k + 1) * P.alpha, l + 1);
    HCUDA(cudaMemcpy2DAsync(out + k * nl * N + lo * N, dn * nl * N * 8, in + lo * N, in_stride * 8, (hi - lo) * N * 8,
                            G, cudaMemcpyDeviceToDevice, st));
  }
}

// D16 for G polynomials: y_g = y + g ys ([l+1+K][N]) -> out_g = out + g os ([l+1][N])
// (accumulate: out += ModDown(y); the finishing (y - t) P^-1 runs in the NTT's pass-2 epilogue)
static void moddown_batch(helrm_ctx* c, const uint64_t* y, size_t ys, int G, uint32_t l, uint64_t* out, size_t os,
                          cudaStream_t st = nullptr, bool accumulate = false) {
  const Params& P = c->P;
  const size_t N = P.N, nq = l + 1;
  const LevelConst& lc = level_const(c, l);
  if (!st) st = c->stream;
  DBuf yp(c, G * P.K * N, st), t(c, G * nq * N, st);
  launch_ntt_inv(c->dc(st), y + nq * N, yp.p, c->scratch, G * P.K, P.map_range(P.L + 1, P.K), ys, P.K * N,
                 lc.moddown_post, pm_lidx(c, G, P.K));
  launch_conv_rows(c->dc(st), lc.moddown_tab, 1, (int)nq, (int)P.K, yp.p, P.K * N, t.p, nq * N, 0, G, P.map_q(l));
  NttEpi epi;
  epi.y = y;
  epi.ys = ys;
  epi.out = out;
  epi.os = os;
  epi.s = lc.pinv;
  epi.sp = lc.pinvs;
  epi.accumulate = accumulate ? 1 : 0;
  launch_ntt_fwd(c->dc(st), t.p, t.p, c->scratch, G * nq, P.map_q(l), 0, 0, true, pm_lidx(c, G, (uint32_t)nq), &epi);
}

static void modup(helrm_ctx* c, const uint64_t* in, uint32_t l, int k, uint64_t* out) {
  const Params& P = c->P;
  const size_t nl = l + 1 + P.K;
  DBuf all(c, (size_t)P.dnum(l) * nl * P.N);
  modup_batch(c, in, 0, 1, l, all.p);
  HCUDA(cudaMemcpyAsync(out, all.p + (size_t)k * nl * P.N, nl * P.N * 8, cudaMemcpyDeviceToDevice, c->stream));
}

static void moddown(helrm_ctx* c, const uint64_t* y, uint32_t l, uint64_t* out) {
  const size_t nl = l + 1 + c->P.K;
  moddown_batch(c, y, nl * c->P.N, 1, l, out, (l + 1) * c->P.N);
}

// D17 on a ciphertext [2][l+1][N] -> out [2][l][N]
// (G contiguous ciphertexts [G][2][l+1][N] -> [G][2][l][N])
static void rescale_ct(helrm_ctx* c, const uint64_t* x, uint32_t l, uint64_t* out, int G = 1) {
  const Params& P = c->P;
  const size_t N = P.N;
  DBuf xl(c, 2 * G * N), r(c, 2 * G * l * N);
  ntt_inv(c, x + l * N, xl.p, 2 * G, P.map_range(l, 1), (l + 1) * N, N);
  launch_rescale_prep(c->dc(), xl.p, N, P.primes[l], r.p, l * N, 2 * G, P.map_q(l - 1));
  const LevelConst& lc = level_const(c, l);
  NttEpi epi;   // x_i' = (x_i - NTT(r)_i) q_l^-1, fused into the NTT's pass 2
  epi.y = x;
  epi.ys = (l + 1) * N;
  epi.out = out;
  epi.os = l * N;
  epi.s = lc.qlinv;
  epi.sp = lc.qlinvs;
  launch_ntt_fwd(c->dc(), r.p, r.p, c->scratch, 2 * G * l, P.map_q(l - 1), 0, 0, false, pm_lidx(c, 2 * G, l), &epi);
}

static uint32_t rot_of_galois(helrm_ctx* c, uint64_t g) {
  need(g < 2 * (uint64_t)c->P.N && (g & 1), HELRM_ERR_CONFIG, "bad Galois element");
  uint32_t r = c->dlog5[g];
  need(r != 0xffffffffu, HELRM_ERR_CONFIG, "Galois element is not a power of 5");
  return r;
}

static uint64_t galois_of_rot(helrm_ctx* c, int64_t k) {
  const uint64_t n = c->P.n, twoN = 2 * (uint64_t)c->P.N;
  uint64_t r = (uint64_t)(((k % (int64_t)n) + (int64_t)n) % (int64_t)n);
  return pow_mod(5, r, twoN);
}

static const uint64_t* key_for(const helrm_rotkeys* rk, uint64_t g) {
  auto it = rk->keys.find(g);
  if (it == rk->keys.end()) throw Error(HELRM_ERR_LAYOUT, "missing rotation key for Galois element " + std::to_string(g));
  return it->second;
}

// KS_g over precomputed digits D [dnum][l+1+K][N] (D18), fused with the
// automorphism; add0/add_mul/add_rows as in KipArgs.
static void kip(helrm_ctx* c, const uint64_t* D, uint32_t l, const helrm_rotkeys* rk, uint64_t g, const uint64_t* add0,
                int add_rows, const uint64_t* add_mul, uint64_t* out0, uint64_t* out1, bool accumulate,
                cudaStream_t st = nullptr) {
  const Params& P = c->P;
  KipArgs a{};
  a.digits = D;
  a.digit_stride = (size_t)(l + 1 + P.K) * P.N;
  a.dnum = (int)P.dnum(l);
  a.key = key_for(rk, g);
  a.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * P.N;
  a.key_half_stride = (size_t)(P.L + 1 + P.K) * P.N;
  a.add0 = add0;
  a.add_rows = add_rows;
  a.add_mul = add_mul;
  a.rot = rot_of_galois(c, g);
  a.out0 = out0;
  a.out1 = out1;
  a.accumulate = accumulate ? 1 : 0;
  launch_kip(c->dc(st), a, P.map_qp(l));
}

// lazy rotation (P phi(c0) + KS0, KS1) over Q_l P from digits of c1
static void rotate_lazy(helrm_ctx* c, const helrm_ct* in, const uint64_t* D, const helrm_rotkeys* rk, uint64_t g,
                        uint64_t* out0, uint64_t* out1) {
  const uint32_t l = in->level;
  kip(c, D, l, rk, g, ct_c0(in), (int)l + 1, level_const(c, l).pmod, out0, out1, false);
}

// Rotate(ct, k) from digits D of ct.c1 (hoisted): ModDown of both lazy halves
static void rotate_from_digits(helrm_ctx* c, const helrm_ct* in, const uint64_t* D, const helrm_rotkeys* rk, int64_t k,
                               helrm_ct* out) {
  const Params& P = c->P;
  const uint32_t l = in->level;
  const size_t N = P.N, nl = l + 1 + P.K;
  const uint64_t g = galois_of_rot(c, k);
  if (g == 1) {
    HCUDA(cudaMemcpyAsync(out->d, in->d, (size_t)2 * (l + 1) * N * 8, cudaMemcpyDeviceToDevice, c->stream));
    return;
  }
  DBuf t(c, 2 * nl * N);
  rotate_lazy(c, in, D, rk, g, t.p, t.p + nl * N);
  moddown_batch(c, t.p, nl * N, 2, l, out->d, (l + 1) * N);
}

static void rotate(helrm_ctx* c, const helrm_ct* in, const helrm_rotkeys* rk, int64_t k, helrm_ct* out) {
  const uint32_t l = in->level;
  if (galois_of_rot(c, k) == 1) {
    HCUDA(cudaMemcpyAsync(out->d, in->d, (size_t)2 * (l + 1) * c->P.N * 8, cudaMemcpyDeviceToDevice, c->stream));
    return;
  }
  DBuf D(c, (size_t)c->P.dnum(l) * (l + 1 + c->P.K) * c->P.N);
  modup_batch(c, ct_c1(in), 0, 1, l, D.p);
  rotate_from_digits(c, in, D.p, rk, k, out);
}

static void ct_add_inplace(helrm_ctx* c, helrm_ct* acc, const helrm_ct* x) {
  LimbMap m = c->P.map_q(acc->level);
  m.n = 2 * (acc->level + 1);
  for (int i = acc->level + 1; i < m.n; i++) m.pr[i] = m.pr[i - acc->level - 1];
  launch_binary(c->dc(), 0, acc->d, x->d, acc->d, m);
}

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* helrm_last_error(void) { return g_last_error.c_str(); }
const char* helrm_version(void) { return "helrm-b200 0.1 (sm_100a)"; }

helrm_status helrm_params_create(const helrm_params_desc* d, helrm_params** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(d && out, HELRM_ERR_ARG, "null argument");
    need(d->log_n >= 12 && d->log_n <= 16, HELRM_ERR_CONFIG, "log_n must be in [12, 16]");
    std::vector<std::pair<uint32_t, uint32_t>> qg, pg;
    need(d->n_q_groups >= 1 && d->n_q_groups <= 8 && d->n_p_groups >= 1 && d->n_p_groups <= 4, HELRM_ERR_CONFIG,
         "bad prime group counts");
    for (uint32_t i = 0; i < d->n_q_groups; i++) qg.push_back({d->q_bits[i], d->q_count[i]});
    for (uint32_t i = 0; i < d->n_p_groups; i++) pg.push_back({d->p_bits[i], d->p_count[i]});
    Params P;
    P.log_n = d->log_n;
    P.N = 1u << d->log_n;
    P.n = P.N / 2;
    auto q = find_primes(qg, P.N, {});
    auto p = find_primes(pg, P.N, q);
    need(q.size() + p.size() <= (size_t)kMaxLimbs, HELRM_ERR_CONFIG, "too many primes");
    need(p.size() <= (size_t)kMaxDigitPrimes, HELRM_ERR_CONFIG, "at most 8 special primes");
    for (uint64_t x : q) need(x < (1ull << 50), HELRM_ERR_CONFIG, "primes must be below 2^50");
    for (uint64_t x : p) need(x < (1ull << 50), HELRM_ERR_CONFIG, "primes must be below 2^50");
    P.L = (uint32_t)q.size() - 1;
    P.K = (uint32_t)p.size();
    P.alpha = P.K;
    need(P.dnum(P.L) <= 7, HELRM_ERR_CONFIG, "dnum = ceil((L+1)/K) must be <= 7 (key-switch kernels)");
    P.log_scale = d->log_scale;
    need(d->log_scale >= 1 && d->log_scale < 62, HELRM_ERR_CONFIG, "bad log_scale");
    P.primes = q;
    P.primes.insert(P.primes.end(), p.begin(), p.end());
    for (uint64_t x : P.primes) P.psi.push_back(min_psi(x, P.N));
    *out = new helrm_params{P};
  });
}

void helrm_params_destroy(helrm_params* p) { delete p; }

helrm_status helrm_params_info(const helrm_params* p, helrm_params_info_t* out) {
  return guard([&] {
    need(p && out, HELRM_ERR_ARG, "null argument");
    *out = {p->P.N, p->P.n, p->P.L, p->P.K, p->P.dnum(p->P.L), p->P.log_scale};
  });
}

helrm_status helrm_params_moduli(const helrm_params* p, uint64_t* q, uint64_t* pp, uint64_t* psi) {
  return guard([&] {
    need(p, HELRM_ERR_ARG, "null argument");
    const Params& P = p->P;
    if (q) std::copy(P.primes.begin(), P.primes.begin() + P.L + 1, q);
    if (pp) std::copy(P.primes.begin() + P.L + 1, P.primes.end(), pp);
    if (psi) std::copy(P.psi.begin(), P.psi.end(), psi);
  });
}

helrm_status helrm_ctx_create(const helrm_params* p, int device, uintptr_t stream, helrm_ctx** out) {
  if (out) *out = nullptr;
  helrm_ctx* c = nullptr;
  helrm_status st = guard([&] {
    need(p && out, HELRM_ERR_ARG, "null argument");
    HCUDA(cudaSetDevice(device));
    c = new helrm_ctx();
    c->P = p->P;
    c->device = device;
    c->stream = (cudaStream_t)stream;
    HCUDA(cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device));
    {
      int lo_prio = 0, hi_prio = 0;
      HCUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
      // HELRM_PRIO 1: NTT stream high priority; 3: MAC / key-switch streams high (persistent HBM
      // kernels get their SM slots first, the NTT fills the rest); 0: all equal
      const char* e = getenv("HELRM_PRIO");
      const int mode = e ? atoi(e) : 1;
      HCUDA(cudaStreamCreateWithPriority(&c->s_ntt, cudaStreamNonBlocking, mode == 1 ? hi_prio : lo_prio));
      HCUDA(cudaStreamCreateWithPriority(&c->s_kip, cudaStreamNonBlocking, mode == 3 ? hi_prio : lo_prio));
      HCUDA(cudaStreamCreateWithPriority(&c->s_mac, cudaStreamNonBlocking, mode == 3 ? hi_prio : lo_prio));
      HCUDA(cudaStreamCreateWithFlags(&c->s_cap, cudaStreamNonBlocking));
      HCUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
      HCUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    }
    {
      // a private pool: memory freed by the lookup's temporaries is kept for the next
      // lookup (release threshold: unlimited) without changing the device's default
      // pool that other allocators of the process (PyTorch) use; trimmed when plans,
      // key sets or the context are destroyed
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      HCUDA(cudaMemPoolCreate(&c->pool, &props));
      uint64_t thr = UINT64_MAX;
      HCUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
      // stream-ordered reuse across the side streams must not add hidden
      // dependencies (they would serialise the pipelined giant steps)
      int dep = 0;
      HCUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &dep));
    }
    const Params& P = c->P;
    const size_t N = P.N, np = P.primes.size();
    // NTT twiddles as (w, w/q) double pairs; per prime [tw1 256][tw2 N][itw1 256][itw2 N]
    const size_t per = 2 * (2 * N + 512);  // doubles per prime
    std::vector<double> tw(np * per);
    std::vector<uint32_t> br(N);
    for (uint32_t k = 0; k < N; k++) {
      uint32_t r = 0;
      for (uint32_t b = 0; b < P.log_n; b++) r |= ((k >> b) & 1u) << (P.log_n - 1 - b);
      br[k] = r;
    }
    const uint32_t s1 = P.log_n - 8;
#pragma omp parallel for
    for (size_t i = 0; i < np; i++) {
      const uint64_t q = P.primes[i], psi = P.psi[i], ipsi = inv_mod(psi, q);
      std::vector<uint64_t> pw(N), ipw(N);
      pw[0] = ipw[0] = 1;
      for (size_t k = 1; k < N; k++) {
        pw[k] = mulm(pw[k - 1], psi, q);
        ipw[k] = mulm(ipw[k - 1], ipsi, q);
      }
      double* base = &tw[i * per];
      // centred twiddles (|w| <= q/2): the butterflies' mmul then accepts inputs below 4q
      // (kernels_ntt.cu), which halves the lazy reductions
      auto cen = [&](uint64_t w) { return w > q / 2 ? (double)w - (double)q : (double)w; };
      auto put = [&](double* dst, size_t j, size_t idx) {
        const double w = cen(pw[br[idx]]), iw = cen(ipw[br[idx]]);
        dst[2 * j] = w;
        dst[2 * j + 1] = w / (double)q;
        dst[2 * N + 512 + 2 * j] = iw;
        dst[2 * N + 512 + 2 * j + 1] = iw / (double)q;
      };
      for (size_t idx = 0; idx < 256; idx++) put(base, idx, idx);  // pass 1 (natural index < 256)
      double* t2 = base + 512;
      for (size_t B = 0; B < N / 256; B++) {
        for (uint32_t st = 0; st < 4; st++)
          for (uint32_t ii = 0; ii < (1u << st); ii++)
            put(t2, B * 256 + (1u << st) - 1 + ii, (1ull << (s1 + st)) + (B << st) + ii);
        for (uint32_t t = 0; t < 16; t++)
          for (uint32_t st = 4; st < 8; st++)
            for (uint32_t ii = 0; ii < (1u << (st - 4)); ii++)
              put(t2, B * 256 + 15 + 16 * ((1u << (st - 4)) - 1 + ii) + t,
                  (1ull << (s1 + st)) + (B << st) + t * (1ull << (st - 4)) + ii);
      }
    }
    {
      std::vector<uint64_t> bits(tw.size());
      std::memcpy(bits.data(), tw.data(), tw.size() * 8);
      c->dtw = c->upload_u64(bits);
      c->dtwb = reinterpret_cast<const double*>(c->dtw);
    }
    c->hprimes.resize(np);
    for (size_t i = 0; i < np; i++) {
      PrimeDev& d = c->hprimes[i];
      uint64_t q = P.primes[i];
      d.rc.q = q;
      d.rc.mu = (uint64_t)(~0ull / q);
      d.rc.r64 = (uint64_t)(((unsigned __int128)1 << 64) % q);
      d.rc.r64s = shoup_pre(d.rc.r64, q);
      d.ninv = inv_mod(N % q, q);
      d.ninvs = shoup_pre(d.ninv, q);
      d.qd = (double)q;
      d.qinv = 1.0 / (double)q;
      d.ninvd = make_double2((double)d.ninv, (double)d.ninv / (double)q);
      const double* b = reinterpret_cast<const double*>(c->dtw) + i * per;
      d.tw1 = reinterpret_cast<const double2*>(b);
      d.tw2 = reinterpret_cast<const double2*>(b + 512);
      d.itw1 = reinterpret_cast<const double2*>(b + 2 * N + 512);
      d.itw2 = reinterpret_cast<const double2*>(b + 2 * N + 1024);
    }
    c->dprimes = (PrimeDev*)c->dalloc(np * sizeof(PrimeDev));
    c->owned.push_back(c->dprimes);
    HCUDA(cudaMemcpyAsync(c->dprimes, c->hprimes.data(), np * sizeof(PrimeDev), cudaMemcpyHostToDevice, c->stream));
    auto sp = slot_of_bitrev(P.log_n);
    c->dslotpos = (uint32_t*)c->dalloc(N * 4);
    c->owned.push_back(c->dslotpos);
    HCUDA(cudaMemcpyAsync(c->dslotpos, sp.data(), N * 4, cudaMemcpyHostToDevice, c->stream));
    {
      // pass-2 grouping: 256-blocks ordered by (half, slot position mod n/256);
      // per block, elements ordered by slot position
      const uint32_t nb = N / 256, stride = P.n / 256;
      std::vector<std::pair<uint64_t, uint32_t>> key(nb);
      std::vector<uint8_t> einv(N);
      for (uint32_t B = 0; B < nb; B++) {
        const uint32_t p0 = sp[B * 256];
        const uint32_t sig = p0 >= P.n, j = (p0 % P.n) % stride;
        std::vector<std::pair<uint32_t, uint32_t>> pe(256);
        for (uint32_t e = 0; e < 256; e++) {
          const uint32_t p = sp[B * 256 + e];
          need((p >= P.n) == (bool)sig && (p % P.n) % stride == j, HELRM_ERR_CONFIG, "slot grouping invariant");
          pe[e] = {p, e};
        }
        std::sort(pe.begin(), pe.end());
        for (uint32_t tp = 0; tp < 256; tp++) einv[B * 256 + tp] = (uint8_t)pe[tp].second;
        key[B] = {((uint64_t)sig << 32) | j, B};
      }
      std::sort(key.begin(), key.end());
      std::vector<uint32_t> grp(nb);
      for (uint32_t i = 0; i < nb; i++) grp[i] = key[i].second;
      c->dgrp = (uint32_t*)c->dalloc(nb * 4);
      c->owned.push_back(c->dgrp);
      HCUDA(cudaMemcpyAsync(c->dgrp, grp.data(), nb * 4, cudaMemcpyHostToDevice, c->stream));
      ntt_set_grp(P.log_n, grp.data(), nb);
      // rank of each element's slot position within its block (inverse of einv); the
      // pass-2 / pass-A swizzle needs tp(16 t + k) mod 16 distinct over t for every k
      std::vector<uint8_t> tpos(N);
      for (uint32_t B = 0; B < nb; B++)
        for (uint32_t tp = 0; tp < 256; tp++) tpos[B * 256 + einv[B * 256 + tp]] = (uint8_t)tp;
      for (uint32_t B = 0; B < nb; B++)
        for (uint32_t k = 0; k < 16; k++) {
          uint32_t seen = 0;
          for (uint32_t t = 0; t < 16; t++) seen |= 1u << (tpos[B * 256 + 16 * t + k] & 15);
          need(seen == 0xffffu, HELRM_ERR_CONFIG, "slot-order swizzle invariant");
        }
      c->dtpos = (uint8_t*)c->dalloc(N);
      c->owned.push_back(c->dtpos);
      HCUDA(cudaMemcpyAsync(c->dtpos, tpos.data(), N, cudaMemcpyHostToDevice, c->stream));
      HCUDA(cudaStreamSynchronize(c->stream));
    }
    c->dcdt = c->upload_u64(gauss_cdt_table());
    c->scratch = (uint64_t*)c->dalloc(ntt_scratch_words(P.log_n) * 8);
    c->owned.push_back(c->scratch);
    c->dlog5.assign(2 * N, 0xffffffffu);
    uint64_t e = 1;
    for (uint32_t j = 0; j < P.n; j++) {
      c->dlog5[e] = j;
      e = e * 5 % (2 * N);
    }
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = c;
  });
  if (st != HELRM_OK && c) {
    if (c->pool) cudaMemPoolDestroy(c->pool);
    delete c;
  }
  return st;
}

void helrm_ctx_destroy(helrm_ctx* c) {
  if (!c) return;
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != c->device) cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->s_ntt) cudaStreamSynchronize(c->s_ntt);
  if (c->s_kip) cudaStreamSynchronize(c->s_kip);
  if (c->s_mac) cudaStreamSynchronize(c->s_mac);
  for (auto& kv : c->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.pinned) cudaFreeHost(kv.second.pinned);
    c->dfree(kv.second.X);
    c->dfree(kv.second.S);
    c->dfree(kv.second.scratch);
  }
  c->graphs.clear();
  if (c->comm) nccl().commDestroy(c->comm);
  for (void* p : c->owned) cudaFreeAsync(p, c->stream);
  cudaStreamSynchronize(c->stream);
  for (cudaEvent_t e : c->evpool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->hev)
    if (e) cudaEventDestroy(e);
  if (c->s_ntt) cudaStreamDestroy(c->s_ntt);
  if (c->s_kip) cudaStreamDestroy(c->s_kip);
  if (c->s_cap) cudaStreamDestroy(c->s_cap);
  if (c->s_mac) cudaStreamDestroy(c->s_mac);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  if (c->pool) cudaMemPoolDestroy(c->pool);
  delete c;
}

helrm_status helrm_ctx_sync(helrm_ctx* c) {
  return guard([&] {
    need(c, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    HCUDA(cudaStreamSynchronize(c->stream));
  });
}

uint64_t helrm_ctx_launches(const helrm_ctx* c) { return c ? c->launches : 0; }

helrm_status helrm_ctx_profile(helrm_ctx* c, int enable) {
  return guard([&] {
    need(c, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    HCUDA(cudaStreamSynchronize(c->stream));
    for (auto& r : c->prof.recs) {
      c->prof.pool.push_back(r.a);
      c->prof.pool.push_back(r.b);
    }
    c->prof.recs.clear();
    c->prof.on = enable != 0;
  });
}

const char* helrm_ctx_profile_json(helrm_ctx* c) {
  if (!c) return "{}";
  cudaStreamSynchronize(c->stream);
  struct Agg {
    uint64_t n = 0;
    double ms = 0, bytes = 0;
  };
  std::map<std::string, Agg> agg;
  static const bool trace = getenv("HELRM_TRACE") && atoi(getenv("HELRM_TRACE")) != 0;
  for (auto& r : c->prof.recs) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (trace && !c->prof.recs.empty()) {   // timeline: start / end relative to the first record
      float t0 = 0, t1 = 0;
      cudaEventElapsedTime(&t0, c->prof.recs[0].a, r.a);
      cudaEventElapsedTime(&t1, c->prof.recs[0].a, r.b);
      fprintf(stderr, "[trace] %-14s %10.3f %10.3f\n", r.name, t0, t1);
    }
    auto& a = agg[r.name];
    a.n++;
    a.ms += ms;
    a.bytes += r.bytes;
  }
  std::string j = "{";
  for (auto& kv : agg) {
    if (j.size() > 1) j += ", ";
    char buf[200];
    snprintf(buf, sizeof buf, "\"%s\": {\"count\": %llu, \"ms\": %.6f, \"bytes\": %.0f}", kv.first.c_str(),
             (unsigned long long)kv.second.n, kv.second.ms, kv.second.bytes);
    j += buf;
  }
  j += "}";
  c->prof_json = j;
  return c->prof_json.c_str();
}

// ---------------------------------------------------------------------------
// keys
// ---------------------------------------------------------------------------
static void sample_small_ntt(helrm_ctx* c, uint64_t seed, uint64_t stream, int kind, uint64_t* out, const LimbMap& m,
                             int64_t* keep = nullptr) {
  const size_t N = c->P.N;
  DBuf s(c, N);
  launch_sample_small(c->dc(), (int64_t*)s.p, prng_base(seed, stream), kind, c->dcdt);
  launch_reduce_signed(c->dc(), (int64_t*)s.p, out, m);
  if (keep) {
    HCUDA(cudaMemcpyAsync(keep, s.p, N * 8, cudaMemcpyDeviceToHost, c->stream));
    HCUDA(cudaStreamSynchronize(c->stream));
  }
  ntt_fwd(c, out, out, m.n, m);
}

helrm_status helrm_sk_gen(helrm_ctx* c, uint64_t seed, helrm_sk** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    helrm_sk* sk = new helrm_sk{c, nullptr, std::vector<int64_t>(P.N)};
    const uint32_t nall = P.L + 1 + P.K;
    sk->sntt = (uint64_t*)c->dalloc((size_t)nall * P.N * 8);
    sample_small_ntt(c, seed, prng_stream(1, 0, 0, 0), 0, sk->sntt, P.map_range(0, nall), sk->s.data());
    *out = sk;
  });
}

void helrm_sk_destroy(helrm_sk* s) {
  if (!s) return;
  DevGuard dg_(s->c->device);
  s->c->dfree(s->sntt);
  delete s;
}

helrm_status helrm_pk_gen(helrm_ctx* c, const helrm_sk* sk, uint64_t seed, helrm_pk** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && sk && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    const size_t N = P.N, nq = P.L + 1;
    helrm_pk* pk = new helrm_pk{c, (uint64_t*)c->dalloc(2 * nq * N * 8)};
    uint64_t* b = pk->d;
    uint64_t* a = pk->d + nq * N;
    LimbMap m = P.map_q(P.L);
    launch_sample_uniform_ntt(c->dc(), a, m, seed, 2, 0, 0, m);
    DBuf e(c, nq * N), t(c, nq * N);
    sample_small_ntt(c, seed, prng_stream(3, 0, 0, 0), 1, e.p, m);
    launch_binary(c->dc(), 2, a, sk->sntt, t.p, m);   // a s
    launch_binary(c->dc(), 1, e.p, t.p, b, m);        // e - a s
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = pk;
  });
}

void helrm_pk_destroy(helrm_pk* p) {
  if (!p) return;
  DevGuard dg_(p->c->device);
  p->c->dfree(p->d);
  delete p;
}

helrm_status helrm_rotkeys_gen(helrm_ctx* c, const helrm_sk* sk, const uint64_t* galois, size_t n, uint64_t seed,
                               helrm_rotkeys** out) {
  if (out) *out = nullptr;
  helrm_rotkeys* rk = nullptr;
  helrm_status st = guard([&] {
    need(c && sk && out && (galois || n == 0), HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    const size_t N = P.N, nall = P.L + 1 + P.K, dn = P.dnum(P.L);
    rk = new helrm_rotkeys{c, {}, dn * 2 * nall * N};
    LimbMap m = P.map_range(0, (uint32_t)nall);
    DBuf e(c, nall * N), t(c, nall * N), phis(c, nall * N);
    const LevelConst& lc = level_const(c, P.L);
    for (size_t gi = 0; gi < n; gi++) {
      const uint64_t g = galois[gi];
      if (rk->keys.count(g)) continue;
      const uint32_t r = rot_of_galois(c, g);
      uint64_t* key = (uint64_t*)c->dalloc(rk->words_per_key * 8);
      rk->keys[g] = key;
      launch_automorph(c->dc(), sk->sntt, phis.p, m, r, 0);   // phi_g(s)
      for (size_t k = 0; k < dn; k++) {
        uint64_t* b = key + k * 2 * nall * N;
        uint64_t* a = b + nall * N;
        launch_sample_uniform_ntt(c->dc(), a, m, seed, 4, g, k, m);
        sample_small_ntt(c, seed, prng_stream(5, g, k, 0), 1, e.p, m);
        launch_binary(c->dc(), 2, a, sk->sntt, t.p, m);
        launch_binary(c->dc(), 1, e.p, t.p, b, m);            // -a s + e
        // + [q_i in digit k] [P]_{q_i} phi_g(s)
        const uint32_t lo = k * P.alpha, hi = std::min((uint32_t)(k + 1) * P.alpha, P.L + 1);
        LimbMap dm = P.map_range(lo, hi - lo);
        launch_scalar_mul(c->dc(), phis.p + lo * N, t.p, dm, lc.pmod + lo, lc.pmods + lo);
        launch_binary(c->dc(), 0, b + lo * N, t.p, b + lo * N, dm);
      }
      launch_dform(c->dc(), key, rk->words_per_key, m, 1);   // keys live in D-form (FP64 MACs)
    }
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = rk;
  });
  if (st != HELRM_OK && rk) helrm_rotkeys_destroy(rk);
  return st;
}

void helrm_rotkeys_destroy(helrm_rotkeys* r) {
  if (!r) return;
  DevGuard dg_(r->c->device);
  r->c->drop_graphs(r->id);
  for (auto& kv : r->keys) r->c->dfree(kv.second);
  r->c->trim();
  delete r;
}

size_t helrm_rotkeys_bytes(const helrm_rotkeys* r) { return r ? r->keys.size() * r->words_per_key * 8 : 0; }

helrm_status helrm_sk_export(helrm_ctx* c, const helrm_sk* s, int64_t* coeff, size_t n_words) {
  return guard([&] {
    need(c && s && coeff && n_words >= c->P.N, HELRM_ERR_ARG, "bad argument");
    DevGuard dg_(c->device);
    std::copy(s->s.begin(), s->s.end(), coeff);
  });
}

static void export_ntt(helrm_ctx* c, const uint64_t* d, size_t npolys, const LimbMap& m, uint64_t* host) {
  const size_t N = c->P.N;
  DBuf t(c, npolys * m.n * N);
  ntt_inv(c, d, t.p, npolys * m.n, m);
  HCUDA(cudaMemcpyAsync(host, t.p, npolys * m.n * N * 8, cudaMemcpyDeviceToHost, c->stream));
  HCUDA(cudaStreamSynchronize(c->stream));
}

helrm_status helrm_pk_export(helrm_ctx* c, const helrm_pk* p, uint64_t* coeff, size_t n_words) {
  return guard([&] {
    need(c && p && coeff && n_words >= (size_t)2 * (c->P.L + 1) * c->P.N, HELRM_ERR_ARG, "bad argument");
    DevGuard dg_(c->device);
    export_ntt(c, p->d, 2, c->P.map_q(c->P.L), coeff);
  });
}

helrm_status helrm_rotkeys_export(helrm_ctx* c, const helrm_rotkeys* r, uint64_t g, uint64_t* coeff, size_t n_words) {
  return guard([&] {
    need(c && r && coeff && n_words >= r->words_per_key, HELRM_ERR_ARG, "bad argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    DBuf tmp(c, r->words_per_key);
    HCUDA(cudaMemcpyAsync(tmp.p, key_for(r, g), r->words_per_key * 8, cudaMemcpyDeviceToDevice, c->stream));
    launch_dform(c->dc(), tmp.p, r->words_per_key, P.map_range(0, P.L + 1 + P.K), 0);
    export_ntt(c, tmp.p, 2 * P.dnum(P.L), P.map_range(0, P.L + 1 + P.K), coeff);
  });
}

// ---------------------------------------------------------------------------
// key import (client keys generated elsewhere, e.g. by the CPU oracle): the
// canonical coefficient form of the *_export calls
// ---------------------------------------------------------------------------
// every word of npolys polynomials of map's limbs is a residue in [0, q)
static void check_canonical(helrm_ctx* c, const uint64_t* h, size_t npolys, const LimbMap& m) {
  const size_t N = c->P.N;
  for (size_t p = 0; p < npolys; p++)
    for (int l = 0; l < m.n; l++) {
      const uint64_t q = c->P.primes[m.pr[l]];
      const uint64_t* row = h + (p * m.n + l) * N;
      for (size_t i = 0; i < N; i++)
        if (row[i] >= q) throw Error(HELRM_ERR_RANGE, "imported word is not a residue in [0, q)");
    }
}

static void upload_ntt(helrm_ctx* c, const uint64_t* host, size_t npolys, const LimbMap& m, uint64_t* d) {
  check_canonical(c, host, npolys, m);
  HCUDA(cudaMemcpyAsync(d, host, npolys * m.n * c->P.N * 8, cudaMemcpyHostToDevice, c->stream));
  ntt_fwd(c, d, d, npolys * m.n, m);
}

helrm_status helrm_sk_import(helrm_ctx* c, const int64_t* coeff, size_t n_words, helrm_sk** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && coeff && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    need(n_words >= P.N, HELRM_ERR_ARG, "buffer too small");
    for (size_t i = 0; i < P.N; i++)
      need(coeff[i] >= -((int64_t)1 << 40) && coeff[i] <= ((int64_t)1 << 40), HELRM_ERR_RANGE,
           "secret coefficient outside [-2^40, 2^40]");
    helrm_sk* sk = new helrm_sk{c, nullptr, std::vector<int64_t>(coeff, coeff + P.N)};
    const uint32_t nall = P.L + 1 + P.K;
    sk->sntt = (uint64_t*)c->dalloc((size_t)nall * P.N * 8);
    DBuf s(c, P.N);
    HCUDA(cudaMemcpyAsync(s.p, coeff, P.N * 8, cudaMemcpyHostToDevice, c->stream));
    const LimbMap m = P.map_range(0, nall);
    launch_reduce_signed(c->dc(), (const int64_t*)s.p, sk->sntt, m);
    ntt_fwd(c, sk->sntt, sk->sntt, m.n, m);
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = sk;
  });
}

helrm_status helrm_pk_import(helrm_ctx* c, const uint64_t* coeff, size_t n_words, helrm_pk** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && coeff && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    const size_t words = (size_t)2 * (P.L + 1) * P.N;
    need(n_words >= words, HELRM_ERR_ARG, "buffer too small");
    helrm_pk* pk = new helrm_pk{c, (uint64_t*)c->dalloc(words * 8)};
    try {
      upload_ntt(c, coeff, 2, P.map_q(P.L), pk->d);
      HCUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
      helrm_pk_destroy(pk);
      throw;
    }
    *out = pk;
  });
}

// one key [dnum(L)][2][L+1+K][N] (coefficient form) into rk under Galois element g
static void rotkey_upload(helrm_ctx* c, helrm_rotkeys* rk, uint64_t g, const uint64_t* coeff) {
  const Params& P = c->P;
  need(g % 2 == 1 && g < 2 * (uint64_t)P.N, HELRM_ERR_ARG, "Galois element must be odd and < 2N");
  (void)rot_of_galois(c, g);   // a power of 5 (the rotations of D8)
  const LimbMap m = P.map_range(0, P.L + 1 + P.K);
  uint64_t* key = (uint64_t*)c->dalloc(rk->words_per_key * 8);
  try {
    upload_ntt(c, coeff, 2 * P.dnum(P.L), m, key);
  } catch (...) {
    c->dfree(key);
    throw;
  }
  launch_dform(c->dc(), key, rk->words_per_key, m, 1);   // keys live in D-form (FP64 MACs)
  auto it = rk->keys.find(g);
  if (it != rk->keys.end()) c->dfree(it->second);
  rk->keys[g] = key;
  c->drop_graphs(rk->id);   // captured lookups point at the replaced key
}

helrm_status helrm_rotkeys_import(helrm_ctx* c, const uint64_t* galois, size_t n, const uint64_t* const* coeff,
                                  size_t words_per_key, helrm_rotkeys** out) {
  if (out) *out = nullptr;
  helrm_rotkeys* rk = nullptr;
  helrm_status st = guard([&] {
    need(c && out && ((galois && coeff) || n == 0), HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    rk = new helrm_rotkeys{c, {}, (size_t)P.dnum(P.L) * 2 * (P.L + 1 + P.K) * P.N};
    need(words_per_key >= rk->words_per_key, HELRM_ERR_ARG, "buffer too small");
    for (size_t i = 0; i < n; i++) {
      need(coeff[i] != nullptr, HELRM_ERR_ARG, "null key buffer");
      rotkey_upload(c, rk, galois[i], coeff[i]);
    }
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = rk;
  });
  if (st != HELRM_OK && rk) helrm_rotkeys_destroy(rk);
  return st;
}

helrm_status helrm_rotkeys_upload(helrm_ctx* c, helrm_rotkeys* rk, uint64_t g, const uint64_t* coeff,
                                  size_t n_words) {
  return guard([&] {
    need(c && rk && coeff && rk->c == c, HELRM_ERR_ARG, "bad argument");
    DevGuard dg_(c->device);
    need(n_words >= rk->words_per_key, HELRM_ERR_ARG, "buffer too small");
    rotkey_upload(c, rk, g, coeff);
    HCUDA(cudaStreamSynchronize(c->stream));
  });
}

helrm_status helrm_rotkeys_galois(const helrm_rotkeys* r, uint64_t* g, size_t cap, size_t* n) {
  return guard([&] {
    need(r && n, HELRM_ERR_ARG, "null argument");
    *n = r->keys.size();
    need(g || cap == 0, HELRM_ERR_ARG, "null argument");
    size_t i = 0;
    for (auto& kv : r->keys) {
      if (i >= cap) break;
      g[i++] = kv.first;
    }
  });
}

// ---------------------------------------------------------------------------
// tables and query encoding (S0)
// ---------------------------------------------------------------------------
helrm_status helrm_tables_create(const helrm_params* p, const helrm_table_desc* t, size_t n_tables, uint32_t n_dense,
                                 helrm_tables** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(p && t && out && n_tables > 0, HELRM_ERR_ARG, "null argument");
    helrm_tables* T = new helrm_tables();
    T->P = p->P;
    T->n_dense = n_dense;
    std::map<const double*, int> seen;
    int64_t I = n_dense, R = 0;
    for (size_t b = 0; b < n_tables; b++) {
      const helrm_table_desc& d = t[b];
      need(d.k >= 1 && d.d >= 1 && d.p >= 0 && d.l >= 0 && d.w, HELRM_ERR_CONFIG, "bad table description");
      Block B{};
      B.k = d.k;
      B.d = d.d;
      B.p = d.p;
      B.comp = d.p != 0 && (d.k > d.p || d.l > 0);
      B.l = 1;
      if (B.comp) {
        need(d.p >= 2, HELRM_ERR_CONFIG, "digit base must be >= 2");
        __int128 cap = d.p;
        while (cap < d.k) { cap *= d.p; B.l++; }
        if (d.l > 0) {   // explicit digit count: p^l >= k, i.e. l >= ceil(log_p k)
          need(d.l >= B.l, HELRM_ERR_LAYOUT, "p^l < k");
          need(d.p * d.l <= ((int64_t)1 << 40), HELRM_ERR_CONFIG, "digit segment too wide");
          B.l = d.l;
        }
      }
      B.w = B.comp ? d.p * B.l : d.k;
      B.I = d.in_off < 0 ? I : d.in_off;
      B.R = d.out_off < 0 ? R : d.out_off;
      auto it = seen.find(d.w);
      if (it == seen.end()) {
        T->weights.emplace_back(d.w, d.w + (size_t)B.w * d.d);
        B.wid = (int)T->weights.size() - 1;
        seen[d.w] = B.wid;
      } else {
        B.wid = it->second;
        need((int64_t)T->weights[B.wid].size() == B.w * B.d, HELRM_ERR_LAYOUT, "shared weights with different shapes");
      }
      I = B.I + B.w;
      R = B.R + B.d;
      T->blocks.push_back(B);
    }
    T->K = 0;
    T->M = 0;
    for (auto& B : T->blocks) {
      T->K = std::max(T->K, B.I + B.w);
      T->M = std::max(T->M, B.R + B.d);
    }
    // overlapping segments / outputs are a layout error
    std::vector<std::pair<int64_t, int64_t>> in, outv;
    for (auto& B : T->blocks) {
      in.push_back({B.I, B.I + B.w});
      outv.push_back({B.R, B.R + B.d});
    }
    in.push_back({0, (int64_t)n_dense});
    for (auto* v : {&in, &outv}) {
      std::sort(v->begin(), v->end());
      for (size_t i = 1; i < v->size(); i++)
        need((*v)[i].first >= (*v)[i - 1].second, HELRM_ERR_LAYOUT, "overlapping table offsets");
    }
    *out = T;
  });
}

void helrm_tables_destroy(helrm_tables* t) { delete t; }

helrm_status helrm_tables_info(const helrm_tables* t, int64_t* K, int64_t* M) {
  return guard([&] {
    need(t, HELRM_ERR_ARG, "null argument");
    if (K) *K = t->K;
    if (M) *M = t->M;
  });
}

helrm_status helrm_encode_query(const helrm_tables* t, const int64_t* idx, const double* dense, double* slots,
                                size_t n_slots) {
  return guard([&] {
    need(t && idx && slots, HELRM_ERR_ARG, "null argument");
    need((int64_t)n_slots >= t->K, HELRM_ERR_CAPACITY, "slot buffer smaller than K");
    std::fill(slots, slots + n_slots, 0.0);
    for (uint32_t i = 0; i < t->n_dense; i++) slots[i] = dense ? dense[i] : 0.0;
    for (size_t b = 0; b < t->blocks.size(); b++) {
      const Block& B = t->blocks[b];
      int64_t i = idx[b];
      need(i >= 0 && i < B.k, HELRM_ERR_RANGE, "index outside [0, k)");
      if (!B.comp) {
        slots[B.I + i] = 1.0;
      } else {
        for (int64_t dgt = 0; dgt < B.l; dgt++) {  // least-significant digit first
          slots[B.I + dgt * B.p + i % B.p] = 1.0;
          i /= B.p;
        }
      }
    }
  });
}

// ---------------------------------------------------------------------------
// ciphertexts
// ---------------------------------------------------------------------------
static void encode_to_device(helrm_ctx* c, const double* slots, size_t n_slots, double delta, uint64_t* out,
                             const LimbMap& m) {
  const Params& P = c->P;
  std::vector<double> z(P.n, 0.0);
  std::copy(slots, slots + n_slots, z.begin());
  std::vector<int64_t> coef(P.N);
  int st = encode_slots(z.data(), n_slots, P.log_n, delta, coef.data());
  need(st == 0, HELRM_ERR_CONFIG, "|encoded coefficient| >= 2^62");
  DBuf d(c, P.N);
  HCUDA(cudaMemcpyAsync(d.p, coef.data(), P.N * 8, cudaMemcpyHostToDevice, c->stream));
  launch_reduce_signed(c->dc(), (const int64_t*)d.p, out, m);
  ntt_fwd(c, out, out, m.n, m);
  HCUDA(cudaStreamSynchronize(c->stream));
}

helrm_status helrm_encrypt(helrm_ctx* c, const helrm_pk* pk, const double* slots, size_t n_slots, uint32_t level,
                           uint64_t seed, helrm_ct** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && pk && slots && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    need(n_slots <= P.n, HELRM_ERR_CAPACITY, "more slots than N/2");
    need(level <= P.L, HELRM_ERR_LEVEL, "level above L");
    const size_t N = P.N, nq = level + 1;
    LimbMap m = P.map_q(level);
    helrm_ct* ct = new_ct(c, level, std::ldexp(1.0, P.log_scale));
    DBuf mm(c, nq * N), v(c, nq * N), e0(c, nq * N), e1(c, nq * N);
    encode_to_device(c, slots, n_slots, std::ldexp(1.0, P.log_scale), mm.p, m);
    sample_small_ntt(c, seed, prng_stream(6, 0, 0, 0), 0, v.p, m);
    sample_small_ntt(c, seed, prng_stream(7, 0, 0, 0), 1, e0.p, m);
    sample_small_ntt(c, seed, prng_stream(8, 0, 0, 0), 1, e1.p, m);
    const uint64_t* pkb = pk->d;
    const uint64_t* pka = pk->d + (size_t)(P.L + 1) * N;
    launch_binary(c->dc(), 2, v.p, pkb, ct_c0(ct), m);
    launch_binary(c->dc(), 0, ct_c0(ct), e0.p, ct_c0(ct), m);
    launch_binary(c->dc(), 0, ct_c0(ct), mm.p, ct_c0(ct), m);
    launch_binary(c->dc(), 2, v.p, pka, ct_c1(ct), m);
    launch_binary(c->dc(), 0, ct_c1(ct), e1.p, ct_c1(ct), m);
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = ct;
  });
}

helrm_status helrm_ct_alloc(helrm_ctx* c, uint32_t level, double scale, helrm_ct** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(level <= c->P.L, HELRM_ERR_LEVEL, "level above L");
    *out = new_ct(c, level, scale);
  });
}

helrm_status helrm_ct_import(helrm_ctx* c, const uint64_t* coeff, uint32_t level, double scale, helrm_ct** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && coeff && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(level <= c->P.L, HELRM_ERR_LEVEL, "level above L");
    helrm_ct* ct = new_ct(c, level, scale);
    const size_t words = (size_t)2 * (level + 1) * c->P.N;
    HCUDA(cudaMemcpyAsync(ct->d, coeff, words * 8, cudaMemcpyHostToDevice, c->stream));
    ntt_fwd(c, ct->d, ct->d, 2 * (level + 1), c->P.map_q(level));
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = ct;
  });
}

helrm_status helrm_ct_export(helrm_ctx* c, const helrm_ct* ct, uint64_t* coeff, size_t n_words) {
  return guard([&] {
    need(c && ct && coeff, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(n_words >= (size_t)2 * (ct->level + 1) * c->P.N, HELRM_ERR_ARG, "buffer too small");
    export_ntt(c, ct->d, 2, c->P.map_q(ct->level), coeff);
  });
}

helrm_status helrm_ct_info(const helrm_ct* ct, uint32_t* level, double* scale) {
  return guard([&] {
    need(ct, HELRM_ERR_ARG, "null argument");
    if (level) *level = ct->level;
    if (scale) *scale = ct->scale;
  });
}

helrm_status helrm_ct_device_ptr(const helrm_ct* ct, uint64_t** dev) {
  return guard([&] {
    need(ct && dev, HELRM_ERR_ARG, "null argument");
    *dev = ct->d;
  });
}

void helrm_ct_destroy(helrm_ct* ct) {
  if (!ct) return;
  DevGuard dg_(ct->c->device);
  ct->c->dfree(ct->d);
  delete ct;
}

helrm_status helrm_decrypt_decode(helrm_ctx* c, const helrm_sk* sk, const helrm_ct* ct, double* slots,
                                  size_t n_slots) {
  return guard([&] {
    need(c && sk && ct && slots, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    const size_t N = P.N, nq = ct->level + 1;
    LimbMap m = P.map_q(ct->level);
    DBuf t(c, nq * N);
    launch_binary(c->dc(), 2, ct_c1(ct), sk->sntt, t.p, m);
    launch_binary(c->dc(), 0, t.p, ct_c0(ct), t.p, m);
    ntt_inv(c, t.p, t.p, nq, m);
    std::vector<uint64_t> h(nq * N);
    HCUDA(cudaMemcpyAsync(h.data(), t.p, nq * N * 8, cudaMemcpyDeviceToHost, c->stream));
    HCUDA(cudaStreamSynchronize(c->stream));
    std::vector<int64_t> mm(N);
    crt_small(h.data(), P.primes.data(), nq, N, mm.data());
    decode_coeffs(mm.data(), P.log_n, ct->scale, slots, std::min(n_slots, (size_t)P.n));
  });
}

// ---------------------------------------------------------------------------
// plan (server setup, D19)
// ---------------------------------------------------------------------------
static int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p *= 2;
  return p;
}

helrm_status helrm_plan_create(helrm_ctx* c, const helrm_tables* T, uint32_t level, uint32_t n1_req, uint32_t mode,
                               helrm_plan** out) {
  if (out) *out = nullptr;
  helrm_plan* pl = nullptr;
  helrm_status st = guard([&] {
    need(c && T && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    need(level >= 1 && level <= P.L, HELRM_ERR_LEVEL, "lookup needs 1 <= level <= L");
    const bool compact = (mode & HELRM_PLAN_COMPACT) != 0;
    mode &= ~(uint32_t)HELRM_PLAN_COMPACT;
    need(mode == HELRM_MODE_DOUBLE || mode == HELRM_MODE_SINGLE, HELRM_ERR_ARG, "bad mode");
    need(!compact || mode == HELRM_MODE_DOUBLE, HELRM_ERR_ARG, "compact plans run the double-hoisted mode");
    const int64_t n = P.n;
    pl = new helrm_plan();
    pl->c = c;
    pl->level = level;
    pl->mode = mode;
    pl->compact = compact;
    pl->K = T->K;
    pl->M = T->M;
    pl->mbar = std::min(next_pow2(T->M), n);
    pl->O = (T->M + n - 1) / n;
    pl->C = (T->K + n - 1) / n;
    // hybrid diagonals: each non-zero W[r][u] lands in exactly one (o, c, t, s)
    std::map<std::tuple<int64_t, int64_t, int64_t>, std::vector<double>> diags;
    for (const Block& B : T->blocks) {
      const std::vector<double>& S = T->weights[B.wid];
      for (int64_t row = 0; row < B.w; row++)
        for (int64_t col = 0; col < B.d; col++) {
          const double v = S[row * B.d + col];
          if (v == 0.0) continue;
          const int64_t r = B.R + col, u = B.I + row;
          const int64_t o = r / n, cc = u / n, ul = u % n;
          int64_t t, s;
          if (pl->mbar < n) {
            t = ((ul - r % pl->mbar) % pl->mbar + pl->mbar) % pl->mbar;
            s = ((ul - t) % n + n) % n;
          } else {
            s = r % n;
            t = ((ul - s) % n + n) % n;
          }
          auto& vec = diags[{o, cc, t}];
          if (vec.empty()) vec.assign(n, 0.0);
          vec[s] += v;
        }
    }
    for (auto it = diags.begin(); it != diags.end();) {
      bool nz = std::any_of(it->second.begin(), it->second.end(), [](double x) { return x != 0.0; });
      it = nz ? std::next(it) : diags.erase(it);
    }
    pl->n_diag = (int64_t)diags.size();
    need(pl->n_diag > 0, HELRM_ERR_LAYOUT, "the packed matrix is zero");
    // BSGS split per output block: minimal cyclic interval, n1, n2
    std::vector<std::pair<int64_t, int64_t>> iv(pl->O);
    int64_t maxspan = 0;
    for (int64_t o = 0; o < pl->O; o++) {
      std::vector<int64_t> ts;
      for (auto& kv : diags)
        if (std::get<0>(kv.first) == o) ts.push_back(std::get<2>(kv.first));
      std::sort(ts.begin(), ts.end());
      ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
      int64_t best_span = -1, best_t0 = 0;
      for (size_t a = 0; a < ts.size(); a++) {
        const int64_t prev = ts[(a + ts.size() - 1) % ts.size()];
        const int64_t span = ts.size() == 1 ? 1 : ((prev - ts[a]) % n + n) % n + 1;
        if (best_span < 0 || span < best_span || (span == best_span && ts[a] < best_t0)) {
          best_span = span;
          best_t0 = ts[a];
        }
      }
      iv[o] = {best_t0, best_span};
      maxspan = std::max(maxspan, best_span);
    }
    int64_t n1 = n1_req;
    if (n1 == 0) {
      n1 = 1;
      while (n1 * n1 < maxspan) n1 *= 2;
    }
    pl->n1 = n1;
    std::vector<std::vector<double>> uniq;
    std::unordered_map<uint64_t, std::vector<int>> by_hash;
    std::vector<std::set<int>> bab(pl->C);
    pl->entries.resize(pl->O);
    pl->giants.resize(pl->O);
    for (int64_t o = 0; o < pl->O; o++) {
      const int64_t t0 = iv[o].first, span = iv[o].second, n2 = (span + n1 - 1) / n1;
      pl->t0.push_back(t0);
      pl->span.push_back(span);
      pl->n2.push_back(n2);
      pl->entries[o].resize(n2);
      for (int64_t i = 0; i < n2; i++) pl->giants[o].push_back((t0 + i * n1) % n);
      for (auto& kv : diags) {
        if (std::get<0>(kv.first) != o) continue;
        const int64_t cc = std::get<1>(kv.first), t = std::get<2>(kv.first);
        const int64_t r = ((t - t0) % n + n) % n, j = r % n1, i = r / n1, g = pl->giants[o][i];
        std::vector<double> u(n);
        for (int64_t s = 0; s < n; s++) u[s] = kv.second[((s - g) % n + n) % n];  // rot(diag, -g)
        uint64_t h = 1469598103934665603ull;
        const unsigned char* bytes = (const unsigned char*)u.data();
        for (size_t b = 0; b < u.size() * 8; b++) h = (h ^ bytes[b]) * 1099511628211ull;
        int uid = -1;
        for (int cand : by_hash[h])
          if (uniq[cand] == u) { uid = cand; break; }
        if (uid < 0) {
          uid = (int)uniq.size();
          uniq.push_back(std::move(u));
          by_hash[h].push_back(uid);
        }
        pl->entries[o][i].push_back(Entry{(int)cc, (int)j, uid});
        bab[cc].insert((int)j);
      }
    }
    for (auto& s : bab) pl->babies.emplace_back(s.begin(), s.end());
    // rotation amounts: babies != 0, non-empty giants != 0, RotSum
    std::set<int64_t> am;
    for (auto& bl : pl->babies)
      for (int j : bl)
        if (j) am.insert(j);
    for (int64_t o = 0; o < pl->O; o++)
      for (size_t i = 0; i < pl->giants[o].size(); i++)
        if (pl->giants[o][i] % n && !pl->entries[o][i].empty()) am.insert(pl->giants[o][i]);
    for (int64_t r = pl->mbar; r < n; r *= 2) am.insert(r);
    pl->rotations.assign(am.begin(), am.end());
    // encode the unique pre-rotated diagonals at Delta_pt = q_level, upload, NTT
    pl->n_unique = (int64_t)uniq.size();
    pl->nl = mode == HELRM_MODE_DOUBLE ? level + 1 + P.K : level + 1;
    LimbMap m = mode == HELRM_MODE_DOUBLE ? P.map_qp(level) : P.map_q(level);
    const size_t N = P.N;
    if (compact) pl->coef = (int64_t*)c->dalloc((size_t)pl->n_unique * N * 8);
    else pl->diag = (uint64_t*)c->dalloc((size_t)pl->n_unique * pl->nl * N * 8);
    const double delta_pt = (double)P.primes[level];
    const int64_t chunk = 64;
    std::vector<int64_t> coef((size_t)chunk * N);
    DBuf dcoef(c, (size_t)chunk * N);
    for (int64_t u0 = 0; u0 < pl->n_unique; u0 += chunk) {
      const int64_t cnt = std::min(chunk, pl->n_unique - u0);
      int bad = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
      for (int64_t k = 0; k < cnt; k++) bad |= encode_slots(uniq[u0 + k].data(), 0, P.log_n, delta_pt, &coef[k * N]);
      need(bad == 0, HELRM_ERR_CONFIG, "|encoded diagonal coefficient| >= 2^62");
      HCUDA(cudaStreamSynchronize(c->stream));
      if (compact) {   // the lookup expands them (reduce, NTT, D-form) just before its inner sums
        HCUDA(cudaMemcpyAsync(pl->coef + (size_t)u0 * N, coef.data(), (size_t)cnt * N * 8, cudaMemcpyHostToDevice,
                              c->stream));
        continue;
      }
      HCUDA(cudaMemcpyAsync(dcoef.p, coef.data(), (size_t)cnt * N * 8, cudaMemcpyHostToDevice, c->stream));
      for (int64_t k = 0; k < cnt; k++) {
        uint64_t* dst = pl->diag + (size_t)(u0 + k) * pl->nl * N;
        launch_reduce_signed(c->dc(), (const int64_t*)(dcoef.p + k * N), dst, m);
      }
      ntt_fwd(c, pl->diag + (size_t)u0 * pl->nl * N, pl->diag + (size_t)u0 * pl->nl * N, (size_t)cnt * pl->nl, m);
      launch_dform(c->dc(), pl->diag + (size_t)u0 * pl->nl * N, (size_t)cnt * pl->nl * N, m, 1);  // stored in D-form
    }
    HCUDA(cudaStreamSynchronize(c->stream));
    *out = pl;
  });
  if (st != HELRM_OK && pl) helrm_plan_destroy(pl);
  return st;
}

void helrm_plan_destroy(helrm_plan* p) {
  if (!p) return;
  DevGuard dg_(p->c->device);
  p->c->drop_graphs(p->id);
  p->c->dfree(p->diag);
  p->c->dfree(p->coef);
  p->c->trim();
  delete p;
}

helrm_status helrm_plan_info(const helrm_plan* p, helrm_plan_info_t* out) {
  return guard([&] {
    need(p && out, HELRM_ERR_ARG, "null argument");
    helrm_plan_info_t r{};
    r.K = p->K;
    r.M = p->M;
    r.mbar = p->mbar;
    r.n_in_cts = p->C;
    r.n_out_cts = p->O;
    r.n_diag = p->n_diag;
    r.n_unique = p->n_unique;
    r.n1 = p->n1;
    r.n2_max = *std::max_element(p->n2.begin(), p->n2.end());
    r.n_rotations = (int64_t)p->rotations.size();
    r.level = p->level;
    r.mode = p->mode | (p->compact ? HELRM_PLAN_COMPACT : 0);
    r.diag_bytes = (uint64_t)p->n_unique * (p->compact ? 1 : p->nl) * p->c->P.N * 8;
    *out = r;
  });
}

helrm_status helrm_plan_rotations(const helrm_plan* p, int64_t* amounts, size_t cap, size_t* n) {
  return guard([&] {
    need(p && n, HELRM_ERR_ARG, "null argument");
    *n = p->rotations.size();
    if (amounts) {
      need(cap >= p->rotations.size(), HELRM_ERR_ARG, "buffer too small");
      std::copy(p->rotations.begin(), p->rotations.end(), amounts);
    }
  });
}

helrm_status helrm_plan_galois(const helrm_plan* p, uint64_t* g, size_t cap, size_t* n) {
  return guard([&] {
    need(p && n, HELRM_ERR_ARG, "null argument");
    // D19 Galois list {5^a mod 2N : a in the rotation amounts}, ascending
    std::vector<uint64_t> v;
    for (int64_t a : p->rotations) v.push_back(galois_of_rot(p->c, a));
    std::sort(v.begin(), v.end());
    *n = v.size();
    need(g || cap == 0, HELRM_ERR_ARG, "null argument");
    for (size_t i = 0; i < v.size() && i < cap; i++) g[i] = v[i];
  });
}

// ---------------------------------------------------------------------------
// the lookup (D20 / D22, D21)
// ---------------------------------------------------------------------------
static void rot_sum(helrm_ctx* c, helrm_ct* ct, int64_t mbar, const helrm_rotkeys* rk) {
  const int64_t n = c->P.n;
  if (mbar >= n) return;
  helrm_ct* tmp = new_ct(c, ct->level, ct->scale);
  for (int64_t r = mbar; r < n; r *= 2) {
    rotate(c, ct, rk, r, tmp);
    ct_add_inplace(c, ct, tmp);
  }
  helrm_ct_destroy(tmp);
}

static LimbMap map_twice(const LimbMap& m) {
  LimbMap r = m;
  r.n = 2 * m.n;
  for (int i = 0; i < m.n; i++) r.pr[m.n + i] = m.pr[i];
  return r;
}

// host-side L3 work list: output pair z per non-empty (o, i) (in o, i order),
// giants packed kGiantPack at a time, one term per baby pair used by the pack
struct MacList {
  int gp = kGiantPack;              // giants per pack (kGiantPack or kWidePack)
  std::vector<char> terms;          // MacTermT<gp> records
  size_t term_size = 0, n_terms = 0;
  std::vector<int4> groups;
  std::vector<std::pair<int64_t, int64_t>> oi;   // (o, i) of each output pair
  double n_u = 0, n_x = 0;   // plaintext limb-sets read, distinct baby pairs read
  std::vector<double> gu;    // plaintexts per group
};

}  // extern "C" (templates below)

template <int GP, class XF>
static MacList build_macs_t(const helrm_plan* pl, size_t diag_stride, XF xptr, int64_t z_lo, int64_t z_hi) {
  using Term = MacTermT<GP>;
  MacList ml;
  ml.gp = GP;
  ml.term_size = sizeof(Term);
  std::set<std::pair<int, int>> xs;   // distinct (c, j) baby pairs
  int64_t zg = 0;   // global index of the non-empty (o, i) pairs
  for (int64_t o = 0; o < pl->O; o++) {
    std::vector<int64_t> gi;
    for (size_t i = 0; i < pl->entries[o].size(); i++)
      if (!pl->entries[o][i].empty()) {
        if (zg >= z_lo && zg < z_hi) gi.push_back((int64_t)i);
        zg++;
      }
    for (size_t g0 = 0; g0 < gi.size(); g0 += GP) {
      const int ng = (int)std::min<size_t>(GP, gi.size() - g0);
      const int z0 = (int)ml.oi.size();
      double gu = 0;
      std::map<std::pair<int, int>, Term> tm;
      for (int g = 0; g < ng; g++) {
        ml.oi.push_back({o, gi[g0 + g]});
        for (const Entry& e : pl->entries[o][gi[g0 + g]]) {
          auto it = tm.find({e.c, e.j});
          if (it == tm.end()) {
            Term t{};
            auto x = xptr(e.c, e.j);
            t.x0 = x.first;
            t.x1 = x.second;
            it = tm.emplace(std::make_pair(e.c, e.j), t).first;
          }
          it->second.u[g] = pl->diag + (size_t)e.uid * diag_stride;
          ml.n_u += 1;
          gu += 1;
        }
      }
      ml.groups.push_back(make_int4((int)ml.n_terms, (int)tm.size(), z0, ng));
      ml.gu.push_back(gu);
      for (auto& kv : tm) {
        const char* b = reinterpret_cast<const char*>(&kv.second);
        ml.terms.insert(ml.terms.end(), b, b + sizeof(Term));
        ml.n_terms++;
        xs.insert(kv.first);
      }
    }
  }
  ml.n_x = (double)xs.size();
  return ml;
}

template <class XF>
static MacList build_macs(const helrm_plan* pl, size_t diag_stride, XF xptr, int64_t z_lo = 0,
                          int64_t z_hi = INT64_MAX, bool wide = false) {
  return wide ? build_macs_t<kWidePack>(pl, diag_stride, xptr, z_lo, z_hi)
              : build_macs_t<kGiantPack>(pl, diag_stride, xptr, z_lo, z_hi);
}

extern "C" {

// the MAC work list on the device (uploaded once per lookup)
// (pinned != null: the list is staged in pinned host memory owned by the
// caller, at least mac_list_bytes() -- a copy from pinned memory can be
// captured into a CUDA graph)
struct MacDev {
  DBuf terms, groups, extra;
  MacDev(helrm_ctx* c, const MacList& ml, void** pinned = nullptr, const std::vector<char>& xtra = {})
      : terms(c, (ml.terms.size() + 7) / 8 + 1), groups(c, 2 * ml.groups.size() + 1),
        extra(c, (xtra.size() + 7) / 8 + 1) {
    const size_t tb = ml.terms.size(), gb = ml.groups.size() * sizeof(int4), xb = xtra.size();
    const void* ht = ml.terms.data();
    const void* hg = ml.groups.data();
    const void* hx = xtra.data();
    if (pinned) {   // allocated by the caller before the capture (mac_list_bytes)
      need(*pinned != nullptr, HELRM_ERR_ARG, "pinned MAC staging buffer missing");
      std::memcpy(*pinned, ht, tb);
      std::memcpy((char*)*pinned + tb, hg, gb);
      if (xb) std::memcpy((char*)*pinned + tb + gb, hx, xb);
      ht = *pinned;
      hg = (const char*)*pinned + tb;
      hx = (const char*)*pinned + tb + gb;
    }
    HostTimer ht_("MacDev upload");
    HCUDA(cudaMemcpyAsync(terms.p, ht, tb, cudaMemcpyHostToDevice, c->stream));
    HCUDA(cudaMemcpyAsync(groups.p, hg, gb, cudaMemcpyHostToDevice, c->stream));
    if (xb) HCUDA(cudaMemcpyAsync(extra.p, hx, xb, cudaMemcpyHostToDevice, c->stream));
  }
};

// run the batched MAC of groups [g0, g1) into out (pair z at out + z out_stride)
static void run_macs(helrm_ctx* c, const MacList& ml, const MacDev& md, size_t g0, size_t g1, uint64_t* out,
                     size_t out_stride, const LimbMap& map, bool x_dform, int nq = 1, size_t xq = 0, size_t oq = 0,
                     cudaStream_t st = nullptr, int pers = 0) {
  if (g1 <= g0) return;
  double nu = 0;
  int nout = 0;
  for (size_t g = g0; g < g1; g++) {
    nu += ml.gu[g];
    nout += ml.groups[g].w;
  }
  // algorithmic bytes: plaintexts of the groups, each distinct baby pair once per lookup (charged to the
  // first launch), the outputs
  const double nx = g0 == 0 ? ml.n_x : 0.0;
  launch_diag_mac(c->dc(st, pers), md.terms.p, (const int4*)md.groups.p + g0, (int)(g1 - g0), nu, nx, nout, out,
                  out_stride, map, x_dform, nq, xq, oq, ml.gp == kWidePack);
}

static void run_macs_all(helrm_ctx* c, const MacList& ml, uint64_t* out, size_t out_stride, const LimbMap& map,
                         bool x_dform) {
  MacDev md(c, ml);
  run_macs(c, ml, md, 0, ml.groups.size(), out, out_stride, map, x_dform);
}

// Compact plans (HELRM_PLAN_COMPACT), one query: D20 L1-L3 with the input
// cts in groups and the diagonals expanded chunk by chunk.  For each group
// of input cts: ModUp of their c1 and their baby steps (one k_kip_multi with
// the cts as "queries" when they share the baby set); then the unique
// diagonals those cts' terms use, `uc` at a time, are expanded from the
// plan's int64 coefficients (reduce into every Q_l P limb, NTT, D-form) and
// the inner sums of the terms that use them are accumulated into AB (pair z
// of ml.oi at AB + z 2 nlN, zeroed by the caller).  Exact modular sums in
// another order: the same bits as the stored-diagonal path.
static void compact_l1_l3(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const uint64_t* X,
                          const std::vector<std::pair<int64_t, int64_t>>& oi, uint64_t* AB) {
  const Params& P = c->P;
  const uint32_t l = pl->level;
  const size_t N = P.N, nq = l + 1, nl = l + 1 + P.K, nlN = nl * N, nqN = nq * N, dn = P.dnum(l);
  const LimbMap mqp = P.map_qp(l), mq = P.map_q(l);
  const LevelConst& lc = level_const(c, l);
  const int64_t C = pl->C;
  size_t fr = 0, tot = 0;
  HCUDA(cudaMemGetInfo(&fr, &tot));
  // device budgets: baby pairs + digits of a ct group, and the expansion buffer
  static const double grp_gib = getenv("HELRM_COMPACT_GROUP_GIB") ? atof(getenv("HELRM_COMPACT_GROUP_GIB")) : 0;
  static const double exp_gib = getenv("HELRM_COMPACT_EXP_GIB") ? atof(getenv("HELRM_COMPACT_EXP_GIB")) : 4;
  const size_t gbudget = grp_gib > 0 ? (size_t)(grp_gib * (1 << 30)) : std::min<size_t>(fr / 3, (size_t)40 << 30);
  size_t nb_max = 1;
  for (auto& b : pl->babies) nb_max = std::max(nb_max, b.size());
  const size_t per_ct = 8 * (dn * nlN + nb_max * 2 * nlN);
  const int64_t G = std::max<int64_t>(1, std::min<int64_t>(C, (int64_t)(gbudget / per_ct)));
  const size_t uc = std::max<size_t>(1, std::min<size_t>({(size_t)pl->n_unique, (size_t)65535,
                                                          (size_t)(exp_gib * (1 << 30)) / (8 * nlN)}));
  DBuf E(c, uc * nlN);
  for (int64_t c0 = 0; c0 < C; c0 += G) {
    const int64_t g = std::min(G, C - c0);
    DBuf Dg(c, (size_t)g * dn * nlN), Bg(c, (size_t)g * nb_max * 2 * nlN);
    // L1: digits of the group's c1 (ct ci at X + ci 2 nqN)
    modup_batch(c, X + c0 * 2 * nqN + nqN, 2 * nqN, (int)g, l, Dg.p, nullptr, false);
    // L2: baby pair (ci, j) at Bg + ((ci - c0) nb_max + jj) 2 nlN
    std::map<std::pair<int64_t, int>, uint64_t*> ab;
    bool same = true;
    for (int64_t ci = c0 + 1; ci < c0 + g; ci++) same = same && pl->babies[ci] == pl->babies[c0];
    const int64_t runs = same ? 1 : g;   // one kip_multi over the group (cts as queries), or one per ct
    for (int64_t r = 0; r < runs; r++) {
      const int64_t cf = c0 + (same ? 0 : r), nct = same ? g : 1;
      const uint64_t* xc = X + cf * 2 * nqN;
      KipMulti km{};
      km.own = xc + nqN;
      km.ownq = 2 * nqN;
      km.alpha = (int)P.alpha;
      km.digits = Dg.p + (cf - c0) * dn * nlN;
      km.digit_stride = nlN;
      km.dnum = (int)dn;
      km.c0 = xc;
      km.p_mod = lc.pmod;
      km.level = l;
      km.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
      km.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
      km.out_half = nlN;
      km.nq = (int)nct;
      km.qk = std::min((int)nct, 4);
      km.zfast = nct > 4 ? 1 : 0;
      km.dq = dn * nlN;
      km.cq = 2 * nqN;
      km.oq = nb_max * 2 * nlN;
      const std::vector<int>& bl = pl->babies[cf];
      for (size_t jj = 0; jj < bl.size(); jj++) {
        const int j = bl[jj];
        uint64_t* a = Bg.p + ((cf - c0) * nb_max + jj) * 2 * nlN;
        for (int64_t k = 0; k < nct; k++) ab[{cf + k, j}] = a + k * nb_max * 2 * nlN;
        if (j == 0) {   // (P c0, P c1) in D-form, P limbs 0
          for (int64_t k = 0; k < nct; k++) HCUDA(cudaMemsetAsync(a + k * nb_max * 2 * nlN, 0, 2 * nlN * 8, c->stream));
          launch_scalar_mul(c->dc(), xc, a, mq, lc.pmod, lc.pmods, 1, (int)nct, 2 * nqN, nb_max * 2 * nlN);
          launch_scalar_mul(c->dc(), xc + nqN, a + nlN, mq, lc.pmod, lc.pmods, 1, (int)nct, 2 * nqN, nb_max * 2 * nlN);
        } else {
          need(km.n < kMaxBabies, HELRM_ERR_CAPACITY, "too many baby steps");
          const uint64_t ge = galois_of_rot(c, j);
          km.rot[km.n] = rot_of_galois(c, ge);
          km.key[km.n] = key_for(rk, ge);
          km.out[km.n] = a;
          km.max_rot = std::max(km.max_rot, km.rot[km.n]);
          km.n++;
        }
      }
      if (km.n) launch_kip_multi(c->dc(), km, mqp);
    }
    // L3: the unique diagonals of this group's terms, uc at a time
    std::vector<uint32_t> uids;
    for (auto& zo : oi)
      for (const Entry& e : pl->entries[zo.first][zo.second])
        if (e.c >= c0 && e.c < c0 + g) uids.push_back((uint32_t)e.uid);
    std::sort(uids.begin(), uids.end());
    uids.erase(std::unique(uids.begin(), uids.end()), uids.end());
    for (size_t u0 = 0; u0 < uids.size(); u0 += uc) {
      const size_t cnt = std::min(uc, uids.size() - u0);
      std::unordered_map<uint32_t, size_t> slot;
      for (size_t k = 0; k < cnt; k++) slot[uids[u0 + k]] = k;
      DBuf du(c, (cnt + 1) / 2);
      HCUDA(cudaMemcpyAsync(du.p, uids.data() + u0, cnt * 4, cudaMemcpyHostToDevice, c->stream));
      launch_expand_coef(c->dc(), pl->coef, (const uint32_t*)du.p, cnt, E.p, mqp);
      ntt_fwd(c, E.p, E.p, cnt * nl, mqp);
      launch_dform(c->dc(), E.p, cnt * nlN, mqp, 1);
      // work list: packs of <= kGiantPack consecutive pairs of one output block
      std::vector<MacTerm> terms;
      std::vector<int4> groups;
      double nu = 0;
      for (size_t z0 = 0; z0 < oi.size();) {
        size_t z1 = z0 + 1;
        while (z1 < oi.size() && z1 - z0 < (size_t)kGiantPack && oi[z1].first == oi[z0].first) z1++;
        std::map<std::pair<int64_t, int>, MacTerm> tm;
        for (size_t z = z0; z < z1; z++)
          for (const Entry& e : pl->entries[oi[z].first][oi[z].second]) {
            if (e.c < c0 || e.c >= c0 + g) continue;
            auto it = slot.find((uint32_t)e.uid);
            if (it == slot.end()) continue;
            auto ti = tm.find({e.c, e.j});
            if (ti == tm.end()) {
              MacTerm t{};
              t.x0 = ab.at({e.c, e.j});
              t.x1 = t.x0 + nlN;
              ti = tm.emplace(std::make_pair((int64_t)e.c, e.j), t).first;
            }
            ti->second.u[z - z0] = E.p + it->second * nlN;
            nu += 1;
          }
        if (!tm.empty()) {
          groups.push_back(make_int4((int)terms.size(), (int)tm.size(), (int)z0, (int)(z1 - z0)));
          for (auto& kv : tm) terms.push_back(kv.second);
        }
        z0 = z1;
      }
      if (groups.empty()) continue;
      DBuf dt(c, (terms.size() * sizeof(MacTerm) + 7) / 8), dg(c, groups.size() * 2);
      HCUDA(cudaMemcpyAsync(dt.p, terms.data(), terms.size() * sizeof(MacTerm), cudaMemcpyHostToDevice, c->stream));
      HCUDA(cudaMemcpyAsync(dg.p, groups.data(), groups.size() * sizeof(int4), cudaMemcpyHostToDevice, c->stream));
      {
        const DevCtx dcx = c->dc();
        ProfScope ps_(dcx, "diag_mac", 8.0 * N * nl * (nu + 2.0 * terms.size() + 4.0 * oi.size()));
        need(launch_diag_mac_bulk(dcx, (const MacTerm*)dt.p, (const int4*)dg.p, (int)groups.size(), AB, 2 * nlN, nlN,
                                  mqp, 1, 0, 0, 1),
             HELRM_ERR_CONFIG, "compact plans need N divisible by the MAC tile");
      }
      // host vectors are copied before the next chunk reuses them (pageable copies are staged)
      HCUDA(cudaStreamSynchronize(c->stream));
    }
  }
}

// D20 L1-L4 for Qc queries (in[q C + c]) and the giant pairs z in [z_lo, z_hi)
// of the non-empty (o, i) enumeration: accumulates into Oall [O][Qc][2][l+1+K][N]
// (zeroed by the caller).  With z over everything this is the whole lookup up
// to L5; split over ranks the partial O's sum exactly to the full one (D23).
// The queries of a call share every key and plaintext read: the key switches
// load each key value once and apply it to all queries (kip_multi stages up
// to 4 queries' digit tiles per CTA), the diagonal MAC re-reads its plaintext
// tiles from L2 for the second and later queries.
static void lookup_double_part(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const uint64_t* X,
                               int Qc, int64_t z_lo, int64_t z_hi, uint64_t* Oall, void** pinned = nullptr) {
  const Params& P = c->P;
  const uint32_t l = pl->level;
  const size_t N = P.N, nq = l + 1, nl = l + 1 + P.K, nlN = nl * N, nqN = nq * N, dn = P.dnum(l);
  const size_t C = pl->C;
  const LimbMap mqp = P.map_qp(l), mq = P.map_q(l);
  const LevelConst& lc = level_const(c, l);
  c->evnext = 0;
  // inputs: ct (q, ci) at X + (q C + ci) 2 nqN (staged by the caller)
  const size_t xs = C * 2 * nqN;   // query stride of the inputs
  std::unique_ptr<NvtxRange> nv12(new NvtxRange("helrm L1-L2 ModUp + baby steps"));
  // L1 (hoist #1): digits of every input c1 [ci][q][dn][nl][N];  L2: lazy baby steps over Q_l P,
  // baby b of query q at babies + (b Qc + q) 2 nlN
  std::vector<std::map<int, uint64_t*>> ab(C);
  size_t n_baby = 0;
  for (auto& bl : pl->babies) n_baby += bl.size();
  need(!pl->compact || Qc == 1, HELRM_ERR_ARG, "compact plans look up one query at a time");
  // compact plans: L1-L2 happen per ct group inside compact_l1_l3 (after the work list)
  DBuf D(c, pl->compact ? 1 : C * Qc * dn * nlN);
  DBuf babies(c, pl->compact ? 1 : std::max<size_t>(1, n_baby) * Qc * 2 * nlN);
  size_t bi = 0;
  bool same_babies = Qc == 1 && C > 1 && !pl->compact;
  for (size_t ci = 1; same_babies && ci < C; ci++) same_babies = pl->babies[ci] == pl->babies[0];
  if (same_babies) {
    // one query, C input cts with the same baby steps (LLM layout L2): the cts take the
    // query role -- one batched ModUp, one baby kernel reading every key once for all C
    const size_t nb = pl->babies[0].size();
    modup_batch(c, X + nqN, 2 * nqN, (int)C, l, D.p, nullptr, false);
    KipMulti km{};
    km.own = X + nqN;
    km.ownq = 2 * nqN;
    km.alpha = (int)P.alpha;
    km.digits = D.p;
    km.digit_stride = nlN;
    km.dnum = (int)dn;
    km.c0 = X;
    km.p_mod = lc.pmod;
    km.level = l;
    km.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
    km.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
    km.out_half = nlN;
    km.nq = (int)C;
    km.qk = std::min((int)C, 4);
    // many input cts: their CTAs of one (tile, limb) run side by side and share the key tiles in L2
    static const int zf = getenv("HELRM_KM_ZFAST") ? atoi(getenv("HELRM_KM_ZFAST")) : 1;
    km.zfast = zf && C > 4 ? 1 : 0;
    km.dq = dn * nlN;
    km.cq = 2 * nqN;
    km.oq = nb * 2 * nlN;
    for (size_t jj = 0; jj < nb; jj++) {
      const int j = pl->babies[0][jj];
      uint64_t* a = babies.p + jj * 2 * nlN;   // baby (ci, j) at babies + (ci nb + jj) 2 nlN
      for (size_t ci = 0; ci < C; ci++) ab[ci][j] = a + ci * nb * 2 * nlN;
      if (j == 0) {
        for (size_t ci = 0; ci < C; ci++)
          HCUDA(cudaMemsetAsync(a + ci * nb * 2 * nlN, 0, 2 * nlN * 8, c->stream));
        launch_scalar_mul(c->dc(), X, a, mq, lc.pmod, lc.pmods, 1, (int)C, 2 * nqN, nb * 2 * nlN);
        launch_scalar_mul(c->dc(), X + nqN, a + nlN, mq, lc.pmod, lc.pmods, 1, (int)C, 2 * nqN, nb * 2 * nlN);
      } else {
        need(km.n < kMaxBabies, HELRM_ERR_CAPACITY, "too many baby steps");
        const uint64_t g = galois_of_rot(c, j);
        km.rot[km.n] = rot_of_galois(c, g);
        km.key[km.n] = key_for(rk, g);
        km.out[km.n] = a;
        km.max_rot = std::max(km.max_rot, km.rot[km.n]);
        km.n++;
      }
    }
    if (km.n) launch_kip_multi(c->dc(), km, mqp);
  }
  for (size_t ci = 0; !same_babies && !pl->compact && ci < C; ci++) {
    const uint64_t* c0 = X + ci * 2 * nqN;
    uint64_t* Dc = D.p + ci * Qc * dn * nlN;
    modup_batch(c, c0 + nqN, xs, Qc, l, Dc, nullptr, false);
    KipMulti km{};
    km.own = c0 + nqN;
    km.ownq = xs;
    km.alpha = (int)P.alpha;
    km.digits = Dc;
    km.digit_stride = nlN;
    km.dnum = (int)dn;
    km.c0 = c0;
    km.p_mod = lc.pmod;
    km.level = l;
    km.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
    km.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
    km.out_half = nlN;
    km.nq = Qc;
    km.qk = std::min(Qc, 4);
    km.dq = dn * nlN;
    km.cq = xs;
    km.oq = 2 * nlN;
    for (int j : pl->babies[ci]) {
      uint64_t* a = babies.p + bi++ * Qc * 2 * nlN;
      if (j == 0) {  // (P c0, P c1): Q limbs scaled by [P]_q, P limbs 0
        HCUDA(cudaMemsetAsync(a, 0, (size_t)Qc * 2 * nlN * 8, c->stream));
        launch_scalar_mul(c->dc(), c0, a, mq, lc.pmod, lc.pmods, 1, Qc, xs, 2 * nlN);   // baby pairs are in D-form
        launch_scalar_mul(c->dc(), c0 + nqN, a + nlN, mq, lc.pmod, lc.pmods, 1, Qc, xs, 2 * nlN);
      } else {
        need(km.n < kMaxBabies, HELRM_ERR_CAPACITY, "too many baby steps");
        const uint64_t g = galois_of_rot(c, j);
        km.rot[km.n] = rot_of_galois(c, g);
        km.key[km.n] = key_for(rk, g);
        km.out[km.n] = a;
        km.max_rot = std::max(km.max_rot, km.rot[km.n]);
        km.n++;
      }
      ab[ci][j] = a;
    }
    if (km.n) launch_kip_multi(c->dc(), km, mqp);
  }
  nv12.reset();
  NvtxRange nv34("helrm L3-L4 inner sums + giant steps");
  // L3 + L4, pipelined over the MAC groups (packs of kGiantPack giants):
  //   context stream: the inner sums (A, B) of a chunk of groups (HBM-bound)
  //   s_ntt:          ModDown(B) + ModUp(B') of the previous one (FP64-bound, hoist #2)
  //   s_kip:          phi(A) + KS(B') into O                     (HBM-bound)
  // Every (A, B) pair and digit set has its own buffer, so the three streams
  // only meet at the events; O is only touched by s_kip.  Pair z of query q
  // lives at AB + (z Qc + q) 2 nlN, so a run of pairs is one strided batch.
  const MacList ml = build_macs(pl, nlN, [&](int ci, int j) {
    if (pl->compact) return std::make_pair((const uint64_t*)nullptr, (const uint64_t*)nullptr);   // unused
    uint64_t* a = ab[ci].at(j);
    return std::make_pair((const uint64_t*)a, (const uint64_t*)(a + nlN));
  }, z_lo, z_hi);
  const int n_out = (int)ml.oi.size();
  if (n_out == 0) return;
  const size_t zq = (size_t)Qc;   // pairs per z
  DBuf AB(c, (size_t)n_out * zq * 2 * nlN), Bp(c, (size_t)n_out * zq * nqN), D2(c, (size_t)n_out * zq * dn * nlN);
  if (pl->compact) {
    HCUDA(cudaMemsetAsync(AB.p, 0, (size_t)n_out * zq * 2 * nlN * 8, c->stream));
    compact_l1_l3(c, pl, rk, X, ml.oi, AB.p);
  }
  const MacDev md(c, pl->compact ? MacList{} : ml, pinned);
  // (serialised while the per-kernel profiler is on, so each kernel's events time it alone)
  // default: on for batched chunks (measured 158 vs 148 lookups/s at batch 64), off for batch 1
  // (7.16 vs 7.22 ms); HELRM_PIPE overrides
  static const int pipe_env = getenv("HELRM_PIPE") ? atoi(getenv("HELRM_PIPE")) : -1;
  static const bool trace_pipe = getenv("HELRM_TRACE_PIPE") && atoi(getenv("HELRM_TRACE_PIPE")) != 0;
  const bool pipe = (pipe_env < 0 ? Qc > 1 : pipe_env != 0) && (!c->prof.on || trace_pipe);
  cudaStream_t sn = pipe ? c->s_ntt : c->stream, sk = pipe ? c->s_kip : c->stream, sm = pipe ? c->s_mac : c->stream;
  const int pers = pipe ? c->persist : 0;
  if (pipe) {
    c->join(sn, c->stream);
    c->join(sk, c->stream);   // O zeroed, babies ready
    c->join(sm, c->stream);
  }
  const LimbMap m2 = map_twice(mqp);
  auto Oq = [&](int z) { return Oall + (size_t)ml.oi[z].first * zq * 2 * nlN; };
  auto zero_giant = [&](int z) {   // O_o += (A, B)_z for every query
    for (int q = 0; q < Qc; q++)
      launch_binary(c->dc(sk), 0, Oq(z) + (size_t)q * 2 * nlN, AB.p + ((size_t)z * zq + q) * 2 * nlN,
                    Oq(z) + (size_t)q * 2 * nlN, m2);
  };
  static const int mac_ch = getenv("HELRM_MACCH") ? atoi(getenv("HELRM_MACCH")) : 4;   // MAC groups per launch
  static const int ntt_env = getenv("HELRM_NTTCH") ? atoi(getenv("HELRM_NTTCH")) : 0;
  const int ntt_ch = ntt_env > 0 ? ntt_env : (Qc > 1 ? 8 : 16);   // giants per ModDown/ModUp batch
  // Output blocks that repeat block 0's work list with the baby pairs of their own input ct
  // (LLM layout L2: the 4 blocks share all 1279 plaintexts) run as one MAC launch in which
  // the blocks take the query role, so each plaintext value is loaded once per 2 blocks.
  size_t g_blk = ml.groups.size();
  bool periodic = !pl->compact && same_babies && pl->O == (int64_t)C && pl->O > 1 && ml.groups.size() % pl->O == 0;
  if (periodic) {
    g_blk = ml.groups.size() / pl->O;
    const size_t ts = ml.term_size, nbb = pl->babies[0].size();
    const int zb = ml.groups[g_blk].z;
    for (int64_t o = 1; periodic && o < pl->O; o++)
      for (size_t g = 0; periodic && g < g_blk; g++) {
        const int4 a = ml.groups[g], b = ml.groups[o * g_blk + g];
        periodic = b.y == a.y && b.w == a.w && b.z == a.z + (int)o * zb;
        for (int t = 0; periodic && t < a.y; t++) {
          const MacTerm* ta = reinterpret_cast<const MacTerm*>(&ml.terms[(size_t)(a.x + t) * ts]);
          const MacTerm* tb = reinterpret_cast<const MacTerm*>(&ml.terms[(size_t)(b.x + t) * ts]);
          periodic = tb->x0 == ta->x0 + o * nbb * 2 * nlN && tb->x1 == ta->x1 + o * nbb * 2 * nlN;
          for (int u = 0; periodic && u < kGiantPack; u++) periodic = tb->u[u] == ta->u[u];
        }
      }
    for (int z = 0; periodic && z < zb; z++)
      for (int64_t o = 1; periodic && o < pl->O; o++)
        periodic = pl->giants[o][ml.oi[z + o * zb].second] == pl->giants[0][ml.oi[z].second];
    if (periodic)
      run_macs(c, ml, md, 0, g_blk, AB.p, zq * 2 * nlN, mqp, true, (int)pl->O, nbb * 2 * nlN, (size_t)zb * 2 * nlN,
               sm, pers);
  }
  if (periodic) {
    // giant steps of every block, then one key switch per giant with the blocks as queries
    const int zb = ml.groups[g_blk].z;
    if (pipe) c->join(sn, sm);
    std::vector<int> rot;
    for (int z = 0; z < n_out; z++)
      if (pl->giants[ml.oi[z].first][ml.oi[z].second] % (int64_t)P.n != 0) rot.push_back(z);
    for (size_t r0 = 0; r0 < rot.size();) {
      size_t r1 = r0 + 1;
      while (r1 < rot.size() && rot[r1] == rot[r1 - 1] + 1 && (int)(r1 - r0) < ntt_ch) r1++;
      const size_t za = rot[r0], G = r1 - r0;
      moddown_batch(c, AB.p + za * 2 * nlN + nlN, 2 * nlN, (int)G, l, Bp.p + za * nqN, nqN, sn);
      modup_batch(c, Bp.p + za * nqN, nqN, (int)G, l, D2.p + za * dn * nlN, sn, false);
      r0 = r1;
    }
    if (pipe) c->join(sk, sn);
    if (pipe) c->join(sk, sm);
    // runs of giants accumulated in registers, the blocks sharing every key value (KipGiants
    // with nq = O): the output blocks are read and written once per run instead of per giant
    static const bool kgrun_p = getenv("HELRM_KIP_RUN") ? atoi(getenv("HELRM_KIP_RUN")) != 0 : true;
    const bool runs = kgrun_p && (pl->O == 1 || pl->O == 2 || pl->O == 4);
    KipGiants kg{};
    auto flush = [&]() {
      if (kg.n == 0) return;
      kg.digit_stride = nlN;
      kg.dnum = (int)dn;
      kg.add_rows = (int)nl;
      kg.alpha = (int)P.alpha;
      kg.level = (int)l;
      kg.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
      kg.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
      kg.out0 = Oall;
      kg.out1 = Oall + nlN;
      kg.nq = (int)pl->O;
      kg.dq = (size_t)zb * dn * nlN;
      kg.ownq = (size_t)zb * nqN;
      kg.aq = (size_t)zb * 2 * nlN;
      kg.oq = 2 * nlN;
      launch_kip_giants(c->dc(sk), kg, mqp);
      kg.n = 0;
    };
    for (int z = 0; z < zb; z++) {
      const int64_t gi = pl->giants[0][ml.oi[z].second];
      if (gi % (int64_t)P.n == 0) {
        for (int64_t o = 0; o < pl->O; o++) zero_giant(z + (int)o * zb);
        continue;
      }
      if (runs) {
        const uint64_t g = galois_of_rot(c, gi);
        kg.digits[kg.n] = D2.p + (size_t)z * dn * nlN;
        kg.own[kg.n] = Bp.p + (size_t)z * nqN;
        kg.key[kg.n] = key_for(rk, g);
        kg.add0[kg.n] = AB.p + (size_t)z * 2 * nlN;
        kg.rot[kg.n] = rot_of_galois(c, g);
        if (++kg.n == kMaxGiantRun) flush();
        continue;
      }
      KipArgs a{};
      a.digits = D2.p + (size_t)z * dn * nlN;
      a.digit_stride = nlN;
      a.dnum = (int)dn;
      a.key = key_for(rk, galois_of_rot(c, gi));
      a.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
      a.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
      a.add0 = AB.p + (size_t)z * 2 * nlN;
      a.add_rows = (int)nl;
      a.rot = rot_of_galois(c, galois_of_rot(c, gi));
      a.out0 = Oall;
      a.out1 = Oall + nlN;
      a.accumulate = 1;
      a.nq = (int)pl->O;
      a.dq = (size_t)zb * dn * nlN;
      a.aq = (size_t)zb * 2 * nlN;
      a.oq = 2 * nlN;
      a.own = Bp.p + (size_t)z * nqN;
      a.ownq = (size_t)zb * nqN;
      a.alpha = (int)P.alpha;
      a.level = (int)l;
      launch_kip(c->dc(sk, pers), a, mqp);
    }
    flush();
  }
  for (size_t gp = 0; !periodic && gp < ml.groups.size(); gp += mac_ch) {
    const size_t gq = std::min(ml.groups.size(), gp + (size_t)mac_ch);
    const int z0 = ml.groups[gp].z, z1 = ml.groups[gq - 1].z + ml.groups[gq - 1].w;
    if (!periodic && !pl->compact)
      run_macs(c, ml, md, gp, gq, AB.p, zq * 2 * nlN, mqp, true, Qc, 2 * nlN, 2 * nlN, sm, pers);
    if (pipe) c->join(sn, sm);
    std::vector<int> rot;   // rotating pairs of the chunk (zero giants need no key switch)
    for (int z = z0; z < z1; z++)
      if (pl->giants[ml.oi[z].first][ml.oi[z].second] % (int64_t)P.n != 0) rot.push_back(z);
    int zdone = z0;   // pairs [z0, zdone) handed to s_kip
    for (size_t r0 = 0; r0 < rot.size();) {   // runs of consecutive rotating pairs, at most ntt_ch long
      size_t r1 = r0 + 1;
      while (r1 < rot.size() && rot[r1] == rot[r1 - 1] + 1 && (int)(r1 - r0) < ntt_ch) r1++;
      const size_t za = rot[r0], G = (r1 - r0) * zq;
      moddown_batch(c, AB.p + za * zq * 2 * nlN + nlN, 2 * nlN, (int)G, l, Bp.p + za * zq * nqN, nqN, sn);
      modup_batch(c, Bp.p + za * zq * nqN, nqN, (int)G, l, D2.p + za * zq * dn * nlN, sn, false);
      if (pipe) c->join(sk, sn);
      const int zend = r1 < rot.size() ? rot[r1] : z1;
      static const bool kgrun = getenv("HELRM_KIP_RUN") ? atoi(getenv("HELRM_KIP_RUN")) != 0 : true;
      if (Qc == 1 && kgrun) {   // one accumulating key-switch pass per run of giants of an output block
        KipGiants kg{};
        auto flush = [&](int64_t o) {
          if (kg.n == 0) return;
          kg.digit_stride = nlN;
          kg.dnum = (int)dn;
          kg.add_rows = (int)nl;
          kg.alpha = (int)P.alpha;
          kg.level = (int)l;
          kg.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
          kg.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
          kg.out0 = Oall + (size_t)o * 2 * nlN;
          kg.out1 = kg.out0 + nlN;
          launch_kip_giants(c->dc(sk), kg, mqp);
          kg.n = 0;
        };
        int64_t cur_o = -1;
        for (int z = zdone; z < zend; z++) {
          const int64_t o = ml.oi[z].first, gi = pl->giants[o][ml.oi[z].second];
          if (gi % (int64_t)P.n == 0) {
            zero_giant(z);
            continue;
          }
          if (o != cur_o || kg.n == kMaxGiantRun) {
            flush(cur_o);
            cur_o = o;
          }
          const uint64_t g = galois_of_rot(c, gi);
          kg.digits[kg.n] = D2.p + (size_t)z * dn * nlN;
          kg.own[kg.n] = Bp.p + (size_t)z * nqN;
          kg.key[kg.n] = key_for(rk, g);
          kg.add0[kg.n] = AB.p + (size_t)z * 2 * nlN;
          kg.rot[kg.n] = rot_of_galois(c, g);
          kg.n++;
        }
        flush(cur_o);
        zdone = zend;
        r0 = r1;
        continue;
      }
      for (int z = zdone; z < zend; z++) {
        const int64_t gi = pl->giants[ml.oi[z].first][ml.oi[z].second];
        if (gi % (int64_t)P.n == 0) {
          zero_giant(z);
        } else {
          KipArgs a{};
          a.digits = D2.p + (size_t)z * zq * dn * nlN;
          a.digit_stride = nlN;
          a.dnum = (int)dn;
          a.key = key_for(rk, galois_of_rot(c, gi));
          a.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
          a.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
          a.add0 = AB.p + (size_t)z * zq * 2 * nlN;
          a.add_rows = (int)nl;
          a.rot = rot_of_galois(c, galois_of_rot(c, gi));
          a.out0 = Oq(z);
          a.out1 = Oq(z) + nlN;
          a.accumulate = 1;
          a.nq = Qc;
          a.dq = dn * nlN;
          a.aq = 2 * nlN;
          a.oq = 2 * nlN;
          a.own = Bp.p + (size_t)z * zq * nqN;
          a.ownq = nqN;
          a.alpha = (int)P.alpha;
          a.level = (int)l;
          launch_kip(c->dc(sk, pers), a, mqp);
        }
      }
      zdone = zend;
      r0 = r1;
    }
    if (pipe) c->join(sk, sm);
    for (int z = zdone; z < z1; z++) zero_giant(z);   // zero giants with no rotating pair after them
  }
  if (pipe) {
    c->join(c->stream, sn);
    c->join(c->stream, sk);
    c->join(c->stream, sm);
  }
}

// D21 RotSum on Qc contiguous ciphertexts S [Qc][2][l+1][N] at level l:
// ct += Rotate(ct, mbar 2^r), each rotation batched over the queries (one
// key read for all of them)
static void rot_sum_batch(helrm_ctx* c, uint64_t* S, int Qc, uint32_t l, int64_t mbar, const helrm_rotkeys* rk) {
  const Params& P = c->P;
  const int64_t n = P.n;
  if (mbar >= n) return;
  const size_t N = P.N, nq = l + 1, nqN = nq * N, nl = l + 1 + P.K, nlN = nl * N, dn = P.dnum(l);
  const LevelConst& lc = level_const(c, l);
  // (splitting every rotation into a c1 chain on the context stream and a c0 chain on a side
  // stream, the halves of each key switch separate, measured slower: 7.23 vs 6.91-7.06 ms per
  // Criteo lookup -- the digits are read twice and the ModDowns lose their 2-poly batching)
  {
    DBuf D(c, (size_t)Qc * dn * nlN), T(c, (size_t)Qc * 2 * nlN);
    for (int64_t r = mbar; r < n; r *= 2) {
      const uint64_t g = galois_of_rot(c, r);
      modup_batch(c, S + nqN, 2 * nqN, Qc, l, D.p, nullptr, false);
      KipArgs a{};
      a.own = S + nqN;
      a.ownq = 2 * nqN;
      a.alpha = (int)P.alpha;
      a.level = (int)l;
      a.digits = D.p;
      a.digit_stride = nlN;
      a.dnum = (int)dn;
      a.key = key_for(rk, g);
      a.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
      a.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
      a.add0 = S;                       // lazy rotation: P phi(c0) + KS0, KS1
      a.add_rows = (int)nq;
      a.add_mul = lc.pmod;
      a.rot = rot_of_galois(c, g);
      a.out0 = T.p;
      a.out1 = T.p + nlN;
      a.accumulate = 0;
      a.nq = Qc;
      a.dq = dn * nlN;
      a.aq = 2 * nqN;
      a.oq = 2 * nlN;
      launch_kip(c->dc(), a, P.map_qp(l));
      moddown_batch(c, T.p, nlN, 2 * Qc, l, S, nqN, nullptr, true);   // S += Rotate(S)
    }
  }
}

// D20 L6-L8 per output block for Qc queries (Oall [O][Qc][2][l+1+K][N]):
// ModDown both halves (scale Delta q_l), rescale (scale Delta), RotSum when
// mbar < n; results into S [O][Qc][2][l][N]
static void lookup_finish(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const uint64_t* Oall, int Qc,
                          uint64_t* S) {
  NvtxRange nv_("helrm L6-L8 ModDown, rescale, RotSum");
  const Params& P = c->P;
  const uint32_t l = pl->level;
  const size_t N = P.N, nq = l + 1, nlN = (size_t)(l + 1 + P.K) * N, oN = 2 * (size_t)l * N;
  for (int64_t o = 0; o < pl->O; o++) {
    DBuf r(c, (size_t)Qc * 2 * nq * N);
    uint64_t* So = S + (size_t)o * Qc * oN;
    moddown_batch(c, Oall + (size_t)o * Qc * 2 * nlN, nlN, 2 * Qc, l, r.p, nq * N);
    rescale_ct(c, r.p, l, So, Qc);
    rot_sum_batch(c, So, Qc, l - 1, pl->mbar, rk);
  }
}

// the whole double-hoisted lookup of Qc staged queries X -> S (no host
// synchronisation inside: this is what a CUDA graph captures)
static void lookup_chunk(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const uint64_t* X, int Qc,
                         uint64_t* S, void** pinned) {
  const size_t nlN = (size_t)(pl->level + 1 + c->P.K) * c->P.N;
  DBuf O(c, (size_t)pl->O * Qc * 2 * nlN);
  HCUDA(cudaMemsetAsync(O.p, 0, (size_t)pl->O * Qc * 2 * nlN * 8, c->stream));
  lookup_double_part(c, pl, rk, X, Qc, 0, INT64_MAX, O.p, pinned);
  lookup_finish(c, pl, rk, O.p, Qc, S);
}

static void stage_inputs(helrm_ctx* c, const helrm_ct* const* in, size_t n, size_t words, uint64_t* X) {
  for (size_t i = 0; i < n; i++)
    HCUDA(cudaMemcpyAsync(X + i * words, in[i]->d, words * 8, cudaMemcpyDeviceToDevice, c->stream));
}

// output ciphertexts of a chunk: out[q O + o] <- S [o][q]
static void emit_outputs(helrm_ctx* c, const helrm_plan* pl, const uint64_t* S, int Qc, double scale,
                         helrm_ct** out) {
  const size_t oN = 2 * (size_t)pl->level * c->P.N;
  for (int64_t o = 0; o < pl->O; o++)
    for (int q = 0; q < Qc; q++) {
      helrm_ct* s = new_ct(c, pl->level - 1, scale);
      HCUDA(cudaMemcpyAsync(s->d, S + ((size_t)o * Qc + q) * oN, oN * 8, cudaMemcpyDeviceToDevice, c->stream));
      out[(size_t)q * pl->O + o] = s;
    }
}

static int64_t count_pairs(const helrm_plan* pl) {
  int64_t n = 0;
  for (auto& eo : pl->entries)
    for (auto& e : eo) n += !e.empty();
  return n;
}

// graph cache entry of (plan, key set, chunk size): persistent staged inputs
// X [Qc][C][2][l+1][N] and outputs S [O][Qc][2][l][N]
static helrm_ctx::LookupGraph& graph_entry(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, int Qc,
                                           int slot = 0) {
  helrm_ctx::LookupGraph& G = c->graphs[std::make_tuple(pl->id, rk->id, Qc + 1000 * slot)];
  if (!G.X) {
    const size_t nqN = (size_t)(pl->level + 1) * c->P.N, oN = 2 * (size_t)pl->level * c->P.N;
    G.X = (uint64_t*)c->dalloc((size_t)Qc * pl->C * 2 * nqN * 8);
    G.S = (uint64_t*)c->dalloc((size_t)pl->O * Qc * oN * 8);
    // MAC work list bound: every term carries >= 1 plaintext, every group >= 1 pair
    size_t nbb = 0;
    for (auto& b : pl->babies) nbb = std::max(nbb, b.size());
    HCUDA(cudaMallocHost(&G.pinned, (size_t)pl->n_diag * sizeof(MacTermW) + count_pairs(pl) * sizeof(int4) +
                                        (size_t)count_pairs(pl) * nbb * 8 + 64));
  }
  return G;
}

// G.X -> G.S on the context stream: eagerly on the first use (creates every
// cached constant), captured into a CUDA graph on the second, replayed after
// G.X -> G.S through body(pinned) on the context stream: eagerly on the first
// use (creates every cached constant), captured into a CUDA graph on the
// second, replayed after.  body enqueues on c->stream only (side streams are
// forked from and joined back to it); pinned != null during the capture (host
// work lists are staged there, so the graph re-uploads them from pinned memory).
}  // extern "C" (template below)
template <class F>
static void run_graph(helrm_ctx* c, helrm_ctx::LookupGraph& G, F body) {
  if (G.exec) {
    HCUDA(cudaGraphLaunch(G.exec, c->stream));
    c->launches += G.launches;
  } else if (G.uses == 0 || G.failed) {
    body((void**)nullptr);
  } else {
    // capture on the private stream (the context stream may be the legacy
    // default stream, which cannot be captured), ordered after the staging
    cudaGraph_t graph = nullptr;
    cudaStream_t user = c->stream;
    c->join(c->s_cap, user);
    c->stream = c->s_cap;
    const uint64_t l0 = c->launches;
    cudaError_t e = cudaStreamBeginCapture(c->s_cap, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      try {
        body(&G.pinned);
      } catch (...) {
        cudaStreamEndCapture(c->s_cap, &graph);
        if (graph) cudaGraphDestroy(graph);
        graph = nullptr;
        cudaGetLastError();
        e = cudaErrorStreamCaptureInvalidated;
      }
    }
    if (e == cudaSuccess) e = cudaStreamEndCapture(c->s_cap, &graph);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&G.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    if (graph) cudaGraphDestroy(graph);
    c->stream = user;
    if (e != cudaSuccess) {   // not capturable here: run eagerly from now on
      cudaGetLastError();
      G.exec = nullptr;
      G.failed = true;
      c->launches = l0;
      body((void**)nullptr);
    } else {
      G.launches = c->launches - l0;
      HCUDA(cudaGraphLaunch(G.exec, c->stream));
    }
  }
  G.uses++;
}

extern "C" {

static void run_graph_chunk(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, helrm_ctx::LookupGraph& G,
                            int Qc) {
  run_graph(c, G, [&](void** pinned) { lookup_chunk(c, pl, rk, G.X, Qc, G.S, pinned); });
}

// device words one query of a batched double-hoisted lookup keeps live
static size_t query_words(helrm_ctx* c, const helrm_plan* pl) {
  const Params& P = c->P;
  const size_t l = pl->level, N = P.N, nq = l + 1, nl = l + 1 + P.K, dn = P.dnum(l);
  size_t nb = 0, pairs = (size_t)count_pairs(pl);
  for (auto& b : pl->babies) nb += b.size();
  return N * (pl->C * (2 * nq + dn * nl) + nb * 2 * nl + pairs * (2 * nl + nq + dn * nl) + pl->O * 2 * nl +
              pl->O * 4 * nq);
}

// D20: the double-hoisted BSGS lookup of `batch` queries (C input cts -> O
// outputs each), in chunks of queries that share every key and plaintext
// read.  Chunks of <= 2 queries replay a captured CUDA graph from the second
// call on (the first call runs eagerly and creates every cached constant).
static void lookup_double(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const helrm_ct* const* in,
                          size_t batch, helrm_ct** out) {
  const Params& P = c->P;
  const size_t nqN = (size_t)(pl->level + 1) * P.N, oN = 2 * (size_t)pl->level * P.N;
  size_t qc = 1;
  if (batch > 1) {
    size_t fr = 0, tot = 0;
    HCUDA(cudaMemGetInfo(&fr, &tot));
    const size_t budget = std::min<size_t>(fr / 2, (size_t)48 << 30);
    qc = std::max<size_t>(1, std::min(batch, budget / (8 * query_words(c, pl))));
    if (getenv("HELRM_QCHUNK")) qc = std::max(1, atoi(getenv("HELRM_QCHUNK")));
    qc = std::min(qc, batch);
  }
  if (pl->compact) qc = 1;   // compact plans: one query at a time, eagerly (chunked host work lists)
  static const bool graphs = getenv("HELRM_GRAPH") ? atoi(getenv("HELRM_GRAPH")) != 0 : true;
  for (size_t q0 = 0; q0 < batch; q0 += qc) {
    const int Qc = (int)std::min(qc, batch - q0);
    const size_t nin = (size_t)Qc * pl->C;
    const double scale = in[q0 * pl->C]->scale;
    if (!graphs || c->prof.on || Qc > 2 || pl->compact) {
      DBuf X(c, nin * 2 * nqN), S(c, (size_t)pl->O * Qc * oN);
      stage_inputs(c, in + q0 * pl->C, nin, 2 * nqN, X.p);
      lookup_chunk(c, pl, rk, X.p, Qc, S.p, nullptr);
      emit_outputs(c, pl, S.p, Qc, scale, out + q0 * pl->O);
      continue;
    }
    helrm_ctx::LookupGraph& G = graph_entry(c, pl, rk, Qc);
    stage_inputs(c, in + q0 * pl->C, nin, 2 * nqN, G.X);
    run_graph_chunk(c, pl, rk, G, Qc);
    emit_outputs(c, pl, G.S, Qc, scale, out + q0 * pl->O);
  }
}

// D22: single-hoisted cross-check mode (full rotations in Q_l)
static void lookup_single(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const helrm_ct* const* in,
                          helrm_ct** out) {
  const Params& P = c->P;
  const uint32_t l = pl->level;
  const size_t N = P.N, nq = l + 1, nqN = nq * N;
  const LimbMap mq = P.map_q(l);
  std::vector<std::map<int, helrm_ct*>> rots(pl->C);
  for (int64_t ci = 0; ci < pl->C; ci++) {
    const helrm_ct* ct = in[ci];
    DBuf D(c, (size_t)P.dnum(l) * (l + 1 + P.K) * N);
    modup_batch(c, ct_c1(ct), 0, 1, l, D.p);
    for (int j : pl->babies[ci]) {
      helrm_ct* r = new_ct(c, l, ct->scale);
      rotate_from_digits(c, ct, D.p, rk, j, r);
      rots[ci][j] = r;
    }
  }
  const MacList ml = build_macs(pl, nqN, [&](int ci, int j) {
    helrm_ct* x = rots[ci].at(j);
    return std::make_pair((const uint64_t*)ct_c0(x), (const uint64_t*)ct_c1(x));
  });
  const int n_out = (int)ml.oi.size();
  DBuf ABbuf(c, (size_t)n_out * 2 * nqN);
  run_macs_all(c, ml, ABbuf.p, 2 * nqN, mq, false);
  std::vector<helrm_ct> AB(n_out);
  for (int z = 0; z < n_out; z++) AB[z] = helrm_ct{c, l, in[0]->scale, ABbuf.p + (size_t)z * 2 * nqN};
  helrm_ct* R = new_ct(c, l, in[0]->scale);
  for (int64_t o = 0; o < pl->O; o++) {
    helrm_ct* acc = new_ct(c, l, in[0]->scale * (double)P.primes[l]);
    HCUDA(cudaMemsetAsync(acc->d, 0, 2 * nqN * 8, c->stream));
    for (int z = 0; z < n_out; z++) {
      if (ml.oi[z].first != o) continue;
      rotate(c, &AB[z], rk, pl->giants[o][ml.oi[z].second], R);
      ct_add_inplace(c, acc, R);
    }
    helrm_ct* s = new_ct(c, l - 1, in[0]->scale);
    rescale_ct(c, acc->d, l, s->d);
    helrm_ct_destroy(acc);
    rot_sum(c, s, pl->mbar, rk);
    out[o] = s;
  }
  helrm_ct_destroy(R);
  for (auto& m : rots)
    for (auto& kv : m) helrm_ct_destroy(kv.second);
}

helrm_status helrm_lookup_host(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                               const uint64_t* const* in, double scale, size_t batch, uint64_t* const* out) {
  return guard([&] {
    need(c && p && rk && (in || batch == 0) && (out || batch == 0), HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(p->mode == HELRM_MODE_DOUBLE && !p->compact, HELRM_ERR_ARG,
         "helrm_lookup_host runs stored-diagonal double-hoisted plans");
    for (int64_t a : p->rotations) (void)key_for(rk, galois_of_rot(c, a));
    const Params& P = c->P;
    const uint32_t l = p->level;
    const size_t nqN = (size_t)(l + 1) * P.N, oN = 2 * (size_t)l * P.N, C = p->C, O = p->O;
    (void)scale;   // the lookup's arithmetic does not depend on the input scale (D20: output scale Delta)
    // Two serving slots: query q runs on slot q & 1 (its own graph, buffers, NTT scratch and
    // stream), so one query's latency-bound tail (final ModDown, rescale, RotSum chain) overlaps
    // the next query's HBM-bound baby steps and inner sums.
    static const int nslot = std::max(1, std::min(3, getenv("HELRM_SLOTS") ? atoi(getenv("HELRM_SLOTS")) : 2));
    helrm_ctx::LookupGraph* Gs[3] = {};
    for (int k = 0; k < nslot; k++) {
      Gs[k] = &graph_entry(c, p, rk, 1, k);
      if (k > 0 && !Gs[k]->scratch) Gs[k]->scratch = (uint64_t*)c->dalloc(ntt_scratch_words(P.log_n) * 8);
    }
    cudaStream_t user = c->stream;
    uint64_t* base_scratch = c->scratch;
    cudaStream_t ss[3] = {user, c->s_mac, c->s_kip};
    uint64_t* scr[3] = {base_scratch, Gs[1] ? Gs[1]->scratch : nullptr, Gs[2] ? Gs[2]->scratch : nullptr};
    // per-slot device staging: H[s] inputs (coefficient form), D[s] outputs
    std::vector<std::unique_ptr<DBuf>> HB, DB;
    uint64_t* H[3] = {};
    uint64_t* D[3] = {};
    for (int k = 0; k < nslot; k++) {
      HB.emplace_back(new DBuf(c, C * 2 * nqN));
      DB.emplace_back(new DBuf(c, O * oN));
      H[k] = HB.back()->p;
      D[k] = DB.back()->p;
    }
    if (!c->hev[0])
      for (auto& e : c->hev) HCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t* h2d = c->hev;       // 3 each
    cudaEvent_t* used = c->hev + 3;
    cudaEvent_t* exp_ = c->hev + 6;
    cudaEvent_t* d2h = c->hev + 9;
    c->join(c->s_h2d, user);   // staging buffers allocated on the context stream
    for (int k = 1; k < nslot; k++) c->join(ss[k], user);
    struct Restore {
      helrm_ctx* c;
      cudaStream_t st;
      uint64_t* sc;
      ~Restore() {
        c->stream = st;
        c->scratch = sc;
      }
    } restore{c, user, base_scratch};
    for (size_t q = 0; q < batch; q++) {
      const int b = (int)(q % nslot);
      helrm_ctx::LookupGraph& G = *Gs[b];
      if (q >= (size_t)nslot) HCUDA(cudaStreamWaitEvent(c->s_h2d, used[b], 0));
      for (size_t ci = 0; ci < C; ci++)
        HCUDA(cudaMemcpyAsync(H[b] + ci * 2 * nqN, in[q * C + ci], 2 * nqN * 8, cudaMemcpyHostToDevice, c->s_h2d));
      HCUDA(cudaEventRecord(h2d[b], c->s_h2d));
      c->stream = ss[b];
      c->scratch = scr[b];
      HCUDA(cudaStreamWaitEvent(c->stream, h2d[b], 0));
      ntt_fwd(c, H[b], G.X, 2 * C * (l + 1), P.map_q(l));   // coefficient -> NTT form, into the graph's inputs
      HCUDA(cudaEventRecord(used[b], c->stream));
      run_graph_chunk(c, p, rk, G, 1);
      if (q >= (size_t)nslot) HCUDA(cudaStreamWaitEvent(c->stream, d2h[b], 0));
      ntt_inv(c, G.S, D[b], 2 * O * l, P.map_q(l - 1));    // outputs back to coefficient form
      HCUDA(cudaEventRecord(exp_[b], c->stream));
      HCUDA(cudaStreamWaitEvent(c->s_d2h, exp_[b], 0));
      for (size_t o = 0; o < O; o++)
        HCUDA(cudaMemcpyAsync(out[q * O + o], D[b] + o * oN, oN * 8, cudaMemcpyDeviceToHost, c->s_d2h));
      HCUDA(cudaEventRecord(d2h[b], c->s_d2h));
      c->stream = user;
      c->scratch = base_scratch;
    }
    for (int k = 1; k < nslot; k++) c->join(user, ss[k]);
    c->join(c->stream, c->s_d2h);
    c->join(c->stream, c->s_h2d);
    HCUDA(cudaStreamSynchronize(c->stream));
  });
}

helrm_status helrm_lookup(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk, const helrm_ct* const* in,
                          size_t batch, helrm_ct** out) {
  if (out)
    for (size_t i = 0; i < batch * (p ? p->O : 0); i++) out[i] = nullptr;
  return guard([&] {
    need(c && p && rk && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    for (int64_t a : p->rotations) (void)key_for(rk, galois_of_rot(c, a));
    for (size_t q = 0; q < batch; q++) {
      c->evnext = 0;
      for (int64_t ci = 0; ci < p->C; ci++) {
        need(in[q * p->C + ci] != nullptr, HELRM_ERR_ARG, "null input ciphertext");
        need(in[q * p->C + ci]->level == p->level, HELRM_ERR_LEVEL, "input level differs from the plan's level");
      }
      if (p->mode != HELRM_MODE_DOUBLE) lookup_single(c, p, rk, in + q * p->C, out + q * p->O);
    }
    if (p->mode == HELRM_MODE_DOUBLE) {
      HostTimer ht_("helrm_lookup(total)");
      lookup_double(c, p, rk, in, batch, out);
    }
    hostprof_dump("helrm_lookup");
  });
}

// ---------------------------------------------------------------------------
// primitives
// ---------------------------------------------------------------------------
helrm_status helrm_ntt_fwd(helrm_ctx* c, uint64_t* dev, uint32_t first, uint32_t n_limbs, size_t n_polys) {
  return guard([&] {
    need(c && dev, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(first + n_limbs <= c->P.primes.size() && n_limbs >= 1, HELRM_ERR_ARG, "prime range outside the chain");
    ntt_fwd(c, dev, dev, (size_t)n_limbs * n_polys, c->P.map_range(first, n_limbs));
  });
}

helrm_status helrm_ntt_inv(helrm_ctx* c, uint64_t* dev, uint32_t first, uint32_t n_limbs, size_t n_polys) {
  return guard([&] {
    need(c && dev, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(first + n_limbs <= c->P.primes.size() && n_limbs >= 1, HELRM_ERR_ARG, "prime range outside the chain");
    ntt_inv(c, dev, dev, (size_t)n_limbs * n_polys, c->P.map_range(first, n_limbs));
  });
}

helrm_status helrm_modup(helrm_ctx* c, const uint64_t* in, uint32_t level, uint32_t digit, uint64_t* out) {
  return guard([&] {
    need(c && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(level <= c->P.L && digit < c->P.dnum(level), HELRM_ERR_LEVEL, "bad level/digit");
    modup(c, in, level, (int)digit, out);
  });
}

helrm_status helrm_moddown(helrm_ctx* c, const uint64_t* in, uint32_t level, uint64_t* out) {
  return guard([&] {
    need(c && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(level <= c->P.L, HELRM_ERR_LEVEL, "bad level");
    moddown(c, in, level, out);
  });
}

helrm_status helrm_rescale(helrm_ctx* c, const helrm_ct* in, helrm_ct** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(in->level >= 1, HELRM_ERR_LEVEL, "rescale at level 0");
    helrm_ct* r = new_ct(c, in->level - 1, in->scale / (double)c->P.primes[in->level]);
    rescale_ct(c, in->d, in->level, r->d);
    *out = r;
  });
}

helrm_status helrm_rotate(helrm_ctx* c, const helrm_rotkeys* rk, const helrm_ct* in, int64_t k, helrm_ct** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && rk && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    helrm_ct* r = new_ct(c, in->level, in->scale);
    rotate(c, in, rk, k, r);
    *out = r;
  });
}

helrm_status helrm_rotate_hoisted(helrm_ctx* c, const helrm_rotkeys* rk, const helrm_ct* in, const int64_t* amounts,
                                  size_t n_amounts, helrm_ct* const* ring, size_t n_ring) {
  return guard([&] {
    need(c && rk && in && amounts && ring && n_ring > 0, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    const uint32_t l = in->level;
    for (size_t i = 0; i < n_ring; i++) need(ring[i] && ring[i]->level == l, HELRM_ERR_LEVEL, "ring ct level");
    DBuf D(c, (size_t)c->P.dnum(l) * (l + 1 + c->P.K) * c->P.N);
    modup_batch(c, ct_c1(in), 0, 1, l, D.p);
    for (size_t i = 0; i < n_amounts; i++) rotate_from_digits(c, in, D.p, rk, amounts[i], ring[i % n_ring]);
  });
}

// SURVEY.md 8(d) "hoisted rotation, keys amortised": ModUp of every input ct
// once (hoist), then per amount ONE key switch over all cts (k_kip with the
// cts as queries: each key value is loaded once for all of them, lazy
// P phi(c0) added) and one ModDown batched over the 2 n polynomials, written
// straight into the caller's device ring: (amount i, ct j) ->
// out + ((i n + j) % ring) 2 (l+1) N, NTT slot order.
helrm_status helrm_rotate_hoisted_batch(helrm_ctx* c, const helrm_rotkeys* rk, const helrm_ct* const* in, size_t n,
                                        const int64_t* amounts, size_t n_amounts, uint64_t* out, size_t ring) {
  return guard([&] {
    need(c && rk && in && amounts && out && n > 0 && ring > 0 && ring % n == 0, HELRM_ERR_ARG,
         "bad argument (ring must be a multiple of the number of cts)");
    DevGuard dg_(c->device);
    const Params& P = c->P;
    const uint32_t l = in[0]->level;
    for (size_t j = 0; j < n; j++) need(in[j] && in[j]->level == l, HELRM_ERR_LEVEL, "input cts at different levels");
    const size_t N = P.N, nq = l + 1, nqN = nq * N, nl = l + 1 + P.K, nlN = nl * N, dn = P.dnum(l);
    const LevelConst& lc = level_const(c, l);
    DBuf X(c, n * 2 * nqN), D(c, n * dn * nlN), T(c, n * 2 * nlN);
    stage_inputs(c, in, n, 2 * nqN, X.p);
    modup_batch(c, X.p + nqN, 2 * nqN, (int)n, l, D.p, nullptr, false);   // hoisted: once per ct
    for (size_t i = 0; i < n_amounts; i++) {
      uint64_t* o = out + ((i * n) % ring) * 2 * nqN;
      const uint64_t g = galois_of_rot(c, amounts[i]);
      if (g == 1) {   // Rotate(ct, 0) = ct
        HCUDA(cudaMemcpyAsync(o, X.p, n * 2 * nqN * 8, cudaMemcpyDeviceToDevice, c->stream));
        continue;
      }
      KipArgs a{};
      a.digits = D.p;
      a.digit_stride = nlN;
      a.dnum = (int)dn;
      a.key = key_for(rk, g);
      a.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
      a.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
      a.add0 = X.p;                     // lazy rotation: P phi(c0) + KS0, KS1
      a.add_rows = (int)nq;
      a.add_mul = lc.pmod;
      a.rot = rot_of_galois(c, g);
      a.out0 = T.p;
      a.out1 = T.p + nlN;
      a.nq = (int)n;
      a.dq = dn * nlN;
      a.aq = 2 * nqN;
      a.oq = 2 * nlN;
      a.own = X.p + nqN;
      a.ownq = 2 * nqN;
      a.alpha = (int)P.alpha;
      a.level = (int)l;
      launch_kip(c->dc(), a, P.map_qp(l));
      moddown_batch(c, T.p, nlN, (int)(2 * n), l, o, nqN);
    }
  });
}

helrm_status helrm_ct_random(helrm_ctx* c, uint64_t seed, uint32_t ct_index, uint32_t level, helrm_ct** out) {
  if (out) *out = nullptr;
  return guard([&] {
    need(c && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(level <= c->P.L, HELRM_ERR_LEVEL, "level above L");
    helrm_ct* ct = new_ct(c, level, std::ldexp(1.0, c->P.log_scale));
    LimbMap m = c->P.map_q(level);
    for (int poly = 0; poly < 2; poly++)
      launch_sample_uniform_ntt(c->dc(), ct->d + (size_t)poly * (level + 1) * c->P.N, m, seed, 9, ct_index, poly, m);
    *out = ct;
  });
}

// ---------------------------------------------------------------------------
// multi-GPU (D23): giant-range partition + uint64 all-reduce
// ---------------------------------------------------------------------------
helrm_status helrm_dist_range(int64_t n_items, int world, int rank, int64_t* lo, int64_t* hi) {
  return guard([&] {
    need(lo && hi && world >= 1 && rank >= 0 && rank < world && n_items >= 0, HELRM_ERR_ARG, "bad argument");
    // contiguous, as even as possible: the first (n mod world) ranks get one more
    const int64_t q = n_items / world, r = n_items % world;
    *lo = rank * q + std::min<int64_t>(rank, r);
    *hi = *lo + q + (rank < r ? 1 : 0);
  });
}

helrm_status helrm_comm_unique_id(uint8_t* id) {
  return guard([&] {
    need(id, HELRM_ERR_ARG, "null argument");
    ncclUniqueId u;
    HNCCL(nccl().getUniqueId(&u));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
  });
}

helrm_status helrm_comm_init(helrm_ctx* c, const uint8_t* id, int rank, int world) {
  return guard([&] {
    need(c && id && world >= 1 && rank >= 0 && rank < world, HELRM_ERR_ARG, "bad argument");
    DevGuard dg_(c->device);
    HCUDA(cudaSetDevice(c->device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (c->comm) nccl().commDestroy(c->comm);
    c->comm = nullptr;
    HNCCL(nccl().commInitRank(&c->comm, world, u, rank));
    c->rank = rank;
    c->world = world;
  });
}

// the communicator's asynchronous error state (a peer failure, a network error)
static void nccl_check_async(helrm_ctx* c) {
  if (!c->comm) return;
  ncclResult_t r = ncclSuccess;
  HNCCL(nccl().commGetAsyncError(c->comm, &r));
  if (r != ncclSuccess && r != ncclInProgress)
    throw Error(HELRM_ERR_NCCL, std::string("NCCL asynchronous error: ") + nccl().getErrorString(r));
}

// D20 with the giant pairs split over `parts` partitions: partition r
// computes the partial Q_l P accumulators of its giant range
// (helrm_dist_range), the partials are summed as uint64 words without
// reduction (what ncclAllReduce(ncclUint64, ncclSum) does), k_modred reduces
// them, and L6-L8 finish.  world > 1: this rank's partition, NCCL combine;
// virt > 0: all `virt` partitions in this process, one after another on the
// context stream, summed by a device kernel (the emulation of the collective
// on one GPU: nothing waits on another rank).
static void lookup_split(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk, const helrm_ct* const* in,
                         size_t batch, helrm_ct** out, int virt) {
  need(p->mode == HELRM_MODE_DOUBLE, HELRM_ERR_ARG, "the distributed lookup runs the double-hoisted mode");
  for (int64_t a : p->rotations) (void)key_for(rk, galois_of_rot(c, a));
  const Params& P = c->P;
  const size_t nlN = (size_t)(p->level + 1 + P.K) * P.N, nqN = (size_t)(p->level + 1) * P.N;
  const size_t owords = (size_t)p->O * 2 * nlN;
  const int parts = virt > 0 ? virt : c->world;
  // graph entry of (plan, key set, split): staged inputs X, outputs S, one pinned MAC-list region per part
  helrm_ctx::LookupGraph& G = c->graphs[std::make_tuple(p->id, rk->id, 300000 + parts * 10 + (virt > 0 ? 1 : 0))];
  size_t nbb = 0;
  for (auto& b : p->babies) nbb = std::max(nbb, b.size());
  const size_t per_part = (size_t)p->n_diag * sizeof(MacTermW) + count_pairs(p) * sizeof(int4) +
                          (size_t)count_pairs(p) * nbb * 8 + 64;
  if (!G.X) {
    G.X = (uint64_t*)c->dalloc((size_t)p->C * 2 * nqN * 8);
    G.S = (uint64_t*)c->dalloc((size_t)p->O * 2 * p->level * P.N * 8);
    HCUDA(cudaMallocHost(&G.pinned, per_part * parts));
  }
  auto body = [&](void** pinned) {
    DBuf O(c, owords);
    HCUDA(cudaMemsetAsync(O.p, 0, owords * 8, c->stream));
    if (virt > 0) {
      DBuf part(c, owords);
      for (int r = 0; r < virt; r++) {
        int64_t lo = 0, hi = 0;
        (void)helrm_dist_range(count_pairs(p), virt, r, &lo, &hi);
        HCUDA(cudaMemsetAsync(part.p, 0, owords * 8, c->stream));
        void* pr = pinned ? (char*)*pinned + (size_t)r * per_part : nullptr;
        lookup_double_part(c, p, rk, G.X, 1, lo, hi, part.p, pinned ? &pr : nullptr);
        launch_add_u64(c->dc(), O.p, part.p, owords);   // the all-reduce's exact uint64 sum
      }
    } else {
      int64_t lo = 0, hi = INT64_MAX;
      (void)helrm_dist_range(count_pairs(p), c->world, c->rank, &lo, &hi);
      lookup_double_part(c, p, rk, G.X, 1, lo, hi, O.p, pinned);
      if (c->world > 1) HNCCL(nccl().allReduce(O.p, O.p, owords, ncclUint64, ncclSum, c->comm, c->stream));
    }
    // L5: each partial word is < q, so the sum is < parts q < 2^64 (parts < 2^13); reduce mod q
    if (parts > 1)
      for (int64_t h = 0; h < 2 * p->O; h++) launch_modred(c->dc(), O.p + (size_t)h * nlN, P.map_qp(p->level));
    lookup_finish(c, p, rk, O.p, 1, G.S);
  };
  static const bool graphs = getenv("HELRM_GRAPH") ? atoi(getenv("HELRM_GRAPH")) != 0 : true;
  for (size_t q = 0; q < batch; q++) {
    const helrm_ct* const* cin = in + q * p->C;
    for (int64_t ci = 0; ci < p->C; ci++) {
      need(cin[ci] != nullptr && cin[ci]->level == p->level, HELRM_ERR_LEVEL, "input level differs from the plan's");
      if (virt == 0 && c->world > 1)   // the query lives on rank 0: broadcast it into every rank's staging buffer
        HNCCL(nccl().broadcast(cin[ci]->d, G.X + ci * 2 * nqN, 2 * nqN, ncclUint64, 0, c->comm, c->stream));
      else
        HCUDA(cudaMemcpyAsync(G.X + ci * 2 * nqN, cin[ci]->d, 2 * nqN * 8, cudaMemcpyDeviceToDevice, c->stream));
    }
    if (graphs && !c->prof.on && !p->compact) run_graph(c, G, body);
    else body(nullptr);
    if (virt == 0 && c->world > 1) nccl_check_async(c);
    emit_outputs(c, p, G.S, 1, cin[0]->scale, out + q * p->O);
  }
}

// the batch-1 lookup with the Q_l P limbs split
// over `parts` ranks (rank r owns rows [lo_r, hi_r) of helrm_dist_range(l+1+K)),
// emulated one rank after another in this process.  What every rank does:
//   replicated (FP64): ModUp of the input c1s, each giant's ModDown + ModUp,
//     the final ModDown / rescale / RotSum;
//   own rows only (HBM): the baby key switches (k_kip_multi, row slice), the
//     inner sums (bulk MAC, row slice) and the giant key switches
//     (k_kip_giants, row slice) -- so each rank streams 1/G of the rotation
//     keys and plaintext diagonals;
//   exchange (an all-gather on a multi-GPU node): each giant pair's B rows
//     before its ModDown, and the output accumulators before the finish.
// Every rank's baby pairs, inner sums and accumulators live in private slice
// buffers [2][rows][N]; the all-gathers are explicit copies of the slices into
// full buffers.  Per-limb work is independent, so the result is bit-identical
// to helrm_lookup (D23: only the limb placement changes).
static void limbsplit_body(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const uint64_t* Xin,
                           uint64_t* Sout, int parts, bool real, int only_rank, void** pinned);

// per-rank pinned staging of the MAC work lists (graph capture of the limb split)
static size_t limbsplit_pinned_per_rank(const helrm_plan* pl) {
  return (size_t)pl->n_diag * sizeof(MacTerm) + (size_t)count_pairs(pl) * sizeof(int4) + 256;
}

static void lookup_limbsplit(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const helrm_ct* const* in,
                             size_t batch, helrm_ct** out, int parts, bool real, int only_rank = -1) {
  need(pl->mode == HELRM_MODE_DOUBLE && !pl->compact, HELRM_ERR_ARG,
       "the limb-partitioned lookup runs stored-diagonal double-hoisted plans");
  for (int64_t a : pl->rotations) (void)key_for(rk, galois_of_rot(c, a));
  const Params& P = c->P;
  const uint32_t l = pl->level;
  const size_t N = P.N, nqN = (size_t)(l + 1) * N, oN = 2 * (size_t)l * N;
  const int64_t C = pl->C, O = pl->O;
  if (real) parts = c->world;
  need(parts >= 1 && (size_t)parts <= l + 1 + P.K, HELRM_ERR_ARG, "1 <= parts <= l + 1 + K");
  // one graph per (plan, key set, partition, mode): staged inputs X, outputs S
  const int mode = only_rank >= 0 ? 2 : real ? 1 : 0;
  helrm_ctx::LookupGraph& G = c->graphs[std::make_tuple(pl->id, rk->id, 100000 + parts * 1000 + mode * 100 +
                                                          std::max(0, only_rank))];
  if (!G.X) {
    G.X = (uint64_t*)c->dalloc((size_t)C * 2 * nqN * 8);
    G.S = (uint64_t*)c->dalloc((size_t)O * oN * 8);
    HCUDA(cudaMallocHost(&G.pinned, limbsplit_pinned_per_rank(pl) * parts));
  }
  static const bool graphs = getenv("HELRM_GRAPH") ? atoi(getenv("HELRM_GRAPH")) != 0 : true;
  for (size_t qy = 0; qy < batch; qy++) {
    const helrm_ct* const* cin = in + qy * C;
    for (int64_t ci = 0; ci < C; ci++) {
      need(cin[ci] != nullptr && cin[ci]->level == l, HELRM_ERR_LEVEL, "input level differs from the plan's");
      if (real && parts > 1)   // the query lives on rank 0
        HNCCL(nccl().broadcast(cin[ci]->d, G.X + ci * 2 * nqN, 2 * nqN, ncclUint64, 0, c->comm, c->stream));
      else
        HCUDA(cudaMemcpyAsync(G.X + ci * 2 * nqN, cin[ci]->d, 2 * nqN * 8, cudaMemcpyDeviceToDevice, c->stream));
    }
    auto body = [&](void** pinned) { limbsplit_body(c, pl, rk, G.X, G.S, parts, real, only_rank, pinned); };
    if (graphs && !c->prof.on) run_graph(c, G, body);
    else body(nullptr);
    emit_outputs(c, pl, G.S, 1, cin[0]->scale, out + qy * O);
  }
}

// the whole limb-partitioned lookup of one staged query Xin -> Sout [O][2][l][N]
static void limbsplit_body(helrm_ctx* c, const helrm_plan* pl, const helrm_rotkeys* rk, const uint64_t* Xin,
                           uint64_t* Sout, int parts, bool real, int only_rank, void** pinned) {
  const Params& P = c->P;
  const uint32_t l = pl->level;
  const size_t N = P.N, nq = l + 1, nl = l + 1 + P.K, nlN = nl * N, nqN = nq * N, dn = P.dnum(l);
  const LimbMap mqp = P.map_qp(l), mq = P.map_q(l);
  const LevelConst& lc = level_const(c, l);
  const int64_t C = pl->C, O = pl->O;
  // equal slices of rp = ceil(nl / parts) rows (the last ones shorter or empty), so that one
  // ncclAllGather of the padded slices lays the rows out in order
  const size_t rp = (nl + parts - 1) / parts;
  std::vector<int64_t> lo(parts), hi(parts);
  for (int r = 0; r < parts; r++) {
    lo[r] = std::min<int64_t>((int64_t)nl, (int64_t)(r * rp));
    hi[r] = std::min<int64_t>((int64_t)nl, (int64_t)((r + 1) * rp));
  }
  std::vector<int> mine;   // the ranks this process computes
  const bool timing = only_rank >= 0;   // one rank's kernels only, exchanges skipped (a timing harness)
  if (timing) mine.push_back(only_rank);
  else if (real) mine.push_back(c->rank);
  else
    for (int r = 0; r < parts; r++) mine.push_back(r);
  auto sub = [&](int r) {   // the LimbMap of rank r's rows (for the row-agnostic element-wise kernels)
    LimbMap m{};
    m.n = (int)(hi[r] - lo[r]);
    for (int i = 0; i < m.n; i++) m.pr[i] = mqp.pr[lo[r] + i];
    return m;
  };
  {
    struct {
      const uint64_t* p;
    } X{Xin};
    // L1: every rank converts the (replicated) y-form of the input c1s into its own rows of
    // the digits: D row r of digit k is written by the rank owning row r
    DBuf D(c, (size_t)C * dn * nlN), Y(c, (size_t)C * nqN);
    launch_ntt_inv(c->dc(), X.p + nqN, Y.p, c->scratch, (size_t)C * nq, mq, 2 * nqN, nqN, lc.modup_post,
                   pm_lidx(c, (int)C, (uint32_t)nq));
    for (int r : mine) {
      if (hi[r] == lo[r]) continue;
      const helrm_ctx::SliceTabs& st = slice_tabs(c, l, (int)lo[r], (int)hi[r], (int)C);
      launch_conv_rows(c->dc(), st.up_tab, (int)dn, st.up_rows, (int)P.alpha, Y.p, nqN, D.p, dn * nlN, nlN, (int)C,
                       mqp);
      if (st.n_up) launch_ntt_fwd(c->dc(), D.p, D.p, c->scratch, st.n_up, mqp, 0, 0, true, st.up_lidx);
    }
    // (P c0, P c1) of every ct (replicated, cheap): the baby pair of rotation 0
    DBuf P0(c, (size_t)C * 2 * nlN);
    HCUDA(cudaMemsetAsync(P0.p, 0, (size_t)C * 2 * nlN * 8, c->stream));
    launch_scalar_mul(c->dc(), X.p, P0.p, mq, lc.pmod, lc.pmods, 1, (int)C, 2 * nqN, 2 * nlN);
    launch_scalar_mul(c->dc(), X.p + nqN, P0.p + nlN, mq, lc.pmod, lc.pmods, 1, (int)C, 2 * nqN, 2 * nlN);
    // the non-empty giant pairs z (o, i)
    std::vector<std::pair<int64_t, int64_t>> oi;
    for (int64_t o = 0; o < O; o++)
      for (size_t i = 0; i < pl->entries[o].size(); i++)
        if (!pl->entries[o][i].empty()) oi.push_back({o, (int64_t)i});
    const size_t nz = oi.size();
    size_t nb_tot = 0;
    for (auto& b : pl->babies) nb_tot += b.size();
    // rank slices: babies [b][2][rows][N], inner sums [z][2][rows][N], accumulators [o][2][rows][N]
    // (slices hold rp rows; a rank with rows < rp leaves the tail unused)
    std::vector<std::unique_ptr<DBuf>> SB(parts), SAB(parts), SO(parts);
    std::vector<uint64_t*> sab(parts, nullptr), so(parts, nullptr);
    for (int r : mine) {
      SB[r].reset(new DBuf(c, std::max<size_t>(1, nb_tot) * 2 * rp * N));
      SAB[r].reset(new DBuf(c, std::max<size_t>(1, nz) * 2 * rp * N));
      SO[r].reset(new DBuf(c, (size_t)O * 2 * rp * N));
      sab[r] = SAB[r]->p;
      so[r] = SO[r]->p;
      HCUDA(cudaMemsetAsync(so[r], 0, (size_t)O * 2 * rp * N * 8, c->stream));
      if (hi[r] == lo[r]) HCUDA(cudaMemsetAsync(sab[r], 0, std::max<size_t>(1, nz) * 2 * rp * N * 8, c->stream));
    }
    for (int r : mine) {
      if (hi[r] == lo[r]) continue;   // an empty slice (parts does not divide into l + 1 + K evenly)
      const size_t rows = rp;         // slice stride (rows actually computed: hi - lo)
      const size_t r0N = (size_t)lo[r] * N;
      // L2 (own rows): baby pairs of every ct, baby (ci, j) at slice + b 2 rows N
      std::map<std::pair<int64_t, int>, uint64_t*> ab;
      size_t b = 0;
      for (int64_t ci = 0; ci < C; ci++) {
        KipMulti km{};
        km.row0 = (int)lo[r];
        km.rows = (int)(hi[r] - lo[r]);
        km.own = X.p + ci * 2 * nqN + nqN;
        km.alpha = (int)P.alpha;
        km.digits = D.p + ci * dn * nlN;
        km.digit_stride = nlN;
        km.dnum = (int)dn;
        km.c0 = X.p + ci * 2 * nqN;
        km.p_mod = lc.pmod;
        km.level = l;
        km.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
        km.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
        km.out_half = rows * N;
        for (int j : pl->babies[ci]) {
          uint64_t* a = SB[r]->p + b++ * 2 * rows * N;
          ab[{ci, j}] = a;
          if (j == 0) {   // this rank's rows of (P c0, P c1)
            for (int h = 0; h < 2; h++)
              HCUDA(cudaMemcpyAsync(a + h * rows * N, P0.p + ci * 2 * nlN + h * nlN + r0N, (hi[r] - lo[r]) * N * 8,
                                    cudaMemcpyDeviceToDevice, c->stream));
            continue;
          }
          need(km.n < kMaxBabies, HELRM_ERR_CAPACITY, "too many baby steps");
          const uint64_t g = galois_of_rot(c, j);
          km.rot[km.n] = rot_of_galois(c, g);
          km.key[km.n] = key_for(rk, g);
          km.out[km.n] = a - r0N;   // the kernel addresses row l at out + l N
          km.max_rot = std::max(km.max_rot, km.rot[km.n]);
          km.n++;
        }
        if (km.n) launch_kip_multi(c->dc(), km, mqp);
      }
      // L3 (own rows): inner sums of every giant pair into the rank's slice
      const MacList ml = build_macs(pl, nlN, [&](int ci, int j) {
        uint64_t* a = ab.at({ci, j}) - r0N;
        return std::make_pair((const uint64_t*)a, (const uint64_t*)(a + rows * N));
      });
      need(ml.oi.size() == nz, HELRM_ERR_CONFIG, "work list differs from the pair enumeration");
      void* pr = pinned ? (char*)*pinned + (size_t)r * limbsplit_pinned_per_rank(pl) : nullptr;
      MacDev md(c, ml, pinned ? &pr : nullptr);
      {
        const DevCtx dcx = c->dc();
        ProfScope ps_(dcx, "diag_mac", 8.0 * N * (hi[r] - lo[r]) * (ml.n_u + 2.0 * ml.n_x + 2.0 * nz));
        need(launch_diag_mac_bulk(dcx, (const MacTerm*)md.terms.p, (const int4*)md.groups.p, (int)ml.groups.size(),
                                  sab[r] - r0N, 2 * rows * N, rows * N, mqp, 1, 0, 0, 0, (int)lo[r],
                                  (int)(hi[r] - lo[r])),
             HELRM_ERR_CONFIG, "the limb partition needs N divisible by the MAC tile");
      }
    }
    // L4, batched over the rotating giant pairs: all-gather every pair's B rows, ModDown of
    // all of them on each rank's Q rows, B' to y-form on those rows, all-gather, each rank's
    // rows of the digits of every B', then the giant key switches in runs on own rows.
    std::vector<size_t> rot;   // rotating pairs (g_i != 0)
    for (size_t z = 0; z < nz; z++) {
      const int64_t o = oi[z].first, gi = pl->giants[o][oi[z].second];
      if (gi % (int64_t)P.n != 0) {
        rot.push_back(z);
        continue;
      }
      for (int r : mine) {   // O_o += (A, B)_z on own rows
        if (hi[r] == lo[r]) continue;
        const LimbMap sm = sub(r);
        for (int h = 0; h < 2; h++)
          launch_binary(c->dc(), 0, so[r] + (o * 2 + h) * rp * N, sab[r] + (z * 2 + h) * rp * N,
                        so[r] + (o * 2 + h) * rp * N, sm);
      }
    }
    const size_t nr = rot.size(), fs = (size_t)parts * rp * N;   // padded full stride per polynomial
    if (nr) {
      DBuf Bf(c, nr * fs), Bp(c, nr * nqN), D2(c, nr * dn * nlN), Y2(c, nr * fs), yP(c, nr * P.K * N),
          T(c, nr * nqN);
      // all-gather of every rotating pair's B rows: slice r of pair t at Bf + t fs + r rp N
      if (real && parts > 1) {
        HNCCL(nccl().groupStart());
        for (size_t t = 0; t < nr; t++)
          HNCCL(nccl().allGather(sab[c->rank] + (rot[t] * 2 + 1) * rp * N, Bf.p + t * fs, rp * N, ncclUint64, c->comm,
                                 c->stream));
        HNCCL(nccl().groupEnd());
      } else {
        for (int r : mine)
          for (size_t t = 0; t < nr; t++)
            HCUDA(cudaMemcpyAsync(Bf.p + t * fs + r * rp * N, sab[r] + (rot[t] * 2 + 1) * rp * N, rp * N * 8,
                                  cudaMemcpyDeviceToDevice, c->stream));
      }
      // ModDown (D16): every B's P rows to y-form (replicated), own Q rows converted + NTT + epilogue
      launch_ntt_inv(c->dc(), Bf.p + nqN, yP.p, c->scratch, nr * P.K, P.map_range(P.L + 1, P.K), fs, P.K * N,
                     lc.moddown_post, nullptr);
      for (int r : mine) {
        const helrm_ctx::SliceTabs& st = slice_tabs(c, l, (int)lo[r], (int)hi[r], (int)nr);
        if (st.n_q == 0) continue;
        launch_conv_rows(c->dc(), st.dn_tab, 1, st.dn_rows, (int)P.K, yP.p, P.K * N, T.p, nqN, 0, (int)nr, mq);
        NttEpi epi;
        epi.y = Bf.p;
        epi.ys = fs;
        epi.out = Bp.p;
        epi.os = nqN;
        epi.s = lc.pinv;
        epi.sp = lc.pinvs;
        launch_ntt_fwd(c->dc(), T.p, T.p, c->scratch, st.n_q, mq, 0, 0, true, st.q_lidx, &epi);
        // ModUp (D15) of B': own Q rows into y-form, rows at the padded positions of Y2
        launch_ntt_inv(c->dc(), Bp.p, Y2.p, c->scratch, st.n_q, mq, nqN, fs, lc.modup_post, st.q_lidx);
      }
      if (real && parts > 1) {   // all-gather of the y-form rows (in place: slice r at r rp rows)
        HNCCL(nccl().groupStart());
        for (size_t t = 0; t < nr; t++)
          HNCCL(nccl().allGather(Y2.p + t * fs + (size_t)c->rank * rp * N, Y2.p + t * fs, rp * N, ncclUint64, c->comm,
                                 c->stream));
        HNCCL(nccl().groupEnd());
      }
      for (int r : mine) {   // each rank's rows of the digits of every B'
        if (hi[r] == lo[r]) continue;
        const helrm_ctx::SliceTabs& st = slice_tabs(c, l, (int)lo[r], (int)hi[r], (int)nr);
        launch_conv_rows(c->dc(), st.up_tab, (int)dn, st.up_rows, (int)P.alpha, Y2.p, fs, D2.p, dn * nlN, nlN,
                         (int)nr, mqp);
        if (st.n_up) launch_ntt_fwd(c->dc(), D2.p, D2.p, c->scratch, st.n_up, mqp, 0, 0, true, st.up_lidx);
      }
      // giant key switches on own rows, in runs of one output block (k_kip_giants row slice)
      for (int r : mine) {
        if (hi[r] == lo[r]) continue;
        const size_t rows = rp;
        const size_t r0N = (size_t)lo[r] * N;
        KipGiants kg{};
        int64_t cur_o = -1;
        auto flush = [&]() {
          if (kg.n == 0) return;
          kg.row0 = (int)lo[r];
          kg.rows = (int)(hi[r] - lo[r]);
          kg.digit_stride = nlN;
          kg.dnum = (int)dn;
          kg.add_rows = (int)nl;
          kg.alpha = (int)P.alpha;
          kg.level = (int)l;
          kg.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
          kg.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
          kg.out0 = so[r] + cur_o * 2 * rows * N - r0N;
          kg.out1 = kg.out0 + rows * N;
          launch_kip_giants(c->dc(), kg, mqp);
          kg.n = 0;
        };
        for (size_t t = 0; t < nr; t++) {
          const size_t z = rot[t];
          const int64_t o = oi[z].first, gi = pl->giants[o][oi[z].second];
          if (o != cur_o || kg.n == kMaxGiantRun) {
            flush();
            cur_o = o;
          }
          const uint64_t g = galois_of_rot(c, gi);
          kg.digits[kg.n] = D2.p + t * dn * nlN;
          kg.own[kg.n] = Bp.p + t * nqN;
          kg.key[kg.n] = key_for(rk, g);
          kg.add0[kg.n] = sab[r] + z * 2 * rows * N - r0N;   // A's rows
          kg.rot[kg.n] = rot_of_galois(c, g);
          kg.n++;
        }
        flush();
      }
    }
    // all-gather of the accumulators
    DBuf Of(c, (size_t)O * 2 * nlN);
    std::unique_ptr<DBuf> Og;
    std::vector<const uint64_t*> src(parts, nullptr);
    if (real && parts > 1) {   // [rank][O][2][rp][N]
      Og.reset(new DBuf(c, (size_t)parts * O * 2 * rp * N));
      HNCCL(nccl().allGather(so[c->rank], Og->p, (size_t)O * 2 * rp * N, ncclUint64, c->comm, c->stream));
      nccl_check_async(c);
      for (int r = 0; r < parts; r++) src[r] = Og->p + (size_t)r * O * 2 * rp * N;
    } else {
      for (int r : mine) src[r] = so[r];
    }
    for (int r = 0; r < parts; r++) {
      if (hi[r] == lo[r] || !src[r]) continue;   // (timing harness: the other ranks' rows are absent)
      for (int64_t k = 0; k < 2 * O; k++)
        HCUDA(cudaMemcpyAsync(Of.p + k * nlN + (size_t)lo[r] * N, src[r] + k * rp * N, (hi[r] - lo[r]) * N * 8,
                              cudaMemcpyDeviceToDevice, c->stream));
    }
    // L6-L8 on each rank's rows.  Ownership follows the primes: at level l - 1 (after the
    // rescale drops q_l) rank r owns rows [lo1, hi1) = its rows with those above l moved down.
    const uint32_t l1 = l - 1;
    const size_t nq1 = l, nl1 = l + P.K, nl1N = nl1 * N, nq1N = nq1 * N, dn1 = P.dnum(l1);
    const LimbMap mq1 = P.map_q(l1), mqp1 = P.map_qp(l1);
    const LevelConst& lc1 = level_const(c, l1);
    std::vector<int64_t> lo1(parts), hi1(parts);
    for (int r = 0; r < parts; r++) {
      lo1[r] = lo[r] - (lo[r] > (int64_t)l ? 1 : 0);
      hi1[r] = hi[r] - (hi[r] > (int64_t)l ? 1 : 0);
    }
    // exchange: every rank's rows [a_r, b_r) of npoly polynomials (poly stride ps) to all ranks
    // (one ncclBroadcast per owner, grouped); the emulation's ranks share the buffer already
    auto share = [&](uint64_t* buf, const std::vector<int64_t>& a, const std::vector<int64_t>& b, int npoly,
                     size_t ps) {
      if (!(real && parts > 1)) return;
      HNCCL(nccl().groupStart());
      for (int r = 0; r < parts; r++)
        for (int k = 0; k < npoly; k++)
          if (b[r] > a[r])
            HNCCL(nccl().broadcast(buf + k * ps + (size_t)a[r] * N, buf + k * ps + (size_t)a[r] * N,
                                   (size_t)(b[r] - a[r]) * N, ncclUint64, r, c->comm, c->stream));
      HNCCL(nccl().groupEnd());
    };
    std::vector<int64_t> qa(parts), qb(parts), pa(parts), pb(parts), la(parts), lb(parts);
    DBuf R(c, 2 * nqN), S1(c, (size_t)O * 2 * nq1N), yP2(c, 2 * (size_t)P.K * N), T2(c, 2 * nqN), xl(c, 2 * N),
        rr(c, 2 * nq1N), Yr(c, nq1N), Dr(c, dn1 * nl1N), K2(c, 2 * nl1N);
    for (int64_t o = 0; o < O; o++) {
      const uint64_t* Oo = Of.p + o * 2 * nlN;
      uint64_t* So = S1.p + o * 2 * nq1N;
      // L6 ModDown of both halves: P rows to y-form (replicated), own Q rows converted + NTT
      launch_ntt_inv(c->dc(), Oo + nqN, yP2.p, c->scratch, 2 * P.K, P.map_range(P.L + 1, P.K), nlN, P.K * N,
                     lc.moddown_post, nullptr);
      for (int r : mine) {
        const helrm_ctx::SliceTabs& st = slice_tabs(c, l, (int)lo[r], (int)hi[r], 2);
        if (st.n_q == 0) continue;
        launch_conv_rows(c->dc(), st.dn_tab, 1, st.dn_rows, (int)P.K, yP2.p, P.K * N, T2.p, nqN, 0, 2, mq);
        NttEpi epi;
        epi.y = Oo;
        epi.ys = nlN;
        epi.out = R.p;
        epi.os = nqN;
        epi.s = lc.pinv;
        epi.sp = lc.pinvs;
        launch_ntt_fwd(c->dc(), T2.p, T2.p, c->scratch, st.n_q, mq, 0, 0, true, st.q_lidx, &epi);
      }
      // L7 rescale: row l of both halves (its owner's) to everyone, then each rank's rows i < l
      for (int r = 0; r < parts; r++) {
        la[r] = std::max<int64_t>(lo[r], (int64_t)l);
        lb[r] = std::min<int64_t>(hi[r], (int64_t)l + 1);
      }
      if (!timing) share(R.p, la, lb, 2, nqN);
      ntt_inv(c, R.p + (size_t)l * N, xl.p, 2, P.map_range(l, 1), nqN, N);
      launch_rescale_prep(c->dc(), xl.p, N, P.primes[l], rr.p, nq1N, 2, mq1);
      for (int r : mine) {
        const helrm_ctx::SliceTabs& st = slice_tabs(c, l1, (int)lo1[r], (int)hi1[r], 2);
        if (st.n_q == 0) continue;
        NttEpi epi;
        epi.y = R.p;
        epi.ys = nqN;
        epi.out = So;
        epi.os = nq1N;
        epi.s = lc.qlinv;
        epi.sp = lc.qlinvs;
        launch_ntt_fwd(c->dc(), rr.p, rr.p, c->scratch, st.n_q, mq1, 0, 0, false, st.q_lidx, &epi);
      }
      // L8 RotSum at level l - 1, every rotation on the ranks' rows
      for (int r = 0; r < parts; r++) {
        qa[r] = lo1[r];
        qb[r] = std::min<int64_t>(hi1[r], (int64_t)nq1);
        pa[r] = std::max<int64_t>(lo1[r], (int64_t)nq1);
        pb[r] = hi1[r];
      }
      for (int64_t amt = pl->mbar; amt < (int64_t)P.n; amt *= 2) {
        const uint64_t g = galois_of_rot(c, amt);
        // ModUp of c1: own Q rows to y-form, shared, own rows of the digits
        for (int r : mine) {
          const helrm_ctx::SliceTabs& st = slice_tabs(c, l1, (int)lo1[r], (int)hi1[r], 1);
          if (st.n_q) launch_ntt_inv(c->dc(), So + nq1N, Yr.p, c->scratch, st.n_q, mq1, nq1N, nq1N, lc1.modup_post,
                                     st.q_lidx);
        }
        if (!timing) share(Yr.p, qa, qb, 1, nq1N);
        for (int r : mine) {
          if (hi1[r] == lo1[r]) continue;
          const helrm_ctx::SliceTabs& st = slice_tabs(c, l1, (int)lo1[r], (int)hi1[r], 1);
          launch_conv_rows(c->dc(), st.up_tab, (int)dn1, st.up_rows, (int)P.alpha, Yr.p, nq1N, Dr.p, dn1 * nl1N,
                           nl1N, 1, mqp1);
          if (st.n_up) launch_ntt_fwd(c->dc(), Dr.p, Dr.p, c->scratch, st.n_up, mqp1, 0, 0, true, st.up_lidx);
          // lazy key switch on own rows: (P phi(c0) + KS0, KS1)
          KipArgs a{};
          a.row0 = (int)lo1[r];
          a.rows = (int)(hi1[r] - lo1[r]);
          a.digits = Dr.p;
          a.digit_stride = nl1N;
          a.dnum = (int)dn1;
          a.key = key_for(rk, g);
          a.key_digit_stride = (size_t)2 * (P.L + 1 + P.K) * N;
          a.key_half_stride = (size_t)(P.L + 1 + P.K) * N;
          a.add0 = So;
          a.add_rows = (int)nq1;
          a.add_mul = lc1.pmod;
          a.rot = rot_of_galois(c, g);
          a.out0 = K2.p;
          a.out1 = K2.p + nl1N;
          a.own = So + nq1N;
          a.alpha = (int)P.alpha;
          a.level = (int)l1;
          launch_kip(c->dc(), a, mqp1);
        }
        // ModDown of (KS0, KS1): their P rows shared, own Q rows accumulated into the ct
        if (!timing) share(K2.p, pa, pb, 2, nl1N);
        launch_ntt_inv(c->dc(), K2.p + nq1N, yP2.p, c->scratch, 2 * P.K, P.map_range(P.L + 1, P.K), nl1N, P.K * N,
                       lc1.moddown_post, nullptr);
        for (int r : mine) {
          const helrm_ctx::SliceTabs& st = slice_tabs(c, l1, (int)lo1[r], (int)hi1[r], 2);
          if (st.n_q == 0) continue;
          launch_conv_rows(c->dc(), st.dn_tab, 1, st.dn_rows, (int)P.K, yP2.p, P.K * N, T2.p, nq1N, 0, 2, mq1);
          NttEpi epi;
          epi.y = K2.p;
          epi.ys = nl1N;
          epi.out = So;
          epi.os = nq1N;
          epi.s = lc1.pinv;
          epi.sp = lc1.pinvs;
          epi.accumulate = 1;   // ct += Rotate(ct)
          launch_ntt_fwd(c->dc(), T2.p, T2.p, c->scratch, st.n_q, mq1, 0, 0, true, st.q_lidx, &epi);
        }
      }
      if (!timing) share(So, qa, qb, 2, nq1N);   // the output ct's rows to every rank
    }
    HCUDA(cudaMemcpyAsync(Sout, S1.p, (size_t)O * 2 * nq1N * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
}

helrm_status helrm_lookup_limbsplit_virtual(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                            const helrm_ct* const* in, size_t batch, int parts, helrm_ct** out) {
  if (out)
    for (size_t i = 0; i < batch * (p ? p->O : 0); i++) out[i] = nullptr;
  return guard([&] {
    need(c && p && rk && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    lookup_limbsplit(c, p, rk, in, batch, out, parts, false);
  });
}

helrm_status helrm_limbsplit_rank_work(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                       const helrm_ct* const* in, int parts, int rank, helrm_ct** out) {
  if (out)
    for (int64_t i = 0; i < (p ? p->O : 0); i++) out[i] = nullptr;
  return guard([&] {
    need(c && p && rk && in && out && parts >= 1 && rank >= 0 && rank < parts, HELRM_ERR_ARG, "bad argument");
    DevGuard dg_(c->device);
    lookup_limbsplit(c, p, rk, in, 1, out, parts, false, rank);
  });
}

helrm_status helrm_lookup_limbsplit(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                   const helrm_ct* const* in, size_t batch, helrm_ct** out) {
  if (out)
    for (size_t i = 0; i < batch * (p ? p->O : 0); i++) out[i] = nullptr;
  return guard([&] {
    need(c && p && rk && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(c->world == 1 || c->comm, HELRM_ERR_ARG, "helrm_comm_init first");
    lookup_limbsplit(c, p, rk, in, batch, out, c->world, true);
  });
}

helrm_status helrm_lookup_dist(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk, const helrm_ct* const* in,
                               size_t batch, helrm_ct** out) {
  if (out)
    for (size_t i = 0; i < batch * (p ? p->O : 0); i++) out[i] = nullptr;
  return guard([&] {
    need(c && p && rk && in && out, HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    lookup_split(c, p, rk, in, batch, out, 0);
  });
}

helrm_status helrm_lookup_dist_virtual(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                       const helrm_ct* const* in, size_t batch, int parts, helrm_ct** out) {
  if (out)
    for (size_t i = 0; i < batch * (p ? p->O : 0); i++) out[i] = nullptr;
  return guard([&] {
    need(c && p && rk && in && out && parts >= 1 && parts < 8192, HELRM_ERR_ARG, "bad argument");
    DevGuard dg_(c->device);
    lookup_split(c, p, rk, in, batch, out, parts);
  });
}

helrm_status helrm_modred(helrm_ctx* c, uint64_t* dev, uint32_t level, size_t n_polys) {
  return guard([&] {
    need(c && (dev || n_polys == 0), HELRM_ERR_ARG, "null argument");
    DevGuard dg_(c->device);
    need(level <= c->P.L, HELRM_ERR_LEVEL, "level above L");
    const LimbMap m = c->P.map_qp(level);
    for (size_t i = 0; i < n_polys; i++) launch_modred(c->dc(), dev + i * m.n * c->P.N, m);
    HCUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
