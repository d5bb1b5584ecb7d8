// internal.h -- library-internal types shared by the host engine and the
// kernels.  Nothing here crosses the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <nccl.h>

#include "arith.cuh"
#include "../../include/helrm.h"

namespace helrm {

constexpr int kMaxLimbs = 64;
constexpr int kMaxDigitPrimes = 8;

struct Error : std::runtime_error {
  helrm_status code;
  Error(helrm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define HCUDA(x)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess)                                                                    \
      throw ::helrm::Error(HELRM_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));  \
  } while (0)

// Constants of one prime of the chain q_0..q_L, p_0..p_{K-1}, on the device.
struct PrimeDev {
  RedConst rc;
  uint64_t ninv, ninvs;         // N^-1 and its shoup companion
  double qd, qinv;              // q and 1/q as doubles (NTT butterflies on the FP64 pipe)
  double2 ninvd;                // (N^-1, N^-1 / q)
  // NTT twiddles as (w, w/q) doubles, w = psi^(+-bitrev_logN(idx)):
  const double2* tw1;           // [256] pass 1, natural index idx < 256
  const double2* tw2;           // [N] pass 2, per 256-block B: [B][j], j in per-thread order
  const double2* itw1;          // inverse twiddles, same layouts
  const double2* itw2;
};

// Global chain index of each limb of a polynomial (by value as kernel arg).
struct LimbMap {
  int n;
  uint8_t pr[kMaxLimbs];
};

// one output row of a base conversion: out[out_row] = sum_b y_{row0+b} cf[b]
// mod q_out (out_row < 0: padding, nothing written), evaluated on the FP64
// pipe: cf as (w, w / q_out) pairs
struct ConvRowDev {
  int src_row0, nb, out_row;
  double q, qinv;
  double2 cf[kMaxDigitPrimes];
};

struct Params {
  uint32_t log_n = 0, N = 0, n = 0, L = 0, K = 0, alpha = 0, log_scale = 0;
  std::vector<uint64_t> primes;  // q_0..q_L, p_0..p_{K-1}
  std::vector<uint64_t> psi;
  uint32_t dnum(uint32_t level) const { return (level + 1 + alpha - 1) / alpha; }
  // chain index of limb `l` of an R_{Q_level P} polynomial
  uint32_t qp_chain(uint32_t level, uint32_t l) const { return l <= level ? l : L + 1 + (l - level - 1); }
  LimbMap map_q(uint32_t level) const {
    LimbMap m{};
    m.n = level + 1;
    for (uint32_t i = 0; i <= level; i++) m.pr[i] = (uint8_t)i;
    return m;
  }
  LimbMap map_qp(uint32_t level) const {
    LimbMap m{};
    m.n = level + 1 + K;
    for (uint32_t i = 0; i < (uint32_t)m.n; i++) m.pr[i] = (uint8_t)qp_chain(level, i);
    return m;
  }
  LimbMap map_range(uint32_t first, uint32_t count) const {
    LimbMap m{};
    m.n = count;
    for (uint32_t i = 0; i < count; i++) m.pr[i] = (uint8_t)(first + i);
    return m;
  }
};

// NCCL, resolved at run time (nccl_dl.cpp)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
};
NcclApi& nccl();
#define HNCCL(x)                                                                                       \
  do {                                                                                                 \
    ncclResult_t r_ = (x);                                                                             \
    if (r_ != ncclSuccess)                                                                             \
      throw ::helrm::Error(HELRM_ERR_NCCL, std::string(#x) + ": " + ::helrm::nccl().getErrorString(r_)); \
  } while (0)

// host math (host_math.cpp)
bool is_prime_u64(uint64_t n);
std::vector<uint64_t> find_primes(const std::vector<std::pair<uint32_t, uint32_t>>& groups, uint64_t N,
                                  std::vector<uint64_t> taken);
uint64_t min_psi(uint64_t q, uint64_t N);
uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t q);
uint64_t inv_mod(uint64_t a, uint64_t q);
uint64_t mulm(uint64_t a, uint64_t b, uint64_t q);
// D6: correctly rounded encode (double-double FFT + binary128 recheck)
int encode_slots(const double* z, size_t n_nonzero_hint, uint32_t log_n, double delta, int64_t* out);
// D7 decode (fp64)
void decode_coeffs(const int64_t* m, uint32_t log_n, double delta, double* z, size_t n_slots);
// centered CRT of small values into int64 (|m| < 2^62 assumed)
void crt_small(const uint64_t* res, const uint64_t* primes, size_t n_limbs, size_t N, int64_t* out);
// the slot-order permutation: slot position of bit-reversed NTT index r
std::vector<uint32_t> slot_of_bitrev(uint32_t log_n);
std::vector<uint64_t> gauss_cdt_table();

// ---------------- kernel launchers (kernels_*.cu) ----------------
// Optional per-kernel CUDA-event timing (helrm_ctx_profile): each launcher
// brackets its launch with events on the context stream.
struct Profiler {
  bool on = false;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
    double bytes;                 // algorithmic HBM bytes of the launch
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get();
};

struct DevCtx {
  const PrimeDev* primes;     // device array, chain-indexed
  const uint32_t* slotpos;    // [N] slot position of bitrev index r
  const uint32_t* ntt_grp;    // [N/256] 256-blocks ordered by (half, slot residue): 16 per pass-2 CTA
  const double* ntt_twb;      // NTT twiddle tables of every prime, 4 N + 1024 doubles per prime
  const uint8_t* ntt_tpos;    // [N] per block: rank of element e's slot position within the block
  uint32_t log_n, N;
  cudaStream_t stream;
  int persist;                // > 0: HBM-bound MAC / key-switch kernels run persistent, persist CTAs per SM
  int n_sm;                   // multiprocessors of the context's device (148 on B200)
  uint64_t* launches;         // host counter
  Profiler* prof;
};

// Programmatic dependent launch (HELRM_PDL=1; off by default: measured neutral).  A kernel launched
// with launch_pdl may be scheduled while its stream predecessor is finishing:
// its CTAs become resident and wait in pdl_wait_trigger() (griddepcontrol.wait)
// until the predecessor has completed and its writes are visible, so a chain
// of small dependent kernels (RotSum, ModUp/ModDown) does not pay a launch
// gap per boundary.  Every kernel launched this way calls pdl_wait_trigger()
// before touching memory; the trigger lets its own successor be scheduled
// once all of its CTAs are running.
bool pdl_on();
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait_trigger() {
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = pdl_on() ? at : nullptr;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  HCUDA(cudaLaunchKernelEx(&cfg, k, args...));
}
#endif

// NVTX range per lookup stage (D20 L1..L8), visible in Nsight tools and usable
// as an ncu --nvtx filter; a push/pop pair on the host thread
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
};

// host-side time per call site (HELRM_HOSTPROF=1; diagnostics of launch overhead)
bool hostprof_on();
void hostprof_add(const char* name, double us);
double hostprof_now_us();
struct HostTimer {
  const char* name;
  double t0;
  explicit HostTimer(const char* n) : name(n), t0(hostprof_on() ? hostprof_now_us() : 0) {}
  ~HostTimer() {
    if (hostprof_on()) hostprof_add(name, hostprof_now_us() - t0);
  }
};

// RAII: records a start event now and a stop event at scope exit
struct ProfScope {
  const DevCtx& c;
  int idx = -1;
  HostTimer ht;
  ProfScope(const DevCtx& c_, const char* name, double bytes = 0);
  ~ProfScope();
};

// Optional epilogue of the forward NTT (the last step of ModDown D16 and of
// rescale D17): instead of storing t = NTT(.) the pass-2 kernel stores, for
// limb l of poly g,  out[g][l] (+)= (y[g][l] - t[g][l]) * s[l]  mod q_l.
struct NttEpi {
  const uint64_t* y = nullptr;   // y + g ys + l N
  size_t ys = 0;
  uint64_t* out = nullptr;       // out + g os + l N
  size_t os = 0;
  const uint64_t* s = nullptr;   // per-limb factor and its Shoup companion
  const uint64_t* sp = nullptr;
  int accumulate = 0;            // out += instead of out =
};
// NTT over n_total limbs: limb y = (poly y / map.n, limb y % map.n) lives at
// src + (y / map.n) * src_stride + (y % map.n) * N (same for dst; stride 0 =
// contiguous polys of map.n limbs).  src == dst allowed.
// din: the source limbs hold centred integer-valued doubles (k_conv_rows output)
// lidx (optional device table): launch limb v is layout limb lidx[v]
void launch_ntt_fwd(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, size_t n_total,
                    const LimbMap& map, size_t src_stride = 0, size_t dst_stride = 0, bool din = false,
                    const uint32_t* lidx = nullptr, const NttEpi* epi = nullptr);
// pass-2 / pass-A block grouping into constant memory (a function of log N only)
void ntt_set_grp(uint32_t log_n, const uint32_t* grp, size_t n);
// post (optional, per limb of map): final factor (w, w/q) replacing N^-1
void launch_ntt_inv(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, size_t n_total,
                    const LimbMap& map, size_t src_stride = 0, size_t dst_stride = 0,
                    const double2* post = nullptr, const uint32_t* lidx = nullptr);
// D14 base conversion from y-form sources (coefficients times [(B/b)^-1]_b,
// folded into the INTT): for polynomial g and conversion k, every output row
// r of the table: out_gk[r] = sum_b y_g[row0 + b] cf_kr[b] mod q_r, written
// as centred integer-valued doubles (coefficient form; a din NTT follows).
// z = g ncv + k.
void launch_conv_rows(const DevCtx& c, const ConvRowDev* tab, int ncv, int rows, int nb_max, const uint64_t* y,
                      size_t y_stride, uint64_t* out, size_t out_stride_g, size_t out_stride_k, int G,
                      const LimbMap& out_map);
size_t ntt_scratch_words(int log_n);

void launch_reduce_signed(const DevCtx& c, const int64_t* m, uint64_t* out, const LimbMap& map);
void launch_sample_uniform_ntt(const DevCtx& c, uint64_t* out, const LimbMap& map, uint64_t seed, uint64_t purpose,
                               uint64_t a, uint64_t b, const LimbMap& ids);
void launch_sample_small(const DevCtx& c, int64_t* out, uint64_t base, int kind, const uint64_t* cdt);
// op 0: a + b, 1: a - b, 2: a * b, 3: -a
void launch_binary(const DevCtx& c, int op, const uint64_t* a, const uint64_t* b, uint64_t* out, const LimbMap& map);
void launch_scalar_mul(const DevCtx& c, const uint64_t* a, uint64_t* out, const LimbMap& map, const uint64_t* s,
                       const uint64_t* sp, int dform_out = 0, int G = 1, size_t a_stride = 0,
                       size_t out_stride = 0);
// in place: dir 1 -> D-form (fmath.cuh), dir 0 -> canonical; word i is in limb
// (i / N) mod map.n of a repeating [map.n][N] layout
void launch_dform(const DevCtx& c, uint64_t* x, size_t n, const LimbMap& map, int dir);
void launch_automorph(const DevCtx& c, const uint64_t* a, uint64_t* out, const LimbMap& map, uint32_t rot,
                      int accumulate);
// out[l] = in[l] mod q_l for in < 2^64 (after a uint64 sum all-reduce)
void launch_modred(const DevCtx& c, uint64_t* x, const LimbMap& map);
// compact plans: out + (k map.n + l) N = coef[uids[k]] mod q_l (signed -> canonical), k < n
void launch_expand_coef(const DevCtx& c, const int64_t* coef, const uint32_t* uids, size_t n, uint64_t* out,
                        const LimbMap& map);
// x[i] += y[i] as uint64 words, i < n (the exact sum of the all-reduce)
void launch_add_u64(const DevCtx& c, uint64_t* x, const uint64_t* y, size_t n);
void launch_rescale_prep(const DevCtx& c, const uint64_t* xl, size_t xs, uint64_t ql, uint64_t* out, size_t os, int G,
                         const LimbMap& map);

struct KipArgs {
  int row0 = 0, rows = 0;     // limb rows [row0, row0 + rows) only (rows = 0: all of map)
  const uint64_t* digits;     // digit k of the switched polynomial at digits + k digit_stride ([nl][N], NTT slot order)
  size_t digit_stride;
  int dnum;
  const uint64_t* key;        // key for g: [digit][2][L+1+K][N], D-form
  size_t key_digit_stride;    // words between digits of the key
  size_t key_half_stride;     // words between b and a of a digit
  const uint64_t* add0;       // optional: out0 += mul_l phi(add0)[l] for l < add_rows
  int add_rows;
  const uint64_t* add_mul;    // [add_rows] per-limb multiplier (device) or null for 1
  uint32_t rot;               // slot rotation amount (phi_{5^rot})
  uint64_t* out0;             // [nl][N]
  uint64_t* out1;
  int accumulate;             // out += result (else out = result)
  int halves = 3;             // 1: out0 only (b keys, add0), 2: out1 only (a keys), 3: both
  // queries sharing the key (batched lookups): query q uses digits + q dq,
  // add0 + q aq and writes out0/out1 + q oq; the key is loaded once for all
  int nq = 1;
  size_t dq = 0, aq = 0, oq = 0;
  // digit k's own limbs (rows k alpha .. of Q_l) are read from the switched
  // polynomial itself (NTT form) when own != null: own + q ownq + row N
  const uint64_t* own = nullptr;
  size_t ownq = 0;
  int alpha = 1, level = 0;
};
void launch_kip(const DevCtx& c, const KipArgs& a, const LimbMap& map);

// Several giant steps of one output block in one pass (D20 L4):
//   out0 += sum_g [ phi_g(A_g) + sum_k phi_g(D_{g,k}) b_{g,k} ],  out1 += sum_g sum_k phi_g(D_{g,k}) a_{g,k}
// so the accumulators are read and written once for the run instead of once
// per giant.  Common fields as KipArgs (add_mul = 1, accumulate = 1, nq = 1).
constexpr int kMaxGiantRun = 16;
struct KipGiants {
  // rows [row0, row0 + rows) of the Q_l P limbs only (rows = 0: all of map): the RNS-limb
  // partition of the lookup gives each rank a slice of the limbs
  int row0 = 0, rows = 0;
  size_t digit_stride;
  int dnum, add_rows, alpha, level, n;
  size_t key_digit_stride, key_half_stride;
  uint64_t* out0;
  uint64_t* out1;
  // nq queries (output blocks) share every key value: query r reads digits[g] + r dq,
  // own[g] + r ownq, add0[g] + r aq and accumulates into out + r oq (nq = 1: strides unused)
  int nq = 1;
  size_t dq = 0, ownq = 0, aq = 0, oq = 0;
  const uint64_t* digits[kMaxGiantRun];
  const uint64_t* own[kMaxGiantRun];
  const uint64_t* key[kMaxGiantRun];
  const uint64_t* add0[kMaxGiantRun];
  uint32_t rot[kMaxGiantRun];
};
void launch_kip_giants(const DevCtx& c, const KipGiants& a, const LimbMap& map);

// all babies of one ciphertext (k_kip_multi)
constexpr int kMaxBabies = 128;
struct KipMulti {
  int row0 = 0, rows = 0;     // limb rows [row0, row0 + rows) only (rows = 0: all of map)
  const uint64_t* digits;     // digit k at digits + k digit_stride ([nl][N])
  size_t digit_stride;
  int dnum;
  const uint64_t* c0;         // [level+1][N]
  const uint64_t* p_mod;      // [level+1] P mod q_l
  uint32_t level;
  size_t key_digit_stride, key_half_stride;
  size_t out_half;            // words from a_j to b_j
  int n;                      // number of babies
  uint32_t max_rot;
  uint32_t rot[kMaxBabies];
  const uint64_t* key[kMaxBabies];
  uint64_t* out[kMaxBabies];
  // queries sharing the keys: query q has digits + q dq, c0 + q cq and writes
  // out[j] + q oq; a CTA stages qk queries' tiles and applies each key value to all
  int nq = 1, qk = 1;
  size_t dq = 0, cq = 0, oq = 0;
  int zfast = 0;                   // query groups fastest in the grid (their key reads meet in L2)
  const uint64_t* own = nullptr;   // as KipArgs::own (the c1 of each query)
  size_t ownq = 0;
  int alpha = 1;
};
void launch_kip_multi(const DevCtx& c, const KipMulti& a, const LimbMap& map);

// D20 L3 work list.  Giants are packed kGiantPack at a time: a term is one
// baby pair x = (x0, x1) with the plaintext u of each giant of the pack that
// uses it (null if none), so every baby value is loaded once per pack.  The
// query-batched kernel packs kWidePack giants (all of a Criteo output block)
// so that each baby value is read once per query.
constexpr int kGiantPack = 4;
constexpr int kWidePack = 16;
template <int GP>
struct MacTermT {
  const uint64_t* x0;         // [nl][N]
  const uint64_t* x1;
  const uint64_t* u[GP];      // plaintext [nl][N] (D-form) or null
};
using MacTerm = MacTermT<kGiantPack>;
using MacTermW = MacTermT<kWidePack>;
// group z: terms [g.x, g.x + g.y), output pairs g.z .. g.z + g.w - 1, each
// written to out + pair out_stride (A) and + nl N (B).  u in D-form; x in
// D-form iff x_dform (else canonical).
// nq queries: query q reads x + q xq and writes out + q oq (plaintexts shared).
// wide: terms are MacTermW (batched kernel, nq >= 1), else MacTerm.
// batch-1 inner sums fed by bulk async copies (kernels_mac_bulk.cu); false if it does not apply
// accumulate: out (+)= the inner sums (compact plans sum a pair's terms over several launches)
// rows [row0, row0 + rows) of map only (rows = 0: all)
bool launch_diag_mac_bulk(const DevCtx& c, const MacTerm* terms, const int4* groups, int n_groups, uint64_t* out,
                          size_t out_stride, size_t half, const LimbMap& map, int nq = 1, size_t xq = 0,
                          size_t oq = 0, int accumulate = 0, int row0 = 0, int rows = 0);
void launch_diag_mac(const DevCtx& c, const void* terms, const int4* groups, int n_groups, double n_u_total,
                     double n_x_distinct, int n_out, uint64_t* out, size_t out_stride, const LimbMap& map,
                     bool x_dform, int nq = 1, size_t xq = 0, size_t oq = 0, bool wide = false);

}  // namespace helrm
