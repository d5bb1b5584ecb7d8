// kernels_ntt_cl.cu -- single-kernel forward NTT for N = 2^16 on a cluster of
// 4 CTAs (sm_100a thread-block clusters + distributed shared memory).
//
// Same transform, twiddles, FP64 butterflies and slot-order output as the
// two-pass k_ntt_fwd<8, 0|2> + k_ntt_fwd<8, 1> (kernels_ntt.cu), but the
// 256 x 256 intermediate never leaves the SMs: CTA r of the cluster
//   pass 1: loads columns [64 r, 64 r + 64) of the limb (256 rows each) and
//           runs the first 8 stages on them into its shared-memory tile;
//   cluster barrier;
//   pass 2: takes 64 of the 256 rows (256-blocks grp[64 r ..]) and reads each
//           row's 4 quarters from the 4 tiles through DSMEM, runs the last 8
//           stages and writes the slot-order output (same swizzled
//           shared-memory permutation as k_ntt_fwd<8, 1>).
// HBM sees exactly one read and one write per coefficient (no scratch round
// trip), and a launch covers any number of limbs (no chunking).
#include <cooperative_groups.h>

#include "internal.h"
#include "fmath.cuh"

namespace cg = cooperative_groups;

namespace helrm {

namespace {
constexpr int kClT = 1024;             // threads per CTA
constexpr int kClPad = 256 + 16;       // pass-2 block stride in shared memory (1 pad word per 16)
constexpr size_t kClSmem = (size_t)64 * kClPad * 8;   // 139,264 B (>= the 128 KiB pass-1 tile)

__device__ __forceinline__ int cpidx(int e) { return e + (e >> 4); }

__device__ __forceinline__ void cl_bfly(double& x, double& y, double2 w, double q) {
  const double r = fm::mmul(y, w.x, w.y, q);
  const double a = x;
  x = a + r;
  y = a - r;
}
}  // namespace

// DIN: source limbs hold centred integer-valued doubles (conversion output)
template <bool DIN>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kClT, 1)
    k_ntt_fwd_cl(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, const PrimeDev* __restrict__ primes,
                 const __grid_constant__ LimbMap map, size_t ss, size_t ds, const uint32_t* __restrict__ grp,
                 const uint8_t* __restrict__ tpos, const uint32_t* __restrict__ lidx,
                 const __grid_constant__ NttEpi epi) {
  extern __shared__ double tile[];
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const size_t limb = blockIdx.x / 4;
  const size_t gl = lidx ? lidx[limb] : limb;
  const PrimeDev& P = primes[map.pr[gl % map.n]];
  const double q = P.qd, qi = P.qinv;
  constexpr int N = 1 << 16;
  const int tid = threadIdx.x;
  double r[16];

  // ---------------- pass 1: columns 64 cr + sub, the first 8 stages ----------------
  {
    const int sub = tid % 64, t = tid / 64;
    const uint64_t* s = src + (gl / map.n) * ss + (gl % map.n) * (size_t)N + 64 * cr + sub;
    const double2* __restrict__ tw = P.tw1;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const uint64_t v = s[(size_t)(t + 16 * k) * 256];
      r[k] = DIN ? fm::bits2d(v) : fm::u2d(v);
    }
#pragma unroll
    for (int st = 0; st < 4; st++) {
      const int half = 8 >> st;
#pragma unroll
      for (int k = 0; k < 16; k++)
        if ((k & half) == 0) cl_bfly(r[k], r[k + half], tw[(1 << st) + (k >> (4 - st))], q);
      if (st & 1) {
#pragma unroll
        for (int k = 0; k < 16; k++) r[k] = fm::cred(r[k], q, qi);
      }
    }
#pragma unroll
    for (int k = 0; k < 16; k++) tile[(t + 16 * k) * 64 + sub] = r[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) r[k] = tile[(16 * t + k) * 64 + sub];
#pragma unroll
    for (int st = 4; st < 8; st++) {
      const int half = 256 >> (st + 1);
#pragma unroll
      for (int k = 0; k < 16; k++)
        if ((k & half) == 0) cl_bfly(r[k], r[k + half], tw[(1 << st) + ((16 * t + k) >> (8 - st))], q);
      if (st & 1) {
#pragma unroll
        for (int k = 0; k < 16; k++) r[k] = fm::cred(r[k], q, qi);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) tile[(16 * t + k) * 64 + sub] = r[k];   // tile[row e][local column]
  }
  cluster.sync();

  // ---------------- pass 2: rows grp[64 cr + sub2], the last 8 stages ----------------
  const int sub2 = tid / 16, t2 = tid % 16;
  const int B = (int)grp[64 * cr + sub2];
#pragma unroll
  for (int k = 0; k < 16; k++) {   // column c = t2 + 16 k lives in CTA c / 64 = k / 4
    const double* rt = cluster.map_shared_rank(tile, k / 4);
    r[k] = rt[B * 64 + ((t2 + 16 * k) & 63)];
  }
  cluster.sync();   // every remote read done before the tiles are reused
  double* sm = tile;
  const double2* __restrict__ twA = P.tw2 + (size_t)B * 256;
#pragma unroll
  for (int st = 0; st < 4; st++) {
    const int half = 8 >> st;
#pragma unroll
    for (int k = 0; k < 16; k++)
      if ((k & half) == 0) cl_bfly(r[k], r[k + half], twA[(1 << st) - 1 + (k >> (4 - st))], q);
    if (st & 1) {
#pragma unroll
      for (int k = 0; k < 16; k++) r[k] = fm::cred(r[k], q, qi);
    }
  }
#pragma unroll
  for (int k = 0; k < 16; k++) sm[sub2 * kClPad + cpidx(t2 + 16 * k)] = r[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 16; k++) r[k] = sm[sub2 * kClPad + cpidx(16 * t2 + k)];
  const double2* __restrict__ twB = twA + 15 + t2;   // phase-B twiddle j of thread t2 at 15 + 16 j + t2
#pragma unroll
  for (int st = 4; st < 8; st++) {
    const int half = 256 >> (st + 1);
#pragma unroll
    for (int k = 0; k < 16; k++)
      if ((k & half) == 0) cl_bfly(r[k], r[k + half], twB[((1 << (st - 4)) - 1 + (k >> (8 - st))) * 16], q);
    if (st & 1) {
#pragma unroll
      for (int k = 0; k < 16; k++) r[k] = fm::cred(r[k], q, qi);
    }
  }
  // slot-order store (kernels_ntt.cu, k_ntt_fwd<8, 1>): 4 groups of 16 interleaving blocks,
  // group gg at smu + 4096 gg, element of rank tp of block i at tp 16 + (i ^ (tp & 15))
  const uint4 tv = *reinterpret_cast<const uint4*>(tpos + (size_t)B * 256 + 16 * t2);
  const uint32_t tw4[4] = {tv.x, tv.y, tv.z, tv.w};
  __syncthreads();
  uint64_t* smu = reinterpret_cast<uint64_t*>(sm);
  {
    const int gg = sub2 / 16, i = sub2 % 16;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const int tp = (tw4[k >> 2] >> (8 * (k & 3))) & 0xff;
      smu[gg * 4096 + tp * 16 + (i ^ (tp & 15))] = fm::d2u(r[k], q, qi, P.rc.q);
    }
  }
  __syncthreads();
  constexpr int n = N >> 1, lgs = 16 - 9, stride = 1 << lgs;
  const int i = tid % 16;
  const uint64_t qq = P.rc.q;
  if (epi.out == nullptr) {
    uint64_t* d = dst + (gl / map.n) * ds + (gl % map.n) * (size_t)N;
#pragma unroll 4
    for (int it = 0; it < 16; it++) {
      const int gg = it / 4, tp = tid / 16 + 64 * (it % 4);
      const int g = 16 * (4 * cr + gg) + i;
      d[(size_t)(g >> lgs) * n + (g & (stride - 1)) + ((size_t)tp << lgs)] = smu[gg * 4096 + tp * 16 + (i ^ (tp & 15))];
    }
  } else {   // fused ModDown / rescale finish: out (+)= (y - t) s mod q
    const size_t pg = gl / map.n, lg = gl % map.n;
    const uint64_t sv = epi.s[lg], svp = epi.sp[lg];
    const uint64_t* yg = epi.y + pg * epi.ys + lg * (size_t)N;
    uint64_t* og = epi.out + pg * epi.os + lg * (size_t)N;
#pragma unroll 4
    for (int it = 0; it < 16; it++) {
      const int gg = it / 4, tp = tid / 16 + 64 * (it % 4);
      const int g = 16 * (4 * cr + gg) + i;
      const size_t at = (size_t)(g >> lgs) * n + (g & (stride - 1)) + ((size_t)tp << lgs);
      uint64_t v = shoup(sub_mod(yg[at], smu[gg * 4096 + tp * 16 + (i ^ (tp & 15))], qq), sv, svp, qq);
      if (epi.accumulate) v = add_mod(v, og[at], qq);
      og[at] = v;
    }
  }
}

bool ntt_fwd_cluster(const DevCtx& c, const uint64_t* src, uint64_t* dst, size_t n_total, const LimbMap& map,
                     size_t ss, size_t ds, bool din, const uint32_t* lidx, const NttEpi& epi) {
  if (c.log_n != 16 || n_total == 0 || n_total > (1u << 29)) return false;
  // measured 46% slower than the two-pass kernels (1 CTA of 1024 threads per SM cannot hide the
  // phase latencies; profiles/r01_ab_cluster.txt): off unless HELRM_NTT_CLUSTER=1
  static const int enabled = getenv("HELRM_NTT_CLUSTER") ? atoi(getenv("HELRM_NTT_CLUSTER")) : 0;
  // small launches (latency-bound chains such as RotSum's ModDown) may still prefer one kernel
  static const size_t small_max = getenv("HELRM_NTT_CLUSTER_MAX") ? (size_t)atoi(getenv("HELRM_NTT_CLUSTER_MAX")) : 0;
  if (!enabled && n_total > small_max) return false;
  auto k = din ? k_ntt_fwd_cl<true> : k_ntt_fwd_cl<false>;
  static bool attr_done[2] = {false, false};
  if (!attr_done[din]) {
    HCUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kClSmem));
    attr_done[din] = true;
  }
  ProfScope ps_(c, "ntt_fwd_cl", 16.0 * c.N * n_total);
  k<<<(unsigned)(4 * n_total), kClT, kClSmem, c.stream>>>(src, dst, c.primes, map, ss, ds, c.ntt_grp, c.ntt_tpos, lidx,
                                                         epi);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
  return true;
}

}  // namespace helrm
