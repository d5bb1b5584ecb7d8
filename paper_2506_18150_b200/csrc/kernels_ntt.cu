// kernels_ntt.cu -- negacyclic NTT / INTT over 64-bit RNS limbs (sm_100a).
//
// D4: NTT_q(a)_i = sum_j a_j psi^{(2i+1) j}.  The library
// keeps NTT-form data in "slot order": position s < N/2 holds the evaluation
// at psi^(5^s), position N/2 + s the one at psi^(-5^s) (D5), so every Galois
// automorphism phi_{5^r} is a cyclic shift by r inside each half -- the
// rotations of the lookup become offset loads instead of gathers.
//
// Forward = Cooley-Tukey with the psi-twist merged into the twiddles
// (psi^bitrev(m+i)), natural input -> bit-reversed output, in two passes of
// batched 2^s-point sub-transforms (N = 2^s1 x 2^8):
//   pass 1: 2^8 column transforms of 2^s1 points (stride 2^8), the first s1
//           stages;  pass 2: 2^s1 row transforms of 256 contiguous points,
//           the last 8 stages, written through bit-reversed -> slot order.
// Each sub-transform is held by S/16 threads x 16 registers: 4 radix-2 stages
// in registers, one shared-memory transpose, the remaining stages in
// registers.  Pass-2 CTAs own the 16 blocks whose slot positions interleave
// (same half, consecutive residues mod N/512), so the permuted stores are
// contiguous runs; pass-2 twiddles are stored in per-block, per-thread order
// so each thread reads its 15 phase-B twiddles contiguously.  Inverse = the
// Gentleman-Sande mirror.  Between the passes the data live in a scratch
// buffer of up to 512 limbs (256 MiB at N = 2^16) per launch: launches up to
// ~200 limbs keep it in the 126 MB L2, the large ModUp launches do not (ncu:
// 1.96 MB of DRAM traffic per limb transform against the algorithmic
// 1 MiB); 64 MiB chunks keep it in L2 but lose more to partial waves
// (profiles/r01_ab_chunk.txt).
//
// Butterfly arithmetic runs on the FP64 pipe (fmath.cuh, q < 2^51): residues
// are exact integer-valued doubles, the product Y W = h + l is split exactly
// with an FMA, the quotient k = rint(Y W / q) comes from one FMA against the
// precomputed W/q (round-to-nearest via the 1.5 2^52 shift), and
// r = (h - k q) + l is exact.  The twiddles are stored centred (|W| <= q/2,
// |W/q| <= 1/2), so mmul accepts any |Y| < 4q < 2^52 and returns |r| <= 0.75 q;
// values stay below 4q by centred reductions (every fourth forward stage on
// the additive inputs, every other inverse stage on the sums).  Measured on B200: ~2.7x the modmul throughput of 64-bit
// integer Shoup (profiles/r01_peak_int.txt).
//
// Limb selection: limb v of a launch is limb lidx[v] of the layout when a
// device table is given (ModUp skips the digit's own limbs this way), else v.
// (A prime-major variant whose pass-2 CTAs loop over several limbs of one
// prime to reuse their twiddles measured slower on B200 -- 2 CTAs/SM instead
// of 4 -- and was dropped, profiles/r01_ab_ntt.txt.)
#include "internal.h"
#include "fmath.cuh"

#include <algorithm>
#include <cstdlib>

namespace helrm {

// pass-2 / pass-A block grouping per log N (12..16): read through the constant
// cache at CTA start instead of a dependent global load
__constant__ uint32_t c_ntt_grp[5][256];

void ntt_set_grp(uint32_t log_n, const uint32_t* grp, size_t n) {
  if (log_n < 12 || log_n > 16 || n > 256) throw Error(HELRM_ERR_CONFIG, "NTT supports 12 <= log N <= 16");
  HCUDA(cudaMemcpyToSymbol(c_ntt_grp, grp, n * 4, (size_t)(log_n - 12) * 256 * 4));
}

namespace {
constexpr int kEPT = 16;                     // elements per thread
constexpr int kTileElems = 4096;             // elements per CTA
constexpr int kThreads = kTileElems / kEPT;  // 256
constexpr int kBlkPad = 256 + 16;            // pass-2 smem block stride (1 pad word per 16)

using fm::cred;
using fm::d2u;
using fm::mmul;
using fm::u2d;

__device__ __forceinline__ int pidx(int e) { return e + (e >> 4); }

__device__ __forceinline__ void ct_bfly(double& x, double& y, double2 w, double q) {
  const double r = mmul(y, w.x, w.y, q);
  const double a = x;
  x = a + r;
  y = a - r;
}
// R: reduce the sum.  Alternating R = true / false from the first stage of a
// pass keeps |x|, |y| < 1.5 q before a reducing stage (so |x - y| < 3q) and
// < 0.75 q + ... before a lazy one; every pass ends below 1.5 q.
template <bool R>
__device__ __forceinline__ void gs_bfly(double& x, double& y, double2 w, double q, double qi) {
  const double s = x + y, dd = x - y;
  x = R ? cred(s, q, qi) : s;
  y = mmul(dd, w.x, w.y, q);
}
}  // namespace

// Forward sub-transforms of S = 2^SLOG points, 16 per thread, TS = S/16
// threads per sub-transform.
//   MODE 0 (pass 1): sub-transform = column (stride 256); twiddles tw1[2^st + i].
//   MODE 1 (pass 2): sub-transform = 256-block B; twiddles tw2[B][...]:
//     [0, 15): phase A, 2^st - 1 + i_loc;  15 + 16 j + t: thread t's phase-B twiddle j.
// The body of one CTA: tile bx of launch limb `limb`; the pass-1 -> pass-2
// intermediate of that limb lives at scratch + slot N.  (A persistent,
// double-buffered variant that prefetched the next tile with cp.async while
// computing this one measured slower: 3 CTAs/SM instead of 4, 7.26 vs 6.81 ms
// per Criteo lookup, 1640 vs 2091 GB/s in the microbenchmark.)
template <int SLOG, int MODE>
__device__ __forceinline__ void ntt_fwd_body(double* sm, unsigned bx, size_t limb, size_t slot,
                                             const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                             const PrimeDev* __restrict__ primes, const LimbMap& map, size_t limb0,
                                             size_t gstride, int log_n, const double* __restrict__ twb,
                                             const uint8_t* __restrict__ tpos, const uint32_t* __restrict__ lidx,
                                             const NttEpi& epi) {
  constexpr int S = 1 << SLOG, TS = S / kEPT, SUBS = kThreads / TS;
  constexpr bool P1 = MODE != 1;  // MODE 2: pass 1 on integer-valued doubles below 4q (conversion output)
  const int N = 1 << log_n;
  const size_t gl = lidx ? lidx[limb0 + limb] : limb0 + limb;
  const int pr = map.pr[gl % map.n];
  const PrimeDev& P = primes[pr];
  const double q = P.qd, qi = P.qinv;
  const double* tb = twb + (size_t)pr * (4 * (size_t)N + 1024);   // [tw1 256][tw2 N][itw1 256][itw2 N] (w, w/q)
  const size_t goff = (gl / map.n) * gstride + (gl % map.n) * (size_t)N;
  const uint64_t* s = src + (P1 ? goff : slot * N);  // pass 1 reads the caller's limb
  uint64_t* d = dst + (P1 ? slot * N : goff);        // pass 2 writes the caller's limb
  const int tid = threadIdx.x;
  const int sub = P1 ? tid % SUBS : tid / TS;
  const int t = P1 ? tid / SUBS : tid % TS;
  const int gsub = P1 ? bx * SUBS + sub : (int)c_ntt_grp[log_n - 12][bx * SUBS + sub];
  const double2* __restrict__ tw1 = reinterpret_cast<const double2*>(tb);
  const double2* __restrict__ twA = P1 ? tw1 : reinterpret_cast<const double2*>(tb + 512) + (size_t)gsub * 256;
  double r[kEPT];
  {
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int e = t + TS * k;
      if (MODE == 2) {
        r[k] = __longlong_as_double((long long)s[(size_t)e * 256 + gsub]);
      } else if (MODE == 0) {
        r[k] = u2d(s[(size_t)e * 256 + gsub]);
      } else {
        r[k] = __longlong_as_double((long long)s[(size_t)gsub * 256 + e]);
      }
    }
  }
  if (!P1 && epi.out != nullptr && (tid & 15) == 0) {
    // fused ModDown / rescale epilogue: its y (and out) lines towards L2 now, so the reads at
    // the end of the CTA do not add an HBM round trip (one thread per 128-byte line)
    const int lgs = log_n - 9, g = (int)bx * 16;
    const size_t pbase = (size_t)(g >> lgs) * (size_t)(N >> 1) + (g & ((1 << lgs) - 1));
    const size_t gstep = (size_t)16 << lgs, pg = gl / map.n, lg = gl % map.n;
    const uint64_t* yg = epi.y + pg * epi.ys + lg * (size_t)N + pbase + ((size_t)(tid / 16) << lgs);
    const uint64_t* og = epi.out + pg * epi.os + lg * (size_t)N + pbase + ((size_t)(tid / 16) << lgs);
#pragma unroll
    for (int it = 0; it < 16; it++) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(yg + it * gstep));
      if (epi.accumulate) asm volatile("prefetch.global.L2 [%0];" ::"l"(og + it * gstep));
    }
  }
  // phase A: stages 0..3 on layout e = t + TS k (twiddles independent of t)
  // Lazy reduction: a butterfly's product term is reduced by mmul (|r| <= 0.75 q for any
  // |y| < 4q, centred twiddles), so only the additive inputs grow, by 0.75 q per stage.
  // Reducing the additive inputs (half the elements) before stages 0 and 4 keeps every
  // value below 0.5 q + 4 x 0.75 q = 3.5 q < 2^52 (q < 2^50).
#pragma unroll
  for (int st = 0; st < 4; st++) {
    const int half = 8 >> st;
    if ((st & 3) == 0) {
#pragma unroll
      for (int k = 0; k < kEPT; k++)
        if ((k & half) == 0) r[k] = cred(r[k], q, qi);
    }
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      if ((k & half) == 0) {
        // MODE 0: tw1[2^st + i]; MODE 1: tw2[B][2^st - 1 + i]
        const double2 w = P1 ? twA[(1 << st) + (k >> (4 - st))] : twA[(1 << st) - 1 + (k >> (4 - st))];
        ct_bfly(r[k], r[k + half], w, q);
      }
    }
  }
  if (SLOG > 4) {
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int e = t + TS * k;
      if (P1) sm[e * SUBS + sub] = r[k];
      else sm[sub * kBlkPad + pidx(e)] = r[k];
    }
    // pass 2: a 256-point block is held by 16 consecutive threads (half a warp) in its own
    // shared-memory rows, so the exchange only needs the warp; pass 1's columns span the CTA
    if (P1) __syncthreads();
    else __syncwarp();
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int e = kEPT * t + k;
      r[k] = P1 ? sm[e * SUBS + sub] : sm[sub * kBlkPad + pidx(e)];
    }
    const double2* __restrict__ twB = P1 ? tw1 : twA + 15 + t;  // phase-B twiddle j of thread t at 15 + 16 j + t
#pragma unroll
    for (int st = 4; st < SLOG; st++) {
      const int half = S >> (st + 1);
      if ((st & 3) == 0) {
#pragma unroll
        for (int k = 0; k < kEPT; k++)
          if ((k & half) == 0) r[k] = cred(r[k], q, qi);
      }
#pragma unroll
      for (int k = 0; k < kEPT; k++) {
        if ((k & half) == 0) {
          const int e = kEPT * t + k;
          double2 w;
          if (P1) w = twB[(1 << st) + (e >> (SLOG - st))];
          else w = twB[((1 << (st - 4)) - 1 + (k >> (SLOG - st))) * 16];
          ct_bfly(r[k], r[k + half], w, q);
        }
      }
    }
  }
  // pass 1 hands values below 3.5 q to pass 2 (whose first stage reduces its additive inputs);
  // pass 2 reduces everything once before canonicalising
  if (!P1) {
#pragma unroll
    for (int k = 0; k < kEPT; k++) r[k] = cred(r[k], q, qi);
  }
  if (P1) {
    // centred doubles into the scratch, natural row positions
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int e = SLOG > 4 ? kEPT * t + k : t + TS * k;
      d[(size_t)e * 256 + gsub] = (uint64_t)__double_as_longlong(r[k]);
    }
  } else {
    // slot-order store through shared memory: element e of block `sub` has
    // rank tp(e) among its block's slot positions; it goes to
    // smem[tp 16 + (sub ^ (tp & 15))].  tp(16 t + k) mod 16 is distinct over
    // the 16 threads t of a block for every k (checked for every block at
    // context creation), so the swizzled scatter and the row-wise read are
    // both bank-conflict free.
    const uint4 tv = *reinterpret_cast<const uint4*>(tpos + (size_t)gsub * 256 + kEPT * t);
    const uint32_t tw4[4] = {tv.x, tv.y, tv.z, tv.w};
    __syncthreads();
    uint64_t* smu = reinterpret_cast<uint64_t*>(sm);
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int tp = (tw4[k >> 2] >> (8 * (k & 3))) & 0xff;
      smu[tp * 16 + (sub ^ (tp & 15))] = fm::c2u(r[k], P.rc.q);   // centred by the last stage's reduction
    }
    __syncthreads();
    // block of rank g = 16 cta + i lives at slot positions (g / stride) n +
    // (g % stride) + stride tp; for a given tp the 16 blocks are adjacent
    const int n = N >> 1, lgs = log_n - 9, stride = 1 << lgs;
    const int i = tid % 16, g = (int)bx * 16 + i;   // idx % 16 == tid % 16
    const size_t pbase = (size_t)(g >> lgs) * n + (g & (stride - 1));
    // thread tid handles tp = tid / 16 + 16 it: tp & 15 is constant per thread, so the shared
    // index advances by 256 and the global one by 16 << lgs per iteration
    const int tp0 = tid / 16;
    const uint64_t* sp0 = smu + tp0 * 16 + (i ^ (tp0 & 15));
    const size_t gstep = (size_t)16 << lgs;
    if (epi.out == nullptr) {
      uint64_t* dg = d + pbase + ((size_t)tp0 << lgs);
#pragma unroll
      for (int it = 0; it < 16; it++) dg[it * gstep] = sp0[256 * it];
    } else {   // fused ModDown / rescale finish: out (+)= (y - t) s mod q
      const size_t pg = gl / map.n, lg = gl % map.n;
      const uint64_t qq = P.rc.q, sv = epi.s[lg], svp = epi.sp[lg];
      const uint64_t* yg = epi.y + pg * epi.ys + lg * (size_t)N + pbase + ((size_t)tp0 << lgs);
      uint64_t* og = epi.out + pg * epi.os + lg * (size_t)N + pbase + ((size_t)tp0 << lgs);
      // all 16 loads of y (and of out when accumulating) in flight at once: the epilogue's
      // HBM reads otherwise serialise per 4-element group at the end of every CTA
      uint64_t yv[16];
#pragma unroll
      for (int it = 0; it < 16; it++) yv[it] = yg[it * gstep];
#pragma unroll
      for (int it = 0; it < 16; it++) {
        uint64_t v = shoup(sub_mod(yv[it], sp0[256 * it], qq), sv, svp, qq);
        if (epi.accumulate) v = add_mod(v, og[it * gstep], qq);
        og[it * gstep] = v;
      }
    }
  }
}

template <int SLOG, int MODE>
__global__ void __launch_bounds__(kThreads, 4) k_ntt_fwd(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                      const PrimeDev* __restrict__ primes,
                                                      const __grid_constant__ LimbMap map, size_t limb0, size_t gstride, int log_n,
                                                      const uint32_t* __restrict__ grp,
                                                      const double* __restrict__ twb,
                                                      const uint8_t* __restrict__ tpos,
                                                      const uint32_t* __restrict__ lidx,
                                                      const __grid_constant__ NttEpi epi) {
  pdl_wait_trigger();
  __shared__ double sm[MODE != 1 ? kTileElems : 16 * kBlkPad];
  (void)grp;
  ntt_fwd_body<SLOG, MODE>(sm, blockIdx.x, blockIdx.y, blockIdx.y, src, dst, primes, map, limb0, gstride, log_n, twb,
                           tpos, lidx, epi);
}

// Inverse (Gentleman-Sande), mirror of k_ntt_fwd.
//   MODE 1 (pass A): blocks gathered from slot order, the last 8 stages;
//   MODE 0 (pass B): columns, the first s1 stages, times N^-1, natural order.
template <int SLOG, int MODE>
__global__ void __launch_bounds__(kThreads, 4) k_ntt_inv(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                      const PrimeDev* __restrict__ primes,
                                                      const __grid_constant__ LimbMap map, size_t limb0, size_t gstride, int log_n,
                                                      const uint32_t* __restrict__ grp,
                                                      const double* __restrict__ twb,
                                                      const uint8_t* __restrict__ tpos,
                                                      const double2* __restrict__ post,
                                                      const uint32_t* __restrict__ lidx) {
  pdl_wait_trigger();
  constexpr int S = 1 << SLOG, TS = S / kEPT, SUBS = kThreads / TS;
  __shared__ double sm[MODE == 0 ? kTileElems : 16 * kBlkPad];
  const int N = 1 << log_n;
  const size_t limb = blockIdx.y;
  const size_t gl = lidx ? lidx[limb0 + limb] : limb0 + limb;
  const int pr = map.pr[gl % map.n];
  const PrimeDev& P = primes[pr];
  const double q = P.qd, qi = P.qinv;
  const double* tb = twb + (size_t)pr * (4 * (size_t)N + 1024) + 2 * (size_t)N + 512;   // itw1, itw2
  const size_t goff = (gl / map.n) * gstride + (gl % map.n) * (size_t)N;
  const uint64_t* s = src + (MODE == 1 ? goff : limb * N);  // pass A gathers the caller's limb
  uint64_t* d = dst + (MODE == 1 ? limb * N : goff);        // pass B writes the caller's limb
  const int tid = threadIdx.x;
  const int sub = MODE == 0 ? tid % SUBS : tid / TS;
  const int t = MODE == 0 ? tid / SUBS : tid % TS;
  const int gsub = MODE == 0 ? blockIdx.x * SUBS + sub : (int)c_ntt_grp[log_n - 12][blockIdx.x * SUBS + sub];
  const double2* __restrict__ itw1 = reinterpret_cast<const double2*>(tb);
  const double2* __restrict__ twA = MODE == 0 ? itw1 : reinterpret_cast<const double2*>(tb + 512) + (size_t)gsub * 256;
  if (MODE == 1) {   // the block's 4 KiB of twiddles towards L1 early, 2 lines per thread of the block
    // (pass A 0.41 -> 0.39 ms per Criteo lookup; the same prefetch slows the forward pass 2)
    const char* tl = reinterpret_cast<const char*>(twA);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(tl + 128 * t));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(tl + 128 * (t + 16)));
  }
  double r[kEPT];
  if (MODE == 1) {
    const int n = N >> 1, lgs = log_n - 9, stride = 1 << lgs;
    const int i = tid % 16, g = blockIdx.x * 16 + i;
    const uint64_t* sg = s + (size_t)(g >> lgs) * n + (g & (stride - 1));
#pragma unroll
    for (int idx = tid; idx < kTileElems; idx += kThreads) {   // swizzled gather, as the forward store
      const int tp = idx / 16;
      sm[tp * 16 + (i ^ (tp & 15))] = u2d(sg[(size_t)tp << lgs]);
    }
    const uint4 tv = *reinterpret_cast<const uint4*>(tpos + (size_t)gsub * 256 + kEPT * t);
    const uint32_t tw4[4] = {tv.x, tv.y, tv.z, tv.w};
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int tp = (tw4[k >> 2] >> (8 * (k & 3))) & 0xff;
      r[k] = sm[tp * 16 + (sub ^ (tp & 15))];
    }
  } else {
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int e = SLOG > 4 ? kEPT * t + k : t + TS * k;
      r[k] = __longlong_as_double((long long)s[(size_t)e * 256 + gsub]);
    }
  }
  if (SLOG > 4) {
    const double2* __restrict__ twB = MODE == 0 ? itw1 : twA + 15 + t;  // phase-B twiddle j of thread t at 15 + 16 j + t
#pragma unroll
    for (int st = SLOG - 1; st >= 4; st--) {
      const int half = S >> (st + 1);
#pragma unroll
      for (int k = 0; k < kEPT; k++) {
        if ((k & half) == 0) {
          const int e = kEPT * t + k;
          double2 w;
          if (MODE == 0) w = twB[(1 << st) + (e >> (SLOG - st))];
          else w = twB[((1 << (st - 4)) - 1 + (k >> (SLOG - st))) * 16];
          if (((SLOG - 1 - st) & 1) == 0) gs_bfly<true>(r[k], r[k + half], w, q, qi);
          else gs_bfly<false>(r[k], r[k + half], w, q, qi);
        }
      }
    }
    if (MODE == 1) __syncthreads();
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int e = kEPT * t + k;
      if (MODE == 0) sm[e * SUBS + sub] = r[k];
      else sm[sub * kBlkPad + pidx(e)] = r[k];
    }
    if (MODE == 0) __syncthreads();
    else __syncwarp();   // pass A: each block's rows belong to its half-warp (as the forward pass 2)
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const int e = t + TS * k;
      r[k] = MODE == 0 ? sm[e * SUBS + sub] : sm[sub * kBlkPad + pidx(e)];
    }
  }
#pragma unroll
  for (int st = 3; st >= 0; st--) {
    const int half = 8 >> st;
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      if ((k & half) == 0) {
        const double2 w = MODE == 0 ? twA[(1 << st) + (k >> (4 - st))] : twA[(1 << st) - 1 + (k >> (4 - st))];
        if (((SLOG - 1 - st) & 1) == 0) gs_bfly<true>(r[k], r[k + half], w, q, qi);
        else gs_bfly<false>(r[k], r[k + half], w, q, qi);
      }
    }
  }
  if (MODE == 1) {
#pragma unroll
    for (int k = 0; k < kEPT; k++) d[(size_t)gsub * 256 + t + TS * k] = (uint64_t)__double_as_longlong(r[k]);
  } else {
    // N^-1, or N^-1 times a per-limb factor (the y-form of a base conversion)
    const double2 nm = post ? post[gl % map.n] : P.ninvd;
#pragma unroll
    for (int k = 0; k < kEPT; k++) {
      const double v = mmul(r[k], nm.x, nm.y, q);
      d[(size_t)(t + TS * k) * 256 + gsub] = fm::c2u(v, P.rc.q);   // |v| <= 0.75 q after mmul
    }
  }
}

// ---------------------------------------------------------------- launchers
static size_t chunk_limbs(int N) {
  static const size_t env = getenv("HELRM_NTT_CHUNK") ? (size_t)atoi(getenv("HELRM_NTT_CHUNK")) : 0;
  // 256 MiB of scratch per chunk (512 limbs at N = 2^16): larger launches lose less to partial
  // waves; measured 8.66 -> 8.32 ms per Criteo lookup against 64 MiB chunks (profiles/r01_ab_chunk.txt)
  size_t ch = (env ? env : 512) * 65536 / (size_t)N;
  return ch > 65535 ? 65535 : ch;
}

size_t ntt_scratch_words(int log_n) { return chunk_limbs(1 << log_n) * ((size_t)1 << log_n); }

template <int SLOG>
static void fwd_chunk(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, unsigned cnt,
                      const LimbMap& map, size_t off, size_t ss, size_t ds, bool din, const uint32_t* lidx,
                      const NttEpi& epi) {
  constexpr int TS = (1 << SLOG) / kEPT;
  const int g1 = TS, g2 = (c.N / 256) / 16;
  {
    ProfScope ps_(c, "ntt_fwd_p1", 8.0 * c.N * cnt);
    auto k1 = din ? k_ntt_fwd<SLOG, 2> : k_ntt_fwd<SLOG, 0>;
    launch_pdl(k1, dim3(g1, cnt), dim3(kThreads), 0, c.stream, src, scratch, c.primes, map, off, ss, c.log_n,
               c.ntt_grp, c.ntt_twb, c.ntt_tpos, lidx, epi);
  }
  {
    ProfScope ps_(c, "ntt_fwd_p2", 8.0 * c.N * cnt);
    launch_pdl(k_ntt_fwd<8, 1>, dim3(dim3(g2, cnt)), dim3(kThreads), 0, c.stream, scratch, dst, c.primes, map, off, ds,
               c.log_n, c.ntt_grp, c.ntt_twb, c.ntt_tpos, lidx, epi);
  }
  *c.launches += 2;
}

template <int SLOG>
static void inv_chunk(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, unsigned cnt,
                      const LimbMap& map, size_t off, size_t ss, size_t ds, const double2* post,
                      const uint32_t* lidx) {
  constexpr int TS = (1 << SLOG) / kEPT;
  const int g1 = TS, g2 = (c.N / 256) / 16;
  {
    ProfScope ps_(c, "ntt_inv_pa", 8.0 * c.N * cnt);
    launch_pdl(k_ntt_inv<8, 1>, dim3(dim3(g2, cnt)), dim3(kThreads), 0, c.stream, src, scratch, c.primes, map, off, ss, c.log_n, c.ntt_grp, c.ntt_twb, c.ntt_tpos, nullptr, lidx);
  }
  {
    ProfScope ps_(c, "ntt_inv_pb", 8.0 * c.N * cnt);
    launch_pdl(k_ntt_inv<SLOG, 0>, dim3(dim3(g1, cnt)), dim3(kThreads), 0, c.stream, scratch, dst, c.primes, map, off, ds, c.log_n, c.ntt_grp, c.ntt_twb, c.ntt_tpos, post, lidx);
  }
  *c.launches += 2;
}

template <bool FWD>
static void ntt_any(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, size_t n_total,
                    const LimbMap& map, size_t ss, size_t ds, const double2* post, bool din, const uint32_t* lidx,
                    const NttEpi& epi = NttEpi{}) {
  if (ss == 0) ss = (size_t)map.n * c.N;
  if (ds == 0) ds = (size_t)map.n * c.N;
  const size_t ch = chunk_limbs(c.N);
  for (size_t off = 0; off < n_total; off += ch) {
    const unsigned cnt = (unsigned)std::min(ch, n_total - off);
#define HELRM_NTT_CASE(LG, SL)                                                  \
  case LG:                                                                      \
    if (FWD) fwd_chunk<SL>(c, src, dst, scratch, cnt, map, off, ss, ds, din, lidx, epi);        \
    else inv_chunk<SL>(c, src, dst, scratch, cnt, map, off, ss, ds, post, lidx);        \
    break;
    switch (c.log_n) {
      HELRM_NTT_CASE(12, 4)
      HELRM_NTT_CASE(13, 5)
      HELRM_NTT_CASE(14, 6)
      HELRM_NTT_CASE(15, 7)
      HELRM_NTT_CASE(16, 8)
      default: throw Error(HELRM_ERR_CONFIG, "NTT supports 12 <= log N <= 16");
    }
#undef HELRM_NTT_CASE
  }
  HCUDA(cudaGetLastError());
}

void launch_ntt_fwd(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, size_t n_total,
                    const LimbMap& map, size_t ss, size_t ds, bool din, const uint32_t* lidx, const NttEpi* epi) {
  ntt_any<true>(c, src, dst, scratch, n_total, map, ss, ds, nullptr, din, lidx, epi ? *epi : NttEpi{});
}

void launch_ntt_inv(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, size_t n_total,
                    const LimbMap& map, size_t ss, size_t ds, const double2* post, const uint32_t* lidx) {
  ntt_any<false>(c, src, dst, scratch, n_total, map, ss, ds, post, false, lidx);
}

}  // namespace helrm
