// kernels_rns.cu -- element-wise RNS kernels of the lookup (sm_100a):
// samplers (D9/D10), signed reduction, modular add/sub/mul, Galois
// automorphisms as slot-order shifts (D8), the ModDown / rescale finishing steps
// (D16/D17), the key inner product with fused automorphism (D18), and the
// plaintext-diagonal multiply-accumulate of the BSGS inner sums (D20 L3).
//
// Layout: polynomials are [limb][N] uint64, NTT form in slot order; one
// thread per coefficient, blockIdx.y = limb, coalesced 8-byte accesses.
#include <cuda_pipeline.h>

#include "internal.h"
#include "fmath.cuh"

namespace helrm {

namespace {
constexpr int kT = 256;

__device__ __forceinline__ uint32_t rot_src(uint32_t p, uint32_t rot, uint32_t n) {
  // phi_{5^rot} in slot order: out[(s, j)] = in[(s, j + rot mod n)]
  uint32_t half = p >= n ? n : 0;
  uint32_t j = p - half + rot;
  j = j >= n ? j - n : j;
  return half + j;
}
}  // namespace

__global__ void k_reduce_signed(const int64_t* __restrict__ m, uint64_t* __restrict__ out,
                                const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const uint64_t q = primes[map.pr[l]].rc.q;
  const int64_t v = m[i];
  uint64_t r;
  if (v >= 0) {
    r = (uint64_t)v % q;
  } else {
    r = (uint64_t)(-v) % q;
    r = r ? q - r : 0;
  }
  out[(size_t)l * N + i] = r;
}

// UniformMod(q) of natural NTT index i = (w_{2i} 2^64 + w_{2i+1}) mod q, placed
// at its slot-order position.
__global__ void k_sample_uniform_ntt(uint64_t* __restrict__ out, const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map,
                                     uint32_t log_n, const uint32_t* __restrict__ slotpos, uint64_t seed,
                                     uint64_t purpose, uint64_t a, uint64_t b, const __grid_constant__ LimbMap ids) {
  const uint32_t N = 1u << log_n;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const RedConst rc = primes[map.pr[l]].rc;
  const uint64_t base = prng_base(seed, prng_stream(purpose, a, b, ids.pr[l]));
  const uint64_t w0 = prng_word(base, 2ull * i), w1 = prng_word(base, 2ull * i + 1);
  const uint32_t r = __brev(i) >> (32 - log_n);
  out[(size_t)l * N + slotpos[r]] = reduce128(w0, w1, rc);
}

// kind 0: ternary (w mod 3 -> 0, +1, -1); kind 1: CDT Gaussian (D10)
__global__ void k_sample_small(int64_t* __restrict__ out, uint32_t N, uint64_t base, int kind,
                               const uint64_t* __restrict__ cdt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const uint64_t w0 = prng_word(base, 2ull * i);
  if (kind == 0) {
    const uint64_t r = w0 % 3;
    out[i] = r == 0 ? 0 : (r == 1 ? 1 : -1);
  } else {
    const uint64_t w1 = prng_word(base, 2ull * i + 1);
    int64_t mag = 19;
    for (int k = 0; k < 19; k++)
      if (w0 < cdt[k]) { mag = k; break; }
    out[i] = ((w1 & 1) && mag > 0) ? -mag : mag;
  }
}

// op 0: a + b, 1: a - b, 2: a * b, 3: -a
__global__ void k_binary(int op, const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                         uint64_t* __restrict__ out, const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N) {
  pdl_wait_trigger();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const RedConst rc = primes[map.pr[l]].rc;
  const size_t o = (size_t)l * N + i;
  const uint64_t x = a[o];
  uint64_t r;
  switch (op) {
    case 0: r = add_mod(x, b[o], rc.q); break;
    case 1: r = sub_mod(x, b[o], rc.q); break;
    case 2: r = mul_mod(x, b[o], rc); break;
    default: r = x ? rc.q - x : 0; break;
  }
  out[o] = r;
}

// out[l] = a[l] * s[l] (shoup constants per limb)
__global__ void k_scalar_mul(const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                             const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N,
                             const uint64_t* __restrict__ s, const uint64_t* __restrict__ sp, int dform_out,
                             size_t as, size_t os) {
  pdl_wait_trigger();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const uint64_t q = primes[map.pr[l]].rc.q;
  const size_t o = (size_t)l * N + i;
  const uint64_t v = shoup(a[blockIdx.z * as + o], s[l], sp[l], q);
  out[blockIdx.z * os + o] = dform_out ? fm::d2bits(fm::u2c(v, (double)q)) : v;
}

// in-place conversion to (dir 1) / from (dir 0) D-form; word i belongs to limb
// (i / N) mod map.n of a repeating [map.n][N] layout
__global__ void k_dform(uint64_t* __restrict__ x, size_t n, uint32_t log_n, const PrimeDev* __restrict__ primes,
                        const __grid_constant__ LimbMap map, int dir) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const PrimeDev& P = primes[map.pr[(i >> log_n) % map.n]];
    x[i] = dir ? fm::d2bits(fm::u2c(x[i], P.qd)) : fm::c2u(fm::bits2d(x[i]), P.rc.q);
  }
}

// out[l][p] = a[l][rot_src(p)]  (+ out if accumulate)
__global__ void k_automorph(const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                            const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N, uint32_t rot,
                            int accumulate) {
  pdl_wait_trigger();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (p >= N) return;
  const uint64_t v = a[(size_t)l * N + rot_src(p, rot, N / 2)];
  const size_t o = (size_t)l * N + p;
  out[o] = accumulate ? add_mod(out[o], v, primes[map.pr[l]].rc.q) : v;
}

// D14 from y-form sources: out_gk[r][i] = sum_b y_g[row0 + b][i] cf_kr[b] mod q_r (as an
// integer-valued double below 4q, not yet reduced when nb <= 4) for
// every row r (the table also reproduces a digit's own rows); the CTA stages
// its conversion's table in shared memory, each thread loads its nb sources
// once and produces all rows.  grid (N/256, G ncv).

template <int NB, int PT = 1>
__global__ void __launch_bounds__(256) k_conv_rows(const ConvRowDev* __restrict__ tab, int ncv, int rows,
                                                   const uint64_t* __restrict__ y, size_t y_stride,
                                                   uint64_t* __restrict__ out, size_t osg, size_t osk, uint32_t N) {
  pdl_wait_trigger();
  __shared__ ConvRowDev st[kMaxLimbs];
  const int g = blockIdx.y / ncv, k = blockIdx.y % ncv;
  const ConvRowDev* tk = tab + (size_t)k * rows;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) st[r] = tk[r];
  __syncthreads();
  // PT positions per thread, 256 apart (each table row read from shared memory once per PT outputs)
  const uint32_t i = blockIdx.x * blockDim.x * PT + threadIdx.x;
  if (i >= N) return;
  const int nb = st[0].nb;
  const uint64_t* src = y + (size_t)g * y_stride + (size_t)st[0].src_row0 * N + i;
  double v[PT][NB];
#pragma unroll
  for (int u = 0; u < PT; u++)
#pragma unroll
    for (int b = 0; b < NB; b++) v[u][b] = b < nb ? fm::u2d(src[(size_t)b * N + 256 * u]) : 0.0;  // missing sources = 0
  uint64_t* o = out + (size_t)g * osg + (size_t)k * osk + i;
#pragma unroll 2
  for (int r = 0; r < rows; r++) {
    const int orow = st[r].out_row;
    if (orow < 0) continue;
    const double q = st[r].q, qi = st[r].qinv;
    double2 cf[NB];
#pragma unroll
    for (int b = 0; b < NB; b++) cf[b] = st[r].cf[b];
#pragma unroll
    for (int u = 0; u < PT; u++) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < NB; b++) acc += fm::mmul(v[u][b], cf[b].x, cf[b].y, q);  // each |.| <= 0.75 q
      // every conversion output feeds a forward NTT (MODE 2), whose butterflies take inputs
      // below 4q: with NB <= 4 terms |acc| <= 3q, so the final reduction is left to it
      o[(size_t)orow * N + 256 * u] = (uint64_t)__double_as_longlong(NB <= 4 ? acc : fm::cred(acc, q, qi));
    }
  }
}

// D17: r = ((x + h) mod q_l) - h, then r mod q_i for the remaining limbs; z = polynomial
__global__ void k_rescale_prep(const uint64_t* __restrict__ xl, size_t xs, uint64_t ql, uint64_t* __restrict__ out,
                               size_t os, const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map,
                               uint32_t N) {
  pdl_wait_trigger();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const uint64_t h = (ql - 1) / 2;
  const uint64_t v = xl[blockIdx.z * xs + i];
  const uint64_t q = primes[map.pr[l]].rc.q;
  uint64_t r;
  if (v <= h) {
    r = v % q;                          // r = v >= 0
  } else {
    const uint64_t mag = (ql - v) % q;  // r = v - ql < 0
    r = mag ? q - mag : 0;
  }
  out[blockIdx.z * os + (size_t)l * N + i] = r;
}

// D18 key inner product with the automorphism fused into the loads:
//   out0[l][p] (+)= [l < add_rows] mul_l phi(add0)[l][p] + sum_k phi(D_k)[l][p] b_k[l][p]
//   out1[l][p] (+)= sum_k phi(D_k)[l][p] a_k[l][p]
// (add0 = c0 with mul = [P]_q for a lazy rotation; add0 = A with mul = 1 for
// the giant step's phi(A) + KS(B'), D20 L4).  Keys in D-form; the products
// are exact FP64 MACs (fmath.cuh), dnum + 1 <= kFAccTerms terms.
// DNUM is a template parameter so that all 3 DNUM loads of a thread are in
// flight before the first product (a runtime bound made the compiler convert
// each digit right after its load, serialising the memory latency).
template <int DNUM, int QR>
__global__ void __launch_bounds__(256, QR == 1 ? 4 : 3) k_kip(const __grid_constant__ KipArgs a, const PrimeDev* __restrict__ primes,
                                             const __grid_constant__ LimbMap map, uint32_t N) {
  pdl_wait_trigger();
  // work item w = (tile, limb); a grid smaller than the work loops (persistent CTAs)
  const uint32_t tiles = N / blockDim.x, total = tiles * (uint32_t)(a.rows ? a.rows : map.n);
  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
  const uint32_t p = (w % tiles) * blockDim.x + threadIdx.x;
  const int l = a.row0 + (int)(w / tiles);
  const uint32_t chain = map.pr[l];
  const PrimeDev& P = primes[chain];
  const double q = P.qd, qi = P.qinv;
  const uint32_t sp = rot_src(p, a.rot, N / 2);
  const uint64_t* kb = a.key + (size_t)chain * N + p;   // D-form key
  const uint64_t* dg = a.digits + (size_t)l * N + sp;
  const int kown = (a.own && l <= a.level) ? l / a.alpha : -1;   // digit whose own limb this row is
  const uint64_t* og = a.own ? a.own + (size_t)l * N + sp : nullptr;
  const bool add = a.add0 != nullptr && l < a.add_rows;
  const double amul = add && a.add_mul ? fm::u2c(a.add_mul[l], q) : 1.0;
  const bool h0 = a.halves & 1, h1 = a.halves & 2;   // which outputs (and key halves) this launch computes
  uint64_t kv0[DNUM], kv1[DNUM];
#pragma unroll
  for (int k = 0; k < DNUM; k++) {
    kv0[k] = kv1[k] = 0;
    if (a.nq == 1) {
      if (h0) kv0[k] = __ldcs(kb + (size_t)k * a.key_digit_stride);
      if (h1) kv1[k] = __ldcs(kb + (size_t)k * a.key_digit_stride + a.key_half_stride);
    } else {
      if (h0) kv0[k] = kb[(size_t)k * a.key_digit_stride];
      if (h1) kv1[k] = kb[(size_t)k * a.key_digit_stride + a.key_half_stride];
    }
  }
  const size_t o = (size_t)l * N + p;
  // QR queries per round: QR (DNUM + 1) loads in flight against the key held in registers
  for (int q0 = 0; q0 < a.nq; q0 += QR) {
    const int nr = a.nq - q0 >= QR ? QR : a.nq - q0;
    uint64_t dv[QR][DNUM], av[QR], pv0[QR], pv1[QR];
#pragma unroll
    for (int r = 0; r < QR; r++) {
      if (r < nr) {
        const uint64_t* dq = dg + (size_t)(q0 + r) * a.dq;
#pragma unroll
        for (int k = 0; k < DNUM; k++)
          dv[r][k] = k == kown ? og[(size_t)(q0 + r) * a.ownq] : dq[(size_t)k * a.digit_stride];
        av[r] = add && h0 ? a.add0[(size_t)(q0 + r) * a.aq + (size_t)l * N + sp] : 0;
        // the accumulated outputs are fetched with the operands (one memory round trip per thread)
        pv0[r] = a.accumulate && h0 ? a.out0[(size_t)(q0 + r) * a.oq + o] : 0;
        pv1[r] = a.accumulate && h1 ? a.out1[(size_t)(q0 + r) * a.oq + o] : 0;
      }
    }
#pragma unroll
    for (int r = 0; r < QR; r++) {
      if (r < nr) {
        fm::FAcc acc0, acc1;
#pragma unroll
        for (int k = 0; k < DNUM; k++) {
          const double d = fm::u2d(dv[r][k]);
          if (h0) fm::fmac(acc0, d, fm::bits2d(kv0[k]));
          if (h1) fm::fmac(acc1, d, fm::bits2d(kv1[k]));
        }
        if (add) fm::fmac(acc0, fm::u2d(av[r]), amul);
        uint64_t r0 = fm::c2u(fm::fred(acc0, q, qi), P.rc.q), r1 = fm::c2u(fm::fred(acc1, q, qi), P.rc.q);
        if (a.accumulate) {
          r0 = add_mod(r0, pv0[r], P.rc.q);
          r1 = add_mod(r1, pv1[r], P.rc.q);
        }
        if (h0) a.out0[(size_t)(q0 + r) * a.oq + o] = r0;
        if (h1) a.out1[(size_t)(q0 + r) * a.oq + o] = r1;
      }
    }
  }
  }
}

// A run of giant steps into one output block (KipGiants): every giant adds
// dnum + 1 exact FP64 MACs per output to the same accumulators (folded every
// 2 giants while 2 (dnum + 1) <= kFAccTerms, else every giant), the output
// block is read once and written once.  NQ queries (the LLM's output blocks)
// share each key value: the key is loaded once per giant for all of them.
template <int DNUM, int NQ>
__global__ void __launch_bounds__(256, NQ > 1 ? 2 : 3) k_kip_giants(const __grid_constant__ KipGiants a,
                                                                   const PrimeDev* __restrict__ primes,
                                                                   const __grid_constant__ LimbMap map, uint32_t N) {
  pdl_wait_trigger();
  constexpr int kFoldEvery = 2 * (DNUM + 1) <= fm::kFAccTerms ? 2 : 1;
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = a.row0 + (int)blockIdx.y;
  const uint32_t chain = map.pr[l];
  const PrimeDev& P = primes[chain];
  const double q = P.qd, qi = P.qinv;
  const size_t o = (size_t)l * N + p;
  uint64_t pv0[NQ], pv1[NQ];
#pragma unroll
  for (int r = 0; r < NQ; r++) {
    pv0[r] = a.out0[(size_t)r * a.oq + o];
    pv1[r] = a.out1[(size_t)r * a.oq + o];
  }
  const int kown = l <= a.level ? l / a.alpha : -1;
  const bool add = l < a.add_rows;
  fm::FAcc acc0[NQ], acc1[NQ];
  for (int g = 0; g < a.n; g++) {
    if (g > 0 && g % kFoldEvery == 0) {
#pragma unroll
      for (int r = 0; r < NQ; r++) {
        fm::fold(acc0[r], q, qi);
        fm::fold(acc1[r], q, qi);
      }
    }
    const uint32_t sp = rot_src(p, a.rot[g], N / 2);
    const uint64_t* kb = a.key[g] + (size_t)chain * N + p;
    const uint64_t* dg = a.digits[g] + (size_t)l * N + sp;
    const uint64_t* og = a.own[g] + (size_t)l * N + sp;
    const uint64_t* ag = a.add0[g] + (size_t)l * N + sp;
    uint64_t kv0[DNUM], kv1[DNUM], dv[NQ][DNUM], av[NQ];
#pragma unroll
    for (int k = 0; k < DNUM; k++) {
      kv0[k] = __ldcs(kb + (size_t)k * a.key_digit_stride);
      kv1[k] = __ldcs(kb + (size_t)k * a.key_digit_stride + a.key_half_stride);
    }
#pragma unroll
    for (int r = 0; r < NQ; r++) {
#pragma unroll
      for (int k = 0; k < DNUM; k++)
        dv[r][k] = k == kown ? og[(size_t)r * a.ownq] : dg[(size_t)r * a.dq + (size_t)k * a.digit_stride];
      av[r] = add ? ag[(size_t)r * a.aq] : 0;
    }
#pragma unroll
    for (int r = 0; r < NQ; r++) {
#pragma unroll
      for (int k = 0; k < DNUM; k++) {
        const double d = fm::u2d(dv[r][k]);
        fm::fmac(acc0[r], d, fm::bits2d(kv0[k]));
        fm::fmac(acc1[r], d, fm::bits2d(kv1[k]));
      }
      if (add) fm::fmac(acc0[r], fm::u2d(av[r]), 1.0);
    }
  }
#pragma unroll
  for (int r = 0; r < NQ; r++) {
    a.out0[(size_t)r * a.oq + o] = add_mod(fm::c2u(fm::fred(acc0[r], q, qi), P.rc.q), pv0[r], P.rc.q);
    a.out1[(size_t)r * a.oq + o] = add_mod(fm::c2u(fm::fred(acc1[r], q, qi), P.rc.q), pv1[r], P.rc.q);
  }
}

void launch_kip_giants(const DevCtx& c, const KipGiants& a, const LimbMap& map) {
  ProfScope ps_(c, "kip",
                8.0 * c.N * (a.n * (2.0 * a.dnum * map.n + a.nq * (a.dnum * map.n + a.add_rows)) + 4.0 * a.nq * map.n));
  decltype(&k_kip_giants<1, 1>) kern = nullptr;
#define HELRM_KG_CASE(D)                                                                        \
  case D:                                                                                       \
    kern = a.nq == 4 ? k_kip_giants<D, 4> : a.nq == 2 ? k_kip_giants<D, 2> : k_kip_giants<D, 1>; \
    break;
  if (a.nq != 1 && a.nq != 2 && a.nq != 4) throw Error(HELRM_ERR_CONFIG, "giant runs support 1, 2 or 4 queries");
  switch (a.dnum) {
    HELRM_KG_CASE(1)
    HELRM_KG_CASE(2)
    HELRM_KG_CASE(3)
    HELRM_KG_CASE(4)
    HELRM_KG_CASE(5)
    HELRM_KG_CASE(6)
    HELRM_KG_CASE(7)
    default: throw Error(HELRM_ERR_CONFIG, "key switch supports dnum <= 7");
  }
#undef HELRM_KG_CASE
  launch_pdl(kern, dim3(dim3(c.N / kT, a.rows ? a.rows : map.n)), dim3(kT), 0, c.stream, a, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

// D20 L2, all baby steps of one input ciphertext in one pass: for each
// baby j (rotation r_j, key K_j), over Q_l P,
//   a_j[l][p] = [l <= level] [P]_{q_l} phi_j(c0)[l][p] + sum_k phi_j(D_k)[l][p] b_{j,k}[l][p]
//   b_j[l][p] = sum_k phi_j(D_k)[l][p] a_{j,k}[l][p]
// The CTA stages its 256-position tile of D_k and c0 plus a halo of max r_j
// positions (cyclic inside the half) in shared memory once (as doubles), then
// streams the D-form keys: the digits are read from HBM once for all babies
// instead of once per baby.  Baby pairs are written in D-form.
template <int DNUM>
__global__ void __launch_bounds__(256, 4) k_kip_multi(const __grid_constant__ KipMulti a,
                                                      const PrimeDev* __restrict__ primes,
                                                      const __grid_constant__ LimbMap map, uint32_t N) {
  pdl_wait_trigger();
  extern __shared__ double shd[];
  const int l = a.row0 + (int)blockIdx.y;
  const uint32_t n = N / 2, tile = blockDim.x;
  const uint32_t zq = (uint32_t)((a.nq + a.qk - 1) / a.qk);
  const uint32_t tix = a.zfast ? blockIdx.x / zq : blockIdx.x, zix = a.zfast ? blockIdx.x % zq : blockIdx.z;
  const uint32_t p0 = tix * tile, half = p0 >= n ? n : 0;
  const uint32_t span = tile + a.max_rot;
  const uint32_t chain = map.pr[l];
  const PrimeDev& P = primes[chain];
  const double q = P.qd, qi = P.qinv;
  const bool has_c0 = l <= (int)a.level;
  const int q0 = (int)zix * a.qk, nqc = min(a.qk, a.nq - q0);   // this CTA's queries
  const int slab = (DNUM + 1) * span;                              // doubles per staged query
  // stage D_k (and c0) tiles + halo of every query of the CTA
  const int kown = (a.own && has_c0) ? l / a.alpha : -1;   // digit whose own limb this row is
  for (int qq = 0; qq < nqc; qq++) {
    const uint64_t* dgq = a.digits + (size_t)(q0 + qq) * a.dq;
    const uint64_t* c0q = a.c0 + (size_t)(q0 + qq) * a.cq;
    const uint64_t* owq = a.own ? a.own + (size_t)(q0 + qq) * a.ownq : nullptr;
    double* sq = shd + qq * slab;
    for (uint32_t e = threadIdx.x; e < span; e += tile) {
      uint32_t j = p0 - half + e;
      j = j >= n ? j - n : j;
      const size_t src = (size_t)l * N + half + j;
#pragma unroll
      for (int k = 0; k < DNUM; k++)
        sq[k * span + e] = fm::u2d(k == kown ? owq[src] : dgq[(size_t)k * a.digit_stride + src]);
      if (has_c0) sq[DNUM * span + e] = fm::u2d(c0q[src]);
    }
  }
  __syncthreads();
  const uint32_t p = p0 + threadIdx.x;
  const double pm = has_c0 ? fm::u2c(a.p_mod[l], q) : 0.0;
  for (int j = 0; j < a.n; j++) {
    const uint64_t* kb = a.key[j] + (size_t)chain * N + p;
    uint64_t kv0[DNUM], kv1[DNUM];
#pragma unroll
    for (int k = 0; k < DNUM; k++) {
      kv0[k] = __ldcs(kb + (size_t)k * a.key_digit_stride);
      kv1[k] = __ldcs(kb + (size_t)k * a.key_digit_stride + a.key_half_stride);
    }
    const uint32_t e = threadIdx.x + a.rot[j];
    for (int qq = 0; qq < nqc; qq++) {
      const double* sq = shd + qq * slab;
      fm::FAcc acc0, acc1;
#pragma unroll
      for (int k = 0; k < DNUM; k++) {
        const double dv = sq[k * span + e];
        fm::fmac(acc0, dv, fm::bits2d(kv0[k]));
        fm::fmac(acc1, dv, fm::bits2d(kv1[k]));
      }
      if (has_c0) fm::fmac(acc0, sq[DNUM * span + e], pm);
      uint64_t* o = a.out[j] + (size_t)(q0 + qq) * a.oq + (size_t)l * N + p;   // baby pairs are stored in D-form
      o[0] = fm::d2bits(fm::fred(acc0, q, qi));
      o[a.out_half] = fm::d2bits(fm::fred(acc1, q, qi));
    }
  }
}

// D20 L3, one query, full grid (tile, pack, limb): the batch-1 form of
// k_diag_mac without the query and work-item loops (fewer instructions per
// MAC; the generic kernel measured 17% slower for batch 1).
template <bool XD>
__global__ void __launch_bounds__(256) k_diag_mac1(const MacTerm* __restrict__ terms, const int4* __restrict__ groups,
                                                  uint64_t* __restrict__ out, size_t out_stride, size_t half,
                                                  const PrimeDev* __restrict__ primes,
                                                  const __grid_constant__ LimbMap map, uint32_t N) {
  pdl_wait_trigger();
  constexpr int G = kGiantPack;
  constexpr int kChunk = 64;
  __shared__ MacTerm tm[kChunk];
  const int4 gr = groups[blockIdx.y];
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.z;
  const PrimeDev& P = primes[map.pr[l]];
  const double q = P.qd, qi = P.qinv;
  const size_t o = (size_t)l * N + p;
  fm::FAcc acc0[G], acc1[G];
  int cnt = 0;
  for (int c0 = 0; c0 < gr.y; c0 += kChunk) {   // term list staged in chunks
    const int nt = min(kChunk, gr.y - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < nt; t += blockDim.x) tm[t] = terms[gr.x + c0 + t];
    __syncthreads();
    if (p >= N) continue;
    // two terms per round: 2 x (2 + G) independent loads in flight
    for (int t = 0; t < nt; t += 2) {
      const int nr = nt - t >= 2 ? 2 : 1;
      uint64_t x0[2], x1[2], u[2][G];
#pragma unroll
      for (int r = 0; r < 2; r++) {
        if (r < nr) {
          const MacTerm& m = tm[t + r];
          x0[r] = m.x0[o];
          x1[r] = m.x1[o];
#pragma unroll
          for (int g = 0; g < G; g++) u[r][g] = m.u[g] ? __ldcs(m.u[g] + o) : 0;  // plaintexts stream once
        } else {
          x0[r] = x1[r] = 0;
#pragma unroll
          for (int g = 0; g < G; g++) u[r][g] = 0;
        }
      }
      if (cnt + 2 > fm::kFAccTerms) {
#pragma unroll
        for (int g = 0; g < G; g++) {
          fm::fold(acc0[g], q, qi);
          fm::fold(acc1[g], q, qi);
        }
        cnt = 0;
      }
      cnt += 2;
#pragma unroll
      for (int r = 0; r < 2; r++) {
        const double xa = XD ? fm::bits2d(x0[r]) : fm::u2c(x0[r], q);
        const double xb = XD ? fm::bits2d(x1[r]) : fm::u2c(x1[r], q);
#pragma unroll
        for (int g = 0; g < G; g++) {
          const double ud = fm::bits2d(u[r][g]);
          fm::fmac(acc0[g], ud, xa);
          fm::fmac(acc1[g], ud, xb);
        }
      }
    }
  }
  if (p >= N) return;
#pragma unroll
  for (int g = 0; g < G; g++) {
    if (g < gr.w) {
      uint64_t* dst = out + (size_t)(gr.z + g) * out_stride;
      dst[o] = fm::c2u(fm::fred(acc0[g], q, qi), P.rc.q);
      dst[half + o] = fm::c2u(fm::fred(acc1[g], q, qi), P.rc.q);
    }
  }
}

// D20 L3: (A, B)_z[l][p] = sum_t u_{z,t}[l][p] (x0_t, x1_t)[l][p] for the
// giants z of a pack.  Work item = (256-position tile fastest, pack, limb
// outermost -- the baby pairs of a limb stay L2-resident); each baby value is
// loaded once per pack of kGiantPack giants.  QN queries share every
// plaintext value a thread loads (batched lookups: QN = 2, so the FP64 work
// per plaintext byte doubles and the kernel stays HBM-bound at half the
// plaintext traffic per query).  Plaintexts u in D-form; x in D-form (XD) or
// canonical (single mode, centred on load).  Exact FP64 MACs, folded every
// kFAccTerms products; the output pairs are canonical.  A grid smaller than
// the work loops (persistent CTAs, HELRM_PERSIST).
template <bool XD, int QN>
__global__ void __launch_bounds__(256) k_diag_mac(const MacTerm* __restrict__ terms, const int4* __restrict__ groups,
                                                  uint64_t* __restrict__ out, size_t out_stride, size_t half,
                                                  const PrimeDev* __restrict__ primes,
                                                  const __grid_constant__ LimbMap map, uint32_t N, int nq, size_t xq,
                                                  size_t oq, int n_groups) {
  pdl_wait_trigger();
  constexpr int G = kGiantPack;
  constexpr int kChunk = 64;
  __shared__ MacTerm tm[kChunk];
  const uint32_t tiles = N / blockDim.x, total = tiles * (uint32_t)n_groups * (uint32_t)map.n;
  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
    // pack fastest: the packs of one (limb, tile) run back to back, so their shared baby
    // pairs come from L2 after the first (per limb they can exceed L2: 256 MB for the LLM)
    const int4 gr = groups[w % n_groups];
    const uint32_t p = ((w / n_groups) % tiles) * blockDim.x + threadIdx.x;
    const int l = (int)(w / (tiles * n_groups));
    const PrimeDev& P = primes[map.pr[l]];
    const double q = P.qd, qi = P.qinv;
    const size_t o = (size_t)l * N + p;
    for (int q0 = 0; q0 < nq; q0 += QN) {
      size_t ox[QN];
#pragma unroll
      for (int r = 0; r < QN; r++) ox[r] = o + (size_t)min(q0 + r, nq - 1) * xq;   // ragged tail: reload, no store
      fm::FAcc acc0[QN][G], acc1[QN][G];
      int cnt = 0;
      for (int c0 = 0; c0 < gr.y; c0 += kChunk) {   // term list staged in chunks
        const int nt = min(kChunk, gr.y - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < nt; t += blockDim.x) tm[t] = terms[gr.x + c0 + t];
        __syncthreads();
        // two terms per round: 2 (2 QN + G) independent loads in flight
        for (int t = 0; t < nt; t += 2) {
          const int nr = nt - t >= 2 ? 2 : 1;
          uint64_t x0[2][QN], x1[2][QN], u[2][G];
#pragma unroll
          for (int r = 0; r < 2; r++) {
            if (r < nr) {
              const MacTerm& m = tm[t + r];
#pragma unroll
              for (int k = 0; k < QN; k++) {
                x0[r][k] = m.x0[ox[k]];
                x1[r][k] = m.x1[ox[k]];
              }
#pragma unroll
              for (int g = 0; g < G; g++)
                u[r][g] = m.u[g] ? (QN == 1 && nq == 1 ? __ldcs(m.u[g] + o) : m.u[g][o]) : 0;
            } else {
#pragma unroll
              for (int k = 0; k < QN; k++) x0[r][k] = x1[r][k] = 0;
#pragma unroll
              for (int g = 0; g < G; g++) u[r][g] = 0;
            }
          }
          if (cnt + 2 > fm::kFAccTerms) {
#pragma unroll
            for (int k = 0; k < QN; k++)
#pragma unroll
              for (int g = 0; g < G; g++) {
                fm::fold(acc0[k][g], q, qi);
                fm::fold(acc1[k][g], q, qi);
              }
            cnt = 0;
          }
          cnt += 2;
#pragma unroll
          for (int r = 0; r < 2; r++) {
#pragma unroll
            for (int k = 0; k < QN; k++) {
              const double xa = XD ? fm::bits2d(x0[r][k]) : fm::u2c(x0[r][k], q);
              const double xb = XD ? fm::bits2d(x1[r][k]) : fm::u2c(x1[r][k], q);
#pragma unroll
              for (int g = 0; g < G; g++) {
                const double ud = fm::bits2d(u[r][g]);
                fm::fmac(acc0[k][g], ud, xa);
                fm::fmac(acc1[k][g], ud, xb);
              }
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < QN; k++) {
        if (q0 + k < nq) {
#pragma unroll
          for (int g = 0; g < G; g++) {
            if (g < gr.w) {
              uint64_t* dst = out + (size_t)(gr.z + g) * out_stride + (size_t)(q0 + k) * oq;
              dst[o] = fm::c2u(fm::fred(acc0[k][g], q, qi), P.rc.q);
              dst[half + o] = fm::c2u(fm::fred(acc1[k][g], q, qi), P.rc.q);
            }
          }
        }
      }
    }
  }
}

// D20 L5: after ncclAllReduce(uint64, sum) of partial Q_l P accumulators
// (each < q, at most 2^13 ranks -> no wrap), reduce every word mod its prime
__global__ void k_modred(uint64_t* __restrict__ x, const PrimeDev* __restrict__ primes,
                         const __grid_constant__ LimbMap map, uint32_t N) {
  pdl_wait_trigger();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const RedConst rc = primes[map.pr[l]].rc;
  const size_t o = (size_t)l * N + i;
  const uint64_t v = x[o];
  x[o] = v - mulhi64(v, rc.mu) * rc.q >= rc.q ? v - mulhi64(v, rc.mu) * rc.q - rc.q : v - mulhi64(v, rc.mu) * rc.q;
}

// Compact plans (HELRM_PLAN_COMPACT): the signed encoded coefficients of
// unique diagonal uids[k] (coef + uids[k] N) reduced into every limb of map:
// out + (k map.n + l) N.  (The NTT and the D-form conversion follow.)
__global__ void k_expand_coef(const int64_t* __restrict__ coef, const uint32_t* __restrict__ uids,
                              uint64_t* __restrict__ out, const PrimeDev* __restrict__ primes,
                              const __grid_constant__ LimbMap map, uint32_t N) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  const size_t k = blockIdx.z;
  if (i >= N) return;
  const uint64_t q = primes[map.pr[l]].rc.q;
  const int64_t v = coef[(size_t)uids[k] * N + i];
  uint64_t r;
  if (v >= 0) {
    r = (uint64_t)v % q;
  } else {
    r = (uint64_t)(-v) % q;
    r = r ? q - r : 0;
  }
  out[(k * map.n + l) * N + i] = r;
}

// x += y as plain uint64 words (the sum ncclAllReduce(ncclUint64, ncclSum) computes)
__global__ void k_add_u64(uint64_t* __restrict__ x, const uint64_t* __restrict__ y, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] += y[i];
}

// ---------------- launchers ----------------
static dim3 grid_for(uint32_t N, int limbs) { return dim3((N + kT - 1) / kT, limbs); }

void launch_reduce_signed(const DevCtx& c, const int64_t* m, uint64_t* out, const LimbMap& map) {
  ProfScope ps_(c, "reduce_signed", 8.0 * c.N * (1 + map.n));
  k_reduce_signed<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(m, out, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_sample_uniform_ntt(const DevCtx& c, uint64_t* out, const LimbMap& map, uint64_t seed, uint64_t purpose,
                               uint64_t a, uint64_t b, const LimbMap& ids) {
  ProfScope ps_(c, "sample_uniform", 8.0 * c.N * map.n);
  k_sample_uniform_ntt<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(out, c.primes, map, c.log_n, c.slotpos, seed,
                                                                  purpose, a, b, ids);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_sample_small(const DevCtx& c, int64_t* out, uint64_t base, int kind, const uint64_t* cdt) {
  ProfScope ps_(c, "sample_small", 8.0 * c.N);
  k_sample_small<<<(c.N + kT - 1) / kT, kT, 0, c.stream>>>(out, c.N, base, kind, cdt);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_binary(const DevCtx& c, int op, const uint64_t* a, const uint64_t* b, uint64_t* out, const LimbMap& map) {
  ProfScope ps_(c, "binary", 8.0 * c.N * map.n * (op == 3 ? 2 : 3));
  launch_pdl(k_binary, dim3(grid_for(c.N, map.n)), dim3(kT), 0, c.stream, op, a, b, out, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_scalar_mul(const DevCtx& c, const uint64_t* a, uint64_t* out, const LimbMap& map, const uint64_t* s,
                       const uint64_t* sp, int dform_out, int G, size_t as, size_t os) {
  ProfScope ps_(c, "scalar_mul", 16.0 * c.N * map.n * G);
  launch_pdl(k_scalar_mul, dim3(dim3((c.N + kT - 1) / kT, map.n, G)), dim3(kT), 0, c.stream, a, out, c.primes, map, c.N, s, sp, dform_out, as, os);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_dform(const DevCtx& c, uint64_t* x, size_t n, const LimbMap& map, int dir) {
  ProfScope ps_(c, "dform", 16.0 * n);
  k_dform<<<c.n_sm * 8, 256, 0, c.stream>>>(x, n, c.log_n, c.primes, map, dir);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_automorph(const DevCtx& c, const uint64_t* a, uint64_t* out, const LimbMap& map, uint32_t rot,
                      int accumulate) {
  ProfScope ps_(c, "automorph", 8.0 * c.N * map.n * (accumulate ? 3 : 2));
  launch_pdl(k_automorph, dim3(grid_for(c.N, map.n)), dim3(kT), 0, c.stream, a, out, c.primes, map, c.N, rot, accumulate);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_conv_rows(const DevCtx& c, const ConvRowDev* tab, int ncv, int rows, int nb_max, const uint64_t* y,
                      size_t y_stride, uint64_t* out, size_t out_stride_g, size_t out_stride_k, int G,
                      const LimbMap& out_map) {
  ProfScope ps_(c, "conv", 8.0 * c.N * (double)G * ncv * (rows + 4));
  static const int pt = getenv("HELRM_CONV_PT") ? atoi(getenv("HELRM_CONV_PT")) : 2;
  auto kern = nb_max <= 1 ? k_conv_rows<1> : nb_max <= 2 ? k_conv_rows<2> : nb_max <= 4 ? k_conv_rows<4>
                                                                                     : k_conv_rows<8>;
  if (pt == 2)
    kern = nb_max <= 1 ? k_conv_rows<1, 2> : nb_max <= 2 ? k_conv_rows<2, 2> : nb_max <= 4 ? k_conv_rows<4, 2>
                                                                                         : k_conv_rows<8, 2>;
  (void)out_map;
  launch_pdl(kern, dim3(dim3(c.N / (256 * pt), G * ncv)), dim3(256), 0, c.stream, tab, ncv, rows, y, y_stride, out, out_stride_g, out_stride_k, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_modred(const DevCtx& c, uint64_t* x, const LimbMap& map) {
  ProfScope ps_(c, "modred", 16.0 * c.N * map.n);
  launch_pdl(k_modred, dim3(grid_for(c.N, map.n)), dim3(kT), 0, c.stream, x, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_expand_coef(const DevCtx& c, const int64_t* coef, const uint32_t* uids, size_t n, uint64_t* out,
                        const LimbMap& map) {
  ProfScope ps_(c, "expand_coef", 8.0 * c.N * n * (1 + map.n));
  k_expand_coef<<<dim3((c.N + kT - 1) / kT, map.n, (unsigned)n), kT, 0, c.stream>>>(coef, uids, out, c.primes, map,
                                                                                    c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_add_u64(const DevCtx& c, uint64_t* x, const uint64_t* y, size_t n) {
  ProfScope ps_(c, "add_u64", 24.0 * n);
  k_add_u64<<<(unsigned)std::min<size_t>((n + kT - 1) / kT, (size_t)c.n_sm * 16), kT, 0, c.stream>>>(x, y, n);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_rescale_prep(const DevCtx& c, const uint64_t* xl, size_t xs, uint64_t ql, uint64_t* out, size_t os, int G,
                         const LimbMap& map) {
  ProfScope ps_(c, "rescale_prep", 8.0 * c.N * (1 + map.n) * G);
  launch_pdl(k_rescale_prep, dim3(dim3((c.N + kT - 1) / kT, map.n, G)), dim3(kT), 0, c.stream, xl, xs, ql, out, os, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_kip(const DevCtx& c, const KipArgs& a, const LimbMap& map) {
  const double nh = a.halves == 3 ? 2.0 : 1.0;
  ProfScope ps_(c, "kip", 8.0 * c.N * (nh * a.dnum * map.n + a.nq * (a.dnum * map.n + (a.add0 ? a.add_rows : 0) +
                                                                      (a.accumulate ? 2 : 1) * nh * map.n)));
  decltype(&k_kip<1, 1>) kern = nullptr;
  const bool b = a.nq > 1;
  switch (a.dnum) {
    case 1: kern = b ? k_kip<1, 2> : k_kip<1, 1>; break;
    case 2: kern = b ? k_kip<2, 2> : k_kip<2, 1>; break;
    case 3: kern = b ? k_kip<3, 2> : k_kip<3, 1>; break;
    case 4: kern = b ? k_kip<4, 2> : k_kip<4, 1>; break;
    case 5: kern = b ? k_kip<5, 2> : k_kip<5, 1>; break;
    case 6: kern = b ? k_kip<6, 2> : k_kip<6, 1>; break;
    case 7: kern = b ? k_kip<7, 2> : k_kip<7, 1>; break;
    default: throw Error(HELRM_ERR_CONFIG, "key switch supports dnum <= 7");
  }
  const unsigned total = (c.N / kT) * (unsigned)(a.rows ? a.rows : map.n);
  const unsigned grid = c.persist > 0 ? std::min<unsigned>(total, (unsigned)c.n_sm * c.persist) : total;
  launch_pdl(kern, dim3(grid), dim3(kT), 0, c.stream, a, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_kip_multi(const DevCtx& c, const KipMulti& a, const LimbMap& map) {
  const double zq = (a.nq + a.qk - 1) / a.qk;   // key passes
  ProfScope ps_(c, "kip_multi", 8.0 * c.N * (a.nq * (a.dnum * map.n + (a.level + 1.0) + a.n * 2.0 * map.n) +
                                             zq * a.n * 2.0 * a.dnum * map.n));
  const uint32_t tile = 256;
  const size_t smem = (size_t)a.qk * (a.dnum + 1) * (tile + a.max_rot) * 8;
  decltype(&k_kip_multi<1>) kern = nullptr;
  switch (a.dnum) {
    case 1: kern = k_kip_multi<1>; break;
    case 2: kern = k_kip_multi<2>; break;
    case 3: kern = k_kip_multi<3>; break;
    case 4: kern = k_kip_multi<4>; break;
    case 5: kern = k_kip_multi<5>; break;
    case 6: kern = k_kip_multi<6>; break;
    case 7: kern = k_kip_multi<7>; break;
    default: throw Error(HELRM_ERR_CONFIG, "key switch supports dnum <= 7");
  }
  if (smem > 48 * 1024) HCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned ny = a.rows ? (unsigned)a.rows : (unsigned)map.n;
  const dim3 grid = a.zfast ? dim3(c.N / tile * (unsigned)zq, ny, 1) : dim3(c.N / tile, ny, (unsigned)zq);
  launch_pdl(kern, grid, dim3(tile), smem, c.stream, a, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_diag_mac(const DevCtx& c, const void* terms, const int4* groups, int n_groups, double n_u_total,
                     double n_x_distinct, int n_out, uint64_t* out, size_t out_stride, const LimbMap& map,
                     bool x_dform, int nq, size_t xq, size_t oq, bool wide) {
  // algorithmic bytes: every plaintext once, every distinct baby pair and output once per query
  ProfScope ps_(c, "diag_mac", 8.0 * c.N * map.n * (n_u_total + nq * (2.0 * n_x_distinct + 2.0 * n_out)));
  (void)wide;
  static const int bulk = getenv("HELRM_MAC_BULK") ? atoi(getenv("HELRM_MAC_BULK")) : 2;
  // bulk-copy kernel: HELRM_MAC_BULK=1 for batch 1 only, 2 for every batch
  if (bulk && (nq == 1 || bulk == 2) && x_dform && !wide && c.persist == 0 &&
      launch_diag_mac_bulk(c, (const MacTerm*)terms, groups, n_groups, out, out_stride, (size_t)map.n * c.N, map, nq,
                           xq, oq))
    return;
  if (nq == 1 && c.persist == 0) {
    auto k1 = x_dform ? k_diag_mac1<true> : k_diag_mac1<false>;
    launch_pdl(k1, dim3(dim3(c.N / kT, n_groups, map.n)), dim3(kT), 0, c.stream, (const MacTerm*)terms, groups, out, out_stride, (size_t)map.n * c.N, c.primes, map, c.N);
    (*c.launches)++;
    HCUDA(cudaGetLastError());
    return;
  }
  // QN queries per plaintext load: 4 when the batch is a multiple of 4 (the LLM's 4 output blocks)
  static const int q4 = getenv("HELRM_MAC_Q4") ? atoi(getenv("HELRM_MAC_Q4")) : 1;
  auto kern = x_dform ? (nq % 4 == 0 && q4 ? k_diag_mac<true, 4> : nq > 1 ? k_diag_mac<true, 2> : k_diag_mac<true, 1>)
                      : (nq % 4 == 0 && q4 ? k_diag_mac<false, 4>
                                           : nq > 1 ? k_diag_mac<false, 2> : k_diag_mac<false, 1>);
  const unsigned total = (c.N / kT) * n_groups * map.n;
  const unsigned grid = c.persist > 0 ? std::min<unsigned>(total, (unsigned)c.n_sm * c.persist) : total;
  launch_pdl(kern, dim3(grid), dim3(kT), 0, c.stream, (const MacTerm*)terms, groups, out, out_stride, (size_t)map.n * c.N, c.primes, map, c.N, nq, xq, oq, n_groups);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

}  // namespace helrm
