// kernels_rns.cu -- element-wise RNS kernels of the lookup (sm_100a):
// samplers (D9/D10), signed reduction, modular add/sub/mul, Galois
// automorphisms as slot-order shifts (D8), fast base conversion (D14, the
// core of ModUp D15 / ModDown D16), the ModDown / rescale finishing steps
// (D16/D17), the key inner product with fused automorphism (D18), and the
// plaintext-diagonal multiply-accumulate of the BSGS inner sums (D20 L3).
//
// Layout: polynomials are [limb][N] uint64, NTT form in slot order; one
// thread per coefficient, blockIdx.y = limb, coalesced 8-byte accesses.
#include "internal.h"

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
                             const uint64_t* __restrict__ s, const uint64_t* __restrict__ sp) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const uint64_t q = primes[map.pr[l]].rc.q;
  const size_t o = (size_t)l * N + i;
  out[o] = shoup(a[o], s[l], sp[l], q);
}

// out[l][p] = a[l][rot_src(p)]  (+ out if accumulate)
__global__ void k_automorph(const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                            const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N, uint32_t rot,
                            int accumulate) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (p >= N) return;
  const uint64_t v = a[(size_t)l * N + rot_src(p, rot, N / 2)];
  const size_t o = (size_t)l * N + p;
  out[o] = accumulate ? add_mod(out[o], v, primes[map.pr[l]].rc.q) : v;
}

// D14 Conv_{B->T}: out[row[t]][i] = (sum_b [x_b (B/b)^-1]_b ((B/b) mod t)) mod t.
struct ConvRows {
  int16_t row[kMaxLimbs];
};
__global__ void k_conv(const ConvDev* __restrict__ cv, const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                       const PrimeDev* __restrict__ primes, uint32_t N, const __grid_constant__ ConvRows rows, int t_per_block) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int nb = cv->nb;
  uint64_t y[kMaxDigitPrimes];
#pragma unroll
  for (int b = 0; b < kMaxDigitPrimes; b++) {
    if (b < nb) {
      const uint64_t qb = primes[cv->bpr[b]].rc.q;
      y[b] = shoup(in[(size_t)b * N + i], cv->binv[b], cv->binvs[b], qb);
    }
  }
  const int t0 = blockIdx.y * t_per_block;
  const int t1 = min(cv->nt, t0 + t_per_block);
  for (int t = t0; t < t1; t++) {
    const RedConst rc = primes[cv->tpr[t]].rc;
    U128 acc{0, 0};
#pragma unroll
    for (int b = 0; b < kMaxDigitPrimes; b++)
      if (b < nb) mac128(acc, y[b], cv->bmod[t][b]);
    out[(size_t)rows.row[t] * N + i] = reduce128(acc.hi, acc.lo, rc);
  }
}

// out[l] = (y[l] - t[l]) * s[l] mod q_l  (ModDown / rescale finish)
__global__ void k_sub_scale(const uint64_t* __restrict__ y, const uint64_t* __restrict__ t, uint64_t* __restrict__ out,
                            const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N,
                            const uint64_t* __restrict__ s, const uint64_t* __restrict__ sp) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const uint64_t q = primes[map.pr[l]].rc.q;
  const size_t o = (size_t)l * N + i;
  out[o] = shoup(sub_mod(y[o], t[o], q), s[l], sp[l], q);
}

// D17: r = ((x + h) mod q_l) - h, then r mod q_i for the remaining limbs
__global__ void k_rescale_prep(const uint64_t* __restrict__ xl, uint64_t ql, uint64_t* __restrict__ out,
                               const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (i >= N) return;
  const uint64_t h = (ql - 1) / 2;
  const uint64_t v = xl[i];
  const uint64_t q = primes[map.pr[l]].rc.q;
  uint64_t r;
  if (v <= h) {
    r = v % q;                       // r = v >= 0
  } else {
    const uint64_t mag = (ql - v) % q;  // r = v - ql < 0
    r = mag ? q - mag : 0;
  }
  out[(size_t)l * N + i] = r;
}

// D18 key inner product with the automorphism fused into the loads:
//   out0[l][p] (+)= [c0] P phi(c0)[l][p] + sum_k phi(D_k)[l][p] b_k[l][p]
//   out1[l][p] (+)= sum_k phi(D_k)[l][p] a_k[l][p]
__global__ void k_kip(const __grid_constant__ KipArgs a, const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (p >= N) return;
  const int nl = map.n;
  const uint32_t chain = map.pr[l];
  const RedConst rc = primes[chain].rc;
  const uint32_t sp = rot_src(p, a.rot, N / 2);
  U128 acc0{0, 0}, acc1{0, 0};
  for (int k = 0; k < a.dnum; k++) {
    const uint64_t d = a.digits[((size_t)k * nl + l) * N + sp];
    const uint64_t* kb = a.key + (size_t)k * a.key_digit_stride + (size_t)chain * N;
    mac128(acc0, d, kb[p]);
    mac128(acc1, d, kb[a.key_half_stride + p]);
  }
  if (a.c0 != nullptr && l <= (int)a.level) mac128(acc0, a.c0[(size_t)l * N + sp], a.p_mod[l]);
  uint64_t r0 = reduce128(acc0.hi, acc0.lo, rc), r1 = reduce128(acc1.hi, acc1.lo, rc);
  const size_t o = (size_t)l * N + p;
  if (a.accumulate) {
    r0 = add_mod(r0, a.out0[o], rc.q);
    r1 = add_mod(r1, a.out1[o], rc.q);
  }
  a.out0[o] = r0;
  a.out1[o] = r1;
}

// D20 L3: (A, B)[l][p] = sum_t u_t[l][p] (x0_t, x1_t)[l][p]
__global__ void k_diag_mac(const MacTerm* __restrict__ terms, int n_terms, uint64_t* __restrict__ out0,
                           uint64_t* __restrict__ out1, const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map,
                           uint32_t N) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (p >= N) return;
  const RedConst rc = primes[map.pr[l]].rc;
  const size_t o = (size_t)l * N + p;
  U128 acc0{0, 0}, acc1{0, 0};
  for (int t = 0; t < n_terms; t++) {
    const MacTerm m = terms[t];
    const uint64_t u = m.u[o];
    mac128(acc0, u, m.x0[o]);
    mac128(acc1, u, m.x1[o]);
  }
  out0[o] = reduce128(acc0.hi, acc0.lo, rc);
  out1[o] = reduce128(acc1.hi, acc1.lo, rc);
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
  k_binary<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(op, a, b, out, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_scalar_mul(const DevCtx& c, const uint64_t* a, uint64_t* out, const LimbMap& map, const uint64_t* s,
                       const uint64_t* sp) {
  ProfScope ps_(c, "scalar_mul", 16.0 * c.N * map.n);
  k_scalar_mul<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(a, out, c.primes, map, c.N, s, sp);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_automorph(const DevCtx& c, const uint64_t* a, uint64_t* out, const LimbMap& map, uint32_t rot,
                      int accumulate) {
  ProfScope ps_(c, "automorph", 8.0 * c.N * map.n * (accumulate ? 3 : 2));
  k_automorph<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(a, out, c.primes, map, c.N, rot, accumulate);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_conv(const DevCtx& c, const ConvDev* cv, int nb, int nt, const int16_t* rows, const uint64_t* in,
                 uint64_t* out) {
  ProfScope ps_(c, "conv", 8.0 * c.N * (nt + nb));
  ConvRows r{};
  for (int t = 0; t < nt; t++) r.row[t] = rows[t];
  const int tpb = 4;
  k_conv<<<dim3((c.N + kT - 1) / kT, (nt + tpb - 1) / tpb), kT, 0, c.stream>>>(cv, in, out, c.primes, c.N, r, tpb);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_sub_scale(const DevCtx& c, const uint64_t* y, const uint64_t* t, uint64_t* out, const LimbMap& map,
                      const uint64_t* s, const uint64_t* sp) {
  ProfScope ps_(c, "sub_scale", 24.0 * c.N * map.n);
  k_sub_scale<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(y, t, out, c.primes, map, c.N, s, sp);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_rescale_prep(const DevCtx& c, const uint64_t* xl, uint64_t ql, uint64_t* out, const LimbMap& map) {
  ProfScope ps_(c, "rescale_prep", 8.0 * c.N * (1 + map.n));
  k_rescale_prep<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(xl, ql, out, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_kip(const DevCtx& c, const KipArgs& a, const LimbMap& map) {
  ProfScope ps_(c, "kip", 8.0 * c.N * (3.0 * a.dnum * map.n + (a.c0 ? a.level + 1 : 0) + (a.accumulate ? 4 : 2) * map.n));
  k_kip<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(a, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

void launch_diag_mac(const DevCtx& c, const MacTerm* terms, int n_terms, uint64_t* out0, uint64_t* out1,
                     const LimbMap& map) {
  ProfScope ps_(c, "diag_mac", 8.0 * c.N * map.n * (3.0 * n_terms + 2));
  k_diag_mac<<<grid_for(c.N, map.n), kT, 0, c.stream>>>(terms, n_terms, out0, out1, c.primes, map, c.N);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

}  // namespace helrm
