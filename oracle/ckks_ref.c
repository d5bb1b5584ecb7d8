/*
 * oracle/ckks_ref.c -- TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * Plain, slow, scalar C for the integer and high-precision steps of the
 * RNS-CKKS lookup that Python cannot do at speed.  Only tests/, smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code with the CUDA path (paper_2506_18150_b200/csrc/).
 *
 * Every modular product here is `(unsigned __int128)a * b % q` -- no Barrett,
 * no Shoup, no lazy reduction -- so that each line can be checked by eye.
 *
 * Definitions followed (SURVEY.md section 8(c) readings of PAPER.md, which is
 * silent on all ring-level conventions):
 *   D4  NTT_q(a)_i = sum_j a_j psi^{(2i+1) j} mod q, natural order
 *       ("R_Q = Z_Q[X]/(X^N+1)", section 2.1.1)
 *   D6  Encode: m_i = RHA((2 Delta / N) sum_j z_j cos(pi e_j i / N)),
 *       e_j = 5^j mod 2N, in binary128 ("inverse Fast
 *       Fourier Transform ... scales each output by Delta ... rounded")
 *   D9  PRNG word(seed, stream, k) = SM((seed ^ SM(stream)) + (k+1) gamma)
 *   D10 samplers (uniform mod q, ternary, CDT Gaussian)
 *   D14 Conv_{B->T}(x)_t = (sum_b [x_b (B/b)^-1]_b (B/b mod t)) mod t
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <quadmath.h>

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + b) % q); }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + q - b) % q); }

static uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = mulmod(r, b, q);
    b = mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}

/* ---------------- D4: negacyclic NTT in natural order ----------------
 * Step 1 (twist): b_j = a_j psi^j.  Step 2: cyclic DFT of b with
 * omega = psi^2 (a plain radix-2 Cooley-Tukey FFT used as a library-style
 * primitive: bit-reverse permutation, then log2 N butterfly passes).
 * Result: A_i = sum_j a_j psi^j omega^{ij} = sum_j a_j psi^{(2i+1) j}. */
static void bitrev_permute(uint64_t* a, size_t N) {
  for (size_t i = 1, j = 0; i < N; i++) {
    size_t bit = N >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) { uint64_t t = a[i]; a[i] = a[j]; a[j] = t; }
  }
}

static void cyclic_dft(uint64_t* a, size_t N, uint64_t q, uint64_t omega) {
  bitrev_permute(a, N);
  for (size_t len = 2; len <= N; len <<= 1) {
    uint64_t wlen = powmod(omega, N / len, q); /* primitive len-th root */
    for (size_t s = 0; s < N; s += len) {
      uint64_t w = 1;
      for (size_t k = 0; k < len / 2; k++) {
        uint64_t u = a[s + k], v = mulmod(a[s + k + len / 2], w, q);
        a[s + k] = addmod(u, v, q);
        a[s + k + len / 2] = submod(u, v, q);
        w = mulmod(w, wlen, q);
      }
    }
  }
}

void or_ntt(uint64_t* a, size_t N, uint64_t q, uint64_t psi) {
  uint64_t pj = 1;
  for (size_t j = 0; j < N; j++) { a[j] = mulmod(a[j], pj, q); pj = mulmod(pj, psi, q); }
  cyclic_dft(a, N, q, mulmod(psi, psi, q));
}

/* INTT: a_j = N^-1 psi^-j sum_i A_i omega^{-ij}  (inverse of or_ntt) */
void or_intt(uint64_t* a, size_t N, uint64_t q, uint64_t psi) {
  uint64_t psi_inv = powmod(psi, q - 2, q);
  uint64_t omega_inv = mulmod(psi_inv, psi_inv, q);
  cyclic_dft(a, N, q, omega_inv);
  uint64_t ninv = powmod((uint64_t)N % q, q - 2, q);
  uint64_t pj = ninv;
  for (size_t j = 0; j < N; j++) { a[j] = mulmod(a[j], pj, q); pj = mulmod(pj, psi_inv, q); }
}

/* D4 by its definition, O(N^2): used only to pin or_ntt on small N. */
void or_ntt_direct(const uint64_t* a, uint64_t* out, size_t N, uint64_t q, uint64_t psi) {
  for (size_t i = 0; i < N; i++) {
    uint64_t acc = 0;
    uint64_t step = powmod(psi, 2 * i + 1, q), w = 1;
    for (size_t j = 0; j < N; j++) { acc = addmod(acc, mulmod(a[j], w, q), q); w = mulmod(w, step, q); }
    out[i] = acc;
  }
}

/* ---------------- element-wise helpers (one limb) ---------------- */
void or_vec_mulmod(const uint64_t* a, const uint64_t* b, uint64_t* out, size_t n, uint64_t q) {
  for (size_t i = 0; i < n; i++) out[i] = mulmod(a[i], b[i], q);
}
void or_vec_mac(const uint64_t* a, const uint64_t* b, uint64_t* acc, size_t n, uint64_t q) {
  for (size_t i = 0; i < n; i++) acc[i] = addmod(acc[i], mulmod(a[i], b[i], q), q);
}
void or_vec_scalar(const uint64_t* a, uint64_t s, uint64_t* out, size_t n, uint64_t q) {
  for (size_t i = 0; i < n; i++) out[i] = mulmod(a[i], s % q, q);
}

/* ---------------- D14: fast base conversion (no correction) ----------------
 * in: nb limbs [nb][N] residues mod bprimes; binv[b] = [(B/b)^-1]_b;
 * bmod[t*nb + b] = (B/b) mod tprimes[t]; out: nt limbs [nt][N]. */
void or_conv(const uint64_t* in, size_t nb, const uint64_t* bprimes, const uint64_t* binv,
             const uint64_t* bmod, size_t nt, const uint64_t* tprimes, uint64_t* out, size_t N) {
  for (size_t i = 0; i < N; i++) {
    for (size_t t = 0; t < nt; t++) {
      uint64_t acc = 0;
      for (size_t b = 0; b < nb; b++) {
        uint64_t y = mulmod(in[b * N + i], binv[b], bprimes[b]);
        acc = addmod(acc, mulmod(y % tprimes[t], bmod[t * nb + b], tprimes[t]), tprimes[t]);
      }
      out[t * N + i] = acc;
    }
  }
}

/* ---------------- D9: counter-based SplitMix64 ---------------- */
static uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t or_prng_word(uint64_t seed, uint64_t stream, uint64_t k) {
  return sm_mix((seed ^ sm_mix(stream)) + (k + 1) * 0x9E3779B97F4A7C15ull);
}

/* ---------------- D10: samplers; coefficient i uses words 2i, 2i+1 -------- */
void or_sample_uniform(uint64_t seed, uint64_t stream, uint64_t q, size_t N, uint64_t* out) {
  for (size_t i = 0; i < N; i++) {
    u128 w = ((u128)or_prng_word(seed, stream, 2 * i) << 64) | or_prng_word(seed, stream, 2 * i + 1);
    out[i] = (uint64_t)(w % q);
  }
}
void or_sample_ternary(uint64_t seed, uint64_t stream, size_t N, int64_t* out) {
  for (size_t i = 0; i < N; i++) {
    uint64_t r = or_prng_word(seed, stream, 2 * i) % 3;
    out[i] = r == 0 ? 0 : (r == 1 ? 1 : -1);
  }
}
/* table[k] for k = 0..19, table[19] stands for 2^64 (passed as 0, never compared) */
void or_sample_gauss(uint64_t seed, uint64_t stream, size_t N, const uint64_t* table, int64_t* out) {
  for (size_t i = 0; i < N; i++) {
    uint64_t w0 = or_prng_word(seed, stream, 2 * i), w1 = or_prng_word(seed, stream, 2 * i + 1);
    int64_t mag = 19;
    for (int k = 0; k < 19; k++) {
      if (w0 < table[k]) { mag = k; break; }
    }
    out[i] = ((w1 & 1) && mag > 0) ? -mag : mag;
  }
}

/* ---------------- D6: Encode in binary128 ----------------
 * z: n = N/2 real slots (double); only non-zero slots enter the sum (adding
 * an exact zero term changes nothing).  delta: the scale (an integer <= 2^53
 * or a power of two, exactly representable).  out: int64 coefficients.
 * tie[i] := 1 when the binary128 value of coefficient i lies within 2^-40 of
 * a half-integer: D6 then requires an exact recomputation (the caller does it
 * with 200-bit mpmath, oracle/textbook.py), since the rounding direction is
 * not decided by a ~113-bit sum there.
 * Returns 0, or 2 (HELRM_ERR_CONFIG) if some |m_i| >= 2^62. */
int or_encode(const double* z, size_t N, double delta, int64_t* out, uint8_t* tie) {
  size_t n = N / 2, twoN = 2 * N;
  __float128* ctab = (__float128*)malloc(sizeof(__float128) * twoN);
  size_t* e = (size_t*)malloc(sizeof(size_t) * n);
  size_t* nz = (size_t*)malloc(sizeof(size_t) * n);
  size_t nnz = 0;
  for (size_t k = 0; k < twoN; k++) ctab[k] = cosq(M_PIq * (__float128)k / (__float128)N);
  size_t ej = 1;
  for (size_t j = 0; j < n; j++) { e[j] = ej; ej = (ej * 5) % twoN; }
  for (size_t j = 0; j < n; j++) if (z[j] != 0.0) nz[nnz++] = j;
  __float128 coef = 2 * (__float128)delta / (__float128)N;
  const __float128 lim = 4611686018427387904.0Q; /* 2^62 */
  const __float128 eps = 9.094947017729282379150390625e-13Q; /* 2^-40 */
  int status = 0;
  for (size_t i = 0; i < N; i++) {
    __float128 acc = 0;
    for (size_t t = 0; t < nnz; t++) {
      size_t j = nz[t];
      acc += (__float128)z[j] * ctab[(uint64_t)((unsigned long long)e[j] * i % twoN)];
    }
    __float128 x = coef * acc;
    tie[i] = fabsq(x - floorq(x) - 0.5Q) < eps;
    __float128 v = roundq(x); /* round half away from zero */
    if (fabsq(v) >= lim) { status = 2; v = 0; }
    out[i] = (int64_t)v;
  }
  free(ctab); free(e); free(nz);
  return status;
}
