// host_math.cpp -- host-side number theory and the client's encode/decode.
//
//  D2  prime search (largest primes < 2^bits with p = 1 mod 2N)
//  D3  psi = smallest primitive 2N-th root of unity mod q
//  D5  slot order: NTT position of psi^(+-5^j)
//  D6  Encode: m_i = RHA((2 Delta/N) sum_j z_j cos(pi e_j i/N)),
//      computed with a double-double (~106-bit) FFT; any coefficient whose
//      fractional part falls within 2^-30 of 1/2 is recomputed by a binary128
//      direct sum, so the result is the correctly rounded integer.
//  D7  Decode (fp64 FFT; tolerance-only)
//  D10 Gaussian CDT table floor(2^64 P(|X| <= k)), sigma = 3.2, |x| <= 19
#include <quadmath.h>

#include <cmath>
#include <complex>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace helrm {

uint64_t mulm(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((unsigned __int128)a * b % q); }

uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  for (; e; e >>= 1) {
    if (e & 1) r = mulm(r, b, q);
    b = mulm(b, b, q);
  }
  return r;
}

uint64_t inv_mod(uint64_t a, uint64_t q) { return pow_mod(a % q, q - 2, q); }  // q prime

bool is_prime_u64(uint64_t n) {
  if (n < 2) return false;
  for (uint64_t p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull})
    if (n % p == 0) return n == p;
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) { d >>= 1; s++; }
  // bases proven sufficient for all n < 2^64
  for (uint64_t a : {2ull, 325ull, 9375ull, 28178ull, 450775ull, 9780504ull, 1795265022ull}) {
    uint64_t x = pow_mod(a, d, n);
    if (x == 0 || x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; r++) {
      x = mulm(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}

std::vector<uint64_t> find_primes(const std::vector<std::pair<uint32_t, uint32_t>>& groups, uint64_t N,
                                  std::vector<uint64_t> taken) {
  std::vector<uint64_t> out;
  const uint64_t step = 2 * N;
  for (auto [bits, count] : groups) {
    if (bits < 20 || bits > 61) throw Error(HELRM_ERR_CONFIG, "prime bit size must be in [20, 61]");
    uint64_t top = (bits == 64) ? ~0ull : ((1ull << bits) - 1);
    uint64_t x = top - ((top - 1) % step);  // largest value = 1 mod 2N that is <= top
    uint32_t got = 0;
    while (got < count) {
      if (x < step) throw Error(HELRM_ERR_CONFIG, "not enough NTT-friendly primes");
      bool used = false;
      for (uint64_t t : taken) used |= (t == x);
      for (uint64_t t : out) used |= (t == x);
      if (!used && is_prime_u64(x)) { out.push_back(x); got++; }
      x -= step;
    }
  }
  return out;
}

uint64_t min_psi(uint64_t q, uint64_t N) {
  uint64_t g = 2;
  while (pow_mod(g, (q - 1) / 2, q) != q - 1) g++;  // quadratic non-residue
  uint64_t psi0 = pow_mod(g, (q - 1) / (2 * N), q);
  if (pow_mod(psi0, N, q) != q - 1) throw Error(HELRM_ERR_CONFIG, "no primitive 2N-th root");
  uint64_t sq = mulm(psi0, psi0, q), best = psi0, cur = psi0;
  for (uint64_t k = 1; k < N; k++) {  // psi0^(2k+1): all primitive 2N-th roots
    cur = mulm(cur, sq, q);
    if (cur < best) best = cur;
  }
  return best;
}

static uint32_t bitrev(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

std::vector<uint32_t> slot_of_bitrev(uint32_t log_n) {
  uint32_t N = 1u << log_n, n = N / 2, twoN = 2 * N;
  std::vector<uint32_t> pos(twoN, 0xffffffffu);
  uint64_t e = 1;
  for (uint32_t j = 0; j < n; j++) {
    pos[e] = j;
    pos[twoN - e] = n + j;
    e = e * 5 % twoN;
  }
  std::vector<uint32_t> out(N);
  for (uint32_t r = 0; r < N; r++) out[r] = pos[2 * bitrev(r, log_n) + 1];
  return out;
}

// ---------------- double-double arithmetic ----------------
struct dd {
  double hi, lo;
};
static inline dd two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
static inline dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
static inline dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi), t = two_sum(x.lo, y.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
static inline dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
static inline dd dd_mul(dd x, dd y) {
  double p = x.hi * y.hi;
  double e = std::fma(x.hi, y.hi, -p);
  e += x.hi * y.lo + x.lo * y.hi;
  return quick_two_sum(p, e);
}
static inline dd dd_from_q(__float128 v) {
  double hi = (double)v;
  double lo = (double)(v - (__float128)hi);
  return {hi, lo};
}
struct cdd {
  dd re, im;
};
static inline cdd cdd_add(cdd a, cdd b) { return {dd_add(a.re, b.re), dd_add(a.im, b.im)}; }
static inline cdd cdd_sub(cdd a, cdd b) { return {dd_add(a.re, dd_neg(b.re)), dd_add(a.im, dd_neg(b.im))}; }
static inline cdd cdd_mul(cdd a, cdd b) {
  return {dd_add(dd_mul(a.re, b.re), dd_neg(dd_mul(a.im, b.im))), dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}

// exp(i pi k / N) for k < N, as double-double (cached per log_n)
static const std::vector<cdd>& zeta_table(uint32_t log_n) {
  static std::mutex mu;
  static std::map<uint32_t, std::vector<cdd>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(log_n);
  if (it != cache.end()) return it->second;
  uint32_t N = 1u << log_n;
  std::vector<cdd> t(N);
  for (uint32_t k = 0; k < N; k++) {
    __float128 a = M_PIq * (__float128)k / (__float128)N;
    t[k] = {dd_from_q(cosq(a)), dd_from_q(sinq(a))};
  }
  return cache.emplace(log_n, std::move(t)).first->second;
}

// X[i] = sum_k x[k] exp(+2 pi i ik/N), in place, radix-2 DIT.
template <typename C, typename Mul, typename Add, typename Sub, typename Tw>
static void fft_pos(std::vector<C>& x, uint32_t log_n, Mul mul, Add add, Sub sub, Tw tw) {
  uint32_t N = 1u << log_n;
  for (uint32_t i = 0; i < N; i++) {
    uint32_t j = bitrev(i, log_n);
    if (i < j) std::swap(x[i], x[j]);
  }
  for (uint32_t len = 2; len <= N; len <<= 1) {
    uint32_t stride = N / len;  // omega_len^k = omega_N^(k stride) = zeta^(2 k stride)
    for (uint32_t s = 0; s < N; s += len)
      for (uint32_t k = 0; k < len / 2; k++) {
        C w = tw(2 * k * stride);
        C u = x[s + k], v = mul(x[s + k + len / 2], w);
        x[s + k] = add(u, v);
        x[s + k + len / 2] = sub(u, v);
      }
  }
}

static __float128 encode_direct_q(const double* z, uint32_t log_n, double delta, uint32_t i) {
  uint64_t N = 1ull << log_n, n = N / 2, twoN = 2 * N;
  __float128 acc = 0;
  uint64_t e = 1;
  for (uint64_t j = 0; j < n; j++) {
    if (z[j] != 0.0) acc += (__float128)z[j] * cosq(M_PIq * (__float128)((e * i) % twoN) / (__float128)N);
    e = e * 5 % twoN;
  }
  return 2 * (__float128)delta / (__float128)N * acc;
}

int encode_slots(const double* z, size_t, uint32_t log_n, double delta, int64_t* out) {
  const uint32_t N = 1u << log_n, n = N / 2, twoN = 2 * N;
  const auto& Z = zeta_table(log_n);
  std::vector<cdd> x(N, cdd{{0, 0}, {0, 0}});
  uint64_t e = 1;
  for (uint32_t j = 0; j < n; j++) {
    if (z[j] != 0.0) {
      x[(e - 1) / 2].re = {z[j], 0};
      x[(twoN - e - 1) / 2].re = {z[j], 0};
    }
    e = e * 5 % twoN;
  }
  fft_pos(x, log_n, cdd_mul, cdd_add, cdd_sub, [&](uint32_t k) { return Z[k]; });
  const double scale = delta / (double)N;  // exact: Delta is an integer < 2^53 or a power of two, N a power of two
  int status = 0;
  for (uint32_t i = 0; i < N; i++) {
    // Re(zeta^i F_i) (Delta/N)
    dd v = dd_add(dd_mul(Z[i].re, x[i].re), dd_neg(dd_mul(Z[i].im, x[i].im)));
    v = dd_mul(v, dd{scale, 0});
    double fh = std::floor(v.hi);
    if (std::fabs(fh) >= 4.0e18) { status = HELRM_ERR_CONFIG; out[i] = 0; continue; }
    int64_t F = (int64_t)fh;
    double r = v.hi - fh;                 // exact, [0, 1)
    double fl = std::floor(v.lo);
    F += (int64_t)fl;
    r += v.lo - fl;                       // [0, 2)
    if (r >= 1.0) { F += 1; r -= 1.0; }
    if (std::fabs(r - 0.5) < 0x1p-30) {   // too close to a tie: binary128 direct sum
      __float128 q = encode_direct_q(z, log_n, delta, i);
      __float128 rq = roundq(q);          // half away from zero
      out[i] = (int64_t)rq;
      if (fabsq(rq) >= 4611686018427387904.0Q) status = HELRM_ERR_CONFIG;
      continue;
    }
    int64_t m = (F >= 0) ? F + (r >= 0.5 ? 1 : 0) : F + (r > 0.5 ? 1 : 0);
    if (m >= (1ll << 62) || m <= -(1ll << 62)) status = HELRM_ERR_CONFIG;
    out[i] = m;
  }
  return status;
}

void decode_coeffs(const int64_t* m, uint32_t log_n, double delta, double* z, size_t n_slots) {
  const uint32_t N = 1u << log_n, n = N / 2, twoN = 2 * N;
  using C = std::complex<double>;
  std::vector<C> x(N);
  std::vector<C> tw(N);
  for (uint32_t k = 0; k < N; k++) tw[k] = std::polar(1.0, M_PI * (double)k / (double)N);
  for (uint32_t i = 0; i < N; i++) x[i] = (double)m[i] * tw[i];
  fft_pos(x, log_n, [](C a, C b) { return a * b; }, [](C a, C b) { return a + b; },
          [](C a, C b) { return a - b; }, [&](uint32_t k) { return tw[k]; });
  uint64_t e = 1;
  for (uint32_t j = 0; j < n && j < n_slots; j++) {
    z[j] = x[(e - 1) / 2].real() / delta;
    e = e * 5 % twoN;
  }
}

void crt_small(const uint64_t* res, const uint64_t* primes, size_t nl, size_t N, int64_t* out) {
  // m = sum_i y_i (Q/q_i) - v Q with y_i = [x_i (Q/q_i)^-1]_{q_i}, v = round(sum y_i / q_i);
  // evaluated mod 2^64 (valid when |m| < 2^63).
  std::vector<uint64_t> inv(nl), qhat64(nl);
  uint64_t Q64 = 1;
  for (size_t i = 0; i < nl; i++) Q64 *= primes[i];
  for (size_t i = 0; i < nl; i++) {
    uint64_t h = 1, h64 = 1;
    for (size_t j = 0; j < nl; j++)
      if (j != i) { h = mulm(h, primes[j] % primes[i], primes[i]); h64 *= primes[j]; }
    inv[i] = inv_mod(h, primes[i]);
    qhat64[i] = h64;
  }
  for (size_t c = 0; c < N; c++) {
    long double f = 0;
    uint64_t acc = 0;
    for (size_t i = 0; i < nl; i++) {
      uint64_t y = mulm(res[i * N + c], inv[i], primes[i]);
      f += (long double)y / (long double)primes[i];
      acc += y * qhat64[i];
    }
    uint64_t v = (uint64_t)llroundl(f);
    out[c] = (int64_t)(acc - v * Q64);
  }
}

std::vector<uint64_t> gauss_cdt_table() {
  const __float128 sig = (__float128)32 / 10, s2 = 2 * sig * sig;
  __float128 rho[20], Z = 0;
  for (int x = 0; x < 20; x++) rho[x] = expq(-(__float128)(x * x) / s2);
  Z = rho[0];
  for (int x = 1; x < 20; x++) Z += 2 * rho[x];
  std::vector<uint64_t> T(20, 0);
  __float128 acc = 0;
  for (int k = 0; k < 19; k++) {
    acc += (k == 0) ? rho[0] : 2 * rho[k];
    T[k] = (uint64_t)floorq(acc / Z * 18446744073709551616.0Q);
  }
  T[19] = 0;  // stands for 2^64 (never compared)
  return T;
}

}  // namespace helrm
