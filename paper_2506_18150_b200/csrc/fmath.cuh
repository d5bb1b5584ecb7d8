// fmath.cuh -- RNS residue arithmetic on the FP64 pipe (device only, q < 2^50).
//
// B200 issues 64-bit integer multiplies as several 32-bit IMADs (a 64x64->128
// modular MAC measured 1.25-1.5 T/s, profiles/r01_peak_int.txt) but runs DFMA
// at 18.1 T/s.  Residues below 2^50 are exact integer-valued doubles, so the
// hot loops of the lookup compute on the FP64 pipe:
//
//  * mmul: Y W mod q for a constant W with its quotient W/q (NTT twiddles,
//    base-conversion factors): exact product split by one FMA, quotient
//    rounded with the 1.5 2^52 shift.
//  * FAcc: exact lazy sums of products x y (|x y| < 2^99).  With
//    M = 1.5 2^102, s = fma(x, y, M) rounds x y onto the 2^50 grid, so
//    h = s - M and l = fma(x, y, -h) = x y - h are both exact (|l| <= 2^49).
//    h's are summed exactly while |sum| < 2^103 (multiples of 2^50 with a
//    53-bit mantissa) and l's while |sum| <= 2^53: at most kFAccTerms
//    products between two folds.  fold() reduces both sums modulo q exactly
//    (the quotient of the h-sum through a 64-bit integer conversion) and
//    leaves a centred value in l.
//
// "D-form": a residue stored as the bit pattern of its centred,
// integer-valued double in [-q/2 - 1, q/2 + 1].  Streamed MAC operands
// (rotation keys, plaintext diagonals, baby-step pairs) live in D-form.
#pragma once
#include <cstdint>

namespace helrm {
namespace fm {

constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;
constexpr double kMacM = 0x1.8p+102;         // 1.5 * 2^102
constexpr int kFAccTerms = 14;                   // products of |x y| < 2^99 between folds

static_assert(kMacM == 1.5 * 5070602400912917605986812821504.0, "M = 1.5 2^102");
static_assert(kMagic == 0x1.8p+52, "1.5 2^52");

// x < 2^52 -> double
__device__ __forceinline__ double u2d(uint64_t x) {
  return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - kTwo52;
}
// centred reduction: |x / q| < 2^51 -> x mod q in [-q/2 - 1, q/2 + 1]
__device__ __forceinline__ double cred(double x, double q, double qi) {
  const double k = __fma_rn(x, qi, kMagic) - kMagic;
  return __fma_rn(-k, q, x);
}
// Y W mod q, exact, centred (|Y| < 2^51)
__device__ __forceinline__ double mmul(double y, double w, double wq, double q) {
  const double h = y * w;
  const double k = __fma_rn(y, wq, kMagic) - kMagic;
  const double l = __fma_rn(y, w, -h);
  return __fma_rn(-k, q, h) + l;
}
// canonical uint64 in [0, q) from an integer-valued double with |x| <= 2^51 q
__device__ __forceinline__ uint64_t d2u(double x, double q, double qi, uint64_t qint) {
  x = cred(x, q, qi);
  const long long v = (long long)(__double_as_longlong(x + kMagic) & 0xFFFFFFFFFFFFFull) - (1ll << 51);
  return (uint64_t)(v < 0 ? v + (long long)qint : v);
}
// centred integer-valued double (|x| < 2^51) -> canonical uint64 in [0, q)
__device__ __forceinline__ uint64_t c2u(double x, uint64_t qint) {
  const long long v = (long long)(__double_as_longlong(x + kMagic) & 0xFFFFFFFFFFFFFull) - (1ll << 51);
  return (uint64_t)(v < 0 ? v + (long long)qint : v);
}
// canonical residue -> centred double
__device__ __forceinline__ double u2c(uint64_t x, double q) {
  const double d = u2d(x);
  return d > 0.5 * q ? d - q : d;
}
__device__ __forceinline__ uint64_t d2bits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double bits2d(uint64_t x) { return __longlong_as_double((long long)x); }

struct FAcc {
  double h = 0.0, l = 0.0;
};

// a += x y  (|x y| < 2^99), exact
__device__ __forceinline__ void fmac(FAcc& a, double x, double y) {
  const double s = __fma_rn(x, y, kMacM);
  const double h = __dsub_rn(s, kMacM);
  const double l = __fma_rn(x, y, -h);
  a.h = __dadd_rn(a.h, h);
  a.l = __dadd_rn(a.l, l);
}

// exact: a <- (0, a mod q centred); valid after <= kFAccTerms products
__device__ __forceinline__ void fold(FAcc& a, double q, double qi) {
  const double k = (double)__double2ll_rn(a.h * qi);   // |a.h / q| < 2^53
  const double hr = __fma_rn(-k, q, a.h);              // exact, |hr| < 4q
  a.l = cred(__dadd_rn(cred(a.l, q, qi), hr), q, qi);
  a.h = 0.0;
}

// final value, centred in [-q/2 - 1, q/2 + 1]
__device__ __forceinline__ double fred(FAcc a, double q, double qi) {
  fold(a, q, qi);
  return a.l;
}

}  // namespace fm
}  // namespace helrm
