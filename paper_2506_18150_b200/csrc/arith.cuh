// arith.cuh -- 64-bit modular arithmetic for RNS limbs (q < 2^62; the
// configs use 30/40/50-bit primes).  Device and host.
//
// Shoup multiplication by a constant w with w' = floor(w 2^64 / q):
//   r = a w - floor(a w' / 2^64) q  (mod 2^64)  lies in [0, 2q) for any a < 2^64.
// Lazy sums of products are accumulated in 128 bits and reduced once
// (reduce128), which is exact because every accumulation here keeps the
// high word below q.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

namespace helrm {

HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

HD uint64_t csub(uint64_t a, uint64_t q) { return a >= q ? a - q : a; }
HD uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
HD uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

// a * w mod q, result in [0, 2q)
HD uint64_t shoup_lazy(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
  return a * w - mulhi64(a, wp) * q;
}
HD uint64_t shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) { return csub(shoup_lazy(a, w, wp, q), q); }

// shoup companion of w (host side)
inline uint64_t shoup_pre(uint64_t w, uint64_t q) { return (uint64_t)(((unsigned __int128)w << 64) / q); }

struct U128 {
  uint64_t lo, hi;
};

HD void mac128(U128& acc, uint64_t a, uint64_t b) {
  uint64_t lo = a * b, hi = mulhi64(a, b);
#if defined(__CUDA_ARCH__)
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(acc.lo), "+l"(acc.hi) : "l"(lo), "l"(hi));
#else
  unsigned __int128 s = ((unsigned __int128)acc.hi << 64 | acc.lo) + ((unsigned __int128)hi << 64 | lo);
  acc.lo = (uint64_t)s;
  acc.hi = (uint64_t)(s >> 64);
#endif
}

// Per-prime constants for reductions.
struct RedConst {
  uint64_t q;
  uint64_t mu;     // floor(2^64 / q)
  uint64_t r64;    // 2^64 mod q
  uint64_t r64s;   // shoup companion of r64
};

// (hi 2^64 + lo) mod q, valid when hi < 2^64 (exact result in [0, q)).
HD uint64_t reduce128(uint64_t hi, uint64_t lo, const RedConst& c) {
  uint64_t t = shoup_lazy(hi, c.r64, c.r64s, c.q);          // hi 2^64 mod q, [0, 2q)
  uint64_t u = lo - mulhi64(lo, c.mu) * c.q;                 // lo mod q, [0, 2q)
  uint64_t s = t + u;                                        // [0, 4q)
  s = csub(s, 2 * c.q);
  return csub(s, c.q);
}

HD uint64_t mul_mod(uint64_t a, uint64_t b, const RedConst& c) { return reduce128(mulhi64(a, b), a * b, c); }

// ---- "split" residues for streaming multiply-accumulates (q < 2^50) ----
// x = x1 2^25 + x0 with x0, x1 < 2^25 is stored as (x1 << 32) | x0, so a
// product of two residues is four 32x32 -> 64-bit IMAD.WIDE with 64-bit
// accumulators c0 += x0 y0, c1 += x0 y1 + x1 y0, c2 += x1 y1 (each term
// < 2^51: 8192 products fit), reduced once: x = c0 + c1 2^25 + c2 2^50.
// Rotation keys, plaintext diagonals and the baby-step pairs live in this
// form on the device.
HD uint64_t to_split(uint64_t x) { return ((x >> 25) << 32) | (x & 0x1FFFFFFull); }
HD uint64_t from_split(uint64_t s) { return ((s >> 32) << 25) | (s & 0xFFFFFFFFull); }

struct Acc3 {
  uint64_t c0 = 0, c1 = 0, c2 = 0;
};

HD void mac_split(Acc3& a, uint64_t xs, uint64_t ys) {
  const uint32_t x0 = (uint32_t)xs, x1 = (uint32_t)(xs >> 32), y0 = (uint32_t)ys, y1 = (uint32_t)(ys >> 32);
  a.c0 += (uint64_t)x0 * y0;
  a.c1 += (uint64_t)x0 * y1;
  a.c1 += (uint64_t)x1 * y0;
  a.c2 += (uint64_t)x1 * y1;
}

// (c0 + c1 2^25 + c2 2^50) mod q
HD uint64_t acc3_reduce(const Acc3& a, const RedConst& rc) {
  uint64_t lo = a.c0, hi = 0;
  uint64_t t = a.c1 << 25;
  lo += t;
  hi += (lo < t) + (a.c1 >> 39);
  t = a.c2 << 50;
  lo += t;
  hi += (lo < t) + (a.c2 >> 14);
  return reduce128(hi, lo, rc);
}

// counter-based SplitMix64 (D9): word(seed, stream, k) = SM((seed ^ SM(stream)) + (k+1) gamma)
HD uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
HD uint64_t prng_word(uint64_t base, uint64_t k) { return sm_mix(base + (k + 1) * 0x9E3779B97F4A7C15ull); }
HD uint64_t prng_base(uint64_t seed, uint64_t stream) { return seed ^ sm_mix(stream); }
HD uint64_t prng_stream(uint64_t purpose, uint64_t a, uint64_t b, uint64_t c) {
  return (purpose << 56) | (a << 32) | (b << 16) | c;
}

}  // namespace helrm
