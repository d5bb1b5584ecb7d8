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
