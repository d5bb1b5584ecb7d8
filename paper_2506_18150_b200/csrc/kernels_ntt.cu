// kernels_ntt.cu -- negacyclic NTT / INTT over 64-bit RNS limbs (sm_100a).
//
// D4: NTT_q(a)_i = sum_j a_j psi^{(2i+1) j}.  The library
// keeps NTT-form data in "slot order": position s < N/2 holds the evaluation
// at psi^(5^s), position N/2 + s the one at psi^(-5^s) (D5), so every Galois
// automorphism phi_{5^r} is a cyclic shift by r inside each half -- the
// rotations of the lookup become offset loads instead of gathers.
//
// Forward: Cooley-Tukey with merged psi-twist (twiddle psi^bitrev(m+i)),
// natural input -> bit-reversed output, split in two passes so each CTA
// works on a 32 KB tile in shared memory:
//   pass 1: the first s1 = log N - 8 stages act on columns {c + 256 h};
//           a CTA loads C consecutive columns (128-byte row segments).
//   pass 2: the last 8 stages act inside contiguous 256-element blocks;
//           the result is written through the bit-reversed -> slot-order
//           permutation.
// Inverse: Gentleman-Sande mirror (gather from slot order, blocks first,
// then columns, times N^-1).
// Between the passes the data live in a scratch buffer that the launcher
// sizes to stay L2-resident (<= 32 MiB per chunk of limbs), so HBM sees one
// read and one write per coefficient.
#include "internal.h"

namespace helrm {

namespace {
constexpr int kTile = 4096;   // elements per CTA (32 KB of shared memory)
constexpr int kThreads = 512;
constexpr int kS2 = 8;        // log2 of the pass-2 block

struct Geo {
  int log_n, N, s1, s2, R, W2, C, G1, NB, G2;
};

Geo geometry(int log_n) {
  Geo g;
  g.log_n = log_n;
  g.N = 1 << log_n;
  g.s2 = log_n < kS2 ? log_n : kS2;
  g.s1 = log_n - g.s2;
  g.R = 1 << g.s1;
  g.W2 = 1 << g.s2;
  g.C = kTile / g.R;
  if (g.C > g.W2) g.C = g.W2;
  g.G1 = g.W2 / g.C;
  g.NB = kTile / g.W2;
  if (g.NB > g.N / g.W2) g.NB = g.N / g.W2;
  g.G2 = (g.N / g.W2) / g.NB;
  return g;
}
}  // namespace

__global__ void __launch_bounds__(kThreads) k_ntt_fwd_p1(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                         const PrimeDev* __restrict__ primes, LimbMap map,
                                                         size_t limb0, Geo g) {
  extern __shared__ uint64_t sm[];
  const size_t limb = blockIdx.y;
  const PrimeDev& P = primes[map.pr[(limb0 + limb) % map.n]];
  const uint64_t q = P.rc.q;
  const uint64_t* s = src + limb * g.N;
  uint64_t* d = dst + limb * g.N;
  const int c0 = blockIdx.x * g.C, tile = g.R * g.C;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) sm[e] = s[(size_t)(e / g.C) * g.W2 + c0 + e % g.C];
  __syncthreads();
  for (int st = 0; st < g.s1; st++) {
    const int m = 1 << st, T = g.R >> (st + 1);
    for (int b = threadIdx.x; b < tile / 2; b += blockDim.x) {
      const int c = b % g.C, bb = b / g.C;
      const int i = bb / T, h = 2 * i * T + bb % T;
      const uint64_t w = P.tw[m + i], wp = P.tws[m + i];
      const uint64_t U = sm[h * g.C + c];
      const uint64_t V = shoup(sm[(h + T) * g.C + c], w, wp, q);
      sm[h * g.C + c] = add_mod(U, V, q);
      sm[(h + T) * g.C + c] = sub_mod(U, V, q);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < tile; e += blockDim.x) d[(size_t)(e / g.C) * g.W2 + c0 + e % g.C] = sm[e];
}

__global__ void __launch_bounds__(kThreads) k_ntt_fwd_p2(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                         const PrimeDev* __restrict__ primes, LimbMap map,
                                                         size_t limb0, Geo g, const uint32_t* __restrict__ slotpos) {
  extern __shared__ uint64_t sm[];
  const size_t limb = blockIdx.y;
  const PrimeDev& P = primes[map.pr[(limb0 + limb) % map.n]];
  const uint64_t q = P.rc.q;
  const uint64_t* s = src + limb * g.N;
  uint64_t* d = dst + limb * g.N;
  const int tile = g.NB * g.W2, base = blockIdx.x * tile;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) sm[e] = s[base + e];
  __syncthreads();
  for (int st = g.s1; st < g.log_n; st++) {
    const int m = 1 << st, t = g.N >> (st + 1);
    for (int b = threadIdx.x; b < tile / 2; b += blockDim.x) {
      const int B = base / 2 + b;
      const int i = B / t, j = 2 * i * t + B % t - base;
      const uint64_t w = P.tw[m + i], wp = P.tws[m + i];
      const uint64_t U = sm[j];
      const uint64_t V = shoup(sm[j + t], w, wp, q);
      sm[j] = add_mod(U, V, q);
      sm[j + t] = sub_mod(U, V, q);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < tile; e += blockDim.x) d[slotpos[base + e]] = sm[e];
}

__global__ void __launch_bounds__(kThreads) k_ntt_inv_pa(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                         const PrimeDev* __restrict__ primes, LimbMap map,
                                                         size_t limb0, Geo g, const uint32_t* __restrict__ slotpos) {
  extern __shared__ uint64_t sm[];
  const size_t limb = blockIdx.y;
  const PrimeDev& P = primes[map.pr[(limb0 + limb) % map.n]];
  const uint64_t q = P.rc.q;
  const uint64_t* s = src + limb * g.N;
  uint64_t* d = dst + limb * g.N;
  const int tile = g.NB * g.W2, base = blockIdx.x * tile;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) sm[e] = s[slotpos[base + e]];
  __syncthreads();
  for (int st = g.log_n - 1; st >= g.s1; st--) {
    const int m = 1 << st, t = g.N >> (st + 1);
    for (int b = threadIdx.x; b < tile / 2; b += blockDim.x) {
      const int B = base / 2 + b;
      const int i = B / t, j = 2 * i * t + B % t - base;
      const uint64_t w = P.itw[m + i], wp = P.itws[m + i];
      const uint64_t U = sm[j], V = sm[j + t];
      sm[j] = add_mod(U, V, q);
      sm[j + t] = shoup(sub_mod(U, V, q), w, wp, q);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < tile; e += blockDim.x) d[base + e] = sm[e];
}

__global__ void __launch_bounds__(kThreads) k_ntt_inv_pb(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                         const PrimeDev* __restrict__ primes, LimbMap map,
                                                         size_t limb0, Geo g) {
  extern __shared__ uint64_t sm[];
  const size_t limb = blockIdx.y;
  const PrimeDev& P = primes[map.pr[(limb0 + limb) % map.n]];
  const uint64_t q = P.rc.q;
  const uint64_t* s = src + limb * g.N;
  uint64_t* d = dst + limb * g.N;
  const int c0 = blockIdx.x * g.C, tile = g.R * g.C;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) sm[e] = s[(size_t)(e / g.C) * g.W2 + c0 + e % g.C];
  __syncthreads();
  for (int st = g.s1 - 1; st >= 0; st--) {
    const int m = 1 << st, T = g.R >> (st + 1);
    for (int b = threadIdx.x; b < tile / 2; b += blockDim.x) {
      const int c = b % g.C, bb = b / g.C;
      const int i = bb / T, h = 2 * i * T + bb % T;
      const uint64_t w = P.itw[m + i], wp = P.itws[m + i];
      const uint64_t U = sm[h * g.C + c], V = sm[(h + T) * g.C + c];
      sm[h * g.C + c] = add_mod(U, V, q);
      sm[(h + T) * g.C + c] = shoup(sub_mod(U, V, q), w, wp, q);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < tile; e += blockDim.x)
    d[(size_t)(e / g.C) * g.W2 + c0 + e % g.C] = shoup(sm[e], P.ninv, P.ninvs, q);
}

static size_t chunk_limbs(int N) {
  size_t ch = ((size_t)64 << 16) / (size_t)N;  // 32 MiB of scratch per chunk
  return ch > 65535 ? 65535 : ch;
}

void launch_ntt_fwd(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, size_t n_total,
                    const LimbMap& map) {
  Geo g = geometry(c.log_n);
  const size_t ch = chunk_limbs(g.N);
  const size_t smem = kTile * sizeof(uint64_t);
  for (size_t off = 0; off < n_total; off += ch) {
    unsigned cnt = (unsigned)std::min(ch, n_total - off);
    {
      ProfScope ps_(c, "ntt_fwd_p1", 8.0 * g.N * cnt);
      k_ntt_fwd_p1<<<dim3(g.G1, cnt), kThreads, smem, c.stream>>>(src + off * g.N, scratch, c.primes, map, off, g);
    }
    {
      ProfScope ps_(c, "ntt_fwd_p2", 8.0 * g.N * cnt);
      k_ntt_fwd_p2<<<dim3(g.G2, cnt), kThreads, smem, c.stream>>>(scratch, dst + off * g.N, c.primes, map, off, g,
                                                                  c.slotpos);
    }
    *c.launches += 2;
  }
  HCUDA(cudaGetLastError());
}

void launch_ntt_inv(const DevCtx& c, const uint64_t* src, uint64_t* dst, uint64_t* scratch, size_t n_total,
                    const LimbMap& map) {
  Geo g = geometry(c.log_n);
  const size_t ch = chunk_limbs(g.N);
  const size_t smem = kTile * sizeof(uint64_t);
  for (size_t off = 0; off < n_total; off += ch) {
    unsigned cnt = (unsigned)std::min(ch, n_total - off);
    {
      ProfScope ps_(c, "ntt_inv_pa", 8.0 * g.N * cnt);
      k_ntt_inv_pa<<<dim3(g.G2, cnt), kThreads, smem, c.stream>>>(src + off * g.N, scratch, c.primes, map, off, g,
                                                                  c.slotpos);
    }
    {
      ProfScope ps_(c, "ntt_inv_pb", 8.0 * g.N * cnt);
      k_ntt_inv_pb<<<dim3(g.G1, cnt), kThreads, smem, c.stream>>>(scratch, dst + off * g.N, c.primes, map, off, g);
    }
    *c.launches += 2;
  }
  HCUDA(cudaGetLastError());
}

size_t ntt_scratch_words(int log_n) { return chunk_limbs(1 << log_n) * ((size_t)1 << log_n); }

}  // namespace helrm
