// kernels_mac_bulk.cu -- D20 L3 inner sums (batch 1) fed by bulk async copies.
//
// Same arithmetic and work order as k_diag_mac1 / k_diag_mac (kernels_rns.cu):
// (A, B)_z[l][p] = sum_t u_{z,t}[l][p] (x0_t, x1_t)[l][p] for the kGiantPack
// giants z of a pack, exact FP64 MACs folded every kFAccTerms products, D-form
// operands, canonical outputs.  What differs is how the operands reach the
// SM: a producer warp streams every term's 256-position tiles (x0, x1 and
// up to four plaintexts, 2 KiB each) into a ring of shared-memory stages with
// cp.async.bulk (the TMA engine's 1-D copies, completion counted on an
// mbarrier), and 256 consumer threads read them from shared memory.
//
// Why: the register-fed kernels need ~24 warps per SM to keep enough bytes in
// flight for HBM, which fills the register file, so an NTT launched
// concurrently on another stream cannot share the SMs (the giant-step
// pipeline measured neutral).  Here the bytes in flight are the ring
// (S x 12 KiB per SM) regardless of the thread count: one 384-thread CTA per
// SM (256 consumers, 4 producer warps, 80 registers: 31 K of the 64 K) streams
// at the same rate as k_diag_mac1 (1.41 vs 1.43 ms per Criteo lookup) and
// leaves room for two NTT CTAs beside it.  Measured: with the giant steps
// pipelined in 4-giant chunks the overlap recovers ~0.35 ms, less than the
// finer chunking costs (7.04-7.3 vs 6.9 ms), so the path is off by default
// (HELRM_MAC_BULK=1; stages HELRM_MACB_STAGES, CTAs per SM HELRM_MACB_CTAS).
#include "internal.h"
#include "fmath.cuh"

namespace helrm {

namespace {
constexpr int kBulkSlots = 2 + kGiantPack;             // x0, x1, u[0..3]
constexpr int kTile = 256;                               // positions per work item (consumer threads)
constexpr uint32_t kSlotBytes = kTile * 8;               // 2 KiB
constexpr uint32_t kStageBytes = kBulkSlots * kSlotBytes;   // 12 KiB
constexpr int kProducers = 4;                           // producer warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16); completion counted on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
}  // namespace

// grid: persistent CTAs; block: 256 consumers + 1 producer warp; dynamic smem:
// stages x 12 KiB ring + 2 stages mbarriers + stage masks.
__global__ void __launch_bounds__(kTile + 32 * kProducers, 2)
    k_diag_mac_bulk(const MacTerm* __restrict__ terms, const int4* __restrict__ groups, int n_groups,
                    uint64_t* __restrict__ out, size_t out_stride, size_t half, const PrimeDev* __restrict__ primes,
                    const __grid_constant__ LimbMap map, uint32_t N, int stages) {
  constexpr int G = kGiantPack;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * kStageBytes);
  uint64_t* empty = full + stages;
  int* smask = reinterpret_cast<int*>(empty + stages);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);        // the producer's arrive (plus the copies' bytes)
      mbar_init(&empty[s], kTile / 32);   // every consumer warp releases the stage
    }
  }
  __syncthreads();
  const uint32_t tiles = N / kTile, total = tiles * (uint32_t)n_groups * (uint32_t)map.n;
  if (tid >= kTile) {
    // ---------------- producer warps ----------------
    // kProducers warps, lane 0 each: term j of the CTA's sequence goes to warp j % kProducers
    // (stages % kProducers == 0, so every stage has one owner and its waits stay in phase
    // order).  An issued bulk copy occupies its warp for a while, so several warps issue in
    // parallel.  Per term: wait for the stage, arm its barrier with the byte count, issue the
    // (up to) six 2 KiB copies.  The next term's pointers are loaded before the wait.
    const int pw = (tid - kTile) >> 5;
    if ((tid & 31) != 0) return;
    uint32_t j = 0;
    for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
      const int4 gr = groups[w % n_groups];   // pack fastest (as k_diag_mac): packs of a tile share baby pairs in L2
      const size_t o0 = (size_t)(w / (tiles * n_groups)) * N + ((w / n_groups) % tiles) * kTile;
      int t = (int)((kProducers + pw - j % kProducers) % kProducers);   // first term of this warp
      j += t;
      MacTerm m{};
      if (t < gr.y) m = terms[gr.x + t];
      for (; t < gr.y; t += kProducers, j += kProducers) {
        const MacTerm cur = m;
        if (t + kProducers < gr.y) m = terms[gr.x + t + kProducers];
        const int stage = (int)(j % (uint32_t)stages);
        const uint32_t phase = (j / (uint32_t)stages) & 1u;
        const uint64_t* src[kBulkSlots] = {cur.x0, cur.x1, cur.u[0], cur.u[1], cur.u[2], cur.u[3]};
        int mask = 0;
#pragma unroll
        for (int k = 0; k < kBulkSlots; k++)
          if (src[k]) mask |= 1 << k;
        mbar_wait(&empty[stage], phase ^ 1);
        smask[stage] = mask;
        mbar_arrive_expect_tx(&full[stage], (uint32_t)__popc(mask) * kSlotBytes);
        unsigned char* st = ring + (size_t)stage * kStageBytes;
#pragma unroll
        for (int k = 0; k < kBulkSlots; k++)
          if (src[k]) bulk_g2s(st + k * kSlotBytes, src[k] + o0, kSlotBytes, &full[stage]);
      }
      j -= (uint32_t)(t - gr.y);   // j = count of terms so far (t overshot gr.y)
    }
    return;
  }
  // ---------------- consumers: one position each ----------------
  int stage = 0;
  uint32_t phase = 0;
  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int4 gr = groups[w % n_groups];
    const int l = (int)(w / (tiles * n_groups));
    const size_t o = (size_t)l * N + ((w / n_groups) % tiles) * kTile + tid;
    const PrimeDev& P = primes[map.pr[l]];
    const double q = P.qd, qi = P.qinv;
    fm::FAcc acc0[G], acc1[G];
    int cnt = 0;
    for (int t = 0; t < gr.y; t++) {
      mbar_wait(&full[stage], phase);
      const int mask = smask[stage];
      const double* st = reinterpret_cast<const double*>(ring + (size_t)stage * kStageBytes);
      const double xa = st[tid], xb = st[kTile + tid];
      double u[G];
#pragma unroll
      for (int g = 0; g < G; g++) u[g] = (mask >> (2 + g)) & 1 ? st[(2 + g) * kTile + tid] : 0.0;
      __syncwarp();   // the warp's operands are in registers: the stage may be refilled
      if ((tid & 31) == 0) mbar_arrive(&empty[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
      if (cnt == fm::kFAccTerms) {
#pragma unroll
        for (int g = 0; g < G; g++) {
          fm::fold(acc0[g], q, qi);
          fm::fold(acc1[g], q, qi);
        }
        cnt = 0;
      }
      cnt++;
#pragma unroll
      for (int g = 0; g < G; g++) {
        fm::fmac(acc0[g], u[g], xa);
        fm::fmac(acc1[g], u[g], xb);
      }
    }
#pragma unroll
    for (int g = 0; g < G; g++) {
      if (g < gr.w) {
        uint64_t* dst = out + (size_t)(gr.z + g) * out_stride;
        dst[o] = fm::c2u(fm::fred(acc0[g], q, qi), P.rc.q);
        dst[half + o] = fm::c2u(fm::fred(acc1[g], q, qi), P.rc.q);
      }
    }
  }
}

bool launch_diag_mac_bulk(const DevCtx& c, const MacTerm* terms, const int4* groups, int n_groups, uint64_t* out,
                          size_t out_stride, size_t half, const LimbMap& map) {
  if (c.N % kTile) return false;
  static const int stages_env = getenv("HELRM_MACB_STAGES") ? atoi(getenv("HELRM_MACB_STAGES")) : 8;
  const int stages = std::max(kProducers, stages_env / kProducers * kProducers);   // a multiple of kProducers
  static const int per_sm = getenv("HELRM_MACB_CTAS") ? atoi(getenv("HELRM_MACB_CTAS")) : 1;
  const size_t smem = (size_t)stages * (kStageBytes + 8 + 8 + 4);
  static bool attr = false;
  if (!attr) {
    HCUDA(cudaFuncSetAttribute(k_diag_mac_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const unsigned total = (c.N / kTile) * (unsigned)n_groups * map.n;
  const unsigned grid = std::min<unsigned>(total, 148u * (unsigned)per_sm);
  k_diag_mac_bulk<<<grid, kTile + 32 * kProducers, smem, c.stream>>>(terms, groups, n_groups, out, out_stride, half, c.primes, map,
                                                        c.N, stages);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
  return true;
}

}  // namespace helrm
