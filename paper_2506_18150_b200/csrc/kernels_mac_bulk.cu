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
// leaves room for two NTT CTAs beside it.  It is the default inner-sum kernel
// for every batch size (HELRM_MAC_BULK=2; 1 = batch 1 only, 0 = the
// register-fed kernels; ring depth HELRM_MACB_STAGES, CTAs per SM
// HELRM_MACB_CTAS).  With the giant steps pipelined in 4-giant chunks the
// overlap recovers ~0.35 ms, less than the finer chunking costs (7.04-7.3 vs
// 6.9 ms), so batch-1 lookups issue the giant steps serially.
#include "internal.h"
#include "fmath.cuh"

namespace helrm {

namespace {
constexpr int kTile = 256;                 // positions per work item (consumer threads)
constexpr uint32_t kSlotBytes = kTile * 8;   // 2 KiB
// producer warps: 4 (2 at QN = 4: its consumers hold 128 accumulator registers; measured
// 5520 against 5420 token lookups/s with 3)
template <int QN>
__host__ __device__ constexpr int bulk_producers() { return QN >= 4 ? 2 : 4; }
// stage: x0 of QN queries, x1 of QN queries, the kGiantPack plaintexts
template <int QN>
__host__ __device__ constexpr int bulk_slots() { return 2 * QN + kGiantPack; }

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

// grid: persistent CTAs; block: 256 consumers + kProducers producer warps;
// dynamic smem: stages x (2 QN + 4) 2 KiB slots + per stage two mbarriers
// and a plaintext mask.  nq queries (a multiple of QN): query k reads its
// baby pairs at x + k xq and writes out + k oq (the plaintexts are shared);
// QN of them per pass over the terms.
// QS consumer threads per position, each taking QN / QS queries (QS = 2 at
// QN = 4 gives 16 consumer warps instead of 8 but measured 5730 against 5850
// token lookups/s: the 576-thread CTA spills; kept at 1)
template <int QN>
__host__ __device__ constexpr int bulk_qsplit() { return 1; }
template <int QN, int kProducers = bulk_producers<QN>(), int QS = bulk_qsplit<QN>()>
__global__ void __launch_bounds__(kTile * QS + 32 * kProducers, 1)
    k_diag_mac_bulk(const MacTerm* __restrict__ terms, const int4* __restrict__ groups, int n_groups,
                    uint64_t* __restrict__ out, size_t out_stride, size_t half, const PrimeDev* __restrict__ primes,
                    const __grid_constant__ LimbMap map, uint32_t N, int stages, int nq, size_t xq, size_t oq,
                    int accumulate, int row0, int nrows) {
  pdl_wait_trigger();
  constexpr int G = kGiantPack, NS = bulk_slots<QN>();
  constexpr uint32_t SB = NS * kSlotBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * SB);
  uint64_t* empty = full + stages;
  int* smask = reinterpret_cast<int*>(empty + stages);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);             // the producer's arrive (plus the copies' bytes)
      mbar_init(&empty[s], kTile * QS / 32);   // every consumer warp releases the stage
    }
  }
  __syncthreads();
  const uint32_t tiles = N / kTile, total = tiles * (uint32_t)n_groups * (uint32_t)nrows;
  const int nqc = nq / QN;   // query chunks per work item
  constexpr int kCons = kTile * QS, QT = QN / QS;   // consumer threads, queries per consumer thread
  if (tid >= kCons) {
    // ---------------- producer warps ----------------
    // Lane 0 of kProducers warps: item j of the CTA's sequence of (query chunk, term) items
    // goes to warp j % kProducers (stages % kProducers == 0, so every stage has one owner
    // and its waits stay in phase order).  An issued bulk copy occupies its warp for a
    // while, so several warps issue in parallel.  Per item: wait for the stage, arm its
    // barrier with the byte count, issue the 2 KiB copies.
    const int pw = (tid - kCons) >> 5;
    if ((tid & 31) != 0) return;
    uint32_t j = 0;
    for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
      const int4 gr = groups[w % n_groups];   // pack fastest (as k_diag_mac): packs of a tile share baby pairs in L2
      const size_t o0 = (size_t)(row0 + w / (tiles * n_groups)) * N + ((w / n_groups) % tiles) * kTile;
      const int items = nqc * gr.y;
      int it = (int)((kProducers + pw - j % kProducers) % kProducers);   // this warp's first item
      j += it;
      for (; it < items; it += kProducers, j += kProducers) {
        const int qc = it / gr.y, t = it % gr.y;
        const MacTerm m = terms[gr.x + t];
        const int stage = (int)(j % (uint32_t)stages);
        const uint32_t phase = (j / (uint32_t)stages) & 1u;
        int mask = 0;
#pragma unroll
        for (int g = 0; g < G; g++)
          if (m.u[g]) mask |= 1 << g;
        mbar_wait(&empty[stage], phase ^ 1);
        smask[stage] = mask;
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(2 * QN + __popc(mask)) * kSlotBytes);
        unsigned char* st = ring + (size_t)stage * SB;
#pragma unroll
        for (int k = 0; k < QN; k++) {
          const size_t xo = o0 + (size_t)(qc * QN + k) * xq;
          bulk_g2s(st + k * kSlotBytes, m.x0 + xo, kSlotBytes, &full[stage]);
          bulk_g2s(st + (QN + k) * kSlotBytes, m.x1 + xo, kSlotBytes, &full[stage]);
        }
#pragma unroll
        for (int g = 0; g < G; g++)
          if (m.u[g]) bulk_g2s(st + (2 * QN + g) * kSlotBytes, m.u[g] + o0, kSlotBytes, &full[stage]);
      }
      j -= (uint32_t)(it - items);   // j = items so far (it overshot by it - items)
    }
    return;
  }
  // ---------------- consumers: one position and QT queries each ----------------
  const int pos = tid % kTile, qh = tid / kTile;   // queries qh QT .. qh QT + QT - 1 of a chunk
  int stage = 0;
  uint32_t phase = 0;
  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int4 gr = groups[w % n_groups];
    const int l = row0 + (int)(w / (tiles * n_groups));
    const size_t o = (size_t)l * N + ((w / n_groups) % tiles) * kTile + pos;
    const PrimeDev& P = primes[map.pr[l]];
    const double q = P.qd, qi = P.qinv;
    for (int qc = 0; qc < nqc; qc++) {
      fm::FAcc acc0[QT][G], acc1[QT][G];
      int cnt = 0;
      for (int t = 0; t < gr.y; t++) {
        mbar_wait(&full[stage], phase);
        const int mask = smask[stage];
        const double* st = reinterpret_cast<const double*>(ring + (size_t)stage * SB);
        double xa[QT], xb[QT], u[G];
#pragma unroll
        for (int k = 0; k < QT; k++) {
          xa[k] = st[(qh * QT + k) * kTile + pos];
          xb[k] = st[(QN + qh * QT + k) * kTile + pos];
        }
#pragma unroll
        for (int g = 0; g < G; g++) u[g] = (mask >> g) & 1 ? st[(2 * QN + g) * kTile + pos] : 0.0;
        __syncwarp();   // the warp's operands are in registers: the stage may be refilled
        if ((tid & 31) == 0) mbar_arrive(&empty[stage]);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
        if (cnt == fm::kFAccTerms) {
#pragma unroll
          for (int k = 0; k < QT; k++)
#pragma unroll
            for (int g = 0; g < G; g++) {
              fm::fold(acc0[k][g], q, qi);
              fm::fold(acc1[k][g], q, qi);
            }
          cnt = 0;
        }
        cnt++;
#pragma unroll
        for (int k = 0; k < QT; k++)
#pragma unroll
          for (int g = 0; g < G; g++) {
            fm::fmac(acc0[k][g], u[g], xa[k]);
            fm::fmac(acc1[k][g], u[g], xb[k]);
          }
      }
#pragma unroll
      for (int k = 0; k < QT; k++)
#pragma unroll
        for (int g = 0; g < G; g++) {
          if (g < gr.w) {
            uint64_t* dst = out + (size_t)(gr.z + g) * out_stride + (size_t)(qc * QN + qh * QT + k) * oq;
            uint64_t v0 = fm::c2u(fm::fred(acc0[k][g], q, qi), P.rc.q);
            uint64_t v1 = fm::c2u(fm::fred(acc1[k][g], q, qi), P.rc.q);
            if (accumulate) {
              v0 = add_mod(v0, dst[o], P.rc.q);
              v1 = add_mod(v1, dst[half + o], P.rc.q);
            }
            dst[o] = v0;
            dst[half + o] = v1;
          }
        }
    }
  }
}

template <int QN>
static void bulk_launch(const DevCtx& c, const MacTerm* terms, const int4* groups, int n_groups, uint64_t* out,
                        size_t out_stride, size_t half, const LimbMap& map, int nq, size_t xq, size_t oq,
                        int accumulate, int row0, int rows) {
  static const int stages_env = getenv("HELRM_MACB_STAGES") ? atoi(getenv("HELRM_MACB_STAGES")) : 0;
  constexpr size_t SB = (size_t)bulk_slots<QN>() * kSlotBytes;
  // default: as many stages as fit in ~200 KiB (16 at 12 KiB, 8 at 24 KiB), a multiple of kProducers
  constexpr int kProducers = bulk_producers<QN>();
  const int want = stages_env > 0 ? stages_env : (int)(200 * 1024 / SB);
  const int stages = std::max(kProducers, want / kProducers * kProducers);
  static const int per_sm = getenv("HELRM_MACB_CTAS") ? atoi(getenv("HELRM_MACB_CTAS")) : 1;
  const size_t smem = (size_t)stages * (SB + 8 + 8 + 4);
  // the attribute is per device: cached per device ordinal
  static size_t attr[64] = {};
  int dev = 0;
  HCUDA(cudaGetDevice(&dev));
  if (dev >= 64 || attr[dev] != smem) {
    HCUDA(cudaFuncSetAttribute(k_diag_mac_bulk<QN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (dev < 64) attr[dev] = smem;
  }
  const unsigned total = (c.N / kTile) * (unsigned)n_groups * (unsigned)rows;
  const unsigned grid = std::min<unsigned>(total, (unsigned)c.n_sm * (unsigned)per_sm);
  launch_pdl(k_diag_mac_bulk<QN>, dim3(grid), dim3(kTile * bulk_qsplit<QN>() + 32 * kProducers), smem, c.stream, terms, groups, n_groups, out, out_stride, half, c.primes, map, c.N, stages, nq, xq, oq, accumulate, row0, rows);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

bool launch_diag_mac_bulk(const DevCtx& c, const MacTerm* terms, const int4* groups, int n_groups, uint64_t* out,
                          size_t out_stride, size_t half, const LimbMap& map, int nq, size_t xq, size_t oq,
                          int accumulate, int row0, int rows) {
  if (c.N % kTile || nq < 1) return false;
  if (rows <= 0) rows = map.n - row0;
  static const int qmax = getenv("HELRM_MACB_QMAX") ? atoi(getenv("HELRM_MACB_QMAX")) : 4;
  if (nq % 4 == 0 && qmax >= 4)
    bulk_launch<4>(c, terms, groups, n_groups, out, out_stride, half, map, nq, xq, oq, accumulate, row0, rows);
  else if (nq % 2 == 0 && qmax >= 2)
    bulk_launch<2>(c, terms, groups, n_groups, out, out_stride, half, map, nq, xq, oq, accumulate, row0, rows);
  else
    bulk_launch<1>(c, terms, groups, n_groups, out, out_stride, half, map, nq, xq, oq, accumulate, row0, rows);
  return true;
}

}  // namespace helrm
