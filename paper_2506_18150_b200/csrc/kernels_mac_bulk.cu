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
                    const __grid_constant__ LimbMap map, uint32_t N, int stages, int nq, size_t xq, size_t oq) {
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
  const uint32_t tiles = N / kTile, total = tiles * (uint32_t)n_groups * (uint32_t)map.n;
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
      const size_t o0 = (size_t)(w / (tiles * n_groups)) * N + ((w / n_groups) % tiles) * kTile;
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
    const int l = (int)(w / (tiles * n_groups));
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
            dst[o] = fm::c2u(fm::fred(acc0[k][g], q, qi), P.rc.q);
            dst[half + o] = fm::c2u(fm::fred(acc1[k][g], q, qi), P.rc.q);
          }
        }
    }
  }
}

template <int QN>
static void bulk_launch(const DevCtx& c, const MacTerm* terms, const int4* groups, int n_groups, uint64_t* out,
                        size_t out_stride, size_t half, const LimbMap& map, int nq, size_t xq, size_t oq) {
  static const int stages_env = getenv("HELRM_MACB_STAGES") ? atoi(getenv("HELRM_MACB_STAGES")) : 0;
  constexpr size_t SB = (size_t)bulk_slots<QN>() * kSlotBytes;
  // default: as many stages as fit in ~200 KiB (16 at 12 KiB, 8 at 24 KiB), a multiple of kProducers
  constexpr int kProducers = bulk_producers<QN>();
  const int want = stages_env > 0 ? stages_env : (int)(200 * 1024 / SB);
  const int stages = std::max(kProducers, want / kProducers * kProducers);
  static const int per_sm = getenv("HELRM_MACB_CTAS") ? atoi(getenv("HELRM_MACB_CTAS")) : 1;
  const size_t smem = (size_t)stages * (SB + 8 + 8 + 4);
  static size_t attr = 0;
  if (attr != smem) {
    HCUDA(cudaFuncSetAttribute(k_diag_mac_bulk<QN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  const unsigned total = (c.N / kTile) * (unsigned)n_groups * map.n;
  const unsigned grid = std::min<unsigned>(total, 148u * (unsigned)per_sm);
  launch_pdl(k_diag_mac_bulk<QN>, dim3(grid), dim3(kTile * bulk_qsplit<QN>() + 32 * kProducers), smem, c.stream, terms, groups, n_groups, out, out_stride, half, c.primes, map, c.N, stages, nq, xq, oq);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
}

bool launch_diag_mac_bulk(const DevCtx& c, const MacTerm* terms, const int4* groups, int n_groups, uint64_t* out,
                          size_t out_stride, size_t half, const LimbMap& map, int nq, size_t xq, size_t oq) {
  if (c.N % kTile || nq < 1) return false;
  static const int qmax = getenv("HELRM_MACB_QMAX") ? atoi(getenv("HELRM_MACB_QMAX")) : 4;
  if (nq % 4 == 0 && qmax >= 4) bulk_launch<4>(c, terms, groups, n_groups, out, out_stride, half, map, nq, xq, oq);
  else if (nq % 2 == 0 && qmax >= 2) bulk_launch<2>(c, terms, groups, n_groups, out, out_stride, half, map, nq, xq, oq);
  else bulk_launch<1>(c, terms, groups, n_groups, out, out_stride, half, map, nq, xq, oq);
  return true;
}

}  // namespace helrm

namespace helrm {

// ---------------------------------------------------------------------------
// D20 L2 + L3 fused for one ciphertext, fed by bulk async copies
// (HELRM_FUSED_BM=2).  Work item = (256-position tile, limb).  The consumers
// stage the tile's digits and c0 (plus the rotation halo) once, compute every
// baby pair of the tile into shared memory from key tiles streamed through
// the ring (2 dnum tiles per baby), then run the inner sums of every giant
// pack against plaintext tiles streamed through the same ring.  The baby pairs
// never go to HBM (against k_kip_multi + k_diag_mac_bulk: 0.87 GB written and
// read back per Criteo lookup).  Same arithmetic as those kernels.
namespace {
constexpr int kFbProducers = 3;
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kTile) : "memory"); }
}  // namespace

template <int DNUM>
__global__ void __launch_bounds__(kTile + 32 * kFbProducers, 1)
    k_baby_mac_bulk(const __grid_constant__ KipMulti a, const __grid_constant__ BabyMacArgs m,
                    const PrimeDev* __restrict__ primes, const __grid_constant__ LimbMap map, uint32_t N, int stages) {
  pdl_wait_trigger();
  constexpr int G = kGiantPack, NS = 2 * DNUM > G ? 2 * DNUM : G;   // ring slots per stage
  constexpr int TPS = NS / G;                                        // MAC terms per stage
  constexpr uint32_t SB = NS * kSlotBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t span = kTile + a.max_rot;
  double* sb = reinterpret_cast<double*>(smem);                  // baby pairs [slot][2][kTile]
  double* sd = sb + (size_t)m.n_slots * 2 * kTile;               // digits + c0 [DNUM + 1][span]
  unsigned char* ring = reinterpret_cast<unsigned char*>(sd + (size_t)(DNUM + 1) * ((span + 15) / 16 * 16));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)stages * SB);
  uint64_t* empty = full + stages;
  int* smask = reinterpret_cast<int*>(empty + stages);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTile / 32);
    }
  }
  __syncthreads();
  const uint32_t n = N / 2, tiles = N / kTile, total = tiles * map.n;
  if (tid >= kTile) {
    // ---------------- producer warps: item j goes to warp j % kFbProducers ----------------
    const int pw = (tid - kTile) >> 5;
    if ((tid & 31) != 0) return;
    uint32_t j = 0;
    auto issue = [&](uint32_t jj, const uint64_t* const* src, int cnt, size_t off) {
      const int stage = (int)(jj % (uint32_t)stages);
      const uint32_t phase = (jj / (uint32_t)stages) & 1u;
      int mask = 0;
      for (int k = 0; k < cnt; k++)
        if (src[k]) mask |= 1 << k;
      mbar_wait(&empty[stage], phase ^ 1);
      smask[stage] = mask;
      mbar_arrive_expect_tx(&full[stage], (uint32_t)__popc(mask) * kSlotBytes);
      unsigned char* st = ring + (size_t)stage * SB;
      for (int k = 0; k < cnt; k++)
        if (src[k]) bulk_g2s(st + k * kSlotBytes, src[k] + off, kSlotBytes, &full[stage]);
    };
    for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
      const int l = (int)(w / tiles);
      const uint32_t p0 = (w % tiles) * kTile;
      const uint32_t chain = map.pr[l];
      for (int b = 0; b < a.n; b++, j++) {   // key tiles of baby b: (a_k, b_k) for every digit k
        if (j % kFbProducers != (uint32_t)pw) continue;
        const uint64_t* src[NS] = {};
        for (int k = 0; k < DNUM; k++) {
          src[2 * k] = a.key[b] + (size_t)k * a.key_digit_stride;
          src[2 * k + 1] = a.key[b] + (size_t)k * a.key_digit_stride + a.key_half_stride;
        }
        issue(j, src, 2 * DNUM, (size_t)chain * N + p0);
      }
      for (int gi = 0; gi < m.n_groups; gi++) {
        const int4 gr = m.groups[gi];
        for (int t = 0; t < gr.y; t += TPS, j++) {   // plaintext tiles of terms t .. t + TPS - 1
          if (j % kFbProducers != (uint32_t)pw) continue;
          const uint64_t* src[NS] = {};
          for (int r = 0; r < TPS && t + r < gr.y; r++) {
            const FusedTerm ft = m.terms[gr.x + t + r];
            for (int g = 0; g < G; g++) src[r * G + g] = ft.u[g];
          }
          issue(j, src, NS, (size_t)l * N + p0);
        }
      }
    }
    return;
  }
  // ---------------- consumers: one position each ----------------
  int stage = 0;
  uint32_t phase = 0;
  auto next = [&]() {
    if (++stage == stages) {
      stage = 0;
      phase ^= 1;
    }
  };
  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int l = (int)(w / tiles);
    const uint32_t p0 = (w % tiles) * kTile, half = p0 >= n ? n : 0, p = p0 + tid;
    const PrimeDev& P = primes[map.pr[l]];
    const double q = P.qd, qi = P.qinv;
    const bool has_c0 = l <= (int)a.level;
    const int kown = (a.own && has_c0) ? l / a.alpha : -1;
    const uint32_t sstride = (span + 15) / 16 * 16;
    cons_sync();   // every consumer is done with the previous item's digit tile
    for (uint32_t e = tid; e < span; e += kTile) {
      uint32_t jj = p0 - half + e;
      jj = jj >= n ? jj - n : jj;
      const size_t src = (size_t)l * N + half + jj;
#pragma unroll
      for (int k = 0; k < DNUM; k++)
        sd[k * sstride + e] = fm::u2d(k == kown ? a.own[src] : a.digits[(size_t)k * a.digit_stride + src]);
      sd[DNUM * sstride + e] = has_c0 ? fm::u2d(a.c0[src]) : 0.0;
    }
    const double pm = has_c0 ? fm::u2c(a.p_mod[l], q) : 0.0;
    if (m.j0 >= 0) {   // rotation-0 pair (P c0, P c1) over Q_l, 0 over P (D20 L2, j = 0)
      double v0 = 0.0, v1 = 0.0;
      if (has_c0) {
        fm::FAcc x0, x1;
        fm::fmac(x0, fm::u2d(a.c0[(size_t)l * N + p]), pm);
        fm::fmac(x1, fm::u2d(m.c1[(size_t)l * N + p]), pm);
        v0 = fm::fred(x0, q, qi);
        v1 = fm::fred(x1, q, qi);
      }
      sb[(m.j0 * 2) * kTile + tid] = v0;
      sb[(m.j0 * 2 + 1) * kTile + tid] = v1;
    }
    cons_sync();   // the digit tile (with its halo) is complete
    for (int b = 0; b < a.n; b++) {
      mbar_wait(&full[stage], phase);
      const double* st = reinterpret_cast<const double*>(ring + (size_t)stage * SB);
      double kv0[DNUM], kv1[DNUM];
#pragma unroll
      for (int k = 0; k < DNUM; k++) {
        kv0[k] = st[(2 * k) * kTile + tid];
        kv1[k] = st[(2 * k + 1) * kTile + tid];
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[stage]);
      next();
      const uint32_t e = tid + a.rot[b];
      fm::FAcc acc0, acc1;
#pragma unroll
      for (int k = 0; k < DNUM; k++) {
        const double dv = sd[k * sstride + e];
        fm::fmac(acc0, dv, kv0[k]);
        fm::fmac(acc1, dv, kv1[k]);
      }
      if (has_c0) fm::fmac(acc0, sd[DNUM * sstride + e], pm);
      const int sl = m.slot0 + b;
      sb[(sl * 2) * kTile + tid] = fm::fred(acc0, q, qi);
      sb[(sl * 2 + 1) * kTile + tid] = fm::fred(acc1, q, qi);
    }
    // inner sums: a thread reads only its own position's baby pairs (no barrier needed)
    const size_t o = (size_t)l * N + p;
    for (int gi = 0; gi < m.n_groups; gi++) {
      const int4 gr = m.groups[gi];
      fm::FAcc acc0[G], acc1[G];
      int cnt = 0;
      for (int t = 0; t < gr.y; t += TPS) {
        int sl[TPS];
#pragma unroll
        for (int r = 0; r < TPS; r++) sl[r] = t + r < gr.y ? m.terms[gr.x + t + r].slot : -1;
        mbar_wait(&full[stage], phase);
        const int mask = smask[stage];
        const double* st = reinterpret_cast<const double*>(ring + (size_t)stage * SB);
        double u[TPS][G];
#pragma unroll
        for (int r = 0; r < TPS; r++)
#pragma unroll
          for (int g = 0; g < G; g++) u[r][g] = (mask >> (r * G + g)) & 1 ? st[(r * G + g) * kTile + tid] : 0.0;
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[stage]);
        next();
#pragma unroll
        for (int r = 0; r < TPS; r++) {
          if (sl[r] < 0) continue;
          const double xa = sb[(sl[r] * 2) * kTile + tid], xb = sb[(sl[r] * 2 + 1) * kTile + tid];
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
            fm::fmac(acc0[g], u[r][g], xa);
            fm::fmac(acc1[g], u[r][g], xb);
          }
        }
      }
#pragma unroll
      for (int g = 0; g < G; g++) {
        if (g < gr.w) {
          uint64_t* dst = m.out + (size_t)(gr.z + g) * m.out_stride;
          dst[o] = fm::c2u(fm::fred(acc0[g], q, qi), P.rc.q);
          dst[m.half + o] = fm::c2u(fm::fred(acc1[g], q, qi), P.rc.q);
        }
      }
    }
  }
}

bool launch_baby_mac_bulk(const DevCtx& c, const KipMulti& a, const BabyMacArgs& m, const LimbMap& map) {
  if (c.N % kTile || a.nq != 1) return false;
  const int NS = std::max(2 * a.dnum, kGiantPack);
  const size_t SB = (size_t)NS * kSlotBytes;
  const size_t span = (kTile + a.max_rot + 15) / 16 * 16;
  const size_t fixed = (size_t)m.n_slots * 2 * kTile * 8 + (size_t)(a.dnum + 1) * span * 8;
  const size_t budget = 225 * 1024;
  if (fixed + 2 * (SB + 20) > budget) return false;
  static const int stages_env = getenv("HELRM_FBM_STAGES") ? atoi(getenv("HELRM_FBM_STAGES")) : 0;
  int stages = (int)((budget - fixed) / (SB + 20));
  if (stages_env > 0) stages = std::min(stages, stages_env);
  stages = std::max(kFbProducers, stages / kFbProducers * kFbProducers);
  if (fixed + (size_t)stages * (SB + 20) > budget) return false;
  const size_t smem = fixed + (size_t)stages * (SB + 20);
  decltype(&k_baby_mac_bulk<1>) kern = nullptr;
  switch (a.dnum) {
    case 1: kern = k_baby_mac_bulk<1>; break;
    case 2: kern = k_baby_mac_bulk<2>; break;
    case 3: kern = k_baby_mac_bulk<3>; break;
    case 4: kern = k_baby_mac_bulk<4>; break;
    case 5: kern = k_baby_mac_bulk<5>; break;
    case 6: kern = k_baby_mac_bulk<6>; break;
    case 7: kern = k_baby_mac_bulk<7>; break;
    default: return false;
  }
  ProfScope ps_(c, "baby_mac", m.bytes);
  HCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned total = (c.N / kTile) * map.n;
  launch_pdl(kern, dim3(std::min<unsigned>(total, 148u)), dim3(kTile + 32 * kFbProducers), smem, c.stream, a, m,
             c.primes, map, c.N, stages);
  (*c.launches)++;
  HCUDA(cudaGetLastError());
  return true;
}

}  // namespace helrm
