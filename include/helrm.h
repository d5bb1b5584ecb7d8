/*
 * helrm.h -- C ABI of the B200-native HE-LRM encrypted embedding lookup.
 *
 * The library computes the server-side hot path of HE-LRM (arxiv 2506.18150):
 * a plaintext, block-diagonally packed, digit-decomposed embedding table times
 * an RNS-CKKS ciphertext holding the client's concatenated one-hot vectors,
 * by hybrid diagonals and double-hoisted baby-step/giant-step rotations.
 *
 *   PAPER.md:248      lookup = OHE(i) . E as a linear transform under FHE
 *   PAPER.md:316-319  client-side base-p digit decomposition, l = ceil(log_p k)
 *   PAPER.md:339-342  block-diagonal multi-table packing, contiguous outputs
 *   PAPER.md:168      BSGS diagonal matrix-vector product (pre-rotated diagonals)
 *   PAPER.md:289,584  double hoisting
 *   PAPER.md:121-151  CKKS ring, encoding, encryption, rotation, key switching
 *
 * The ring-level conventions the paper leaves open are fixed by the readings
 * D1-D23 of SURVEY.md section 8(c) (listed in DESIGN.md); ciphertexts produced
 * here are bit-identical to the independent CPU oracle (oracle/) under them.
 *
 * Conventions for every call:
 *  - Return value: HELRM_OK (0) or an error code below; on error every
 *    `out` handle is set to NULL and helrm_last_error() (thread-local) holds a
 *    one-line message.  No C++ exception crosses this boundary.
 *  - Handles are opaque; each has a destroy function; destroy(NULL) is a no-op.
 *  - Host buffers are caller-owned and only read/written during the call.
 *  - "dev" pointers are device pointers on the context's device (for example
 *    a borrowed torch.uint64 tensor); the library never frees them.
 *  - All GPU work of a context is enqueued on the context's CUDA stream; calls
 *    that return host data synchronise that stream first.
 *  - Residues are uint64 in [0, q).  Polynomials are limb-major [limb][N].
 *    A ciphertext at level l is [2][l+1][N]; in the library's device memory it
 *    is in NTT form, "slot order" (position s < N/2 <-> psi^(5^s), position
 *    N/2 + s <-> psi^(-5^s)); the canonical exchange format of *_export /
 *    *_import is coefficient form.
 */
#ifndef HELRM_H
#define HELRM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (2/3/4 = SPEC.md:648 exit codes) ---------------------- */
typedef int helrm_status;
#define HELRM_OK 0
#define HELRM_ERR_CONFIG 2   /* bad params, missing primes, |encoded coeff| >= 2^62 */
#define HELRM_ERR_LEVEL 3    /* level 0 lookup / rescale, level mismatch */
#define HELRM_ERR_CAPACITY 4 /* more slots than n, sizes beyond limits */
#define HELRM_ERR_RANGE 5    /* index outside [0, k) */
#define HELRM_ERR_LAYOUT 6   /* table/offset/ct-count mismatch */
#define HELRM_ERR_CUDA 7
#define HELRM_ERR_NCCL 8
#define HELRM_ERR_ALLOC 9
#define HELRM_ERR_ARG 10     /* NULL pointer or buffer too small */

#define HELRM_MODE_DOUBLE 0  /* double-hoisted BSGS (the paper's) */
#define HELRM_MODE_SINGLE 1  /* single-hoisted cross-check mode */
/* Flag OR-ed into the plan mode (double-hoisted only): keep the encoded
 * diagonals as int64 coefficients (N words each instead of l+1+K limbs) and
 * expand them (reduce, NTT, D-form) during every lookup, in bounded chunks;
 * input ciphertexts are processed in groups.  For layouts whose QP-NTT
 * diagonals exceed HBM (LLM layout L1: 36,348 diagonals = 426 GiB; the
 * 100-input-ct Criteo model: 700 GiB).  Same bits as the stored form.
 * Lookups on compact plans run query by query, without graph replay. */
#define HELRM_PLAN_COMPACT 2

typedef struct helrm_params helrm_params;
typedef struct helrm_ctx helrm_ctx;
typedef struct helrm_sk helrm_sk;
typedef struct helrm_pk helrm_pk;
typedef struct helrm_rotkeys helrm_rotkeys;
typedef struct helrm_tables helrm_tables;
typedef struct helrm_ct helrm_ct;
typedef struct helrm_plan helrm_plan;

/* ---- parameters (D1-D3) ------------------------------- */
typedef struct {
  uint32_t log_n;          /* ring degree N = 2^log_n, 12 <= log_n <= 16 */
  uint32_t n_q_groups;     /* ciphertext prime groups, in order q_0, q_1, ... */
  uint32_t q_bits[8], q_count[8];
  uint32_t n_p_groups;     /* special prime groups (alpha = K = total count) */
  uint32_t p_bits[4], p_count[4];
  uint32_t log_scale;      /* Delta = 2^log_scale */
} helrm_params_desc;

typedef struct {
  uint32_t N, n_slots, L, K, dnum_top, log_scale;
} helrm_params_info_t;

/* Primes by D2 (largest primes < 2^bits, = 1 mod 2N, group by group), psi by
 * D3 (smallest primitive 2N-th root).  CONFIG if the request cannot be met. */
helrm_status helrm_params_create(const helrm_params_desc* d, helrm_params** out);
void helrm_params_destroy(helrm_params* p);
helrm_status helrm_params_info(const helrm_params* p, helrm_params_info_t* out);
/* q: L+1 words, p: K words, psi: L+1+K words (q's then p's); any may be NULL */
helrm_status helrm_params_moduli(const helrm_params* p, uint64_t* q, uint64_t* pp, uint64_t* psi);

/* ---- context: device tables + stream ------------------------------------ */
/* Builds the device twiddle / conversion tables of every prime on `device`;
 * all later GPU work is enqueued on `cuda_stream` (0 = legacy default). */
helrm_status helrm_ctx_create(const helrm_params* p, int device, uintptr_t cuda_stream, helrm_ctx** out);
/* Frees the context's device memory pool: every handle created on the
 * context (keys, ciphertexts, plans) must be destroyed before it. */
void helrm_ctx_destroy(helrm_ctx* c);
helrm_status helrm_ctx_sync(helrm_ctx* c);
/* Number of library kernels launched on this context since creation. */
uint64_t helrm_ctx_launches(const helrm_ctx* c);
/* Per-kernel timing: when enabled, every library launch is bracketed by CUDA
 * events on the context stream; enabling/disabling clears the records.
 * helrm_ctx_profile_json returns {"kernel": {"count": n, "ms": total}, ...}
 * for the records so far (synchronises; string owned by the context). */
helrm_status helrm_ctx_profile(helrm_ctx* c, int enable);
const char* helrm_ctx_profile_json(helrm_ctx* c);

/* ---- client keys (D9-D11) --------------------- */
/* Deterministic in the seed (counter-based SplitMix64 streams, D9).  Key
 * material is generated by device kernels of this library. */
helrm_status helrm_sk_gen(helrm_ctx* c, uint64_t seed, helrm_sk** out);
helrm_status helrm_pk_gen(helrm_ctx* c, const helrm_sk* sk, uint64_t seed, helrm_pk** out);
/* one key per Galois element g (odd, < 2N), each dnum(L) x 2 x (L+1+K) x N */
helrm_status helrm_rotkeys_gen(helrm_ctx* c, const helrm_sk* sk, const uint64_t* galois, size_t n,
                               uint64_t seed, helrm_rotkeys** out);
void helrm_sk_destroy(helrm_sk* s);
void helrm_pk_destroy(helrm_pk* p);
void helrm_rotkeys_destroy(helrm_rotkeys* r);
/* coefficient-form exports: sk -> int64[N] ternary; pk -> [2][L+1][N]
 * (b, a); rotation key g -> [dnum][2][L+1+K][N] (b_k, a_k). */
helrm_status helrm_sk_export(helrm_ctx* c, const helrm_sk* s, int64_t* coeff, size_t n_words);
helrm_status helrm_pk_export(helrm_ctx* c, const helrm_pk* p, uint64_t* coeff, size_t n_words);
helrm_status helrm_rotkeys_export(helrm_ctx* c, const helrm_rotkeys* r, uint64_t g, uint64_t* coeff, size_t n_words);
size_t helrm_rotkeys_bytes(const helrm_rotkeys* r);
/* Galois elements held by a key set, ascending (n = count; up to cap written) */
helrm_status helrm_rotkeys_galois(const helrm_rotkeys* r, uint64_t* g, size_t cap, size_t* n);

/* Key import: client keys generated elsewhere (keys are client material,
 * PAPER.md:142 "with a given public key", :163 "a unique key is needed for
 * each rotation offset"), in the canonical coefficient form of the exports
 * above.  The words are copied to the context's device and converted to the
 * library's internal form (NTT slot order; rotation keys in D-form).
 * Ownership: the caller keeps its buffers; the handles are the library's.
 * Errors: ARG on a NULL pointer or a short buffer; RANGE if a word is not a
 * residue in [0, q) of its limb (sk: |coefficient| > 2^40); CONFIG if g is
 * not a power of 5 mod 2N (D8).
 *   sk:   int64[N] secret coefficients (D11: ternary)
 *   pk:   uint64 [2][L+1][N] (b, a)
 *   rotation keys: key i for Galois element galois[i] at coeff[i],
 *         uint64 [dnum(L)][2][L+1+K][N] (b_k, a_k) per digit k (D11);
 *         words_per_key >= dnum(L) 2 (L+1+K) N.  A repeated g keeps the last. */
helrm_status helrm_sk_import(helrm_ctx* c, const int64_t* coeff, size_t n_words, helrm_sk** out);
helrm_status helrm_pk_import(helrm_ctx* c, const uint64_t* coeff, size_t n_words, helrm_pk** out);
helrm_status helrm_rotkeys_import(helrm_ctx* c, const uint64_t* galois, size_t n, const uint64_t* const* coeff,
                                  size_t words_per_key, helrm_rotkeys** out);
/* Upload one more key (same form as one key of helrm_rotkeys_import) into
 * an existing key set, e.g. streamed from the client one rotation at a time;
 * replaces a key already held for g. */
helrm_status helrm_rotkeys_upload(helrm_ctx* c, helrm_rotkeys* rk, uint64_t g, const uint64_t* coeff, size_t n_words);

/* ---- tables and client query (S0) --------- */
typedef struct {
  int64_t k;          /* rows of the (virtual) original table, >= 1 */
  int64_t d;          /* embedding dimension, >= 1 */
  int64_t p;          /* digit base; 0 = never compress; compress iff k > p */
  const double* w;    /* (uncompressed ? k : p * l) x d, row-major (l below);
                         rows [t p, (t+1) p) are sub-table t (LSD-first digits) */
  int64_t in_off;     /* input slot offset, -1 = contiguous default (D19) */
  int64_t out_off;    /* output slot offset, -1 = contiguous default */
  int64_t l;          /* digit count: 0 = ceil(log_p k); > 0 (p >= 2): exactly l digits,
                         LAYOUT unless p^l >= k -- shapes whose p^l exceeds the int64 row
                         range, e.g. PAPER.md:361's p = 16, l = 32 (the weights then have
                         p l rows and the high digits of every index are 0) */
} helrm_table_desc;

/* Copies the weights in (blocks sharing one `w` pointer are deduplicated);
 * block order = array order.  LAYOUT on overlapping offsets. */
helrm_status helrm_tables_create(const helrm_params* p, const helrm_table_desc* t, size_t n_tables,
                                 uint32_t n_dense, helrm_tables** out);
void helrm_tables_destroy(helrm_tables* t);
/* K = input slots used, M = output slots used */
helrm_status helrm_tables_info(const helrm_tables* t, int64_t* K, int64_t* M);
/* slots[0..n_slots) := [dense || one-hot segments]; n_slots >= K.
 * RANGE if an index is outside [0, k_b). */
helrm_status helrm_encode_query(const helrm_tables* t, const int64_t* idx, const double* dense,
                                double* slots, size_t n_slots);

/* ---- ciphertexts (D6, D12, D13) ----------------------------------------- */
/* Encode (correctly rounded, >= 100-bit intermediates) at Delta and
 * public-key encrypt at `level`; n_slots <= N/2 (CAPACITY), level <= L (LEVEL). */
helrm_status helrm_encrypt(helrm_ctx* c, const helrm_pk* pk, const double* slots, size_t n_slots,
                           uint32_t level, uint64_t seed, helrm_ct** out);
/* coefficient form [2][level+1][N] <-> device NTT form */
helrm_status helrm_ct_import(helrm_ctx* c, const uint64_t* coeff, uint32_t level, double scale, helrm_ct** out);
helrm_status helrm_ct_export(helrm_ctx* c, const helrm_ct* ct, uint64_t* coeff, size_t n_words);
helrm_status helrm_ct_info(const helrm_ct* ct, uint32_t* level, double* scale);
/* device pointer of the NTT-form (slot order) data, [2][level+1][N] */
helrm_status helrm_ct_device_ptr(const helrm_ct* ct, uint64_t** dev);
void helrm_ct_destroy(helrm_ct* ct);
/* m' = c0 + c1 s (device), centered CRT + decode (host, fp64) */
helrm_status helrm_decrypt_decode(helrm_ctx* c, const helrm_sk* sk, const helrm_ct* ct, double* slots,
                                  size_t n_slots);

/* ---- server setup: the lookup plan (D19) ------- */
typedef struct {
  int64_t K, M, mbar, n_in_cts, n_out_cts, n_diag, n_unique, n1, n2_max, n_rotations;
  uint32_t level, mode;
  uint64_t diag_bytes;    /* device bytes of the encoded diagonals */
} helrm_plan_info_t;

/* Packs W, extracts the hybrid diagonals, splits them BSGS (n1 = 0: smallest
 * power of two with n1^2 >= span), pre-rotates, encodes at Delta_pt = q_level
 * over Q_level P (double) or Q_level (single) and uploads them (device memory
 * owned by the plan; mode | HELRM_PLAN_COMPACT: the int64 coefficients only).
 * LEVEL if level < 1 or > L; ARG for a compact single-hoisted plan. */
helrm_status helrm_plan_create(helrm_ctx* c, const helrm_tables* t, uint32_t level, uint32_t n1, uint32_t mode,
                               helrm_plan** out);
void helrm_plan_destroy(helrm_plan* p);
helrm_status helrm_plan_info(const helrm_plan* p, helrm_plan_info_t* out);
/* rotation amounts needing a key (babies, giants, RotSum), ascending;
 * the Galois element of amount a is 5^a mod 2N */
helrm_status helrm_plan_rotations(const helrm_plan* p, int64_t* amounts, size_t cap, size_t* n);
/* the plan's D19 Galois list {5^a mod 2N : a in helrm_plan_rotations},
 * ascending: the keys the client must generate (n = count, <= cap written) */
helrm_status helrm_plan_galois(const helrm_plan* p, uint64_t* g, size_t cap, size_t* n);

/* ---- the hot path (D20-D22) --------------------------------------------- */
/* in: batch x C ciphertexts (query-major), all at the plan's level; out:
 * batch x O new ciphertexts at level-1, scale Delta, slot s = y[s mod mbar].
 * Asynchronous on the context stream; inputs are not modified.
 * LAYOUT if a key is missing, LEVEL on a level mismatch. */
helrm_status helrm_lookup(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk, const helrm_ct* const* in,
                          size_t batch, helrm_ct** out);

/* Serving form of the lookup on host buffers (coefficient form, the
 * helrm_ct_import / helrm_ct_export exchange format; pinned memory makes the
 * copies asynchronous): in[q C + c] is input ct c of query q,
 * [2][level+1][N] words at the plan's level with scale `scale`; out[q O + o]
 * receives output ct o of query q, [2][level][N] words.  The queries run
 * one after another through the same computation as helrm_lookup (batch 1,
 * double-hoisted mode), pipelined so that the host->device copy of query
 * q+1 and the device->host copy of query q-1 overlap the lookup of query q.
 * Returns after every output has been written.  LAYOUT if a key is missing,
 * ARG for the single-hoisted mode. */
helrm_status helrm_lookup_host(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                               const uint64_t* const* in, double scale, size_t batch, uint64_t* const* out);

/* ---- primitives (parity tests and kernel microbenchmarks) --------------- */
/* In-place negacyclic NTT (coefficient -> slot-order NTT form) / inverse on
 * n_polys x n_limbs limbs of N words at `dev`; limb i of a polynomial uses
 * prime first_prime + i of the chain q_0..q_L, p_0..p_{K-1}. */
helrm_status helrm_ntt_fwd(helrm_ctx* c, uint64_t* dev, uint32_t first_prime, uint32_t n_limbs, size_t n_polys);
helrm_status helrm_ntt_inv(helrm_ctx* c, uint64_t* dev, uint32_t first_prime, uint32_t n_limbs, size_t n_polys);
/* D15: dev_in [level+1][N] NTT form -> dev_out [level+1+K][N] NTT form */
helrm_status helrm_modup(helrm_ctx* c, const uint64_t* dev_in, uint32_t level, uint32_t digit, uint64_t* dev_out);
/* D16: dev_in [level+1+K][N] -> dev_out [level+1][N] (NTT form) */
helrm_status helrm_moddown(helrm_ctx* c, const uint64_t* dev_in, uint32_t level, uint64_t* dev_out);
/* D17 */
helrm_status helrm_rescale(helrm_ctx* c, const helrm_ct* in, helrm_ct** out);
/* D18 Rotate(ct, k): left rotation by k slots */
helrm_status helrm_rotate(helrm_ctx* c, const helrm_rotkeys* rk, const helrm_ct* in, int64_t k, helrm_ct** out);
/* Hoisted rotations of one ct: ModUp once, then for each amount
 * Rotate(ct, a) written to out_ring[i % ring] (caller-created cts at the
 * input's level, e.g. by helrm_ct_import or helrm_ct_alloc). */
helrm_status helrm_rotate_hoisted(helrm_ctx* c, const helrm_rotkeys* rk, const helrm_ct* in, const int64_t* amounts,
                                  size_t n_amounts, helrm_ct* const* out_ring, size_t ring);
/* Hoisted rotations of n cts with the keys amortised over them (SURVEY.md
 * 8(d) microbench unit): every ct's ModUp once; per amount one key switch
 * over all n cts (each key value loaded once) and one batched ModDown.
 * Rotate(in[j], amounts[i]) is written to the device buffer `out` (borrowed,
 * NTT slot order, [ring][2][level+1][N]) at slot (i n + j) % ring; ring must
 * be a multiple of n (ARG); all cts at one level (LEVEL).  Bit-identical to
 * helrm_rotate. */
helrm_status helrm_rotate_hoisted_batch(helrm_ctx* c, const helrm_rotkeys* rk, const helrm_ct* const* in, size_t n,
                                        const int64_t* amounts, size_t n_amounts, uint64_t* out, size_t ring);
helrm_status helrm_ct_alloc(helrm_ctx* c, uint32_t level, double scale, helrm_ct** out);
/* Microbench input: limbs of cts drawn UniformMod from D9 streams
 * (purpose 9, a = ct, b = poly, c = limb), written in NTT form. */
helrm_status helrm_ct_random(helrm_ctx* c, uint64_t seed, uint32_t ct_index, uint32_t level, helrm_ct** out);

/* ---- multi-GPU: one process per GPU ----------------- */
/* Contiguous split of n_items over world ranks: [lo, hi) for `rank`. */
helrm_status helrm_dist_range(int64_t n_items, int world, int rank, int64_t* lo, int64_t* hi);
/* NCCL unique id (128 bytes) to broadcast through torch.distributed. */
helrm_status helrm_comm_unique_id(uint8_t* id);
/* Create the context's communicator (NCCL is loaded at run time). */
helrm_status helrm_comm_init(helrm_ctx* c, const uint8_t* id, int rank, int world);
/* helrm_lookup with the giant steps split over the ranks: rank 0's inputs are
 * broadcast into each rank's staging buffer (every rank passes cts at the
 * plan's level, e.g. from helrm_ct_alloc; none is modified), each rank
 * computes the partial Q_l P accumulators of its giant range,
 * ncclAllReduce(uint64, sum) + a mod-q kernel combine them, and every rank
 * finishes (ModDown, rescale, RotSum).  Bit-identical to helrm_lookup for
 * every world size (only exact modular sums are split, D23). */
helrm_status helrm_lookup_dist(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk, const helrm_ct* const* in,
                               size_t batch, helrm_ct** out);
/* The same partition emulated in one process (parity harness of the
 * multi-GPU combine on one GPU): the `parts` giant ranges run one after
 * another, their partial accumulators are summed as plain uint64 words (the
 * all-reduce's arithmetic) and reduced by the same mod-q kernel, then L6-L8.
 * 1 <= parts < 8192 (ARG otherwise).  Bit-identical to helrm_lookup. */
helrm_status helrm_lookup_dist_virtual(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                       const helrm_ct* const* in, size_t batch, int parts, helrm_ct** out);
/* The RNS-limb partition of the batch-1 lookup
 * emulated in one process: rank r of `parts` owns rows [lo_r, hi_r) of the
 * l+1+K limbs (helrm_dist_range) and computes only those rows of the baby key
 * switches, inner sums and giant key switches (1/parts of the rotation keys
 * and plaintext diagonals streamed per rank); ModUp / ModDown / rescale /
 * RotSum are replicated; each giant's B rows and the output accumulators are
 * all-gathered (explicit copies of the ranks' private slices).  Rank r owns
 * rows [r rp, (r+1) rp), rp = ceil((l+1+K) / parts) (trailing ranks may own
 * none).  Stored-diagonal double-hoisted plans; 1 <= parts <= l+1+K.
 * Bit-identical to helrm_lookup. */
helrm_status helrm_lookup_limbsplit_virtual(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                            const helrm_ct* const* in, size_t batch, int parts, helrm_ct** out);
/* The same partition over the context's communicator (helrm_comm_init), one
 * process per GPU: this rank computes its rows only; rank 0's inputs are
 * broadcast, each giant's B rows and the accumulators are exchanged with
 * ncclAllGather (slices padded to ceil((l+1+K) / world) rows). */
helrm_status helrm_lookup_limbsplit(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                   const helrm_ct* const* in, size_t batch, helrm_ct** out);
/* Timing harness of the partition (no multi-GPU node needed): enqueues
 * exactly the kernels rank `rank` of `parts` runs for one query, with every
 * exchange skipped -- the outputs are NOT a lookup result.  bench.py times it
 * per rank to project the partitioned lookup's device time. */
helrm_status helrm_limbsplit_rank_work(helrm_ctx* c, const helrm_plan* p, const helrm_rotkeys* rk,
                                       const helrm_ct* const* in, int parts, int rank, helrm_ct** out);
/* The combine's reduction alone (D23 L5), in place: n_polys R_{Q_level P}
 * polynomials [n_polys][level+1+K][N] at `dev` whose words are sums of
 * residues (< 2^64) become residues mod their limb's prime. */
helrm_status helrm_modred(helrm_ctx* c, uint64_t* dev, uint32_t level, size_t n_polys);

const char* helrm_last_error(void);
const char* helrm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HELRM_H */
