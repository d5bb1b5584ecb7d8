"""Seeded synthetic workloads for the five BASELINE.json configs.

Shapes and distributions (BASELINE.json `configs`):

  tiny_a / tiny_b  N=2^12, q = 40/30/30-bit + one 40-bit special prime,
                   Delta = 2^30, lookup level 2.  tiny_a: one 256x16 table,
                   U[-1,1], never compressed.  tiny_b: the same index, base 16,
                   two 16x16 sub-tables U[-1,1].  Index ~ U{0..255}.
  uci              N=2^14, 8x40-bit q + 2x40-bit p, Delta = 2^36, level 7.
                   Vocab [2,2,3,4,4,5,8,16], d=16, entries N(0, 0.1^2),
                   base 4; 13 dense features U[0,1].
  criteo           N=2^16, 24x50-bit q + 4x50-bit p (dnum 6), Delta = 2^40,
                   level 23.  26 tables, CRITEO_VOCAB below, d=16, entries
                   N(0, 0.05^2), base 64; indices Zipf(1.1) per table.
  llm              N=2^16, 20x50-bit q + 4x50-bit p (dnum 5), Delta = 2^40,
                   level 19.  One 50257x768 table compressed base 256 into
                   2 sub-tables 256x768, entries N(0, 0.02^2); 128 token ids
                   U[0, 50257); layout L2 (token stride 1024 in and out).
  llm_small        the same layout on the Tiny ring (N=2^12): 64 tokens of a
                   1000x48 table, base 32, stride 128 (4 in / 4 out cts).
  microbench       N=2^16, Criteo's primes; 1024 ciphertexts of uniform limbs
                   (drawn by the D9 PRNG, purpose 9 -- see microbench_seed).

Draw order from numpy.random.default_rng(seed): table weights in block order,
then indices (query-major, block order within a query), then dense features.
No arithmetic of the method lives here (no digit decomposition, packing,
encoding or modular arithmetic).  `subtable_rows` is the one shape rule the
generator needs to know how many rows to draw; both the oracle and the
library re-derive and check it independently.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np

# Criteo-shaped vocabulary: the first seed s >= 0 for
# which round(exp(default_rng(s).uniform(ln 3, ln 1e7, 26))) sums into
# [3.25e7, 3.35e7] with max <= 1e7 is s = 230; stored so that a NumPy stream
# change cannot alter it (tests/test_synth.py re-derives it).
CRITEO_VOCAB = [3, 6970, 2744503, 9007069, 1240, 3227764, 8408764, 2256022, 431, 2246483,
                415, 9, 213122, 1215, 66731, 214456, 425, 55, 240, 3613143, 4875, 17,
                495595, 10, 822, 1375]
CRITEO_VOCAB_SEED = 230

CONFIG_NAMES = ("tiny_a", "tiny_b", "uci", "criteo", "criteo_b64", "criteo_c2", "criteo_c2_small", "llm",
                "llm_small", "llm_gen", "llm_gen_small", "tiny_dnum7", "criteo_c17", "criteo_c9_small", "criteo_l4", "mlp_small",
                "llm_l1", "llm_l1_small", "criteo_c100", "table1", "table1_small",
                "mlp_512x256", "microbench")


def subtable_rows(k: int, p: int) -> int:
    """Number of weight rows drawn for a table of k rows at base p.

    k rows if the table stays uncompressed (p == 0 or k <= p), else p * l with
    l the smallest integer such that p**l >= k (section 5.1).
    """
    if p == 0 or k <= p:
        return k
    l, cap = 1, p
    while cap < k:
        cap *= p
        l += 1
    return p * l


@dataclasses.dataclass
class Table:
    k: int                      # rows of the (virtual) original table
    d: int                      # embedding dimension
    p: int                      # digit base, 0 = never compress
    weights: np.ndarray         # (subtable_rows(k, p), d) float64, row-major
    in_off: int = -1            # explicit input slot offset, -1 = contiguous default
    out_off: int = -1           # explicit output slot offset, -1 = contiguous default
    weight_id: int = -1         # blocks sharing one weight array carry the same id
    l: int = 0                  # explicit digit count (p^l >= k), 0 = ceil(log_p k)


@dataclasses.dataclass
class Config:
    name: str
    log_n: int
    q_groups: List[Tuple[int, int]]   # (bits, count) ciphertext groups, in order
    p_groups: List[Tuple[int, int]]   # (bits, count) special group(s)
    log_scale: int
    level: int
    seed: int
    batch: int = 1

    @property
    def N(self) -> int:
        return 1 << self.log_n

    @property
    def n_slots(self) -> int:
        return 1 << (self.log_n - 1)


@dataclasses.dataclass
class Workload:
    config: Config
    tables: List[Table]
    n_dense: int
    indices: np.ndarray               # (batch, n_blocks) int64
    dense: np.ndarray                 # (batch, n_dense) float64


_CONFIGS = {
    "tiny_a": Config("tiny_a", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    "tiny_b": Config("tiny_b", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    # edge case of the key switch: one special prime (alpha = 1) under 7 ciphertext primes,
    # so dnum = 7 at the lookup level (the largest the library accepts), Tiny-B's table
    "tiny_dnum7": Config("tiny_dnum7", 12, [(40, 1), (30, 6)], [(40, 1)], 30, 6, 1),
    "uci": Config("uci", 14, [(40, 8)], [(40, 2)], 36, 7, 1),
    "criteo": Config("criteo", 16, [(50, 24)], [(50, 4)], 40, 23, 1),
    "criteo_b64": Config("criteo_b64", 16, [(50, 24)], [(50, 4)], 40, 23, 1, batch=64),
    # the lookup where Orion places it in the ReLU DLRM: input level 4, same tables
    "criteo_l4": Config("criteo_l4", 16, [(50, 24)], [(50, 4)], 40, 4, 1),
    # a less compressed Criteo model (PAPER.md:459-463, Table 2 threshold 5e4; :470): tables
    # with vocab <= 5e4 stay one-hot, the rest are digit-decomposed in base 1024 ->
    # 47,798 input slots = 2 input cts and 1024 diagonals (the paper: 47,759 slots,
    # "1024 non-zero diagonals ... two ciphertexts")
    "criteo_c2": Config("criteo_c2", 16, [(50, 24)], [(50, 4)], 40, 23, 1),
    # the same shape scaled to the Tiny ring so the oracle runs it live: vocab sqrt(k),
    # one-hot below 1000 rows, base 32 above -> 2,944 slots = 2 input cts of 2048
    "criteo_c2_small": Config("criteo_c2_small", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    # many input cts on the Tiny ring (every sqrt-vocab table one-hot: 16,529 slots = 9 cts of
    # 2048) so the oracle checks the many-ct paths live
    "criteo_c9_small": Config("criteo_c9_small", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    # the 10^2x model (569,545 slots, 18 input cts): one-hot up to 2.2e5
    # rows, base 1024 above -> 535,963 slots = 17 input cts, 8704 diagonals (119 GiB)
    "criteo_c17": Config("criteo_c17", 16, [(50, 24)], [(50, 4)], 40, 23, 1),
    # the paper's least compressed Criteo model (2,772,109 slots, 85 input
    # cts at n = 2^15): with our seeded vocabularies the nearest threshold keeps every table
    # of <= 2.25e6 rows one-hot (base 1024 above) -> 3,272,921 slots = 100 input cts (85 is
    # not reachable: the next lower threshold gives 33); 51,200 diagonals, kept as int64
    # coefficients (25 GiB instead of 700 GiB in QP-NTT form) and expanded during the lookup.
    # Its many-ct path is checked bit for bit on criteo_c9_small.
    "criteo_c100": Config("criteo_c100", 16, [(50, 24)], [(50, 4)], 40, 23, 1),
    "llm": Config("llm", 16, [(50, 20)], [(50, 4)], 40, 19, 1),
    # the paper-exact LLM layout L1 ("contiguous slot ordering (row-major)",
    # SURVEY.md R23): 128 tokens at input stride 512 (2 digits x 256 one-hot) and output
    # stride 768 -> 2 input / 3 output cts, 36,348 diagonals (426 GiB in QP-NTT form: the
    # plan keeps them as int64 coefficients and expands them during the lookup); and the
    # same layout on the Tiny ring (64 tokens of a 1000 x 48 table, base 32)
    "llm_l1": Config("llm_l1", 16, [(50, 20)], [(50, 4)], 40, 19, 1),
    "llm_l1_small": Config("llm_l1_small", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    # LLM-L2 layout scaled to the Tiny ring so the oracle runs it live: 64 tokens
    # of a 1000 x 48 table (base 32, 2 digits), stride 128 -> 4 in / 4 out cts
    "llm_small": Config("llm_small", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    # LLM generation step: the one sampled token of the 50257 x 768
    # table (base 256, 2 digits) -> a sparse matrix-vector product, 512 one-hot slots in,
    # 768 out; and the same on the Tiny ring (1000 x 48, base 32) for the live oracle
    "llm_gen": Config("llm_gen", 16, [(50, 20)], [(50, 4)], 40, 19, 1),
    "llm_gen_small": Config("llm_gen_small", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    # a dense linear layer on the same BSGS engine (fully connected layers by
    # pre-rotated diagonals and baby/giant steps; the DLRM's bottom/top MLPs, :654): the
    # "table" is the weight matrix W (in x out, one row per input slot), the input a dense
    # encrypted vector x, the output W^T x
    "mlp_small": Config("mlp_small", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    # the paper's Table-1 shape: one GPT-2 table
    # (d = 768) decomposed base p = 16 into l = 32 digits -> p l = 512 one-hot input slots and
    # 768 outputs, one ct each way (the paper: "BSGS 3.17" s on its CPU).  16^32 rows do not
    # fit the boundary's int64 row index, so the table declares k = 2^63 - 1 rows with an
    # explicit digit count l = 32 (Table.l): the server-side matrix (32 sub-tables of
    # 16 x 768) is the paper's, and digits 16..31 of a query are always 0.  LLM ring and
    # level; table1_small: 16^8 rows, base 16 (8 digits), d = 48 on the Tiny ring.
    "table1": Config("table1", 16, [(50, 20)], [(50, 4)], 40, 19, 1),
    "table1_small": Config("table1_small", 12, [(40, 1), (30, 2)], [(40, 1)], 30, 2, 1),
    "mlp_512x256": Config("mlp_512x256", 16, [(50, 24)], [(50, 4)], 40, 23, 1),
    "microbench": Config("microbench", 16, [(50, 24)], [(50, 4)], 40, 23, 1, batch=1024),
}


def config_by_name(name: str) -> Config:
    return dataclasses.replace(_CONFIGS[name])


def _zipf_index(rng: np.random.Generator, k: int, a: float = 1.1) -> int:
    while True:
        r = int(rng.zipf(a))
        if r <= k:
            return r - 1


def make_workload(name: str, batch: Optional[int] = None) -> Workload:
    cfg = config_by_name(name)
    if batch is not None:
        cfg.batch = batch
    rng = np.random.default_rng(cfg.seed)
    B = cfg.batch
    if name in ("tiny_a", "tiny_b", "tiny_dnum7"):
        if name == "tiny_a":
            w = rng.uniform(-1.0, 1.0, size=(256, 16))
            tables = [Table(256, 16, 0, w)]
        else:
            w = rng.uniform(-1.0, 1.0, size=(subtable_rows(256, 16), 16))
            tables = [Table(256, 16, 16, w)]
        idx = rng.integers(0, 256, size=(B, 1))
        return Workload(cfg, tables, 0, idx.astype(np.int64), np.zeros((B, 0)))
    if name == "uci":
        vocab = [2, 2, 3, 4, 4, 5, 8, 16]
        tables = [Table(k, 16, 4, rng.normal(0.0, 0.1, size=(subtable_rows(k, 4), 16))) for k in vocab]
        idx = np.array([[rng.integers(0, k) for k in vocab] for _ in range(B)], dtype=np.int64)
        dense = rng.uniform(0.0, 1.0, size=(B, 13))
        return Workload(cfg, tables, 13, idx, dense)
    if name in ("criteo", "criteo_b64", "criteo_l4"):
        tables = [Table(k, 16, 64, rng.normal(0.0, 0.05, size=(subtable_rows(k, 64), 16))) for k in CRITEO_VOCAB]
        idx = np.array([[_zipf_index(rng, k) for k in CRITEO_VOCAB] for _ in range(B)], dtype=np.int64)
        return Workload(cfg, tables, 0, idx, np.zeros((B, 0)))
    if name in ("criteo_c2", "criteo_c2_small", "criteo_c17", "criteo_c9_small", "criteo_c100"):
        small = name in ("criteo_c2_small", "criteo_c9_small")
        vocab = [max(2, int(round(k ** 0.5))) for k in CRITEO_VOCAB] if small else CRITEO_VOCAB
        thr, base = {"criteo_c2_small": (1000, 32), "criteo_c9_small": (3001, 32), "criteo_c17": (220000, 1024),
                     "criteo_c2": (50000, 1024), "criteo_c100": (2250000, 1024)}[name]
        tables = []
        for k in vocab:
            p = 0 if k <= thr else base
            rows = k if p == 0 else subtable_rows(k, p)
            tables.append(Table(k, 16, p, rng.normal(0.0, 0.05, size=(rows, 16))))
        idx = np.array([[_zipf_index(rng, k) for k in vocab] for _ in range(B)], dtype=np.int64)
        return Workload(cfg, tables, 0, idx, np.zeros((B, 0)))
    if name in ("llm_gen", "llm_gen_small"):
        V, d, p = (50257, 768, 256) if name == "llm_gen" else (1000, 48, 32)
        w = rng.normal(0.0, 0.02, size=(subtable_rows(V, p), d))
        idx = rng.integers(0, V, size=(B, 1)).astype(np.int64)
        return Workload(cfg, [Table(V, d, p, w)], 0, idx, np.zeros((B, 0)))
    if name in ("mlp_small", "mlp_512x256"):
        fan_in, fan_out = (64, 32) if name == "mlp_small" else (512, 256)
        w = rng.normal(0.0, 1.0 / np.sqrt(fan_in), size=(fan_in, fan_out))
        return Workload(cfg, [Table(fan_in, fan_out, 0, w)], 0, np.zeros((B, 1), dtype=np.int64), np.zeros((B, 0)))
    if name in ("table1", "table1_small"):
        k, d, p, l = (2**63 - 1, 768, 16, 32) if name == "table1" else (16**8, 48, 16, 0)
        w = rng.normal(0.0, 0.02, size=(p * (l or 8), d))
        idx = rng.integers(0, k, size=(B, 1), dtype=np.int64)
        return Workload(cfg, [Table(k, d, p, w, l=l)], 0, idx, np.zeros((B, 0)))
    if name in ("llm_l1", "llm_l1_small"):
        V, d, p, m = (50257, 768, 256, 128) if name == "llm_l1" else (1000, 48, 32, 64)
        w = rng.normal(0.0, 0.02, size=(subtable_rows(V, p), d))
        tables = [Table(V, d, p, w, weight_id=0) for _ in range(m)]   # contiguous: stride p l in, d out
        idx = rng.integers(0, V, size=(B, m)).astype(np.int64)
        return Workload(cfg, tables, 0, idx, np.zeros((B, 0)))
    if name in ("llm", "llm_small"):
        V, d, p, m, stride = (50257, 768, 256, 128, 1024) if name == "llm" else (1000, 48, 32, 64, 128)
        w = rng.normal(0.0, 0.02, size=(subtable_rows(V, p), d))
        tables = [Table(V, d, p, w, in_off=stride * t, out_off=stride * t, weight_id=0) for t in range(m)]
        idx = rng.integers(0, V, size=(B, m)).astype(np.int64)
        return Workload(cfg, tables, 0, idx, np.zeros((B, 0)))
    raise KeyError(name)


def microbench_seed() -> int:
    """Seed of the microbench's uniform limbs (D9 purpose 9 streams)."""
    return _CONFIGS["microbench"].seed


def dense_inputs(name: str, batch: int = 1) -> np.ndarray:
    """Encrypted input vectors of the dense linear-layer configs (mlp_*):
    U[-1, 1], one row per query, from the config seed's second stream (the
    weights use the first)."""
    cfg = config_by_name(name)
    fan_in = 64 if name == "mlp_small" else 512
    rng = np.random.default_rng([cfg.seed, 2])
    return rng.uniform(-1.0, 1.0, size=(batch, fan_in))
