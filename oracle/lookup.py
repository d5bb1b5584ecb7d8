"""oracle.lookup -- TEST INFRASTRUCTURE (parity oracle), see oracle/__init__.py.

The HE-LRM server-side lookup, following SURVEY.md D19-D23 (readings of
PAPER.md sections 5.1-5.2 and 2.1.5):

  S0 query encode      digit decomposition (Fig. 6 :329) and
                       concatenated one-hots after the dense slots
                       (Fig. 10 :654)
  D19 layout and plan  block-diagonal packing (PAPER.md:339 torch.block_diag),
                       hybrid diagonals, BSGS split, pre-rotated diagonals
                       ("pre-rotates diagonals")
  D20 lookup, double   double-hoisted BSGS (PAPER.md:289, :584 [bossuat])
  D21 RotSum           Rot-Sum, used as the hybrid fold
  D22 lookup, single   single-hoisted debug/cross-check mode
  gather               the plain definition the lookup approximates:
                       y = W x, i.e. E[i] / sum_t T_t[digit_t(i)]
                       
"""
from __future__ import annotations

import dataclasses
import hashlib
from fractions import Fraction
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import core
from .core import Ciphertext, Params

MODE_DOUBLE, MODE_SINGLE = 0, 1


# --------------------------------------------------------------------------
# S0: client-side digit decomposition and one-hot encoding
# --------------------------------------------------------------------------
def n_digits(k: int, p: int) -> int:
    """l = ceil(log_p k): the smallest l with p^l >= k."""
    l, cap = 1, p
    while cap < k:
        cap *= p
        l += 1
    return l


def digit_decompose(i: int, p: int, l: int) -> Tuple[int, ...]:
    """Base-p digits of i, least-significant first (Fig. 6: 14 -> (2,3) base 4)."""
    if not 0 <= i < p ** l:
        raise ValueError("HELRM_ERR_RANGE")
    out = []
    for _ in range(l):
        out.append(i % p)
        i //= p
    return tuple(out)


@dataclasses.dataclass
class Block:
    k: int
    d: int
    p: int
    compressed: bool
    l: int          # digits (1 if uncompressed)
    w: int          # input segment width
    I: int          # input offset
    R: int          # output offset
    S: np.ndarray   # (w, d) rows of the block (E or the stacked sub-tables)


@dataclasses.dataclass
class Layout:
    blocks: List[Block]
    n_dense: int
    K: int
    M: int


def layout(workload) -> Layout:
    """D19 input/output layout: table b is uncompressed iff k_b <= p_b (or
    p_b = 0) and no digit count is given, segment width k_b; else l_b digits
    (ceil(log_p k_b), or the table's explicit l >= that), width p_b l_b, digit t
    one-hot at [t p_b, (t+1) p_b) of the segment.  Default offsets are the
    paper's contiguous layout."""
    blocks = []
    I, R = workload.n_dense, 0
    for t in workload.tables:
        lx = getattr(t, "l", 0)          # explicit digit count (the boundary's int64 k caps ceil(log_p k))
        comp = t.p != 0 and (t.k > t.p or lx > 0)
        if comp and lx > 0 and t.p ** lx < t.k:
            raise ValueError("HELRM_ERR_LAYOUT: p^l < k")
        l = (lx or n_digits(t.k, t.p)) if comp else 1
        w = t.p * l if comp else t.k
        if t.weights.shape != (w, t.d):
            raise ValueError("HELRM_ERR_LAYOUT: table weights have the wrong shape")
        Ib = I if t.in_off < 0 else t.in_off
        Rb = R if t.out_off < 0 else t.out_off
        blocks.append(Block(t.k, t.d, t.p, comp, l, w, Ib, Rb, np.asarray(t.weights, dtype=np.float64)))
        I, R = Ib + w, Rb + t.d
    K = max(b.I + b.w for b in blocks)
    M = max(b.R + b.d for b in blocks)
    return Layout(blocks, workload.n_dense, K, M)


def encode_query(lay: Layout, idx, dense) -> np.ndarray:
    """Client slot vector x (length K): [dense || seg_1 || ... || seg_B]."""
    x = np.zeros(lay.K)
    x[: lay.n_dense] = dense
    for b, i in zip(lay.blocks, idx):
        i = int(i)
        if not 0 <= i < b.k:
            raise ValueError("HELRM_ERR_RANGE")
        if b.compressed:
            for t, dgt in enumerate(digit_decompose(i, b.p, b.l)):
                x[b.I + t * b.p + dgt] = 1.0
        else:
            x[b.I + i] = 1.0
    return x


def gather(lay: Layout, idx) -> np.ndarray:
    """The plain definition: y[R_b + c] = E_b[i_b][c] (uncompressed) or
    sum_t T_{b,t}[digit_t(i_b)][c] (compressed), zero elsewhere (length M)."""
    y = np.zeros(lay.M)
    for b, i in zip(lay.blocks, idx):
        i = int(i)
        if b.compressed:
            row = np.zeros(b.d)
            for t, dgt in enumerate(digit_decompose(i, b.p, b.l)):
                row += b.S[t * b.p + dgt]
        else:
            row = b.S[i]
        y[b.R: b.R + b.d] += row
    return y


def dense_matrix(lay: Layout) -> np.ndarray:
    """W in R^{M x K}, W[R_b + col][I_b + row] = S_b[row][col] (small configs)."""
    W = np.zeros((lay.M, lay.K))
    for b in lay.blocks:
        W[b.R: b.R + b.d, b.I: b.I + b.w] += b.S.T
    return W


# --------------------------------------------------------------------------
# D19: hybrid diagonals and the BSGS plan
# --------------------------------------------------------------------------
def next_pow2(x: int) -> int:
    p = 1
    while p < x:
        p *= 2
    return p


def _box_offsets(b: Block, o: int, c: int, n: int) -> List[int]:
    """Offsets t (mod n) whose diagonal line s -> (o n + s, c n + (s + t) mod n)
    (mbar = n) can cross block b's box of W: rows [R_b, R_b + d_b) x columns
    [I_b, I_b + w_b), both clipped to output ct o / input ct c.  For s in the
    box's row range [s0, s1) and column position v in [v0, v1), t = v - s."""
    s0, s1 = max(b.R, o * n) - o * n, min(b.R + b.d, (o + 1) * n) - o * n
    v0, v1 = max(b.I, c * n) - c * n, min(b.I + b.w, (c + 1) * n) - c * n
    if s0 >= s1 or v0 >= v1:
        return []
    lo, hi = v0 - (s1 - 1), (v1 - 1) - s0
    if hi - lo + 1 >= n:
        return list(range(n))
    return [t % n for t in range(lo, hi + 1)]


def hybrid_diagonals(lay: Layout, n: int):
    """D19 hybrid diagonals, evaluated from their definition:

        diag_{o,c,t}[s] = W[o n + (s mod mbar)][c n + ((s + t) mod n)]

    for t in [0, mbar), s in [0, n), 0 where the index falls outside W, with
    W[R_b + col][I_b + row] = S_b[row][col] and 0 elsewhere.  Returns mbar, O,
    C and {(o, c, t): vector} for the diagonals that are not identically zero.

    W is zero outside the block boxes, so for each t only the positions s
    whose row o n + (s mod mbar) lies in some block can be non-zero: those s
    are enumerated per block (every s with s mod mbar = r - o n), and W is read
    at (row(s), col(s, t)) there.  When mbar < n every t in [0, mbar) is
    evaluated; when mbar = n (O, C may exceed 1) only the offsets whose line
    crosses a block's box (_box_offsets) -- every other t reads W only outside
    the boxes."""
    mbar = min(next_pow2(lay.M), n)
    O = -(-lay.M // n)
    C = -(-lay.K // n)
    # the stacked block entries: S_b[row][col] at flat[off_b + row d_b + col]
    offs, acc = [], 0
    for b in lay.blocks:
        offs.append(acc)
        acc += b.w * b.d
    flat = np.concatenate([b.S.ravel() for b in lay.blocks]) if lay.blocks else np.zeros(0)
    diags: Dict[Tuple[int, int, int], np.ndarray] = {}
    for o in range(O):
        # every (s, W row, block) with row(s) = o n + (s mod mbar) inside a block's rows
        S_, R_, B_ = [], [], []
        for bi, b in enumerate(lay.blocks):
            r = np.arange(max(b.R, o * n), min(b.R + b.d, (o + 1) * n))
            r = r[(r - o * n) < mbar]                   # row(s) never exceeds o n + mbar - 1
            if len(r) == 0:
                continue
            a = np.arange(n // mbar)
            s = ((r - o * n)[:, None] + mbar * a[None, :]).ravel()
            S_.append(s)
            R_.append(np.repeat(r, len(a)))
            B_.append(np.full(len(s), bi))
        if not S_:
            continue
        s_all, r_all, b_all = np.concatenate(S_), np.concatenate(R_), np.concatenate(B_)
        I_b = np.array([b.I for b in lay.blocks])[b_all]
        w_b = np.array([b.w for b in lay.blocks])[b_all]
        d_b = np.array([b.d for b in lay.blocks])[b_all]
        R_b = np.array([b.R for b in lay.blocks])[b_all]
        off_b = np.array(offs)[b_all]
        for c in range(C):
            if mbar < n:
                cand = range(mbar)
            else:
                cand = sorted({t for b in lay.blocks for t in _box_offsets(b, o, c, n)})
            for t in cand:
                u = c * n + (s_all + t) % n             # W column of position s
                inside = (u >= I_b) & (u < I_b + w_b)
                if not inside.any():
                    continue
                vals = flat[off_b[inside] + (u[inside] - I_b[inside]) * d_b[inside] + (r_all[inside] - R_b[inside])]
                vec = np.zeros(n)
                np.add.at(vec, s_all[inside], vals)
                if np.any(vec != 0):
                    diags[(o, c, t)] = vec
    return mbar, O, C, diags


def min_cyclic_interval(offsets: List[int], n: int) -> Tuple[int, int]:
    """Minimal cyclic interval [t0, t0 + span) mod n covering the offsets;
    ties go to the smallest t0."""
    ts = sorted(set(offsets))
    best = None
    for idx, start in enumerate(ts):
        # the interval starting at ts[idx] ends at its cyclic predecessor
        span = (ts[idx - 1] - start) % n + 1 if len(ts) > 1 else 1
        cand = (span, start)
        if best is None or cand < best:
            best = cand
    span, t0 = best
    return t0, span


def choose_n1(span: int) -> int:
    """Smallest power of two n1 with n1^2 >= span."""
    n1 = 1
    while n1 * n1 < span:
        n1 *= 2
    return n1


@dataclasses.dataclass
class Plan:
    level: int
    mode: int
    mbar: int
    O: int
    C: int
    t0: List[int]                     # per output block
    span: List[int]
    n1: int
    n2: List[int]
    # entries[o][i] = list of (c, j, uid); giants[o][i] = g_i (rotation amount)
    entries: List[List[List[Tuple[int, int, int]]]]
    giants: List[List[int]]
    u_slots: List[np.ndarray]         # unique pre-rotated diagonals (length n)
    babies: List[List[int]]           # per input ct, the baby amounts j used
    n_diag: int                       # kept (non-zero) diagonals before dedup

    def rotation_amounts(self, P: Params) -> List[int]:
        """Rotation amounts that need a key: babies j != 0 that occur, giants
        g_i != 0 whose inner sum is not empty, and the RotSum amounts mbar 2^r."""
        amts = set()
        for bl in self.babies:
            amts.update(j for j in bl if j != 0)
        for o, gl in enumerate(self.giants):
            amts.update(g for i, g in enumerate(gl) if g % P.n != 0 and self.entries[o][i])
        r = self.mbar
        while r < P.n:
            amts.add(r)
            r *= 2
        return sorted(amts)

    def galois(self, P: Params) -> List[int]:
        """D19 Galois list {5^a : a in rotation_amounts}."""
        return sorted({core.galois_elt(a, P) for a in self.rotation_amounts(P)})


def make_plan(lay: Layout, n: int, level: int, n1: int = 0, mode: int = MODE_DOUBLE) -> Plan:
    if level < 1:
        raise ValueError("HELRM_ERR_LEVEL")
    mbar, O, C, diags = hybrid_diagonals(lay, n)
    t0s, spans, n2s, entries, giants = [], [], [], [], []
    n1_all = n1
    per_o = {}
    for o in range(O):
        offs = [t for (oo, c, t) in diags if oo == o]
        t0, span = min_cyclic_interval(offs, n)
        per_o[o] = (t0, span)
    if n1_all == 0:
        n1_all = choose_n1(max(sp for _, sp in per_o.values()))
    u_slots: List[np.ndarray] = []
    uid_of: Dict[bytes, int] = {}
    babies = [set() for _ in range(C)]
    for o in range(O):
        t0, span = per_o[o]
        n2 = -(-span // n1_all)
        ent = [[] for _ in range(n2)]
        gl = [(t0 + i * n1_all) % n for i in range(n2)]
        for (oo, c, t), vec in sorted(diags.items()):
            if oo != o:
                continue
            r = (t - t0) % n
            j, i = r % n1_all, r // n1_all
            u = np.roll(vec, gl[i])          # rot(v, -g)[s] = v[(s - g) mod n]
            key = hashlib.sha256(u.tobytes()).digest()
            uid = uid_of.get(key)
            if uid is None:
                uid = len(u_slots)
                uid_of[key] = uid
                u_slots.append(u)
            ent[i].append((c, j, uid))
            babies[c].add(j)
        t0s.append(t0)
        spans.append(span)
        n2s.append(n2)
        entries.append(ent)
        giants.append(gl)
    return Plan(level, mode, mbar, O, C, t0s, spans, n1_all, n2s, entries, giants, u_slots,
                [sorted(b) for b in babies], len(diags))


def simulate_plan_slots(plan: Plan, x: np.ndarray, n: int) -> np.ndarray:
    """float64 slot-level run of exactly the D19/D20 schedule (ckks-vm style,
    SPEC.md:101): babies rot(x_c, j), inner sums with the pre-rotated
    diagonals, giant rotations, then RotSum.  Used to pin the plan against
    the dense W x."""
    rot = lambda v, k: np.roll(v, -k)
    xs = [np.zeros(n) for _ in range(plan.C)]
    for c in range(plan.C):
        seg = x[c * n:(c + 1) * n]
        xs[c][: len(seg)] = seg
    out = []
    for o in range(plan.O):
        acc = np.zeros(n)
        for i, ent in enumerate(plan.entries[o]):
            if not ent:
                continue
            inner = np.zeros(n)
            for (c, j, uid) in ent:
                inner += plan.u_slots[uid] * rot(xs[c], j)
            acc += rot(inner, plan.giants[o][i])
        r = plan.mbar
        while r < n:
            acc = acc + rot(acc, r)
            r *= 2
        out.append(acc)
    return np.concatenate(out)


# --------------------------------------------------------------------------
# Encoded plaintext diagonals (server setup, S2): Encode(u, Delta_pt = q_l)
# over Q_l P (double) or Q_l (single), NTT form
# --------------------------------------------------------------------------
def encode_plan(P: Params, plan: Plan) -> List[np.ndarray]:
    l = plan.level
    primes = P.qp(l) if plan.mode == MODE_DOUBLE else P.q[: l + 1]
    ms = core.encode_many(plan.u_slots, P.q[l], P.N)
    return [core.ntt(core.reduce_signed(m, primes), primes, P) for m in ms]


def query_cts(P: Params, pk, lay: Layout, plan: Plan, idx, dense, level: int, seed: int, query: int) -> List[Ciphertext]:
    """Client: encode the query and encrypt its C ciphertexts; the encryption
    seed of ciphertext c of query q is (seed << 20) | (q C + c)."""
    x = encode_query(lay, idx, dense)
    cts = []
    for c in range(plan.C):
        z = np.zeros(P.n)
        seg = x[c * P.n:(c + 1) * P.n]
        z[: len(seg)] = seg
        cts.append(core.encrypt(P, pk, z, level, (seed << 20) | (query * plan.C + c)))
    return cts


# --------------------------------------------------------------------------
# D20 / D21 / D22: the lookup
# --------------------------------------------------------------------------
def rot_sum(P: Params, ct: Ciphertext, mbar: int, rk) -> Ciphertext:
    """D21: for r = 0..log2(n/mbar)-1: ct <- ct + Rotate(ct, mbar 2^r)."""
    r = mbar
    while r < P.n:
        ct = core.ct_add(P, ct, core.rotate(P, ct, r, rk))
        r *= 2
    return ct


def lookup(P: Params, plan: Plan, u_ntt: List[np.ndarray], rk, cts: List[Ciphertext]) -> List[Ciphertext]:
    if len(cts) != plan.C:
        raise ValueError("HELRM_ERR_LAYOUT")
    for ct in cts:
        if ct.level != plan.level:
            raise ValueError("HELRM_ERR_LEVEL")
    if plan.mode == MODE_SINGLE:
        return _lookup_single(P, plan, u_ntt, rk, cts)
    O = lookup_partial(P, plan, u_ntt, rk, cts, 0, None)
    return lookup_finish(P, plan, rk, O, cts[0].scale)


def giant_pairs(plan: Plan) -> List[Tuple[int, int]]:
    """The non-empty (o, i) giant pairs in (o, i) order -- the unit D23 splits."""
    return [(o, i) for o in range(plan.O) for i, ent in enumerate(plan.entries[o]) if ent]


def lookup_partial(P: Params, plan: Plan, u_ntt, rk, cts: List[Ciphertext], z_lo: int, z_hi: Optional[int]):
    """D20 L1-L4 restricted to the giant pairs z in [z_lo, z_hi) of
    giant_pairs(plan): returns the Q_l P accumulators (O0, O1) per output
    block.  Over all pairs this is the lookup up to L5; the partial results of
    a split sum exactly to it (D23)."""
    l = plan.level
    qp = P.qp(l)
    pairs = giant_pairs(plan)
    mine = set(pairs[z_lo:z_hi] if z_hi is not None else pairs[z_lo:])
    # L1: D^c_k = ModUp_k(c1^c)
    D = [[core.modup(P, ct.c1, l, k) for k in range(P.dnum(l))] for ct in cts]
    # L2: baby steps (a, b)^c_j over Q_l P, lazy (no ModDown)
    ab: List[Dict[int, Tuple[np.ndarray, np.ndarray]]] = []
    for c, ct in enumerate(cts):
        d = {}
        for j in plan.babies[c]:
            if j == 0:
                d[0] = (core.lift_P(P, ct.c0, l), core.lift_P(P, ct.c1, l))
            else:
                d[j] = core.rotate_lazy(P, ct, j, rk, D=D[c])
        ab.append(d)
    outs = []
    for o in range(plan.O):
        O0 = np.zeros((len(qp), P.N), dtype=np.uint64)
        O1 = np.zeros_like(O0)
        for i, ent in enumerate(plan.entries[o]):
            if not ent or (o, i) not in mine:
                continue
            # L3: (A, B)_{o,i} = sum_c sum_j u_{o,c,i,j} (.) (a, b)^c_j
            A = np.zeros_like(O0)
            B = np.zeros_like(O0)
            for (c, j, uid) in ent:
                a, b = ab[c][j]
                A = core.vadd(A, core.vmul(u_ntt[uid], a, qp), qp)
                B = core.vadd(B, core.vmul(u_ntt[uid], b, qp), qp)
            # L4: giant step
            gi = plan.giants[o][i]
            if gi % P.n == 0:
                O0 = core.vadd(O0, A, qp)
                O1 = core.vadd(O1, B, qp)
            else:
                g = core.galois_elt(gi, P)
                Bp = core.moddown(P, B, l)
                G0, G1 = core.keyswitch(P, Bp, g, rk, l)
                O0 = core.vadd(O0, core.vadd(core.automorph_ntt(A, g, P.N), G0, qp), qp)
                O1 = core.vadd(O1, G1, qp)
        outs.append((O0, O1))
    return outs


def lookup_finish(P: Params, plan: Plan, rk, O, scale) -> List[Ciphertext]:
    """D20 L6-L8 per output block: ModDown both halves (scale Delta q_l),
    rescale (scale Delta), RotSum when mbar < n."""
    l = plan.level
    res = []
    for (O0, O1) in O:
        ct = Ciphertext(core.moddown(P, O0, l), core.moddown(P, O1, l), l, Fraction(scale) * P.q[l])
        ct = core.rescale(P, ct)
        if plan.mbar < P.n:
            ct = rot_sum(P, ct, plan.mbar, rk)
        res.append(ct)
    return res


def _lookup_single(P: Params, plan: Plan, u_ntt, rk, cts):
    """D22: babies are full Rotate(ct, j) in Q_l, u over Q_l only,
    O += Rotate((A_i, B_i), g_i); then rescale and RotSum as in D20."""
    l = plan.level
    Q = P.q[: l + 1]
    rots = []
    for c, ct in enumerate(cts):
        D = [core.modup(P, ct.c1, l, k) for k in range(P.dnum(l))]
        rots.append({j: core.rotate(P, ct, j, rk, D=D) for j in plan.babies[c]})
    outs = []
    for o in range(plan.O):
        acc = None
        for i, ent in enumerate(plan.entries[o]):
            if not ent:
                continue
            A = np.zeros((len(Q), P.N), dtype=np.uint64)
            B = np.zeros_like(A)
            for (c, j, uid) in ent:
                r = rots[c][j]
                A = core.vadd(A, core.vmul(u_ntt[uid], r.c0, Q), Q)
                B = core.vadd(B, core.vmul(u_ntt[uid], r.c1, Q), Q)
            part = core.rotate(P, Ciphertext(A, B, l, cts[0].scale), plan.giants[o][i], rk)
            acc = part if acc is None else core.ct_add(P, acc, part)
        ct = Ciphertext(acc.c0, acc.c1, l, Fraction(cts[0].scale) * P.q[l])
        ct = core.rescale(P, ct)
        if plan.mbar < P.n:
            ct = rot_sum(P, ct, plan.mbar, rk)
        outs.append(ct)
    return outs


# --------------------------------------------------------------------------
# Convenience: a whole config end to end (used by tests and golden scripts)
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Run:
    P: Params
    lay: Layout
    plan: Plan
    sk: object
    pk: object
    rk: object
    u_ntt: List[np.ndarray]
    cts: List[List[Ciphertext]]
    outs: List[List[Ciphertext]]


def run_config(workload, n1: int = 0, mode: int = MODE_DOUBLE, queries: Optional[List[int]] = None,
               do_lookup: bool = True) -> Run:
    cfg = workload.config
    P = core.params_from_config(cfg)
    lay = layout(workload)
    plan = make_plan(lay, P.n, cfg.level, n1=n1, mode=mode)
    sk = core.sk_gen(P, cfg.seed)
    pk = core.pk_gen(P, sk, cfg.seed)
    rk = core.rotkeys_gen(P, sk, plan.galois(P), cfg.seed)
    u_ntt = encode_plan(P, plan)
    qs = list(range(workload.indices.shape[0])) if queries is None else queries
    cts = [query_cts(P, pk, lay, plan, workload.indices[q], workload.dense[q], cfg.level, cfg.seed, q) for q in qs]
    outs = [lookup(P, plan, u_ntt, rk, c) for c in cts] if do_lookup else []
    return Run(P, lay, plan, sk, pk, rk, u_ntt, cts, outs)
