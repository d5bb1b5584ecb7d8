"""Pins of the oracle's lookup layer (S0, D19-D22) against the paper's worked
examples and counts, the plain definition (float64 gather / dense W x), and
exact identities.  CPU only."""
import types

import numpy as np
import pytest

import synth
from oracle import core
from oracle import lookup as lk


def test_digit_decomposition_paper_examples():
    assert lk.digit_decompose(14, 4, 2) == (2, 3)             # PAPER.md:329, Fig. 6
    assert lk.digit_decompose(50256, 16, 4) == (0, 5, 4, 12)
    assert lk.digit_decompose(0, 7, 3) == (0, 0, 0)
    with pytest.raises(ValueError):
        lk.digit_decompose(16, 4, 2)
    assert lk.n_digits(10**6, 4) == 10
    assert lk.n_digits(50257, 16) == 4 and lk.n_digits(50257, 256) == 2


@pytest.mark.parametrize("p,l", [(2, 16), (4, 8), (16, 4), (256, 2), (7, 5)])
def test_digit_recomposition_exhaustive(p, l):
    for i in range(min(p ** l, 1 << 16)):
        d = lk.digit_decompose(i, p, l)
        assert sum(x * p ** t for t, x in enumerate(d)) == i and all(0 <= x < p for x in d)


def test_uci_layout_paper_slot_count():
    """5 dense + one-hots of widths [2,4,2,3,2,3,4,3] need 28
    slots (uncompressed).  Our UCI-shaped config (BASELINE.json) instead has 13
    dense and base-4 digits: widths [2,2,3,4,4,8,8,8], K = 52."""
    paper = types.SimpleNamespace(n_dense=5, tables=[synth.Table(k, 4, 0, np.zeros((k, 4)))
                                                     for k in [2, 4, 2, 3, 2, 3, 4, 3]])
    assert lk.layout(paper).K == 28
    lay = lk.layout(synth.make_workload("uci"))
    assert [b.w for b in lay.blocks] == [2, 2, 3, 4, 4, 8, 8, 8] and lay.K == 52 and lay.M == 128


def test_encode_query_invariants():
    w = synth.make_workload("criteo")
    lay = lk.layout(w)
    x = lk.encode_query(lay, w.indices[0], w.dense[0])
    assert lay.K == 4126 and x.sum() == 68
    for b, i in zip(lay.blocks, w.indices[0]):
        seg = x[b.I: b.I + b.w]
        assert seg.sum() == b.l                              # popcount = l per segment
        if b.compressed:
            for t in range(b.l):
                assert seg[t * b.p:(t + 1) * b.p].sum() == 1
    with pytest.raises(ValueError):
        lk.encode_query(lay, [10**8] * 26, [])


@pytest.mark.parametrize("slots,cts", [(569545, 18), (2772109, 85), (128 * 512, 2), (1096, 1), (47759, 2)])
def test_input_ciphertext_counts(slots, cts):
    """PAPER.md:462-463, :472 (18 and 85 cts at n = 2^15), :553 (m p l / n = 2)."""
    lay = lk.Layout([lk.Block(slots, 1, 0, False, 1, slots, 0, 0, np.zeros((1, 1)))], 0, slots, 1)
    assert -(-lay.K // (1 << 15)) == cts
    # the planner's own count
    w = types.SimpleNamespace(n_dense=0, tables=[synth.Table(1, 1, 0, np.ones((1, 1)), in_off=slots - 1)])
    mbar, O, C, diags = lk.hybrid_diagonals(lk.layout(w), 1 << 15)
    assert C == cts


def test_criteo_plan_matches_paper_diagonal_count():
    """the 10^4x / 10^5x Criteo models have 512 non-zero
    diagonals; our Criteo-shaped draw (26 tables of width <= 256, d = 16) under
    the hybrid layout gives exactly 512, span 512 ->
    n1 = 32, n2 = 16, <= 46 BSGS rotations."""
    lay = lk.layout(synth.make_workload("criteo"))
    plan = lk.make_plan(lay, 1 << 15, 23)
    assert plan.n_diag == 512 and len(plan.u_slots) == 512
    assert (plan.mbar, plan.O, plan.C, plan.n1, plan.n2, plan.t0) == (512, 1, 1, 32, [16], [0])
    P = types.SimpleNamespace(n=1 << 15)
    amts = plan.rotation_amounts(P)
    bsgs = [a for a in amts if a < 512]
    assert len(bsgs) <= 46 and len(bsgs) <= plan.n1 + plan.n2[0] - 2
    assert len(amts) == 52                                   # 31 + 15 + 6 RotSum


def test_uci_and_tiny_plans():
    P = types.SimpleNamespace(n=1 << 13)
    plan = lk.make_plan(lk.layout(synth.make_workload("uci")), 1 << 13, 7)
    assert plan.n_diag == 98 and (plan.n1, plan.n2) == (16, [8]) and len(plan.rotation_amounts(P)) == 27
    for name in ("tiny_a", "tiny_b"):
        plan = lk.make_plan(lk.layout(synth.make_workload(name)), 1 << 11, 2)
        assert plan.n_diag == 16 and (plan.n1, plan.n2) == (4, [4])
        assert len(plan.rotation_amounts(types.SimpleNamespace(n=1 << 11))) == 13


@pytest.mark.parametrize("name", ["tiny_a", "tiny_b", "uci", "criteo"])
def test_plan_slot_simulation_equals_dense_matvec(name):
    """The exact D19/D20 schedule run on float64 slots (ckks-vm semantics,
    SPEC.md:101, :246) equals the dense W x and the gather, periodic in mbar."""
    w = synth.make_workload(name)
    lay = lk.layout(w)
    n = w.config.n_slots
    plan = lk.make_plan(lay, n, w.config.level)
    rng = np.random.default_rng(0)
    W = lk.dense_matrix(lay)
    for trial in range(3):
        x = rng.normal(size=lay.K) if trial else lk.encode_query(lay, w.indices[0], w.dense[0])
        y = lk.simulate_plan_slots(plan, x, n)
        assert np.abs(y[: lay.M] - W @ x).max() < 1e-9
        assert np.abs(y[lay.M: plan.mbar]).max(initial=0) < 1e-12
        assert np.allclose(y[: plan.mbar], y[plan.mbar: 2 * plan.mbar] if plan.mbar < n else y[: plan.mbar])
    x = lk.encode_query(lay, w.indices[0], w.dense[0])
    assert np.abs(W @ x - lk.gather(lay, w.indices[0])).max() < 1e-12


def test_plan_scaled_llm_l2_layout():
    """Scaled LLM-L2 (n = 2048, stride 128, shared 32x48 table, 64 tokens):
    4 in / 4 out cts, 79 shared diagonals, t0 = -47 mod n."""
    n, stride, rows, d, m = 2048, 128, 32, 48, 64
    wts = np.random.default_rng(1).normal(size=(rows, d))
    tables = [synth.Table(rows, d, 0, wts, in_off=stride * t, out_off=stride * t) for t in range(m)]
    w = types.SimpleNamespace(n_dense=0, tables=tables)
    lay = lk.layout(w)
    plan = lk.make_plan(lay, n, 1)
    assert (plan.C, plan.O, len(plan.u_slots)) == (4, 4, 79) and plan.t0[0] == n - 47
    x = np.random.default_rng(2).normal(size=lay.K)
    y = lk.simulate_plan_slots(plan, x, n)
    assert np.abs(y[: lay.M] - lk.dense_matrix(lay) @ x).max() < 1e-9


def test_hs_and_bsgs_agree_on_random_matrices():
    """Halevi-Shoup (n1 = 1, every offset a giant) == BSGS == dense."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        k, d = int(rng.integers(1, 40)), int(rng.integers(1, 20))
        w = types.SimpleNamespace(n_dense=int(rng.integers(0, 5)),
                                  tables=[synth.Table(k, d, 0, rng.normal(size=(k, d)))])
        lay = lk.layout(w)
        n = 64
        x = rng.normal(size=lay.K)
        ref = lk.dense_matrix(lay) @ x
        for n1 in (1, 0, 2, 8):
            y = lk.simulate_plan_slots(lk.make_plan(lay, n, 1, n1=n1), x, n)
            assert np.abs(y[: lay.M] - ref).max() < 1e-9


def test_digit_decomposition_identity_exhaustive():
    """North star: per-digit partial lookups sum to the full lookup, which is
    E^[i] = sum_t T_t[digit_t(i)] -- exact on plaintext slots, all i of Tiny-B."""
    w = synth.make_workload("tiny_b")
    lay = lk.layout(w)
    b = lay.blocks[0]
    W = lk.dense_matrix(lay)
    for i in range(256):
        x = lk.encode_query(lay, [i], [])
        full = W @ x
        parts = np.zeros_like(full)
        for t in range(b.l):
            xt = np.zeros_like(x)
            seg = slice(b.I + t * b.p, b.I + (t + 1) * b.p)
            xt[seg] = x[seg]
            parts += W @ xt
        assert np.array_equal(parts, full)
        d = lk.digit_decompose(i, 16, 2)
        assert np.array_equal(full, b.S[d[0]] + b.S[16 + d[1]])


@pytest.fixture(scope="module")
def uci_run():
    return lk.run_config(synth.make_workload("uci"))


@pytest.mark.parametrize("name", ["tiny_a", "tiny_b"])
def test_tiny_lookup_decrypts_to_gather(name):
    w = synth.make_workload(name)
    run = lk.run_config(w)
    out = run.outs[0][0]
    assert out.level == w.config.level - 1 and out.scale == w.config.N // w.config.N * (1 << 30)
    z = core.decrypt_decode(run.P, run.sk, out)
    y = lk.gather(run.lay, w.indices[0])
    assert np.abs(z[: run.lay.M] - y).max() < 1e-3
    # slot s holds y[s mod mbar] everywhere (RotSum periodicity, R20)
    mb = run.plan.mbar
    zz = z.reshape(-1, mb)
    assert np.abs(zz[:, : run.lay.M] - y).max() < 1e-3 and np.abs(zz[:, run.lay.M:]).max(initial=0) < 1e-3


def test_uci_lookup_decrypts_to_gather_and_ignores_dense(uci_run):
    run = uci_run
    w = synth.make_workload("uci")
    z = core.decrypt_decode(run.P, run.sk, run.outs[0][0])
    y = lk.gather(run.lay, w.indices[0])
    assert np.abs(z[: run.lay.M] - y).max() < 1e-3
    # dense slots do not influence y (R19): change them, same decrypted result within noise
    ct2 = lk.query_cts(run.P, run.pk, run.lay, run.plan, w.indices[0], 1 - w.dense[0], 7, 1, 0)
    out2 = lk.lookup(run.P, run.plan, run.u_ntt, run.rk, ct2)[0]
    z2 = core.decrypt_decode(run.P, run.sk, out2)
    assert np.abs(z2[: run.lay.M] - y).max() < 1e-3


def test_single_and_double_modes_agree(uci_run):
    run = uci_run
    w = synth.make_workload("uci")
    plan_s = lk.make_plan(run.lay, run.P.n, 7, mode=lk.MODE_SINGLE)
    u_s = lk.encode_plan(run.P, plan_s)
    out_s = lk.lookup(run.P, plan_s, u_s, run.rk, run.cts[0])[0]
    zs = core.decrypt_decode(run.P, run.sk, out_s)
    zd = core.decrypt_decode(run.P, run.sk, run.outs[0][0])
    assert np.abs(zs - zd).max() < 1e-3
    assert not np.array_equal(out_s.c0, run.outs[0][0].c0)   # different bits, same values (D22)


def test_per_digit_partial_lookups_sum_encrypted():
    """The digit-decomposition identity under encryption (within noise)."""
    w = synth.make_workload("tiny_b")
    run = lk.run_config(w)
    b = run.lay.blocks[0]
    x = lk.encode_query(run.lay, w.indices[0], [])
    total = np.zeros(run.P.n)
    for t in range(b.l):
        xt = np.zeros(run.P.n)
        seg = slice(b.I + t * b.p, b.I + (t + 1) * b.p)
        xt[seg] = x[seg]
        ct = core.encrypt(run.P, run.pk, xt, 2, 1000 + t)
        total += core.decrypt_decode(run.P, run.sk, lk.lookup(run.P, run.plan, run.u_ntt, run.rk, [ct])[0])
    y = lk.gather(run.lay, w.indices[0])
    assert np.abs(total[: run.lay.M] - y).max() < 2e-3


def test_llm_full_size_plan_counts():
    """LLM-L2 at full size (n = 2^15): 1279 distinct diagonals shared by the 4
    blocks (t0 = -767), n1 = 64, n2 = 20, 82 rotation amounts (63 babies + 20
    giants; giant 12 is amount 1, also a baby)."""
    w = synth.make_workload("llm")
    lay = lk.layout(w)
    n = 1 << 15
    plan = lk.make_plan(lay, n, 19)
    assert (plan.C, plan.O, len(plan.u_slots), plan.n1, plan.n2) == (4, 4, 1279, 64, [20] * 4)
    assert plan.t0 == [n - 767] * 4 and plan.n_diag == 4 * 1279
    amts = plan.rotation_amounts(types.SimpleNamespace(n=n))
    assert len(amts) == 82 and (n - 767 + 64 * 12) % n == 1


def test_llm_small_lookup_decrypts_to_gather():
    """LLM-L2 layout (4 input / 4 output cts, shared diagonals, mbar = n, no
    RotSum) on the Tiny ring: every output block decrypts to the gather."""
    w = synth.make_workload("llm_small")
    run = lk.run_config(w)
    assert (run.plan.C, run.plan.O, len(run.plan.u_slots), run.plan.n1) == (4, 4, 111, 16)
    z = np.concatenate([core.decrypt_decode(run.P, run.sk, o) for o in run.outs[0]])
    assert np.abs(z[: run.lay.M] - lk.gather(run.lay, w.indices[0])).max() < 1e-3


def test_criteo_c2_small_lookup_decrypts_to_gather():
    """Two input ciphertexts (the less compressed Criteo model of PAPER.md
    Table 2, scaled to the Tiny ring): 2,944 one-hot slots over 2 cts, 1024
    diagonals (512 per ct), the 15 giant rotations shared by both cts; the
    output decrypts to the float64 gather."""
    w = synth.make_workload("criteo_c2_small")
    run = lk.run_config(w)
    assert (run.plan.C, run.plan.O, len(run.plan.u_slots), run.plan.n1, run.plan.n_diag) == (2, 1, 1024, 32, 1024)
    z = core.decrypt_decode(run.P, run.sk, run.outs[0][0])
    assert np.abs(z[: run.lay.M] - lk.gather(run.lay, w.indices[0])).max() < 1e-3


def test_criteo_c2_full_size_plan_counts():
    """The full-size 2-ct Criteo shape (the 10^3x model "has 1024
    non-zero diagonals and requires two ciphertexts"): 47,798 input slots, C = 2,
    1024 diagonals, n1 = 32, n2 = 16, 52 rotation keys (31 babies + 15 giants +
    RotSum 6 -- the same key set as the 1-ct model)."""
    w = synth.make_workload("criteo_c2")
    lay = lk.layout(w)
    assert sum(len(t.weights) for t in w.tables) == 47798
    n = 1 << 15
    plan = lk.make_plan(lay, n, 23)
    assert (plan.C, plan.O, len(plan.u_slots), plan.n1, plan.n2, plan.n_diag) == (2, 1, 1024, 32, [16], 1024)
    assert len(plan.rotation_amounts(types.SimpleNamespace(n=n))) == 52


def test_llm_gen_small_lookup_decrypts_to_gather():
    """LLM generation step (one sampled token looked up per
    step, a sparse matrix-vector product) on the Tiny ring: 1000 x 48 table,
    base 32 -> 64 one-hot slots, 64 diagonals; decrypts to the gather."""
    w = synth.make_workload("llm_gen_small")
    run = lk.run_config(w)
    assert (run.plan.C, run.plan.O, run.plan.n_diag, run.plan.n1, run.plan.mbar) == (1, 1, 64, 8, 64)
    z = core.decrypt_decode(run.P, run.sk, run.outs[0][0])
    assert np.abs(z[: run.lay.M] - lk.gather(run.lay, w.indices[0])).max() < 1e-3


def test_llm_gen_full_size_plan_counts():
    """Generation step at full size (GPT-2 table, base 256: 512 slots in, 768
    out): mbar = 1024, 1024 diagonals, n1 = 32, n2 = 32, 67 rotation keys
    (31 babies + 31 giants + RotSum log2(n / 1024) = 5)."""
    w = synth.make_workload("llm_gen")
    lay = lk.layout(w)
    n = 1 << 15
    plan = lk.make_plan(lay, n, 19)
    assert (plan.C, plan.O, plan.n_diag, plan.n1, plan.n2, plan.mbar) == (1, 1, 1024, 32, [32], 1024)
    assert len(plan.rotation_amounts(types.SimpleNamespace(n=n))) == 67


def test_tiny_dnum7_lookup_decrypts_to_gather():
    """Key-switch edge case: alpha = K = 1 under 7 ciphertext primes gives
    dnum = 7 digits at the lookup level (the library's maximum); the lookup
    still decrypts to the gather."""
    w = synth.make_workload("tiny_dnum7")
    run = lk.run_config(w)
    assert run.P.dnum(w.config.level) == 7
    z = core.decrypt_decode(run.P, run.sk, run.outs[0][0])
    assert np.abs(z[: run.lay.M] - lk.gather(run.lay, w.indices[0])).max() < 1e-3


def _dense_layer_run(name):
    w = synth.make_workload(name)
    x = synth.dense_inputs(name)[0]
    cfg = w.config
    P = core.params_from_config(cfg)
    lay = lk.layout(w)
    plan = lk.make_plan(lay, P.n, cfg.level)
    sk = core.sk_gen(P, cfg.seed)
    pk = core.pk_gen(P, sk, cfg.seed)
    rk = core.rotkeys_gen(P, sk, plan.galois(P), cfg.seed)
    z = np.zeros(P.n)
    z[: len(x)] = x
    ct = core.encrypt(P, pk, z, cfg.level, cfg.seed << 20)
    out = lk.lookup(P, plan, lk.encode_plan(P, plan), rk, [ct])
    return w, x, P, plan, sk, ct, out


def test_dense_linear_layer_on_the_lookup_engine():
    """fully connected layers run on the same diagonal/BSGS
    machinery.  With the weight matrix W (64 x 32) as the "table" and a dense
    encrypted x, the lookup decrypts to the matrix-vector product x W."""
    w, x, P, plan, sk, ct, out = _dense_layer_run("mlp_small")
    assert (plan.n_diag, plan.n1, plan.mbar) == (32, 8, 32)
    y = core.decrypt_decode(P, sk, out[0])
    assert np.abs(y[:32] - x @ w.tables[0].weights).max() < 1e-3


def _extraction_workloads(w):
    """the server splits the client's [dense || one-hot] vector
    into a dense and a sparse ciphertext.  Mask + rotate is a linear map with a
    single non-zero diagonal, so it runs on the same engine: identity "tables"
    reading slots [0, n_dense) and [n_dense, K) and writing from slot 0."""
    import dataclasses
    lay = lk.layout(w)
    nd, ns = w.n_dense, lay.K - w.n_dense
    dense = dataclasses.replace(w, tables=[synth.Table(nd, nd, 0, np.eye(nd), in_off=0, out_off=0)], n_dense=0)
    sparse = dataclasses.replace(w, tables=[synth.Table(ns, ns, 0, np.eye(ns), in_off=nd, out_off=0)], n_dense=0)
    return lay, dense, sparse


def test_dense_sparse_extraction_on_the_lookup_engine():
    """UCI query: the dense extraction returns the 13 dense features, the
    sparse extraction the one-hot segments moved to slot 0 (each a plan with
    one non-zero diagonal)."""
    w = synth.make_workload("uci")
    lay, dense, sparse = _extraction_workloads(w)
    x = lk.encode_query(lay, w.indices[0], w.dense[0])
    P = core.params_from_config(w.config)
    sk = core.sk_gen(P, w.config.seed)
    pk = core.pk_gen(P, sk, w.config.seed)
    z = np.zeros(P.n)
    z[: len(x)] = x
    ct = core.encrypt(P, pk, z, w.config.level, w.config.seed << 20)
    for wl, want in ((dense, x[: w.n_dense]), (sparse, x[w.n_dense:])):
        plan = lk.make_plan(lk.layout(wl), P.n, w.config.level)
        assert plan.n_diag == 1
        rk = core.rotkeys_gen(P, sk, plan.galois(P), w.config.seed)
        out = lk.lookup(P, plan, lk.encode_plan(P, plan), rk, [ct])
        got = core.decrypt_decode(P, sk, out[0])
        assert np.abs(got[: len(want)] - want).max() < 1e-3


def _diagonals_brute_force(W: np.ndarray, n: int):
    """D19 written out with no shortcut: every t in [0, mbar), every s in
    [0, n), W read at (o n + (s mod mbar), c n + ((s + t) mod n)), 0 outside W."""
    M, K = W.shape
    mbar = min(lk.next_pow2(M), n)
    O, C = -(-M // n), -(-K // n)
    out = {}
    s = np.arange(n)
    for o in range(O):
        for c in range(C):
            for t in range(mbar):
                rows = o * n + s % mbar
                cols = c * n + (s + t) % n
                ok = (rows < M) & (cols < K)
                v = np.zeros(n)
                v[ok] = W[rows[ok], cols[ok]]
                if np.any(v != 0):
                    out[(o, c, t)] = v
    return mbar, O, C, out


def _random_block_layout(rng, n_dense, n_blocks, n, gap=True):
    tables, I, R = [], n_dense, 0
    for _ in range(n_blocks):
        k, d = int(rng.integers(1, 40)), int(rng.integers(1, 24))
        if gap:
            I += int(rng.integers(0, 3 * n // 4))
            R += int(rng.integers(0, n // 2))
        tables.append(synth.Table(k, d, 0, rng.normal(size=(k, d)), in_off=I, out_off=R))
        I, R = I + k, R + d
    return types.SimpleNamespace(n_dense=n_dense, tables=tables)


@pytest.mark.parametrize("name", ["tiny_a", "tiny_b", "uci", "llm_gen_small", "mlp_small"])
def test_hybrid_diagonals_equal_brute_force_configs(name):
    """The planner's D19 extraction equals D19 evaluated at every (o, c, t, s)."""
    w = synth.make_workload(name)
    lay = lk.layout(w)
    n = w.config.n_slots
    got = lk.hybrid_diagonals(lay, n)
    want = _diagonals_brute_force(lk.dense_matrix(lay), n)
    assert got[:3] == want[:3] and got[3].keys() == want[3].keys()
    for k, v in want[3].items():
        assert np.array_equal(got[3][k], v)


def test_hybrid_diagonals_equal_brute_force_random_multi_ct():
    """Random block layouts with gaps: mbar < n and mbar = n with O, C > 1
    (several output and input ciphertexts, blocks straddling ct borders)."""
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.choice([16, 32, 64]))
        w = _random_block_layout(rng, int(rng.integers(0, 5)), int(rng.integers(1, 6)), n, gap=trial % 2 == 0)
        lay = lk.layout(w)
        got = lk.hybrid_diagonals(lay, n)
        want = _diagonals_brute_force(lk.dense_matrix(lay), n)
        assert got[:3] == want[:3] and got[3].keys() == want[3].keys(), trial
        for k, v in want[3].items():
            assert np.array_equal(got[3][k], v)


def test_llm_l1_layout_plan_counts():
    """The paper-exact LLM layout L1 (contiguous row-major slot
    ordering) on the Tiny ring: 64 tokens at input stride 64
    and output stride 48 -> 2 input / 2 output cts; the diagonals equal the
    brute-force D19 evaluation and the plan reproduces the dense W x."""
    w = synth.make_workload("llm_l1_small")
    lay = lk.layout(w)
    n = w.config.n_slots
    assert (lay.K, lay.M) == (64 * 64, 64 * 48)
    got = lk.hybrid_diagonals(lay, n)
    want = _diagonals_brute_force(lk.dense_matrix(lay), n)
    assert got[:3] == want[:3] == (n, 2, 2) and got[3].keys() == want[3].keys() and len(want[3]) == 1325
    plan = lk.make_plan(lay, n, w.config.level)
    x = np.random.default_rng(5).normal(size=lay.K)
    y = lk.simulate_plan_slots(plan, x, n)
    assert np.abs(y[: lay.M] - lk.dense_matrix(lay) @ x).max() < 1e-9
    # full size: 2 input / 3 output cts (m = 128 tokens x 512 slots -> 2 cts)
    lay_f = lk.layout(synth.make_workload("llm_l1"))
    assert (-(-lay_f.K // (1 << 15)), -(-lay_f.M // (1 << 15))) == (2, 3)


def test_criteo_100_ct_layout():
    """The least compressed Criteo model analog: 3,272,921 input slots -> 100
    input cts at n = 2^15 (the paper's 2,772,109 -> 85)."""
    w = synth.make_workload("criteo_c100")
    lay = lk.layout(w)
    assert lay.K == 3272921 and -(-lay.K // (1 << 15)) == 100 and lay.M == 416


def test_table1_shape_layout_and_digits():
    """The paper's Table-1 shape (p = 16, l = 32, d = 768,
    "p l = 512 slots"): 512 one-hot input slots, 768 outputs, one ct each way;
    the query has one 1 per 16-slot digit segment (32 ones, LSD first) and the
    gather is the sum of the 32 sub-table rows.  An explicit l below
    ceil(log_p k) is a layout error."""
    w = synth.make_workload("table1")
    lay = lk.layout(w)
    assert (lay.K, lay.M) == (512, 768)
    b = lay.blocks[0]
    assert (b.compressed, b.l, b.w) == (True, 32, 512)
    i = int(w.indices[0, 0])
    x = lk.encode_query(lay, w.indices[0], w.dense[0])
    digits = lk.digit_decompose(i, 16, 32)
    assert x.sum() == 32 and all(x[t * 16 + dg] == 1 for t, dg in enumerate(digits))
    assert all(dg == 0 for dg in digits[16:])              # i < 2^63 < 16^16
    y = lk.gather(lay, w.indices[0])
    assert np.allclose(y, sum(w.tables[0].weights[t * 16 + dg] for t, dg in enumerate(digits)), atol=0)
    plan = lk.make_plan(lay, 1 << 15, 19)
    assert (plan.C, plan.O, plan.mbar) == (1, 1, 1024)
    bad = types.SimpleNamespace(tables=[synth.Table(1000, 4, 4, np.zeros((16, 4)), l=4)], n_dense=0)
    with pytest.raises(ValueError, match="LAYOUT"):
        lk.layout(bad)                                      # 4^4 = 256 < 1000


def test_table1_small_lookup_decrypts_to_gather():
    """Table-1 shape on the Tiny ring (16^8 rows, base 16, 8 digits, d = 48):
    the oracle lookup decrypts to the digit gather."""
    w = synth.make_workload("table1_small")
    run = lk.run_config(w)
    assert (run.lay.K, run.lay.M, run.lay.blocks[0].l) == (128, 48, 8)
    z = core.decrypt_decode(run.P, run.sk, run.outs[0][0])
    assert np.abs(z[: run.lay.M] - lk.gather(run.lay, w.indices[0])).max() < 1e-3
