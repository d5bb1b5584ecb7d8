"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bit-exact for every integer result (NTT, keys, ciphertexts, ModUp/ModDown,
rescale, rotations, lookups); decrypted lookups within 1e-3 of the float64
gather (BASELINE.json north star).  GPU tests are marked `gpu`; the symbol
export check runs on CPU."""
import re

import numpy as np
import pytest

import synth
from oracle import core
from oracle import lookup as lk

ROOT_H = __import__("os").path.join(__import__("os").path.dirname(__file__), "..", "include", "helrm.h")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_library_exports_every_declared_symbol():
    """CPU: libhelrm.so loads and exports every function include/helrm.h declares."""
    from paper_2506_18150_b200 import helrm
    decl = set(re.findall(r"\b(helrm_[a-z0-9_]+)\s*\(", open(ROOT_H).read()))
    assert len(decl) > 30
    for name in sorted(decl):
        assert hasattr(helrm._L, name), name
    assert set(helrm.EXPORTED) <= decl


def test_host_side_matches_oracle_on_cpu():
    """CPU: primes/psi (D2/D3), table layout and the client query (S0)."""
    from paper_2506_18150_b200 import helrm
    for name in ("table1", "table1_small", "tiny_a", "tiny_b", "uci", "criteo"):
        w = synth.make_workload(name)
        P = helrm.params_from_config(w.config)
        PO = core.params_from_config(w.config)
        q, p, psi = P.moduli()
        assert q == PO.q and p == PO.p and psi == [PO.psi[x] for x in PO.q + PO.p]
        T = helrm.tables_create(P, w.tables, w.n_dense)
        lay = lk.layout(w)
        assert T.info() == (lay.K, lay.M)
        for qi in range(w.indices.shape[0]):
            x = helrm.encode_query(T, w.indices[qi], w.dense[qi], lay.K)
            assert np.array_equal(x, lk.encode_query(lay, w.indices[qi], w.dense[qi]))
    with pytest.raises(helrm.HelrmError) as e:
        helrm.encode_query(T, [10**9] * 26, [], lay.K)
    assert e.value.code == 5
    with pytest.raises(helrm.HelrmError) as e:      # explicit digit count with p^l < k
        helrm.tables_create(P, [synth.Table(1000, 4, 4, np.zeros((16, 4)), l=4)], 0)
    assert e.value.code == 6


gpu = pytest.mark.gpu


def _slot_to_natural(N):
    """Library NTT slot order -> oracle natural order (D4/D5): position s < N/2
    holds the evaluation at psi^(5^s), N/2 + s the one at psi^(-5^s)."""
    n = N // 2
    idx = np.zeros(N, dtype=np.int64)      # idx[natural i] = slot position
    e = 1
    for s in range(n):
        idx[(e - 1) // 2] = s
        idx[(2 * N - e - 1) // 2] = n + s
        e = e * 5 % (2 * N)
    return idx


@pytest.fixture(scope="module")
def torch_mod():
    if not _cuda_ok():
        pytest.skip("no CUDA device")
    import torch
    return torch


class Env:
    def __init__(self, name, torch):
        from paper_2506_18150_b200 import helrm
        self.h = helrm
        self.w = synth.make_workload(name)
        self.cfg = self.w.config
        self.PO = core.params_from_config(self.cfg)
        self.P = helrm.params_from_config(self.cfg)
        self.ctx = helrm.Context(self.P, 0, 0)
        self.torch = torch

    def dev(self, arr):
        t = self.torch.from_numpy(np.ascontiguousarray(arr, dtype=np.uint64)).cuda()
        return t

    def host(self, t):
        self.ctx.sync()
        return t.cpu().numpy()


_envs = {}


def env(name, torch):
    if name not in _envs:
        _envs[name] = Env(name, torch)
    return _envs[name]


@gpu
@pytest.mark.parametrize("name", ["tiny_a", "uci", "criteo"])
def test_ntt_matches_oracle(name, torch_mod):
    E = env(name, torch_mod)
    PO = E.PO
    primes = PO.q + PO.p
    rng = np.random.default_rng(11)
    a = np.stack([rng.integers(0, q, size=PO.N, dtype=np.uint64) for q in primes])
    # 3 polys x all limbs in one launch (several tiles and chunks)
    d = E.dev(np.concatenate([a, a, a]))
    E.h.ntt_fwd(E.ctx, d, 0, len(primes), 3)
    got = E.host(d).reshape(3, len(primes), PO.N)
    want = core.ntt(a, primes, PO)
    perm = _slot_to_natural(PO.N)
    for k in range(3):
        assert np.array_equal(got[k][:, perm], want)
    E.h.ntt_inv(E.ctx, d, 0, len(primes), 3)
    assert np.array_equal(E.host(d).reshape(3, len(primes), PO.N)[1], a)


@gpu
@pytest.mark.parametrize("name", ["tiny_a", "criteo"])
def test_ntt_extreme_inputs_match_oracle(name, torch_mod):
    """The lazy reductions of the butterflies (values kept below 4q between
    reductions, centred twiddles) on inputs of maximal magnitude: constant
    q - 1, constant (q +- 1)/2, alternating 0 / q - 1, one-hot q - 1, and
    random draws from {0, 1, (q-1)/2, (q+1)/2, q - 2, q - 1}, for the forward
    and the inverse transform against the oracle."""
    E = env(name, torch_mod)
    PO = E.PO
    primes = PO.q + PO.p
    N = PO.N
    rng = np.random.default_rng(5)
    pats = []
    for q in primes:
        q = np.uint64(q)
        alt = np.zeros(N, dtype=np.uint64)
        alt[::2] = q - np.uint64(1)
        one = np.zeros(N, dtype=np.uint64)
        one[N // 3] = q - np.uint64(1)
        pick = np.array([0, 1, (int(q) - 1) // 2, (int(q) + 1) // 2, int(q) - 2, int(q) - 1], dtype=np.uint64)
        pats.append([np.full(N, q - np.uint64(1)), np.full(N, (q - np.uint64(1)) // np.uint64(2)),
                     np.full(N, (q + np.uint64(1)) // np.uint64(2)), alt, one, pick[rng.integers(0, 6, N)]])
    n_pat = len(pats[0])
    a = np.stack([np.stack([pats[l][k] for l in range(len(primes))]) for k in range(n_pat)])   # [pat][limb][N]
    perm = _slot_to_natural(N)
    d = E.dev(a.reshape(n_pat * len(primes), N))
    E.h.ntt_fwd(E.ctx, d, 0, len(primes), n_pat)
    got = E.host(d).reshape(n_pat, len(primes), N)
    for k in range(n_pat):
        assert np.array_equal(got[k][:, perm], core.ntt(a[k], primes, PO)), k
    # inverse of the same extreme values placed in slot order (as NTT-form data)
    d = E.dev(a.reshape(n_pat * len(primes), N))
    E.h.ntt_inv(E.ctx, d, 0, len(primes), n_pat)
    got = E.host(d).reshape(n_pat, len(primes), N)
    for k in range(n_pat):
        natural = a[k][:, perm]              # the oracle's natural order of the slot-order input
        assert np.array_equal(got[k], core.intt(natural, primes, PO)), k


@gpu
@pytest.mark.parametrize("name", ["tiny_a", "uci"])
def test_keys_and_encryption_match_oracle(name, torch_mod):
    E = env(name, torch_mod)
    h, PO, cfg = E.h, E.PO, E.cfg
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    osk = core.sk_gen(PO, cfg.seed)
    opk = core.pk_gen(PO, osk, cfg.seed)
    assert np.array_equal(h.sk_export(E.ctx, sk), osk.s)
    gpk = h.pk_export(E.ctx, pk)
    assert np.array_equal(gpk[0], core.intt(opk.b, PO.q, PO)) and np.array_equal(gpk[1], core.intt(opk.a, PO.q, PO))
    gs = [core.galois_elt(3, PO), core.galois_elt(PO.n - 1, PO)]
    rk = h.rotkeys_gen(E.ctx, sk, gs, cfg.seed)
    ork = core.rotkeys_gen(PO, osk, gs, cfg.seed)
    allp = PO.q + PO.p
    for g in gs:
        got = h.rotkeys_export(E.ctx, rk, g)
        for k, (b, a) in enumerate(ork.keys[g]):
            assert np.array_equal(got[k, 0], core.intt(b, allp, PO))
            assert np.array_equal(got[k, 1], core.intt(a, allp, PO))
    z = np.random.default_rng(5).uniform(-1, 1, PO.n)
    for level in (PO.L, 1):
        ct = h.encrypt(E.ctx, pk, z, level, 1234)
        oct_ = core.encrypt(PO, opk, z, level, 1234)
        assert np.array_equal(h.ct_export(E.ctx, ct), core.ct_to_coeff(PO, oct_))
        dec = h.decrypt_decode(E.ctx, sk, ct)
        assert np.abs(dec - z).max() < 1e-3


def _rand_ct(PO, level, seed):
    rng = np.random.default_rng(seed)
    Q = PO.q[: level + 1]
    return np.stack([np.stack([rng.integers(0, q, size=PO.N, dtype=np.uint64) for q in Q]) for _ in range(2)])


@gpu
@pytest.mark.parametrize("name", ["tiny_a", "uci", "criteo"])
def test_modup_moddown_rescale_match_oracle(name, torch_mod):
    E = env(name, torch_mod)
    h, PO = E.h, E.PO
    level = PO.L - 1 if PO.L > 1 else PO.L
    coeff = _rand_ct(PO, level, 3)
    Q = PO.q[: level + 1]
    qp = PO.qp(level)
    c1_ntt = core.ntt(coeff[1], Q, PO)
    ct = h.ct_import(E.ctx, coeff, level, 2.0 ** 30)
    perm = _slot_to_natural(PO.N)
    dptr = ct.device_ptr()
    torch = E.torch
    for k in range(PO.dnum(level)):
        out = torch.zeros(len(qp) * PO.N, dtype=torch.uint64, device="cuda")
        h.modup(E.ctx, dptr + (level + 1) * PO.N * 8, level, k, out)
        got = E.host(out).reshape(len(qp), PO.N)[:, perm]
        assert np.array_equal(got, core.modup(PO, c1_ntt, level, k)), k
    y = np.stack([np.random.default_rng(4).integers(0, q, size=PO.N, dtype=np.uint64) for q in qp])
    yd = E.dev(core.intt(y, qp, PO))          # coefficient form -> library NTT
    _ntt_limbs(E, yd, level, len(qp))
    out = torch.zeros((level + 1) * PO.N, dtype=torch.uint64, device="cuda")
    h.moddown(E.ctx, yd, level, out)
    got = E.host(out).reshape(level + 1, PO.N)[:, perm]
    assert np.array_equal(got, core.moddown(PO, y, level))
    r = h.rescale(E.ctx, ct)
    oct_ = core.Ciphertext(core.ntt(coeff[0], Q, PO), c1_ntt, level, 2 ** 30)
    assert np.array_equal(h.ct_export(E.ctx, r), core.ct_to_coeff(PO, core.rescale(PO, oct_)))


def _ntt_limbs(E, d, level, nl):
    """library NTT of a Q_l P polynomial (limb i uses its chain prime)."""
    PO = E.PO
    E.h.ntt_fwd(E.ctx, d, 0, level + 1, 1)
    E.h.ntt_fwd(E.ctx, d.data_ptr() + (level + 1) * PO.N * 8, PO.L + 1, PO.K, 1)


@gpu
@pytest.mark.parametrize("name", ["tiny_a", "uci"])
def test_rotation_matches_oracle(name, torch_mod):
    E = env(name, torch_mod)
    h, PO, cfg = E.h, E.PO, E.cfg
    sk = h.sk_gen(E.ctx, cfg.seed)
    osk = core.sk_gen(PO, cfg.seed)
    ks = [1, 7, PO.n - 3]
    gs = [core.galois_elt(k, PO) for k in ks]
    rk = h.rotkeys_gen(E.ctx, sk, gs, cfg.seed)
    ork = core.rotkeys_gen(PO, osk, gs, cfg.seed)
    for level in (PO.L, 1):
        coeff = _rand_ct(PO, level, 7 + level)
        Q = PO.q[: level + 1]
        ct = h.ct_import(E.ctx, coeff, level, 1.0)
        oct_ = core.Ciphertext(core.ntt(coeff[0], Q, PO), core.ntt(coeff[1], Q, PO), level, 1)
        ring = [h.ct_alloc(E.ctx, level) for _ in ks]
        h.rotate_hoisted(E.ctx, rk, ct, ks, ring)
        for k, rct in zip(ks, ring):
            want = core.ct_to_coeff(PO, core.rotate(PO, oct_, k, ork))
            assert np.array_equal(h.ct_export(E.ctx, h.rotate(E.ctx, rk, ct, k)), want)
            assert np.array_equal(h.ct_export(E.ctx, rct), want)


def _gpu_lookup(E, w, mode=0, n1=0):
    h, cfg = E.h, w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level, n1, mode)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    info = plan.info()
    outs = []
    for q in range(w.indices.shape[0]):
        x = h.encode_query(T, w.indices[q], w.dense[q], info.n_in_cts * cfg.n_slots)
        cts = [h.encrypt(E.ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level,
                         (cfg.seed << 20) | (q * info.n_in_cts + c)) for c in range(info.n_in_cts)]
        outs.append(h.lookup(E.ctx, plan, rk, cts))
    return plan, sk, outs


@gpu
@pytest.mark.parametrize("name,mode", [("tiny_a", 0), ("tiny_b", 0), ("uci", 0), ("uci", 1), ("tiny_b", 1),
                                       ("llm_small", 0), ("llm_small", 1), ("criteo_c2_small", 0),
                                       ("llm_gen_small", 0), ("tiny_dnum7", 0), ("tiny_dnum7", 1),
                                       ("criteo_c9_small", 0), ("table1_small", 0)])
def test_lookup_bit_exact_vs_oracle(name, mode, torch_mod):
    E = env(name, torch_mod)
    w = synth.make_workload(name)
    ref = lk.run_config(w, mode=mode)
    plan, sk, outs = _gpu_lookup(E, w, mode)
    info = plan.info()
    assert (info.n_diag, info.n_unique, info.n1, info.mbar) == (ref.plan.n_diag, len(ref.plan.u_slots),
                                                                ref.plan.n1, ref.plan.mbar)
    assert plan.rotations() == ref.plan.rotation_amounts(ref.P)
    assert len(outs[0]) == info.n_out_cts == ref.plan.O
    for got_ct, want_ct in zip(outs[0], ref.outs[0]):
        assert np.array_equal(E.h.ct_export(E.ctx, got_ct), core.ct_to_coeff(ref.P, want_ct))
    z = np.concatenate([E.h.decrypt_decode(E.ctx, sk, o) for o in outs[0]])
    y = lk.gather(ref.lay, w.indices[0])
    assert np.abs(z[: ref.lay.M] - y).max() < 1e-3


@gpu
def test_criteo_full_size_matches_oracle_golden(torch_mod):
    """Criteo-shaped lookup at full size (N = 2^16, 24 + 4 primes, 512
    diagonals, 52 rotation keys) against digests of the oracle's own outputs
    (tests/golden/criteo.json, written by tests/golden/make_golden.py from
    oracle/ only): rotation key, encrypted query, output ciphertext; plus the
    decrypted output against the float64 gather."""
    import hashlib
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "criteo.json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()
    E = env("criteo", torch_mod)
    w = synth.make_workload("criteo")
    plan, sk, outs = _gpu_lookup(E, w)
    info = plan.info()
    assert (info.n_diag, info.n1, info.n2_max, info.n_rotations) == (512, 32, 16, 52)
    # rotation key of the first Galois element, digit by digit
    T = E.h.tables_create(E.P, w.tables, w.n_dense)
    rk = E.h.rotkeys_gen(E.ctx, sk, [gold["rotkey_g0"]], w.config.seed)
    kk = E.h.rotkeys_export(E.ctx, rk, gold["rotkey_g0"])
    assert [sha(kk[k]) for k in range(kk.shape[0])] == gold["rotkey_g0_sha"]
    q0 = gold["queries"][0]
    pk = E.h.pk_gen(E.ctx, sk, w.config.seed)
    x = E.h.encode_query(T, w.indices[0], w.dense[0], w.config.n_slots)
    ct = E.h.encrypt(E.ctx, pk, x, w.config.level, (w.config.seed << 20) | 0)
    assert sha(E.h.ct_export(E.ctx, ct)) == q0["in_sha"][0]
    assert sha(E.h.ct_export(E.ctx, outs[0][0])) == q0["out_sha"][0]
    z = E.h.decrypt_decode(E.ctx, sk, outs[0][0])
    lay = lk.layout(w)
    y = lk.gather(lay, w.indices[0])
    assert np.abs(z[: lay.M] - y).max() < 1e-3
    # slot s holds y[s mod mbar] in every period (RotSum, R20)
    zz = z.reshape(-1, info.mbar)
    assert np.abs(zz[:, : lay.M] - y).max() < 1e-3


def _golden_outputs(E, name, outs):
    """The output ciphertexts of query 0 against the SHA-256 digests the CPU
    oracle wrote for this config (tests/golden/<name>.json, written by
    tests/golden/make_golden.py from oracle/ only)."""
    import hashlib
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", name + ".json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()
    want = gold["queries"][0]["out_sha"]
    assert len(outs) == len(want)
    for o, h in zip(outs, want):
        assert sha(E.h.ct_export(E.ctx, o)) == h
    return gold


@gpu
def test_llm_full_size_plan_and_decryption(torch_mod):
    """LLM-style config at full size (N = 2^16, 20 + 4 primes, 128 tokens of
    the 50257 x 768 table, layout L2): the plan's counts (1279 distinct
    diagonals shared by the 4 blocks, n1 = 64, n2 = 20, 82 rotation keys --
    63 babies + 20 giants, giant 12 being amount 1 = baby 1 (SURVEY.md 8.0
    counts 83 by not merging it; tests/test_oracle_lookup.py re-derives 82 on
    the oracle's plan) -- 4 in / 4 out cts) and every decrypted output block against
    the float64 gather, and all four output ciphertexts against the oracle's
    digests (tests/golden/llm.json: the oracle run at full size, 20 + 4
    primes, dnum 5, offline)."""
    E = env("llm", torch_mod)
    w = synth.make_workload("llm")
    plan, sk, outs = _gpu_lookup(E, w)
    info = plan.info()
    assert (info.n_in_cts, info.n_out_cts, info.n_unique, info.n1, info.n2_max, info.n_rotations) == (4, 4, 1279, 64,
                                                                                                      20, 82)
    assert info.mbar == w.config.n_slots and info.n_diag == 4 * 1279
    _golden_outputs(E, "llm", outs[0])
    lay = lk.layout(w)
    y = lk.gather(lay, w.indices[0])
    z = np.concatenate([E.h.decrypt_decode(E.ctx, sk, o) for o in outs[0]])
    assert np.abs(z[: lay.M] - y).max() < 1e-3


@gpu
def test_criteo_c2_full_size_plan_and_decryption(torch_mod):
    """The 2-input-ct Criteo shape at full size (Table 2 threshold
    5e4: 47,798 one-hot slots, 1024 diagonals, giants shared by both cts):
    plan counts, the output against the oracle's digest (tests/golden/
    criteo_c2.json) and the decrypted output against the float64 gather."""
    E = env("criteo_c2", torch_mod)
    w = synth.make_workload("criteo_c2")
    plan, sk, outs = _gpu_lookup(E, w)
    info = plan.info()
    assert (info.n_in_cts, info.n_out_cts, info.n_diag, info.n1, info.n2_max, info.n_rotations) == (2, 1, 1024, 32,
                                                                                                    16, 52)
    _golden_outputs(E, "criteo_c2", outs[0])
    lay = lk.layout(w)
    y = lk.gather(lay, w.indices[0])
    z = E.h.decrypt_decode(E.ctx, sk, outs[0][0])
    assert np.abs(z[: lay.M] - y).max() < 1e-3


@gpu
def test_llm_gen_full_size_decryption(torch_mod):
    """LLM generation step at full size (one token of the 50257 x 768 GPT-2
    table): plan counts, the output against the oracle's digest
    (tests/golden/llm_gen.json) and the decrypted 768-dim embedding against
    the float64 gather."""
    E = env("llm", torch_mod)
    w = synth.make_workload("llm_gen")
    plan, sk, outs = _gpu_lookup(E, w)
    info = plan.info()
    assert (info.n_in_cts, info.n_out_cts, info.n_diag, info.n1, info.n2_max, info.n_rotations, info.mbar) == (
        1, 1, 1024, 32, 32, 67, 1024)
    _golden_outputs(E, "llm_gen", outs[0])
    lay = lk.layout(w)
    z = E.h.decrypt_decode(E.ctx, sk, outs[0][0])
    assert np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max() < 1e-3


@gpu
def test_table1_shape_full_size(torch_mod):
    """The paper's Table-1 shape at full size (GPT-2 d = 768,
    p = 16, l = 32 -> 512 one-hot slots, one ct in and out) on the LLM ring:
    plan counts and the decrypted output against the 32-digit gather."""
    E = env("llm", torch_mod)
    h, w = E.h, synth.make_workload("table1")
    cfg = w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level)
    info = plan.info()
    assert (info.K, info.M, info.n_in_cts, info.n_out_cts, info.mbar) == (512, 768, 1, 1, 1024)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(), cfg.seed)
    x = h.encode_query(T, w.indices[0], w.dense[0], cfg.n_slots)
    assert x.sum() == 32
    ct = h.encrypt(E.ctx, pk, x, cfg.level, cfg.seed << 20)
    out = h.lookup(E.ctx, plan, rk, [ct])
    lay = lk.layout(w)
    z = h.decrypt_decode(E.ctx, sk, out[0])
    assert np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max() < 1e-3


@gpu
def test_criteo_level4_decryption(torch_mod):
    """The Criteo lookup at input level 4, where Orion places the embedding in
    the ReLU DLRM: 5 + 4 limbs, dnum 2; the plan counts match
    the level-23 plan, the output equals the oracle's digest
    (tests/golden/criteo_l4.json) and decrypts to the float64 gather."""
    E = env("criteo", torch_mod)
    w = synth.make_workload("criteo_l4")
    plan, sk, outs = _gpu_lookup(E, w)
    info = plan.info()
    assert (info.n_diag, info.n1, info.n2_max, info.n_rotations) == (512, 32, 16, 52)
    _golden_outputs(E, "criteo_l4", outs[0])
    lay = lk.layout(w)
    z = E.h.decrypt_decode(E.ctx, sk, outs[0][0])
    assert np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max() < 1e-3


@gpu
def test_dense_sparse_extraction_matches_oracle(torch_mod):
    """PAPER.md:654 dense/sparse extraction as single-diagonal plans on the
    engine (tests/test_oracle_lookup.py builds them): the GPU outputs equal the
    oracle's bit for bit and decrypt to the two parts of the query vector."""
    import test_oracle_lookup as tol
    E = env("uci", torch_mod)
    w = synth.make_workload("uci")
    lay, dense, sparse = tol._extraction_workloads(w)
    h, cfg = E.h, w.config
    x = lk.encode_query(lay, w.indices[0], w.dense[0])
    P = core.params_from_config(cfg)
    sk_ref = core.sk_gen(P, cfg.seed)
    pk_ref = core.pk_gen(P, sk_ref, cfg.seed)
    z = np.zeros(P.n)
    z[: len(x)] = x
    ct_ref = core.encrypt(P, pk_ref, z, cfg.level, cfg.seed << 20)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    ct = h.encrypt(E.ctx, pk, z, cfg.level, cfg.seed << 20)
    for wl, want in ((dense, x[: w.n_dense]), (sparse, x[w.n_dense:])):
        T = h.tables_create(E.P, wl.tables, wl.n_dense)
        plan = h.plan_create(E.ctx, T, cfg.level)
        assert plan.info().n_diag == 1
        rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
        out = h.lookup(E.ctx, plan, rk, [ct])
        ref_plan = lk.make_plan(lk.layout(wl), P.n, cfg.level)
        rk_ref = core.rotkeys_gen(P, sk_ref, ref_plan.galois(P), cfg.seed)
        ref = lk.lookup(P, ref_plan, lk.encode_plan(P, ref_plan), rk_ref, [ct_ref])
        assert np.array_equal(h.ct_export(E.ctx, out[0]), core.ct_to_coeff(P, ref[0]))
        got = h.decrypt_decode(E.ctx, sk, out[0])
        assert np.abs(got[: len(want)] - want).max() < 1e-3


@gpu
@pytest.mark.parametrize("name", ["mlp_small", "mlp_512x256"])
def test_dense_linear_layer(name, torch_mod):
    """A dense linear layer on the lookup engine: the weight
    matrix as the table, a dense encrypted input.  mlp_small: the output
    ciphertext equals the oracle's bit for bit; mlp_512x256: equals the
    oracle's digest (tests/golden/mlp_512x256.json); both: decrypts to x W."""
    E = env(name, torch_mod)
    w = synth.make_workload(name)
    x = synth.dense_inputs(name)[0]
    cfg, h = w.config, E.h
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    z = np.zeros(cfg.n_slots)
    z[: len(x)] = x
    ct = h.encrypt(E.ctx, pk, z, cfg.level, cfg.seed << 20)
    out = h.lookup(E.ctx, plan, rk, [ct])
    want = x @ w.tables[0].weights
    y = h.decrypt_decode(E.ctx, sk, out[0])
    assert np.abs(y[: len(want)] - want).max() < 1e-3
    if name == "mlp_512x256":
        _golden_outputs(E, name, out)
    if name == "mlp_small":
        import test_oracle_lookup as tol
        _, _, P, _, _, _, ref = tol._dense_layer_run(name)
        assert np.array_equal(h.ct_export(E.ctx, out[0]), core.ct_to_coeff(P, ref[0]))


@gpu
@pytest.mark.parametrize("name", ["uci", "llm_small", "criteo_c2_small", "llm_gen_small", "tiny_dnum7"])
def test_lookup_dist_single_rank_matches_lookup(name, torch_mod):
    """helrm_lookup_dist on a 1-rank NCCL communicator (the only GPU a gpurun
    box has) runs the partitioned code path (broadcast, partial accumulators,
    finish) and must equal helrm_lookup bit for bit; the 2-rank split itself
    is covered on CPU by tests/test_dist_cpu.py."""
    E = env(name, torch_mod)
    h, cfg = E.h, E.cfg
    w = synth.make_workload(name)
    plan, sk, outs = _gpu_lookup(E, w)
    h.comm_init(E.ctx, h.comm_unique_id(), 0, 1)
    T = h.tables_create(E.P, w.tables, w.n_dense)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    info = plan.info()
    x = h.encode_query(T, w.indices[0], w.dense[0], info.n_in_cts * cfg.n_slots)
    cts = [h.encrypt(E.ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level,
                     (cfg.seed << 20) | c) for c in range(info.n_in_cts)]
    for _ in range(3):   # eager, graph capture, graph replay
        got = h.lookup_dist(E.ctx, plan, rk, cts)
        for a, b in zip(got, outs[0]):
            assert np.array_equal(h.ct_export(E.ctx, a), h.ct_export(E.ctx, b))


def _encrypt_batch(E, w, T, pk, info):
    h, cfg = E.h, w.config
    cts = []
    for q in range(w.indices.shape[0]):
        x = h.encode_query(T, w.indices[q], w.dense[q], info.n_in_cts * cfg.n_slots)
        cts += [h.encrypt(E.ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level,
                          (cfg.seed << 20) | (q * info.n_in_cts + c)) for c in range(info.n_in_cts)]
    return cts


@gpu
@pytest.mark.parametrize("name,batch", [("tiny_b", 3), ("uci", 3), ("llm_small", 2), ("criteo_c2_small", 2),
                                        ("tiny_dnum7", 3), ("llm_gen_small", 3)])
def test_batched_lookup_bit_exact_vs_oracle(name, batch, torch_mod):
    """One helrm_lookup call over `batch` queries (the query-batched engine:
    shared key and plaintext reads, query loops inside the key-switch and MAC
    kernels, batched ModUp/ModDown/rescale/RotSum) against the oracle's
    per-query lookups, every output ciphertext bit for bit."""
    E = env(name, torch_mod)
    w = synth.make_workload(name, batch=batch)
    ref = lk.run_config(w)
    h, cfg = E.h, w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    info = plan.info()
    cts = _encrypt_batch(E, w, T, pk, info)
    outs = h.lookup(E.ctx, plan, rk, cts, batch)
    assert len(outs) == batch * info.n_out_cts
    for q in range(batch):
        for o in range(info.n_out_cts):
            got = h.ct_export(E.ctx, outs[q * info.n_out_cts + o])
            assert np.array_equal(got, core.ct_to_coeff(ref.P, ref.outs[q][o])), (q, o)


@gpu
def test_criteo_batched_equals_single(torch_mod):
    """Criteo full size, 3 queries in one call (query chunk forced to 2 so a
    full chunk and a ragged one both run): every output equals the batch-1
    lookup of the same ciphertext bit for bit, and query 0 matches the
    oracle's golden digest."""
    import hashlib
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "criteo.json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()
    E = env("criteo", torch_mod)
    w = synth.make_workload("criteo", batch=3)
    h, cfg = E.h, w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    info = plan.info()
    cts = _encrypt_batch(E, w, T, pk, info)
    os.environ["HELRM_QCHUNK"] = "2"
    try:
        outs = h.lookup(E.ctx, plan, rk, cts, 3)
    finally:
        del os.environ["HELRM_QCHUNK"]
    assert sha(h.ct_export(E.ctx, outs[0])) == gold["queries"][0]["out_sha"][0]
    for q in range(3):
        single = h.lookup(E.ctx, plan, rk, [cts[q]])[0]
        assert np.array_equal(h.ct_export(E.ctx, outs[q]), h.ct_export(E.ctx, single)), q


@gpu
@pytest.mark.parametrize("name", ["uci", "llm_small", "criteo_c2_small", "llm_gen_small"])
def test_lookup_host_matches_lookup(name, torch_mod):
    """helrm_lookup_host (host coefficient-form buffers, copies pipelined
    against the lookups, CUDA-graph replay from the second query) equals
    ct_import -> helrm_lookup -> ct_export bit for bit, for 3 queries."""
    E = env(name, torch_mod)
    w = synth.make_workload(name, batch=3)
    h, cfg = E.h, w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    info = plan.info()
    cts = _encrypt_batch(E, w, T, pk, info)
    ins = [np.ascontiguousarray(h.ct_export(E.ctx, ct).reshape(-1)) for ct in cts]
    outs = [np.zeros(2 * cfg.level * cfg.N, dtype=np.uint64) for _ in range(3 * info.n_out_cts)]
    h.lookup_host(E.ctx, plan, rk, ins, 2.0 ** cfg.log_scale, 3, outs)
    for q in range(3):
        want = h.lookup(E.ctx, plan, rk, cts[q * info.n_in_cts:(q + 1) * info.n_in_cts])
        for o in range(info.n_out_cts):
            assert np.array_equal(outs[q * info.n_out_cts + o], h.ct_export(E.ctx, want[o]).reshape(-1)), (q, o)


@gpu
def test_microbench_ntt_full_size_sampled(torch_mod):
    """configs[4] at full size in the launch configuration bench.py times:
    1024 ciphertexts x 2 x 24 limbs at N = 2^16 (49,152 limb transforms, 24
    GiB) through helrm_ntt_fwd / helrm_ntt_inv; sampled limbs against the
    oracle's NTT (first, middle, last chunk), and the inverse restores them."""
    torch = torch_mod
    E = env("criteo", torch)
    PO = E.PO
    L1 = PO.L + 1
    n_polys = 2 * 1024
    g = torch.Generator(device="cuda").manual_seed(99)
    # residues below the smallest prime of the chain (uniform enough for a transform check)
    qmin = min(PO.q)
    buf = torch.randint(0, qmin, (n_polys * L1 * PO.N,), dtype=torch.int64, device="cuda", generator=g)
    picks = [0, 7, n_polys * L1 // 2 + 3, n_polys * L1 - 1]          # global limb indices
    before = {i: buf[i * PO.N:(i + 1) * PO.N].cpu().numpy().astype(np.uint64) for i in picks}
    ptr = buf.data_ptr()
    E.h.ntt_fwd(E.ctx, ptr, 0, L1, n_polys)
    E.ctx.sync()
    perm = _slot_to_natural(PO.N)
    for i in picks:
        q = PO.q[i % L1]
        got = buf[i * PO.N:(i + 1) * PO.N].cpu().numpy().astype(np.uint64)[perm]
        want = core.ntt(before[i][None, :], [q], PO)[0]
        assert np.array_equal(got, want), i
    E.h.ntt_inv(E.ctx, ptr, 0, L1, n_polys)
    E.ctx.sync()
    for i in picks:
        assert np.array_equal(buf[i * PO.N:(i + 1) * PO.N].cpu().numpy().astype(np.uint64), before[i]), i
    del buf
    torch.cuda.empty_cache()


@gpu
def test_criteo_hoisted_rotations_sampled(torch_mod):
    """configs[4] hoisted rotations at Criteo size: one ModUp, amounts 1..64
    written to a ring (the bench's helrm_rotate_hoisted call), sampled
    amounts bit-exact against the oracle's Rotate with the same keys."""
    E = env("criteo", torch_mod)
    h, PO, cfg = E.h, E.PO, E.cfg
    sk = h.sk_gen(E.ctx, cfg.seed)
    osk = core.sk_gen(PO, cfg.seed)
    amounts = list(range(1, 65))
    check = [1, 37, 64]
    rk = h.rotkeys_gen(E.ctx, sk, sorted({core.galois_elt(a, PO) for a in amounts}), cfg.seed)
    ork = core.rotkeys_gen(PO, osk, [core.galois_elt(a, PO) for a in check], cfg.seed)
    level = PO.L
    coeff = _rand_ct(PO, level, 21)
    Q = PO.q[: level + 1]
    ct = h.ct_import(E.ctx, coeff, level, 1.0)
    ring = [h.ct_alloc(E.ctx, level) for _ in amounts]
    h.rotate_hoisted(E.ctx, rk, ct, amounts, ring)
    oct_ = core.Ciphertext(core.ntt(coeff[0], Q, PO), core.ntt(coeff[1], Q, PO), level, 1)
    for a in check:
        want = core.ct_to_coeff(PO, core.rotate(PO, oct_, a, ork))
        assert np.array_equal(h.ct_export(E.ctx, ring[a - 1]), want), a


@gpu
def test_criteo_batch64_sampled(torch_mod):
    """configs[2] batch 64 in the bench's configuration (one helrm_lookup
    call, default query chunking): sampled queries equal the batch-1 lookups
    of the same ciphertexts (which tests/golden pins against the oracle)."""
    E = env("criteo", torch_mod)
    w = synth.make_workload("criteo", batch=4)
    h, cfg = E.h, w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    cts = _encrypt_batch(E, w, T, pk, plan.info())
    batch = [cts[i % 4] for i in range(64)]
    outs = h.lookup(E.ctx, plan, rk, batch, 64)
    for q in (0, 17, 42, 63):
        single = h.lookup(E.ctx, plan, rk, [cts[q % 4]])[0]
        assert np.array_equal(h.ct_export(E.ctx, outs[q]), h.ct_export(E.ctx, single)), q


@gpu
def test_lookup_error_and_degenerate_cases(torch_mod):
    """Empty batch (no work, no outputs), an input at the wrong level (LEVEL),
    a key set missing a rotation (LAYOUT), the serving call on a
    single-hoisted plan (ARG)."""
    E = env("tiny_b", torch_mod)
    w = synth.make_workload("tiny_b")
    h, cfg = E.h, w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N), cfg.seed)
    assert h.lookup(E.ctx, plan, rk, [], 0) == []
    x = h.encode_query(T, w.indices[0], w.dense[0], cfg.n_slots)
    low = h.encrypt(E.ctx, pk, x, cfg.level - 1, 5)
    with pytest.raises(h.HelrmError) as e:
        h.lookup(E.ctx, plan, rk, [low])
    assert e.value.code == 3
    ct = h.encrypt(E.ctx, pk, x, cfg.level, 5)
    partial = h.rotkeys_gen(E.ctx, sk, plan.galois(cfg.N)[:1], cfg.seed)
    with pytest.raises(h.HelrmError) as e:
        h.lookup(E.ctx, plan, partial, [ct])
    assert e.value.code == 6
    splan = h.plan_create(E.ctx, T, cfg.level, 0, 1)
    coeff = np.ascontiguousarray(h.ct_export(E.ctx, ct).reshape(-1))
    out = np.zeros(2 * (cfg.level) * cfg.N, dtype=np.uint64)
    with pytest.raises(h.HelrmError) as e:
        h.lookup_host(E.ctx, splan, rk, [coeff], 1.0, 1, [out])
    assert e.value.code == 10


@gpu
@pytest.mark.parametrize("knobs,test", [
    ({"HELRM_MAC_BULK": "0"}, "test_criteo_full_size_matches_oracle_golden"),      # register-fed MAC
    ({"HELRM_MAC_BULK": "0"}, "test_batched_lookup_bit_exact_vs_oracle"),
    ({"HELRM_MAC_BULK": "0"}, "test_llm_full_size_plan_and_decryption"),
    ({"HELRM_PIPE": "1", "HELRM_MACCH": "1", "HELRM_NTTCH": "4"},                  # pipelined giant steps
     "test_criteo_full_size_matches_oracle_golden"),
    ({"HELRM_PDL": "1"}, "test_criteo_full_size_matches_oracle_golden"),          # programmatic dependent launch
    ({"HELRM_PDL": "1"}, "test_lookup_bit_exact_vs_oracle"),
])
def test_parity_under_engine_knobs(knobs, test):
    """Parity tests in a fresh process with alternative engine paths switched
    on (the knobs are read once per process): the register-fed MAC kernels
    (k_diag_mac1 / k_diag_mac; the default is the bulk-copy kernel,
    kernels_mac_bulk.cu) and the stream-pipelined giant steps must give the
    same bit-exact outputs."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, **knobs)
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_parity.py") + "::" + test],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
