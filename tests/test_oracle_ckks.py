"""Pins of the oracle's CKKS layer (D8, D11-D18): big-integer definitions of
ModUp / ModDown / rescale evaluated with Python integers, algebraic
invariants of automorphisms, decryption of key-switched ciphertexts, and the
exact identities that make hoisting bit-exact.  CPU only."""
import math

import numpy as np
import pytest

import synth
from oracle import core


@pytest.fixture(scope="module")
def tiny():
    P = core.params_from_config(synth.config_by_name("tiny_a"))
    sk = core.sk_gen(P, 1)
    pk = core.pk_gen(P, sk, 1)
    return P, sk, pk


@pytest.fixture(scope="module")
def uci():
    P = core.params_from_config(synth.config_by_name("uci"))
    sk = core.sk_gen(P, 1)
    pk = core.pk_gen(P, sk, 1)
    return P, sk, pk


def _rand_poly(P, primes, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, q, size=P.N, dtype=np.uint64) for q in primes])


def _crt(col, primes):
    Q = math.prod(primes)
    return sum(int(v) * (Q // q) * pow(Q // q, -1, q) for v, q in zip(col, primes)) % Q


def test_sizes_match_paper_formula():
    """a polynomial is N (L+1) 8 bytes -> 12,582,912 B for the
    Criteo ring (N = 2^16, 24 limbs); a rotation key is dnum 2 (L+1+K) N 8 B
    = 168 MiB, the paper's "~200 MB each"."""
    P = core.params_from_config(synth.config_by_name("criteo"))
    assert P.N * (P.L + 1) * 8 == 12_582_912
    key = P.dnum(P.L) * 2 * (P.L + 1 + P.K) * P.N * 8
    assert key == 168 * 2**20 and 150e6 < key < 250e6
    assert P.dnum(P.L) == 6


def test_encrypt_decrypt_roundtrip(tiny, uci):
    for P, sk, pk in (tiny, uci):
        z = np.random.default_rng(2).uniform(-1, 1, P.n)
        ct = core.encrypt(P, pk, z, P.L, 99)
        err = np.abs(core.decrypt_decode(P, sk, ct) - z).max()
        # fresh noise: |e0 + e1 s + v e| <~ 6 sigma sqrt(N) (..) / Delta
        bound = 6 * 3.2 * math.sqrt(P.N) * math.sqrt(2 * P.N / 3) * 2 / P.scale
        assert err < bound, (err, bound)


def test_automorphism_invariants(tiny):
    P, sk, pk = tiny
    Q = P.q
    a = _rand_poly(P, Q, 1)
    g, h = core.galois_elt(3, P), core.galois_elt(11, P)
    # phi_g phi_h = phi_{gh}; phi_{5^{N/2}} = id
    assert np.array_equal(core.automorph_coeff(core.automorph_coeff(a, h, Q, P.N), g, Q, P.N),
                          core.automorph_coeff(a, g * h % (2 * P.N), Q, P.N))
    assert pow(5, P.n, 2 * P.N) == 1
    assert np.array_equal(core.automorph_coeff(a, pow(5, P.n, 2 * P.N), Q, P.N), a)
    # coefficient-form and NTT-form application agree
    lhs = core.ntt(core.automorph_coeff(a, g, Q, P.N), Q, P)
    rhs = core.automorph_ntt(core.ntt(a, Q, P), g, P.N)
    assert np.array_equal(lhs, rhs)
    # -1 (conjugation) is also an automorphism and fixes the real encodings
    assert np.array_equal(core.ntt(core.automorph_coeff(a, 2 * P.N - 1, Q, P.N), Q, P),
                          core.automorph_ntt(core.ntt(a, Q, P), 2 * P.N - 1, P.N))


@pytest.mark.parametrize("k", [0, 1, 2])
def test_modup_bigint(uci, k):
    """D15: the integer represented by ModUp_k(c) over Q_l P is x + u Q_k with
    x = [c]_{Q_k} in [0, Q_k) and 0 <= u < |digit k| (the alpha-bounded
    overflow of the uncorrected fast base conversion)."""
    P, sk, pk = uci
    l = 6                                       # not the top level: exercises key slicing too
    Q = P.q[: l + 1]
    c = _rand_poly(P, Q, 10 + k)
    out = core.intt(core.modup(P, c, l, k), P.qp(l), P)
    cc = core.intt(c, Q, P)
    dig = P.digit(l, k)
    Qk = math.prod(P.q[i] for i in dig)
    for i in range(0, P.N, P.N // 16):
        x = _crt([cc[r, i] for r in dig], [P.q[r] for r in dig])
        y = _crt(out[:, i], P.qp(l))
        u, rem = divmod(y - x, Qk)
        assert rem == 0 and 0 <= u < len(dig)
    assert np.array_equal(core.modup(P, c, l, k)[dig], c[dig])


def test_moddown_bigint(uci):
    """D16: ModDown(y) = floor(Y / P) - u (mod Q_l), 0 <= u < K, Y the CRT lift over Q_l P."""
    P, sk, pk = uci
    l = 5
    y = _rand_poly(P, P.qp(l), 3)
    x = core.intt(core.moddown(P, y, l), P.q[: l + 1], P)
    yc = core.intt(y, P.qp(l), P)
    Ql = math.prod(P.q[: l + 1])
    for i in range(0, P.N, P.N // 16):
        Y = _crt(yc[:, i], P.qp(l))
        X = _crt(x[:, i], P.q[: l + 1])
        assert (Y // P.P - X) % Ql < P.K


def test_rescale_bigint(uci):
    """D17: rescale gives exactly round(X / q_l) mod Q_{l-1}; scale / q_l."""
    P, sk, pk = uci
    l = 7
    Q = P.q[: l + 1]
    ct = core.Ciphertext(_rand_poly(P, Q, 4), _rand_poly(P, Q, 5), l, 1 << 36)
    r = core.rescale(P, ct)
    assert r.level == l - 1 and r.scale * Q[l] == 1 << 36
    for src, dst in ((ct.c0, r.c0), (ct.c1, r.c1)):
        xc = core.intt(src, Q, P)
        yc = core.intt(dst, Q[:l], P)
        for i in range(0, P.N, P.N // 16):
            X = _crt(xc[:, i], Q)
            want = (2 * X + Q[l]) // (2 * Q[l])      # round half up; q_l odd: no ties
            assert _crt(yc[:, i], Q[:l]) == want % math.prod(Q[:l])


def test_moddown_of_lift_is_identity(uci):
    """ModDown(P x + y) = x + ModDown(y) exactly (why RotateLazy + ModDown = Rotate)."""
    P, sk, pk = uci
    l = 7
    x = _rand_poly(P, P.q[: l + 1], 6)
    y = _rand_poly(P, P.qp(l), 7)
    lhs = core.moddown(P, core.vadd(core.lift_P(P, x, l), y, P.qp(l)), l)
    rhs = core.vadd(x, core.moddown(P, y, l), P.q[: l + 1])
    assert np.array_equal(lhs, rhs)


@pytest.mark.parametrize("cfg", ["tiny", "uci"])
def test_rotation_decrypts_and_hoisting_is_bit_exact(cfg, tiny, uci):
    P, sk, pk = tiny if cfg == "tiny" else uci
    ks = [1, 5, P.n // 2]
    rk = core.rotkeys_gen(P, sk, [core.galois_elt(k, P) for k in ks], 7)
    z = np.random.default_rng(8).uniform(-1, 1, P.n)
    ct = core.encrypt(P, pk, z, P.L, 5)
    D = [core.modup(P, ct.c1, P.L, k) for k in range(P.dnum(P.L))]
    for k in ks:
        r = core.rotate(P, ct, k, rk)
        got = core.decrypt_decode(P, sk, r)
        assert np.abs(got - np.roll(z, -k)).max() < 1e-3     # rot_k: new slot j = old slot j + k
        # hoisted (shared ModUp) == unhoisted, and ModDown(RotateLazy) == Rotate, bit for bit
        rh = core.rotate(P, ct, k, rk, D=D)
        assert np.array_equal(r.c0, rh.c0) and np.array_equal(r.c1, rh.c1)
        a, b = core.rotate_lazy(P, ct, k, rk, D=D)
        assert np.array_equal(core.moddown(P, a, P.L), r.c0) and np.array_equal(core.moddown(P, b, P.L), r.c1)
    assert core.rotate(P, ct, 0, rk) is ct


def test_rotation_at_lower_level_uses_key_slices(uci):
    """Keys are generated at level L and sliced (limbs q_0..q_l, all p, digits < dnum(l))."""
    P, sk, pk = uci
    rk = core.rotkeys_gen(P, sk, [core.galois_elt(3, P)], 7)
    z = np.random.default_rng(9).uniform(-1, 1, P.n)
    ct = core.encrypt(P, pk, z, 4, 6)
    assert P.dnum(4) == 3
    r = core.rotate(P, ct, 3, rk)
    assert np.abs(core.decrypt_decode(P, sk, r) - np.roll(z, -3)).max() < 1e-3


def test_conv_does_not_commute_with_negation():
    """Why D18 fixes "ModUp, then automorphism": Conv(-x) != -Conv(x)."""
    B, t = [1048193, 1047809], 1046017
    rng = np.random.default_rng(0)
    x = np.stack([rng.integers(1, b, size=200, dtype=np.uint64) for b in B])
    negx = np.stack([(np.uint64(b) - x[i]) % np.uint64(b) for i, b in enumerate(B)])
    c1 = core.conv(x, B, [t])[0]
    c2 = core.conv(negx, B, [t])[0]
    assert np.mean((c1 + c2) % np.uint64(t) != 0) > 0.9
