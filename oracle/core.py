"""oracle.core -- TEST INFRASTRUCTURE (parity oracle), see oracle/__init__.py.

RNS-CKKS primitives D1-D18 of SURVEY.md section 8(c), one function per
definition, in the order and notation of that section.  The paper's own text
for each is cited; the paper is silent on every ring-level convention
(SURVEY.md R1-R10), so the D-numbered readings are the specification.

Representation: a polynomial over an RNS basis is a uint64 numpy array of
shape (n_limbs, N) with residues in [0, q); `primes` lists the modulus of each
row.  Ciphertexts are kept in NTT form, natural order (D4).  The hot loops
(NTT, modular products, base conversion, encoding) run in oracle/ckks_ref.c,
scalar `unsigned __int128 % q`; limbs are independent, so they are farmed out
to a thread pool (ctypes releases the GIL) -- this changes no arithmetic.
"""
from __future__ import annotations

import concurrent.futures
import ctypes
import math
import os
import subprocess
import threading
from fractions import Fraction
from typing import Dict, List, Optional, Sequence

import numpy as np

__all__ = [
    "lib", "set_threads", "threads", "is_prime", "find_primes", "min_psi", "Params", "params_from_config",
    "ntt", "intt", "ntt_direct", "vmul", "vadd", "vsub", "vneg", "vscalar", "reduce_signed",
    "prng_word", "stream", "sample_uniform", "sample_ternary", "sample_gauss", "gauss_cdt",
    "encode", "decode", "crt_centered", "automorph_ntt", "automorph_coeff", "galois_elt",
    "SecretKey", "PublicKey", "RotKeys", "Ciphertext", "sk_gen", "pk_gen", "rotkeys_gen", "encrypt",
    "decrypt", "decrypt_decode", "conv", "modup", "moddown", "rescale", "lift_P", "keyswitch",
    "rotate_lazy", "rotate", "ct_to_coeff",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ckks_ref.c")
_SO = os.path.join(_HERE, "libckks_ref.so")
_LIB = None
_LOCK = threading.Lock()


def build_lib() -> str:
    """Compile oracle/ckks_ref.c (plain gcc, -O2) if the .so is missing/stale."""
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-o", _SO, _SRC, "-lquadmath", "-lm"])
    return _SO


def lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            L = ctypes.CDLL(build_lib())
            u64p = ctypes.POINTER(ctypes.c_uint64)
            i64p = ctypes.POINTER(ctypes.c_int64)
            dp = ctypes.POINTER(ctypes.c_double)
            sz, u64 = ctypes.c_size_t, ctypes.c_uint64
            L.or_ntt.argtypes = [u64p, sz, u64, u64]
            L.or_intt.argtypes = [u64p, sz, u64, u64]
            L.or_ntt_direct.argtypes = [u64p, u64p, sz, u64, u64]
            L.or_vec_mulmod.argtypes = [u64p, u64p, u64p, sz, u64]
            L.or_vec_mac.argtypes = [u64p, u64p, u64p, sz, u64]
            L.or_vec_scalar.argtypes = [u64p, u64, u64p, sz, u64]
            L.or_conv.argtypes = [u64p, sz, u64p, u64p, u64p, sz, u64p, u64p, sz]
            L.or_prng_word.argtypes = [u64, u64, u64]
            L.or_prng_word.restype = u64
            L.or_sample_uniform.argtypes = [u64, u64, u64, sz, u64p]
            L.or_sample_ternary.argtypes = [u64, u64, sz, i64p]
            L.or_sample_gauss.argtypes = [u64, u64, sz, u64p, i64p]
            L.or_encode.argtypes = [dp, sz, ctypes.c_double, i64p, ctypes.POINTER(ctypes.c_uint8)]
            L.or_encode.restype = ctypes.c_int
            _LIB = L
    return _LIB


_POOL: Optional[concurrent.futures.ThreadPoolExecutor] = None
_NTHREADS = int(os.environ.get("ORACLE_THREADS", "0")) or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def set_threads(n: int) -> None:
    """Number of limbs processed concurrently (1 = fully single-threaded)."""
    global _POOL, _NTHREADS
    _NTHREADS = max(1, int(n))
    _POOL = None


def threads() -> int:
    return _NTHREADS


def _map(fn, items):
    global _POOL
    items = list(items)
    if _NTHREADS <= 1 or len(items) <= 1:
        return [fn(x) for x in items]
    if _POOL is None:
        _POOL = concurrent.futures.ThreadPoolExecutor(_NTHREADS)
    return list(_POOL.map(fn, items))


def _p64(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _pi64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


# --------------------------------------------------------------------------
# D1/D2/D3: parameters, primes, roots   (section 2.1.1:
# "R_Q = R/QR ... Q = prod_{i=0}^{L} q_i"; N, L and the primes themselves are
# never stated -- SURVEY.md R1 -- so BASELINE.json's configs and D2 fix them)
# --------------------------------------------------------------------------
def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (bases = first 13 primes)."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_primes(groups: Sequence[Sequence[int]], N: int, taken: Optional[List[int]] = None) -> List[int]:
    """D2: for each (bits, count) group, in order, the `count` largest primes
    < 2^bits with p = 1 mod 2N not already taken, in descending order."""
    taken = list(taken or [])
    out: List[int] = []
    for bits, count in groups:
        x = ((1 << bits) - 1) // (2 * N) * (2 * N) + 1
        while x >= (1 << bits):
            x -= 2 * N
        got = 0
        while got < count:
            if x < 2 * N:
                raise ValueError("HELRM_ERR_CONFIG: not enough primes")
            if is_prime(x) and x not in taken and x not in out:
                out.append(x)
                got += 1
            x -= 2 * N
    return out


def min_psi(q: int, N: int) -> int:
    """D3: the smallest x in [2, q) with x^N = -1 mod q (a primitive 2N-th root)."""
    g = 2
    while pow(g, (q - 1) // 2, q) != q - 1:
        g += 1
    psi0 = pow(g, (q - 1) // (2 * N), q)
    assert pow(psi0, N, q) == q - 1
    sq = psi0 * psi0 % q
    best, cur = psi0, psi0
    for _ in range(N - 1):          # psi0^k for odd k < 2N
        cur = cur * sq % q
        best = min(best, cur)
    return best


class Params:
    """D1: N = 2^logN, n = N/2 slots, q_0..q_L, special p_0..p_{K-1}, alpha = K."""

    def __init__(self, log_n: int, q: List[int], p: List[int], log_scale: int):
        self.log_n = log_n
        self.N = 1 << log_n
        self.n = self.N // 2
        self.q = list(q)
        self.p = list(p)
        self.L = len(q) - 1
        self.K = len(p)
        self.alpha = self.K
        self.log_scale = log_scale
        self.scale = 1 << log_scale
        self.psi: Dict[int, int] = {x: min_psi(x, self.N) for x in self.q + self.p}
        self.P = math.prod(self.p)

    def qp(self, level: int) -> List[int]:
        """Primes of R_{Q_l P}, in limb order q_0..q_l, p_0..p_{K-1}."""
        return self.q[: level + 1] + self.p

    def dnum(self, level: int) -> int:
        return -(-(level + 1) // self.alpha)

    def digit(self, level: int, k: int) -> List[int]:
        """Indices i of the q_i in digit k at level l: k*alpha <= i < min((k+1)*alpha, l+1)."""
        return list(range(k * self.alpha, min((k + 1) * self.alpha, level + 1)))

    def global_limb(self, level: int, limb: int) -> int:
        """Index of QP-limb `limb` (at level l) in the full chain q_0..q_L, p_0..p_{K-1}."""
        return limb if limb <= level else self.L + 1 + (limb - level - 1)


def params_from_config(cfg) -> Params:
    N = 1 << cfg.log_n
    q = find_primes(cfg.q_groups, N)
    p = find_primes(cfg.p_groups, N, taken=q)
    return Params(cfg.log_n, q, p, cfg.log_scale)


# --------------------------------------------------------------------------
# D4: NTT (natural order) and element-wise modular arithmetic
# --------------------------------------------------------------------------
def ntt(a: np.ndarray, primes: Sequence[int], P: Params) -> np.ndarray:
    out = np.array(a, dtype=np.uint64, copy=True, order="C")
    L = lib()

    def one(i):
        L.or_ntt(_p64(out[i]), P.N, primes[i], P.psi[primes[i]])
    _map(one, range(len(primes)))
    return out


def intt(a: np.ndarray, primes: Sequence[int], P: Params) -> np.ndarray:
    out = np.array(a, dtype=np.uint64, copy=True, order="C")
    L = lib()

    def one(i):
        L.or_intt(_p64(out[i]), P.N, primes[i], P.psi[primes[i]])
    _map(one, range(len(primes)))
    return out


def ntt_direct(a: np.ndarray, q: int, psi: int) -> np.ndarray:
    """D4 by its O(N^2) definition (pin for small N)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.zeros_like(a)
    lib().or_ntt_direct(_p64(a), _p64(out), a.shape[0], q, psi)
    return out


def _col(primes) -> np.ndarray:
    return np.array(primes, dtype=np.uint64).reshape(-1, 1)


def vmul(a: np.ndarray, b: np.ndarray, primes: Sequence[int]) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.empty_like(a)
    L = lib()

    def one(i):
        L.or_vec_mulmod(_p64(a[i]), _p64(b[i]), _p64(out[i]), a.shape[1], primes[i])
    _map(one, range(len(primes)))
    return out


def vscalar(a: np.ndarray, s: Sequence[int], primes: Sequence[int]) -> np.ndarray:
    """Limb i times the scalar s[i] mod primes[i]."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    L = lib()
    for i, q in enumerate(primes):
        L.or_vec_scalar(_p64(a[i]), int(s[i]) % q, _p64(out[i]), a.shape[1], q)
    return out


def vadd(a, b, primes):
    return (a + b) % _col(primes)          # residues < 2^62: no uint64 overflow


def vsub(a, b, primes):
    return (a + (_col(primes) - b)) % _col(primes)


def vneg(a, primes):
    return (_col(primes) - a) % _col(primes)


def reduce_signed(m: np.ndarray, primes: Sequence[int]) -> np.ndarray:
    """Signed integer polynomial -> canonical residues [m mod q_i] per limb."""
    m = np.asarray(m, dtype=np.int64)
    return np.stack([np.mod(m, np.int64(q)).astype(np.uint64) for q in primes])


# --------------------------------------------------------------------------
# D8: Galois automorphisms phi_g(a)(X) = a(X^g)   (PAPER.md:149 rotation)
# --------------------------------------------------------------------------
def galois_elt(k: int, P: Params) -> int:
    """rot_k (left by k) <-> g = 5^k mod 2N."""
    return pow(5, k % P.n, 2 * P.N)


def automorph_coeff(a: np.ndarray, g: int, primes: Sequence[int], N: int) -> np.ndarray:
    """Coefficient form: coefficient i moves to g*i mod 2N, negated (and
    reduced by N) when that is >= N."""
    i = np.arange(N, dtype=np.int64)
    dst = (g * i) % (2 * N)
    neg = dst >= N
    dst = dst % N
    out = np.empty_like(a)
    for r, q in enumerate(primes):
        v = a[r].copy()
        v[neg] = (np.uint64(q) - v[neg]) % np.uint64(q)
        out[r, dst] = v
    return out


def automorph_ntt(a: np.ndarray, g: int, N: int) -> np.ndarray:
    """NTT form, natural order: phi_g(a)^_i = a^_{i'} with 2i'+1 = g(2i+1) mod 2N."""
    i = np.arange(N, dtype=np.int64)
    src = ((g * (2 * i + 1)) % (2 * N) - 1) // 2
    return np.ascontiguousarray(a[:, src])


# --------------------------------------------------------------------------
# D9/D10: PRNG and samplers (the paper is silent)
# --------------------------------------------------------------------------
PURPOSE_SK, PURPOSE_PK_A, PURPOSE_PK_E, PURPOSE_RK_A, PURPOSE_RK_E = 1, 2, 3, 4, 5
PURPOSE_ENC_V, PURPOSE_ENC_E0, PURPOSE_ENC_E1, PURPOSE_MICRO = 6, 7, 8, 9


def stream(purpose: int, a: int = 0, b: int = 0, c: int = 0) -> int:
    return (purpose << 56) | (a << 32) | (b << 16) | c


def prng_word(seed: int, strm: int, k: int) -> int:
    return int(lib().or_prng_word(seed & (2**64 - 1), strm, k))


def sample_uniform(seed: int, strm: int, q: int, N: int) -> np.ndarray:
    out = np.empty(N, dtype=np.uint64)
    lib().or_sample_uniform(seed & (2**64 - 1), strm, q, N, _p64(out))
    return out


def sample_ternary(seed: int, strm: int, N: int) -> np.ndarray:
    out = np.empty(N, dtype=np.int64)
    lib().or_sample_ternary(seed & (2**64 - 1), strm, N, _pi64(out))
    return out


_CDT: Optional[List[int]] = None


def gauss_cdt(sigma: float = 3.2, bound: int = 19) -> List[int]:
    """T[k] = floor(2^64 P(|X| <= k)), rho(x) = exp(-x^2/(2 sigma^2)) normalised
    over |x| <= 19, evaluated with mpmath at 200 bits; T[19] = 2^64."""
    global _CDT
    if _CDT is None:
        import mpmath
        with mpmath.workprec(200):
            s = mpmath.mpf(repr(sigma))  # exactly 3.2, not the binary double nearest to it
            rho = [mpmath.exp(-mpmath.mpf(x * x) / (2 * s * s)) for x in range(bound + 1)]
            Z = rho[0] + 2 * sum(rho[1:])
            T = []
            acc = rho[0]
            for k in range(bound + 1):
                if k > 0:
                    acc += 2 * rho[k]
                T.append(int(mpmath.floor(acc / Z * mpmath.mpf(2) ** 64)))
            T[bound] = 1 << 64
        _CDT = T
    return _CDT


def sample_gauss(seed: int, strm: int, N: int) -> np.ndarray:
    T = gauss_cdt()
    tab = np.array(T[:19] + [0], dtype=np.uint64)
    out = np.empty(N, dtype=np.int64)
    lib().or_sample_gauss(seed & (2**64 - 1), strm, N, _p64(tab), _pi64(out))
    return out


# --------------------------------------------------------------------------
# D5/D6/D7: slots, encode, decode   (section 2.1.2
# "Encoding": inverse FFT, scale by Delta, round to nearest integer)
# --------------------------------------------------------------------------
def encode(z: np.ndarray, delta: int, N: int) -> np.ndarray:
    """D6: m_i = RHA((2 Delta/N) sum_j z_j cos(pi e_j i/N)), binary128 sums;
    a coefficient whose binary128 value lies within 2^-40 of a half-integer
    is recomputed exactly (200-bit mpmath, textbook.encode_mp_coeff), as D6
    requires."""
    from . import textbook
    z = np.ascontiguousarray(z, dtype=np.float64)
    assert z.shape == (N // 2,)
    assert float(delta) == delta, "Delta must be exactly representable"
    out = np.empty(N, dtype=np.int64)
    tie = np.zeros(N, dtype=np.uint8)
    st = lib().or_encode(z.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), N, float(delta), _pi64(out),
                         tie.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    if st != 0:
        raise ValueError("HELRM_ERR_CONFIG: |encoded coefficient| >= 2^62")
    for i in np.flatnonzero(tie):
        v = textbook.encode_mp_coeff(z, int(delta), N, int(i))
        if abs(v) >= 1 << 62:
            raise ValueError("HELRM_ERR_CONFIG: |encoded coefficient| >= 2^62")
        out[i] = v
    return out


def encode_many(zs: List[np.ndarray], delta: int, N: int) -> List[np.ndarray]:
    return _map(lambda z: encode(z, delta, N), zs)


def crt_centered(x: np.ndarray, primes: Sequence[int]) -> List[int]:
    """Centered CRT lift of coefficient-form residues into (-Q/2, Q/2]."""
    Q = math.prod(primes)
    terms = []
    for q in primes:
        Qi = Q // q
        terms.append((Qi, pow(Qi, -1, q), q))
    out = []
    cols = [list(map(int, x[r])) for r in range(len(primes))]
    for c in range(x.shape[1]):
        v = 0
        for r, (Qi, inv, q) in enumerate(terms):
            v += (cols[r][c] * inv % q) * Qi
        v %= Q
        if v > Q // 2:
            v -= Q
        out.append(v)
    return out


def decode(m: Sequence[int], delta, N: int) -> np.ndarray:
    """D7: z_j = Re(sum_i m_i zeta^{e_j i}) / Delta, fp64 (tolerance-only).
    The length-N sum uses numpy's FFT as a library step:
    zeta^{e_j i} = zeta^i * omega^{i (e_j - 1)/2}, omega = exp(2 pi i/N)."""
    m = np.array([float(v) for v in m], dtype=np.float64)
    i = np.arange(N)
    u = m * np.exp(1j * np.pi * i / N)
    F = np.fft.ifft(u) * N
    n = N // 2
    e = np.array([pow(5, j, 2 * N) for j in range(n)], dtype=np.int64)
    return F[(e - 1) // 2].real / float(delta)


# --------------------------------------------------------------------------
# D11/D12/D13: keys, encryption, decryption   ("encrypted ...
# with a given public key and the addition of some random noise"
# key switching; "a unique key is needed for each rotation offset")
# --------------------------------------------------------------------------
class SecretKey:
    def __init__(self, P: Params, s: np.ndarray):
        self.P = P
        self.s = s                                              # int64 ternary coefficients
        allp = P.q + P.p
        self.s_ntt_all = ntt(reduce_signed(s, allp), allp, P)   # rows: q_0..q_L, p_0..p_{K-1}

    def s_ntt(self, primes_idx: Sequence[int]) -> np.ndarray:
        return self.s_ntt_all[list(primes_idx)]


class PublicKey:
    def __init__(self, b: np.ndarray, a: np.ndarray):
        self.b, self.a = b, a


class RotKeys:
    """keys[g] = list over digits k of (b_k, a_k), each (L+1+K, N) NTT form."""

    def __init__(self, P: Params):
        self.P = P
        self.keys: Dict[int, List] = {}


def sk_gen(P: Params, seed: int) -> SecretKey:
    return SecretKey(P, sample_ternary(seed, stream(PURPOSE_SK), P.N))


def pk_gen(P: Params, sk: SecretKey, seed: int) -> PublicKey:
    """pk over Q_L: a <- UniformMod per limb (sampled as NTT-domain values,
    natural order -- DESIGN.md reading R-a), e <- Gauss; pk = (-a s + e, a)."""
    primes = P.q
    a = np.stack([sample_uniform(seed, stream(PURPOSE_PK_A, c=l), q, P.N) for l, q in enumerate(primes)])
    e = ntt(reduce_signed(sample_gauss(seed, stream(PURPOSE_PK_E), P.N), primes), primes, P)
    s = sk.s_ntt(range(P.L + 1))
    b = vadd(vneg(vmul(a, s, primes), primes), e, primes)
    return PublicKey(b, a)


def rotkeys_gen(P: Params, sk: SecretKey, galois: Sequence[int], seed: int) -> RotKeys:
    """D11: for each g and digit k < dnum(L), over all L+1+K limbs:
       b_k = -a_k s + e_k + [q_i in digit k] [P]_{q_i} phi_g(s)  (mod q_i)
       b_k = -a_k s + e_k                                          (mod p_j)"""
    rk = RotKeys(P)
    allp = P.q + P.p
    s = sk.s_ntt_all
    for g in galois:
        phis = automorph_ntt(s, g, P.N)
        digits = []
        for k in range(P.dnum(P.L)):
            a = np.stack([sample_uniform(seed, stream(PURPOSE_RK_A, g, k, l), q, P.N) for l, q in enumerate(allp)])
            e = ntt(reduce_signed(sample_gauss(seed, stream(PURPOSE_RK_E, g, k), P.N), allp), allp, P)
            b = vadd(vneg(vmul(a, s, allp), allp), e, allp)
            gad = np.zeros_like(b)
            dig = P.digit(P.L, k)
            gad[dig] = vscalar(phis[dig], [P.P % P.q[i] for i in dig], [P.q[i] for i in dig])
            b = vadd(b, gad, allp)
            digits.append((b, a))
        rk.keys[g] = digits
    return rk


class Ciphertext:
    """(c0, c1) in R_{Q_l}^2, NTT form natural order; level l; scale."""

    def __init__(self, c0: np.ndarray, c1: np.ndarray, level: int, scale):
        self.c0, self.c1, self.level, self.scale = c0, c1, level, scale

    def primes(self, P: Params) -> List[int]:
        return P.q[: self.level + 1]


def encrypt(P: Params, pk: PublicKey, z: np.ndarray, level: int, seed: int, delta=None) -> Ciphertext:
    """D12: m = Encode(z, Delta); v <- Ternary, e0, e1 <- Gauss;
    c0 = v pk0 + e0 + m, c1 = v pk1 + e1 (mod q_i, i <= l)."""
    if level > P.L or level < 0:
        raise ValueError("HELRM_ERR_LEVEL")
    delta = P.scale if delta is None else delta
    primes = P.q[: level + 1]
    zz = np.zeros(P.n)
    zz[: len(z)] = z
    if len(z) > P.n:
        raise ValueError("HELRM_ERR_CAPACITY")
    m = ntt(reduce_signed(encode(zz, delta, P.N), primes), primes, P)
    v = ntt(reduce_signed(sample_ternary(seed, stream(PURPOSE_ENC_V), P.N), primes), primes, P)
    e0 = ntt(reduce_signed(sample_gauss(seed, stream(PURPOSE_ENC_E0), P.N), primes), primes, P)
    e1 = ntt(reduce_signed(sample_gauss(seed, stream(PURPOSE_ENC_E1), P.N), primes), primes, P)
    c0 = vadd(vadd(vmul(v, pk.b[: level + 1], primes), e0, primes), m, primes)
    c1 = vadd(vmul(v, pk.a[: level + 1], primes), e1, primes)
    return Ciphertext(c0, c1, level, delta)


def decrypt(P: Params, sk: SecretKey, ct: Ciphertext) -> List[int]:
    """D13: m' = c0 + c1 s mod Q_l, centered CRT lift (coefficient form)."""
    primes = ct.primes(P)
    m = vadd(ct.c0, vmul(ct.c1, sk.s_ntt(range(ct.level + 1)), primes), primes)
    return crt_centered(intt(m, primes, P), primes)


def decrypt_decode(P: Params, sk: SecretKey, ct: Ciphertext) -> np.ndarray:
    return decode(decrypt(P, sk, ct), ct.scale, P.N)


def ct_to_coeff(P: Params, ct: Ciphertext) -> np.ndarray:
    """Canonical parity format: coefficient form, [2][level+1][N] uint64."""
    primes = ct.primes(P)
    return np.stack([intt(ct.c0, primes, P), intt(ct.c1, primes, P)])


# --------------------------------------------------------------------------
# D14-D18: base conversion, ModUp, ModDown, rescale, key switching
# (PAPER.md:151 key switching, :146-147 rescale; hybrid RNS key switching
# is SURVEY.md reading R8, the rounding conventions R9, the order R10)
# --------------------------------------------------------------------------
def conv(x: np.ndarray, B: Sequence[int], T: Sequence[int]) -> np.ndarray:
    """D14: Conv_{B->T}(x)_t = (sum_b [x_b (B/b)^-1]_b ((B/b) mod t)) mod t,
    coefficient-form input, no correction term."""
    Bprod = math.prod(B)
    binv = np.array([pow(Bprod // b, -1, b) for b in B], dtype=np.uint64)
    bp = np.array(B, dtype=np.uint64)
    x = np.ascontiguousarray(x, dtype=np.uint64)
    N = x.shape[1]
    out = np.empty((len(T), N), dtype=np.uint64)
    L = lib()

    def one(ti):
        t = T[ti]
        bmod = np.array([(Bprod // b) % t for b in B], dtype=np.uint64)
        tp = np.array([t], dtype=np.uint64)
        L.or_conv(_p64(x), len(B), _p64(bp), _p64(binv), _p64(bmod), 1, _p64(tp), _p64(out[ti]), N)
    _map(one, range(len(T)))
    return out


def modup(P: Params, c: np.ndarray, level: int, k: int) -> np.ndarray:
    """D15: ModUp_k(c), c in R_{Q_l} NTT form -> R_{Q_l P} NTT form.
    INTT the digit-k limbs, Conv them to (Q_l minus digit k) u P, NTT the new
    limbs; digit-k limbs are copied unchanged."""
    qp = P.qp(level)
    dig = P.digit(level, k)
    Bp = [P.q[i] for i in dig]
    x = intt(c[dig], Bp, P)
    tgt = [r for r in range(len(qp)) if r not in dig]
    T = [qp[r] for r in tgt]
    y = ntt(conv(x, Bp, T), T, P)
    out = np.empty((len(qp), P.N), dtype=np.uint64)
    out[dig] = c[dig]
    out[tgt] = y
    return out


def moddown(P: Params, y: np.ndarray, level: int) -> np.ndarray:
    """D16: x_i = (y_i - NTT_{q_i}(Conv_{P->Q_l}(INTT_P(y_P)))_i) [P^-1]_{q_i}."""
    Q = P.q[: level + 1]
    yP = intt(y[level + 1:], P.p, P)
    t = ntt(conv(yP, P.p, Q), Q, P)
    d = vsub(y[: level + 1], t, Q)
    return vscalar(d, [pow(P.P, -1, q) for q in Q], Q)


def rescale(P: Params, ct: Ciphertext) -> Ciphertext:
    """D17: h = (q_l - 1)/2, r = ((INTT(x_l) + h) mod q_l) - h in [-h, h],
    x'_i = (x_i - NTT_{q_i}(r mod q_i)) [q_l^-1]_{q_i}, i < l; scale / q_l."""
    l = ct.level
    if l < 1:
        raise ValueError("HELRM_ERR_LEVEL")
    ql = P.q[l]
    Qm = P.q[:l]
    h = (ql - 1) // 2

    def one(x):
        xl = intt(x[l:l + 1], [ql], P)[0]
        r = ((xl + np.uint64(h)) % np.uint64(ql)).astype(np.int64) - np.int64(h)
        rn = ntt(reduce_signed(r, Qm), Qm, P)
        return vscalar(vsub(x[:l], rn, Qm), [pow(ql, -1, q) for q in Qm], Qm)
    return Ciphertext(one(ct.c0), one(ct.c1), l - 1, Fraction(ct.scale) / ql)


def lift_P(P: Params, x: np.ndarray, level: int) -> np.ndarray:
    """P.x: Q-limbs [P]_{q_i} x_i, P-limbs 0."""
    Q = P.q[: level + 1]
    out = np.zeros((len(Q) + P.K, P.N), dtype=np.uint64)
    out[: len(Q)] = vscalar(x, [P.P % q for q in Q], Q)
    return out


def key_at_level(P: Params, key: np.ndarray, level: int) -> np.ndarray:
    """Restrict a full-chain key polynomial to limbs q_0..q_l, p_0..p_{K-1}."""
    return np.concatenate([key[: level + 1], key[P.L + 1:]])


def keyswitch_digits(P: Params, D: List[np.ndarray], g: int, rk: RotKeys, level: int):
    """KS from precomputed digits D_k = ModUp_k(c) (hoisting):
    (sum_k phi_g(D_k) (.) b_{g,k}, sum_k phi_g(D_k) (.) a_{g,k}) in R_{Q_l P}^2."""
    qp = P.qp(level)
    ks0 = np.zeros((len(qp), P.N), dtype=np.uint64)
    ks1 = np.zeros_like(ks0)
    for k, Dk in enumerate(D):
        b, a = rk.keys[g][k]
        phiD = automorph_ntt(Dk, g, P.N)
        ks0 = vadd(ks0, vmul(phiD, key_at_level(P, b, level), qp), qp)
        ks1 = vadd(ks1, vmul(phiD, key_at_level(P, a, level), qp), qp)
    return ks0, ks1


def keyswitch(P: Params, c: np.ndarray, g: int, rk: RotKeys, level: int):
    """D18: KS_g(c) -- ModUp first, then the automorphism."""
    D = [modup(P, c, level, k) for k in range(P.dnum(level))]
    return keyswitch_digits(P, D, g, rk, level)


def rotate_lazy(P: Params, ct: Ciphertext, k: int, rk: RotKeys, D=None):
    """RotateLazy(ct, k) = (P phi_g(c0) + KS_g(c1)_0, KS_g(c1)_1), g = 5^k, over Q_l P."""
    l = ct.level
    g = galois_elt(k, P)
    if D is None:
        D = [modup(P, ct.c1, l, kk) for kk in range(P.dnum(l))]
    ks0, ks1 = keyswitch_digits(P, D, g, rk, l)
    qp = P.qp(l)
    return vadd(lift_P(P, automorph_ntt(ct.c0, g, P.N), l), ks0, qp), ks1


def rotate(P: Params, ct: Ciphertext, k: int, rk: RotKeys, D=None) -> Ciphertext:
    """Rotate(ct, k) = (phi_g(c0) + ModDown(KS0), ModDown(KS1)); Rotate(ct, 0) = ct."""
    if k % P.n == 0:
        return ct
    l = ct.level
    g = galois_elt(k, P)
    if D is None:
        D = [modup(P, ct.c1, l, kk) for kk in range(P.dnum(l))]
    ks0, ks1 = keyswitch_digits(P, D, g, rk, l)
    Q = P.q[: l + 1]
    c0 = vadd(automorph_ntt(ct.c0, g, P.N), moddown(P, ks0, l), Q)
    return Ciphertext(c0, moddown(P, ks1, l), l, ct.scale)


def ct_add(P: Params, x: Ciphertext, y: Ciphertext) -> Ciphertext:
    assert x.level == y.level
    Q = x.primes(P)
    return Ciphertext(vadd(x.c0, y.c0, Q), vadd(x.c1, y.c1, Q), x.level, x.scale)
