"""oracle.textbook -- TEST INFRASTRUCTURE: brute-force textbook definitions
for tiny rings (N <= 64), in pure Python integers / mpmath, used only to pin
the C oracle (tests/test_oracle_pins.py).  Nothing here is fast or clever.

  negacyclic_mul  schoolbook product in Z_q[X]/(X^N + 1)
  ntt_eval        a(psi^{2i+1}) by Horner                   (D4)
  encode_mp       m_i = RHA((2 Delta/N) sum_j z_j cos(pi e_j i/N)) at 200 bits (D6)
  encode_mp_coeff one coefficient of encode_mp (the oracle's exact D6 recomputation)
  decode_mp       z_j = Re(sum_i m_i zeta^{e_j i}) / Delta   (D7)
"""
from __future__ import annotations

from typing import List, Sequence


def negacyclic_mul(a: Sequence[int], b: Sequence[int], q: int) -> List[int]:
    N = len(a)
    out = [0] * N
    for i in range(N):
        for j in range(N):
            k = i + j
            if k < N:
                out[k] = (out[k] + a[i] * b[j]) % q
            else:
                out[k - N] = (out[k - N] - a[i] * b[j]) % q
    return out


def ntt_eval(a: Sequence[int], q: int, psi: int) -> List[int]:
    N = len(a)
    out = []
    for i in range(N):
        x = pow(psi, 2 * i + 1, q)
        acc = 0
        for c in reversed(a):
            acc = (acc * x + c) % q
        out.append(acc)
    return out


def rha(v) -> int:
    """Round half away from zero of an mpmath number."""
    import mpmath
    if v >= 0:
        return int(mpmath.floor(v + mpmath.mpf(1) / 2))
    return -int(mpmath.floor(-v + mpmath.mpf(1) / 2))


def encode_mp(z: Sequence[float], delta: int, N: int, prec: int = 200) -> List[int]:
    import mpmath
    n = N // 2
    e = [pow(5, j, 2 * N) for j in range(n)]
    out = []
    with mpmath.workprec(prec):
        c = mpmath.mpf(2) * delta / N
        cos_tab = [mpmath.cos(mpmath.pi * k / N) for k in range(2 * N)]
        for i in range(N):
            acc = mpmath.mpf(0)
            for j in range(n):
                if z[j] != 0:
                    acc += mpmath.mpf(z[j]) * cos_tab[(e[j] * i) % (2 * N)]
            out.append(rha(c * acc))
    return out


def encode_mp_coeff(z: Sequence[float], delta: int, N: int, i: int, prec: int = 200) -> int:
    """Coefficient i of encode_mp alone (the D6 exact recomputation)."""
    import mpmath
    n = N // 2
    with mpmath.workprec(prec):
        acc = mpmath.mpf(0)
        ej = 1
        for j in range(n):
            if z[j] != 0:
                acc += mpmath.mpf(float(z[j])) * mpmath.cos(mpmath.pi * ((ej * i) % (2 * N)) / N)
            ej = ej * 5 % (2 * N)
        return rha(mpmath.mpf(2) * delta / N * acc)


def encode_mp_frac(z: Sequence[float], delta: int, N: int, prec: int = 200) -> List[float]:
    """Distance of each unrounded coefficient from the nearest half-integer."""
    import mpmath
    n = N // 2
    e = [pow(5, j, 2 * N) for j in range(n)]
    out = []
    with mpmath.workprec(prec):
        c = mpmath.mpf(2) * delta / N
        for i in range(N):
            acc = mpmath.mpf(0)
            for j in range(n):
                if z[j] != 0:
                    acc += mpmath.mpf(z[j]) * mpmath.cos(mpmath.pi * ((e[j] * i) % (2 * N)) / N)
            v = c * acc
            out.append(float(abs(v - mpmath.floor(v) - mpmath.mpf(1) / 2)))
    return out


def decode_mp(m: Sequence[int], delta, N: int, prec: int = 120) -> List[float]:
    import mpmath
    n = N // 2
    out = []
    with mpmath.workprec(prec):
        for j in range(n):
            e = pow(5, j, 2 * N)
            acc = mpmath.mpf(0)
            for i, mi in enumerate(m):
                acc += mi * mpmath.cos(mpmath.pi * ((e * i) % (2 * N)) / N)
            out.append(float(acc / delta))
    return out
