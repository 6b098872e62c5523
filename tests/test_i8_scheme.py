"""The INT8 Gram's modular scheme (R18), checked on the host (no GPU): the moduli the library
uses and the integer width b it picks must make S = X X^T recoverable and every residue step exact.

  * 16 pairwise-coprime odd moduli p <= 253: symmetric residues (and the +-1 quotient slack of the
    FP32 rounding) stay in [-127, 127], int8;
  * prod p > 2 K 2^(2b) for |x| <= 2^b: the signed CRT reconstruction of |S_ij| <= K 2^(2b) is unique;
  * b <= 50: w = x + 2^50 + 2^33 + 2^16 lies in [0, 2^52), the DFMA rounding trick's range;
  * 127^2 2^16 < 2^31: a K-chunk of 2^16 int8 products accumulates exactly in int32;
  * balanced 17-bit digits and balanced constants |c| <= 126: |u0| + |c1 u1| + |c2 u2| < 2^24, so the
    FP32 FFMA chain forming x mod p is exact;
  * the whole scheme reproduces X X^T exactly on random integer matrices (Python big integers: residue
    Grams, Garner mixed radix, signed reconstruction) — the arithmetic the kernels implement.
"""
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def T():
    from paper_1711_06874_b200 import build, tucker
    build.build()
    tucker.load()
    return tucker


@pytest.mark.parametrize("K", [1, 2, 1000, 2 ** 16, 2 ** 20, 2 ** 22, 3 * 2 ** 22, 2 ** 30])
def test_scheme_bounds(T, K):
    mod, b = T.i8_scheme(K)
    assert len(mod) == 16 and all(p % 2 == 1 and 128 < p <= 253 for p in mod)
    for i in range(16):
        for j in range(i):
            assert math.gcd(mod[i], mod[j]) == 1
    P = math.prod(mod)
    assert b <= 50 and P > 2 * K * 2 ** (2 * b)
    assert b >= 40 if K <= 2 ** 30 else True
    assert b == 50 or P <= 2 * K * 2 ** (2 * (b + 1))  # the largest width the moduli allow
    for p in mod:
        assert (p + 1) // 2 <= 127  # |r| <= (p + 1) / 2 with the quotient's +-1 slack
    assert 127 ** 2 * 2 ** 16 < 2 ** 31


def _balanced(r, p):
    return r - p if r > p // 2 else r


def test_fp32_exactness_of_the_limb_combination(T):
    mod, _ = T.i8_scheme(2 ** 20)
    for p in mod:
        c1, c2 = _balanced(pow(2, 17, p), p), _balanced(pow(2, 34, p), p)
        assert abs(c1) <= 126 and abs(c2) <= 126
        umax = 2 ** 16 + 1  # balanced digits (the top one may reach 2^16 + 1 at |x| = 2^50)
        assert umax + abs(c1) * umax < 2 ** 24 and umax + abs(c1) * umax + abs(c2) * umax < 2 ** 24


def test_crt_reconstructs_integer_gram(T):
    rng = np.random.default_rng(5)
    K = 700
    mod, b = T.i8_scheme(K)
    X = [[int(v) for v in row] for row in rng.integers(-(2 ** b), 2 ** b + 1, size=(6, K), dtype=np.int64)]
    X[0][:5] = [2 ** b, -(2 ** b), 2 ** b, -(2 ** b), 2 ** b]  # extremes
    P = math.prod(mod)
    for i in range(6):
        for j in range(i + 1):
            exact = sum(a * c for a, c in zip(X[i], X[j]))
            # residue Grams: symmetric residues, products summed exactly, reduced mod p
            s = []
            for p in mod:
                ri = [_balanced(x % p, p) for x in X[i]]
                rj = [_balanced(x % p, p) for x in X[j]]
                s.append(sum(a * c for a, c in zip(ri, rj)) % p)
            # Garner mixed radix, then Horner from the top digit, then the signed range
            v = list(s)
            for l in range(1, 16):
                for q in range(l):
                    v[l] = ((v[l] - v[q] % mod[l]) * pow(mod[q] % mod[l], -1, mod[l])) % mod[l]
            S = 0
            for l in range(15, -1, -1):
                S = S * mod[l] + v[l]
            if S > P // 2:
                S -= P
            assert S == exact
