"""The INT8 TTM's digit scheme (R22, ttm_i8.cu / err_i8.cu), checked on the host in exact
integer arithmetic (no GPU, none of the library's code):

  * balanced base-256 digits: for |X| <= 2^46, the bytes of X + 0x808080808080 with their top bit
    flipped are six int8 digits x_s with X = sum_s x_s 256^(5-s) exactly (the one-DFMA conversion
    puts X + bias in the low 48 mantissa bits: fma(F, 2^(46-E), 2^52 + bias) rounds once to an
    integer since 2^52 <= 2^52 + bias + X < 2^53);
  * the 26 digit pairs s + t <= 6 reproduce X Y up to the dropped pairs, whose sum is bounded by
    sum_{s+t>6} 128^2 256^(10-s-t) < 2^41 (relative 2^-51 of the 2^92 scale) per product;
  * per TMEM group d the int32 sum of <= 6 pairs over n3 <= 2^14 terms stays below 2^31;
  * the FP64 recombination T1 = sum_d acc_d 2^(E + E_c - 12 - 8 d) equals X Y 2^(E + E_c - 92) for the
    kept pairs (checked with exact rationals).
"""
import random
from fractions import Fraction

BIAS = 0x808080808080


def digits(X):
    w = X + BIAS
    assert 0 <= w < 1 << 48
    out = []
    for s in range(6):  # most significant first
        byte = (w >> (8 * (5 - s))) & 255
        out.append((byte ^ 0x80) - 256 if (byte ^ 0x80) >= 128 else (byte ^ 0x80))
    return out


def test_digits_reconstruct_exactly():
    rng = random.Random(1711)
    vals = [0, 1, -1, 2 ** 46, -2 ** 46, 2 ** 46 - 1, -(2 ** 46) + 1, 0x7F7F7F7F7F7F - 2 ** 45, 127, -128, 128]
    vals += [rng.randint(-2 ** 46, 2 ** 46) for _ in range(20000)]
    for X in vals:
        d = digits(X)
        assert all(-128 <= x <= 127 for x in d)
        assert sum(x * 256 ** (5 - s) for s, x in enumerate(d)) == X


def test_magic_fma_range():
    # 2^52 + bias + X for |X| <= 2^46 lies in [2^52, 2^53): one rounding to an integer, low 48 bits = X + bias
    assert (1 << 52) + BIAS - (1 << 46) >= 1 << 52
    assert (1 << 52) + BIAS + (1 << 46) < 1 << 53
    assert BIAS + (1 << 46) < 1 << 48 and BIAS - (1 << 46) >= 0


def test_truncated_product_and_groups():
    rng = random.Random(874)
    n3 = 1 << 14
    # worst case per group: <= 6 pairs of |x y| <= 128^2 over n3 terms
    assert 6 * 128 * 128 * n3 < 2 ** 31
    dropped_bound = sum(128 * 128 * 256 ** (10 - s - t) for s in range(6) for t in range(6) if s + t > 6)
    assert dropped_bound < 2 ** 41
    for _ in range(2000):
        X, Y = rng.randint(-2 ** 46, 2 ** 46), rng.randint(-2 ** 46, 2 ** 46)
        dx, dy = digits(X), digits(Y)
        acc = [0] * 7
        for s in range(6):
            for t in range(6):
                if s + t <= 6:
                    acc[s + t] += dx[s] * dy[t]
        kept = sum(a * 256 ** (10 - d) for d, a in enumerate(acc))
        assert abs(X * Y - kept) <= dropped_bound
        # FP64-side recombination in exact rationals: T1 = sum_d acc_d 2^(E + Ec - 12 - 8 d) = kept 2^(E + Ec - 92)
        E, Ec = rng.randint(-10, 3), rng.randint(-6, 0)
        t1 = sum(Fraction(a) * Fraction(2) ** (E + Ec - 12 - 8 * d) for d, a in enumerate(acc))
        assert t1 == Fraction(kept) * Fraction(2) ** (E + Ec - 92)
