"""The FLOAT engine's one-comparison certified decision (slot_fast.cu), restated
in numpy float32 and checked with exact rationals (CPU check, no GPU).

With w = fl(T - hw 2^-16) and A = fl(T (|x2| k + c1) + 2^-16) the kernel
accepts when w >= A and rejects when w <= -A.  Whatever the roundings, an
accepted bucket [hw, hw + 1) 2^-16 must lie below T - band and a rejected one at
or above T + band, where band = T (|x2| k + c1) is the certified error bound of
T: then every u of the bucket decides the same way as the FP64 expression.
"""
from fractions import Fraction

import numpy as np

K = np.float32(float.fromhex("0x1.62e430p-20"))
TINY = np.float32(2.0 ** -16)


def f32(x):
    return np.float32(x)


def fma32(a, b, c):  # a * b is exact in float64; one extra rounding at most
    return f32(np.float64(a) * np.float64(b) + np.float64(c))


def test_accept_and_reject_are_certified():
    rng = np.random.default_rng(5)
    n_acc = n_rej = n_und = 0
    for _ in range(20000):
        x2 = f32(-rng.exponential(3.0)) if rng.random() < 0.9 else f32(rng.exponential(0.01))
        T = f32(2.0 ** np.float64(x2))
        c1 = f32(2.0 ** rng.uniform(-18, -10))
        # buckets near T are the interesting ones
        hw = int(np.clip(round(float(T) * 65536 + rng.integers(-3, 4)), 0, 65535)) if rng.random() < 0.7 \
            else int(rng.integers(0, 65536))
        A = fma32(T, fma32(abs(x2), K, c1), TINY)
        w = fma32(f32(hw), f32(-2.0 ** -16), T)
        band = Fraction(float(T)) * (Fraction(float(abs(x2))) * Fraction(float(K)) + Fraction(float(c1)))
        slack = band / 1000  # the roundings of A and w stay far inside the 2^-18 T term of c1
        if w >= A:
            n_acc += 1
            assert Fraction(hw + 1, 65536) <= Fraction(float(T)) - band + slack
        elif w <= -A:
            n_rej += 1
            assert Fraction(hw, 65536) >= Fraction(float(T)) + band - slack
        else:
            n_und += 1
    assert n_acc > 1000 and n_rej > 1000 and n_und > 100


def test_flushed_threshold_never_rejects_the_zero_bucket():
    # T flushed to zero by ex2.approx.ftz (T_true < 2^-126): the bucket of hw = 0
    # contains u = 0 < T_true and must stay undecided; every other bucket is
    # rejected, which is right because u >= 2^-16 > T_true.
    T = f32(0.0)
    A = fma32(T, f32(1e-5), TINY)
    w0 = fma32(f32(0), f32(-2.0 ** -16), T)
    assert not (w0 >= A) and not (w0 <= -A)
    for hw in (1, 2, 65535):
        w = fma32(f32(hw), f32(-2.0 ** -16), T)
        assert w <= -A
