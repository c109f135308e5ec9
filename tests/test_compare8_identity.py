"""Bit-sliced identity behind plane_device.cuh `compare8` (CPU check, no GPU).

The PLANE kernels compare the 8 unconditional planes of 32 lanes' uniforms with
the lanes' threshold planes in two 3-input LOP3 chains (least-significant plane
first).  This restates the chains with the same truth tables (0x8E, 0x90, 0xCA,
operand order a = 0xF0, b = 0xCC, c = 0xAA) and checks them against the
MSB-first lazy comparison of `compare_block` / `compare4_sel` and against the
integer comparison of the 8-bit prefixes.
"""
import numpy as np

MASK = np.uint32(0xFFFFFFFF)


def lop3(lut, a, b, c):
    out = np.zeros_like(a)
    for i in range(8):
        if (lut >> i) & 1:
            ta = a if (i >> 2) & 1 else ~a
            tb = b if (i >> 1) & 1 else ~b
            tc = c if i & 1 else ~c
            out |= ta & tb & tc
    return out & MASK


def sel(m, a1, a0):
    return lop3(0xCA, m, a1, a0)


def compare8(t, r, u):
    lt = t[7] & ~r[7]
    for b in range(6, -1, -1):
        lt = lop3(0x8E, r[b], t[b], lt)
    e = u.copy()
    for b in range(8):
        e = lop3(0x90, e, r[b], t[b])
    return lt, e


def msb_first(t, r, u):
    und, lt = u.copy(), np.zeros_like(u)
    for b in range(8):
        lt |= und & t[b] & ~r[b]
        und &= ~(t[b] ^ r[b])
    return lt & MASK, und & MASK


def test_sel_is_bitwise_mux():
    rng = np.random.default_rng(1)
    m, a1, a0 = (rng.integers(0, 1 << 32, 1000, dtype=np.uint64).astype(np.uint32) for _ in range(3))
    assert np.array_equal(sel(m, a1, a0), (m & a1) | (~m & a0))


def test_compare8_matches_msb_first_and_integers():
    rng = np.random.default_rng(2)
    n = 4000
    for trial in range(4):
        t = [rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32) for _ in range(8)]
        r = [rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32) for _ in range(8)]
        if trial >= 2:  # force many equal prefixes (the undecided case)
            keep = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            r = [(rb & ~keep) | (tb & keep) for rb, tb in zip(r, t)]
        u = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        lt, und = compare8(t, r, u)
        lt_ref, und_ref = msb_first(t, r, u)
        # compare8's lt is only meaningful on the lanes of u
        assert np.array_equal(lt & u, lt_ref)
        assert np.array_equal(und, und_ref)
        # against the integer prefixes, lane by lane (plane 0 = most significant)
        for lane in range(32):
            tv = sum(((t[b] >> lane) & 1).astype(np.int64) << (7 - b) for b in range(8))
            rv = sum(((r[b] >> lane) & 1).astype(np.int64) << (7 - b) for b in range(8))
            on = ((u >> lane) & 1).astype(bool)
            assert np.array_equal(((lt >> lane) & 1).astype(bool)[on], (rv < tv)[on])
            assert np.array_equal(((und >> lane) & 1).astype(bool), on & (rv == tv))
