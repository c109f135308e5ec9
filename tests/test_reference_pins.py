"""Known-answer tests of the reference that pin this path,
applied to the oracle and to the engine library's host-side helpers (the
library loads without a GPU; no kernels run here).

* swap-probability tables        test_engine.cpp:47-58, 68-79 (to 1e-12)
* general rule reductions        test_engine.cpp:85-116
* pair parity / direction        test_engine.cpp:132-178 (free_spin fixture)
* five-node instance constants   test_instances.cpp:123-126
* Philox4x32-10 KATs             tests/golden/philox_kat.json (cuRAND's implementation)
"""
import json
import math
import os

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

P_SWAP = [  # (beta, dp, dg, expected)  test_engine.cpp:47-58
    (1.0, 2.0, 0.0, 1.0), (1.0, 2.0, 4.0, 1.0), (1.0, 2.0, -4.0, 3.354626279025118e-4),
    (0.5, 1.0, -4.0, 0.1353352832366127), (2.0, 0.5, -8.0, 3.354626279025118e-4),
    (1.0, 3.0, 4.0, 1.0), (0.1, 10.0, -4.0, 0.018315638888734176),
    (1.5, 2.0, -2.0, 0.0024787521766663585), (3.0, 1.0, -1.0, 0.049787068367863944),
    (0.25, 4.0, -3.0, 0.049787068367863944),
]
B_SWAP = [  # (dbeta, de, expected)  test_engine.cpp:68-79
    (0.5, 0.0, 1.0), (0.5, 6.0, 1.0), (0.5, -6.0, 0.049787068367863944),
    (0.2, -10.0, 0.13533528323661268), (1.0, -1.0, 0.36787944117144233),
    (0.05, -40.0, 0.13533528323661268), (0.3, 2.5, 1.0), (0.7, -0.5, 0.7046880897187135),
    (0.125, -16.0, 0.1353352832366127), (2.0, -0.25, 0.6065306597126334),
]


def _lib_or_none():
    try:
        from paper_2506_14781_b200 import _lib
        return _lib.lib()
    except Exception:  # noqa: BLE001
        return None


def impls():
    out = [("port", O.p_swap_probability, O.beta_swap_probability, O.general_swap_probability)]
    L = _lib_or_none()
    if L is not None:
        out.append(("engine", L.tg_p_swap_probability, L.tg_beta_swap_probability,
                    L.tg_general_swap_probability))
    return out


@pytest.mark.parametrize("name,pf,bf,gf", impls(), ids=[i[0] for i in impls()])
def test_swap_probability_tables(name, pf, bf, gf):
    for beta, dp, dg, exp in P_SWAP:
        assert pf(beta, dp, dg) == pytest.approx(exp, rel=1e-12)
    for db, de, exp in B_SWAP:
        assert bf(db, de) == pytest.approx(exp, rel=1e-12)


@pytest.mark.parametrize("name,pf,bf,gf", impls(), ids=[i[0] for i in impls()])
def test_general_rule_reduces_to_special_cases(name, pf, bf, gf):
    rng = np.random.default_rng(101)
    for _ in range(1000):
        beta = 0.1 + 3.0 * rng.random()
        pa = 0.5 + 2.0 * rng.random()
        pb = pa + 0.1 + 2.0 * rng.random()
        fa, fb = 10 * rng.random() - 5, 10 * rng.random() - 5
        ga, gb = 4.0 * rng.integers(6), 4.0 * rng.integers(6)
        de_a = (fa + pa * ga) - (fa * 0 + fb + pa * gb)
        de_b = (fb + pb * gb) - (fa + pb * ga)
        assert gf(beta, beta, de_a, de_b) == pytest.approx(pf(beta, pb - pa, gb - ga), rel=1e-12)
        ba = 0.1 + 2.0 * rng.random()
        bb = ba + 0.05 + 2.0 * rng.random()
        ea, eb = 10 * rng.random() - 5, 10 * rng.random() - 5
        assert gf(ba, bb, ea - eb, eb - ea) == pytest.approx(bf(bb - ba, eb - ea), rel=1e-12)


FREE_SPIN = I.Problem.make(1, [], [0.0])


def test_single_row_pair_parity():
    # test_engine.cpp:132-146: g == 0 so every attempted P pair is accepted
    r = O.run(FREE_SPIN, [1.0], [1.0, 2.0, 3.0, 4.0], 2, 1, round_counters=True)
    rates = r.round_acc_p / np.maximum(1, np.array([[1, 0, 1], [1, 1, 1]]))
    np.testing.assert_array_equal(r.round_acc_p, [[1, 0, 1], [1, 1, 1]])
    assert r.round_acc_b.shape[1] == 0
    assert rates.shape == (2, 3)


def test_single_column_pair_parity():
    r = O.run(FREE_SPIN, [0.5, 1.0, 1.5, 2.0], [1.0], 2, 1, round_counters=True)
    np.testing.assert_array_equal(r.round_acc_b, [[1, 0, 1], [1, 1, 1]])


def test_direction_alternates_every_two_rounds():
    # test_engine.cpp:162-178
    r = O.run(FREE_SPIN, [1.0, 2.0], [1.0, 2.0], 6, 1, round_counters=True)
    np.testing.assert_array_equal(r.round_acc_p[0], [1, 1])
    np.testing.assert_array_equal(r.round_acc_b[0], [0, 0])
    np.testing.assert_array_equal(r.round_acc_b[2], [1, 1])
    np.testing.assert_array_equal(r.round_acc_p[3], r.round_acc_p[0])


def test_one_by_one_never_swaps():
    r = O.run(I.k10_pm1(1), [1.0], [2.0], 50, 5, round_counters=True)
    assert r.attempts_p.size == 0 and r.attempts_b.size == 0


def _enumerate(pr, beta, penalty=0.0):
    n = pr.n
    states = ((np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1) * 2 - 1
    e = np.zeros(1 << n)
    for i, j, w in zip(pr.ci, pr.cj, pr.cw):
        e -= w * states[:, i] * states[:, j]
    e -= states @ pr.fields
    g = np.zeros(1 << n)
    for a, b in zip(pr.pa, pr.pb):
        g += (states[:, a] - states[:, b]) ** 2
    tot = e + penalty * g
    w = np.exp(-beta * (tot - tot.min()))
    return w / w.sum(), tot


def test_five_node_instance_constants():
    # test_instances.cpp:123-126: ground state -5.5 at encoding 13, p13 at beta=1
    p, e = _enumerate(I.five_node_complete(), 1.0)
    assert e.min() == pytest.approx(-5.5)
    assert int(np.argmin(e)) == 13
    assert p[13] == pytest.approx(0.21449522432110954, rel=1e-12)


def test_philox_known_answers():
    kat = json.load(open(os.path.join(GOLDEN, "philox_kat.json")))
    for case in kat["cases"]:
        np.testing.assert_array_equal(O.philox(case["ctr"], case["key"]), case["out"])


def test_splitmix_and_stream_contract():
    # mix64 is the SplitMix64 finalizer: first SplitMix64 output for state 0
    assert O.derive_seed(0, 0, 0) != 0
    from ctypes import c_uint64  # noqa: F401
    # derive_seed(m, p, i) = mix64(mix64(m ^ mix64(p)) ^ i)  (rng.hpp:36-40)
    mix = lambda z: _mix64(z)  # noqa: E731
    for m, p, i in [(1, 1, 0), (77, 2, 0), (2**63 + 5, 3, 12345)]:
        assert O.derive_seed(m, p, i) == mix(mix(m ^ mix(p)) ^ i)
    assert _mix64(0) == 0xE220A8397B1DCDAF
    # stream bits: word pairs of one Philox block (philox_ref.h header)
    seed = O.derive_seed(9, 1, 4)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    o = O.philox([0, 0, 0, 0], key)
    assert O.stream_bits(seed, 0) == int(o[0]) | (int(o[1]) << 32)
    assert O.stream_bits(seed, 1) == int(o[2]) | (int(o[3]) << 32)
    # plane uniform: bit `lane` of the four words of block (b>>2) | grp<<4
    pk = O.derive_seed(3, 8, 0)
    pkey = [pk & 0xFFFFFFFF, pk >> 32]
    u = O.plane_u53(pk, 2, 7, 11, 5)
    o0 = O.philox([11, 7, 0, 0 | (2 << 4)], pkey)
    top4 = [(int(o0[q]) >> 5) & 1 for q in range(4)]
    assert [(u >> (52 - b)) & 1 for b in range(4)] == top4


def _mix64(z):
    M = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)
