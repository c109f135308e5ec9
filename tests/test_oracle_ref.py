"""Pin the oracle: the C restatement (oracle/tg_oracle.c) against the
reference's own sources compiled in place (oracle/_ref, built by
oracle/Makefile from /root/reference) and against the reference's known-answer
tests.  CPU only.

* O1  (libtgref_mt)        unmodified reference: determinism / thread-count
                           invariance (test_engine.cpp:214-227, acceptance.cpp:538-563).
* O2  (libtgref_philox*)   reference + Philox shadow rng.hpp: the port must be
                           bit-identical (f, g, digests, final grid, counters).
"""
import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I

needs_ref = pytest.mark.skipif(not O.ref_available("philox"), reason="oracle/_ref not built")


def five_sparse():
    f = I.five_node_complete()
    return I.to_canonical(I.sparsify(5, list(zip(f.ci.tolist(), f.cj.tolist(), f.cw.tolist())),
                                     f.fields.tolist(), 2, 3))


def crit1_problem():
    # acceptance.cpp:48-54: dense 3-node problem over three copies per node
    return I.to_canonical(I.sparsify(3, [(0, 1, 1.2), (0, 2, -1.5), (1, 2, 0.9)],
                                     [0.4, -0.3, 0.5], 3, 3))


CASES = [
    ("five_node", five_sparse, [0.5, 1.0, 1.5], [2.0, 4.0, 6.0, 8.0], 300, 3),
    ("k10", lambda: I.k10_pm1(1), *I.config_schedule("c1"), 200, 1),
    ("crit1_float", crit1_problem, [0.8, 1.0, 1.25], [1.0, 2.0, 4.0], 300, 10),
    ("bip3reg", lambda: I.bipartite_3regular(64, seed=2), [0.3, 1.0, 3.0], [0.0, 0.25, 1.0], 60, 1),
    ("wishart", lambda: I.wishart_planted(6, 0.5, seed=3), [0.2, 1.0, 5.0], [0.0, 0.1, 0.3], 120, 2),
    ("single_row", lambda: I.k10_pm1(2), [1.0], [0.0, 0.5, 1.0, 1.5], 60, 1),
    ("single_col", lambda: I.k10_pm1(2), [0.2, 0.5, 1.0, 3.0], [1.0], 60, 1),
    ("one_by_one", lambda: I.k10_pm1(2), [1.0], [2.0], 40, 4),
]
VARIANTS = [("metropolis", "slot", "philox"), ("heat_bath", "slot", "philox_hb"),
            ("metropolis", "plane", "plane"), ("heat_bath", "plane", "plane_hb"),
            ("metropolis", "float", "pack"), ("heat_bath", "float", "pack_hb")]


@needs_ref
@pytest.mark.parametrize("rule,rng,variant", VARIANTS)
@pytest.mark.parametrize("name,mk,betas,pens,total,sps", CASES, ids=[c[0] for c in CASES])
def test_port_bit_identical_to_reference(name, mk, betas, pens, total, sps, rule, rng, variant):
    pr = mk()
    a = O.run(pr, betas, pens, total, sps, seed=7, rule=rule, rng=rng, round_counters=True)
    r = O.run(pr, betas, pens, total, sps, seed=7, rule=rule, rng=rng, impl="ref:" + variant,
              round_counters=True)
    np.testing.assert_array_equal(a.f, r.f)
    np.testing.assert_array_equal(a.g, r.g)
    np.testing.assert_array_equal(a.feasible, r.feasible)
    np.testing.assert_array_equal(a.digest, r.digest)
    np.testing.assert_array_equal(a.final_grid, r.final_grid)
    np.testing.assert_array_equal(a.accepts_p, r.accepts_p)
    np.testing.assert_array_equal(a.accepts_b, r.accepts_b)
    np.testing.assert_array_equal(a.attempts_p, r.attempts_p)
    np.testing.assert_array_equal(a.round_acc_p, r.round_acc_p)
    np.testing.assert_array_equal(a.round_acc_b, r.round_acc_b)


@needs_ref
def test_reference_thread_count_invariance():
    # test_engine.cpp:214-227 / acceptance criterion 8, on the unmodified reference (O1)
    pr = five_sparse()
    a = O.run(pr, [1.0], [2.0, 4.0, 6.0, 8.0], 2000, 500 // 50, seed=77, impl="ref:mt", threads=1)
    b = O.run(pr, [1.0], [2.0, 4.0, 6.0, 8.0], 2000, 500 // 50, seed=77, impl="ref:mt", threads=4)
    np.testing.assert_array_equal(a.digest, b.digest)
    np.testing.assert_array_equal(a.f, b.f)


@needs_ref
@pytest.mark.parametrize("bad,msg", [
    (dict(betas=[1.0, 1.0]), "strictly increasing"),
    (dict(betas=[]), "non-empty"),
    (dict(pens=[float("inf")]), "finite"),
    (dict(sps=0), "sweeps_per_swap"),
    (dict(total=0), "total_sweeps"),
    (dict(pens=[-1.0]), "penalty must be >= 0"),
])
def test_validation_matches_reference(bad, msg):
    # engine.cpp:41-59, constraints.cpp:123-124
    pr = I.k10_pm1(1)
    kw = dict(betas=[0.5, 1.0], pens=[0.0, 1.0], total=10, sps=1)
    kw.update(bad)
    errs = []
    for impl in ("port", "ref:philox"):
        with pytest.raises(O.OracleError) as ei:
            O.run(pr, kw["betas"], kw["pens"], kw["total"], kw["sps"], impl=impl)
        assert ei.value.code == 2
        assert msg in ei.value.msg
        errs.append(ei.value.msg)
    assert errs[0] == errs[1]


@needs_ref
@pytest.mark.parametrize("n,couplings,fields,copies,deg", [
    (5, [(0, 1, -1.0), (0, 2, -1.0), (0, 3, -2.0), (0, 4, -2.0), (1, 2, -1.0), (1, 3, -1.0),
         (1, 4, -2.0), (2, 3, -1.0), (2, 4, -1.0), (3, 4, -2.0)], [0.5, -1, 0.5, 0.5, -1], 2, 3),
    (3, [(0, 1, 1.2), (0, 2, -1.5), (1, 2, 0.9)], [0.4, -0.3, 0.5], 3, 3),
    (6, [(i, j, 1.0 + 0.1 * i - 0.05 * j) for i in range(6) for j in range(i + 1, 6)], [0.0] * 6, 3, 4),
])
def test_sparsify_matches_reference(n, couplings, fields, copies, deg):
    # python restatement of constraints.cpp:50-120 vs the reference itself
    n_ref, ci, cj, w, h, pa, pb = O.ref_sparsify(n, couplings, fields, copies, deg)
    pr = I.sparsify(n, couplings, fields, copies, deg)
    assert pr.n == n_ref
    got = sorted(zip(pr.ci.tolist(), pr.cj.tolist(), pr.cw.tolist()))
    ref = sorted(zip(ci.tolist(), cj.tolist(), w.tolist()))
    assert got == ref
    np.testing.assert_array_equal(pr.fields, h)
    assert list(zip(pr.pa.tolist(), pr.pb.tolist())) == list(zip(pa.tolist(), pb.tolist()))


@needs_ref
def test_sparsify_refusal_matches_reference():
    # test_constraints.cpp:137-141: capacity c*(D-2)+2 < degree is refused
    cpl = [(i, j, 1.0) for i in range(10) for j in range(i + 1, 10)]
    with pytest.raises(O.OracleError):
        O.ref_sparsify(10, cpl, [0.0] * 10, 3, 4)
    with pytest.raises(I.ConfigError):
        I.sparsify(10, cpl, [0.0] * 10, 3, 4)


def test_port_determinism_and_seed_sensitivity():
    pr = I.k10_pm1(1)
    b, p = I.config_schedule("c1")
    a = O.run(pr, b, p, 100, 1, seed=5)
    c = O.run(pr, b, p, 100, 1, seed=5)
    d = O.run(pr, b, p, 100, 1, seed=6)
    np.testing.assert_array_equal(a.digest, c.digest)
    assert not np.array_equal(a.digest, d.digest)
