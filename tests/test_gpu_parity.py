"""GPU parity: the B200 engine (through the C ABI) against the oracle.

Integer / dyadic instances must match bit for bit: every round's target f, g,
feasibility and state digest, the final configuration of every grid slot and
the cumulative swap-accept counters.  The oracle is the C restatement
(oracle/tg_oracle.c), itself pinned to the reference sources in
tests/test_oracle_ref.py; where oracle/_ref is present the engine is also
compared with the reference build directly.
"""
import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig

pytestmark = pytest.mark.gpu


def engine_run(pr, betas, pens, total, sps, seed, rule, engine):
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(betas, pens)
    recs = []

    def sink(r, n, states, ap, ab):
        for k in range(n):
            recs.append((r[k].round, r[k].f, r[k].g, r[k].feasible, r[k].digest, r[k].target_state))
        return 0

    cfg = RunConfig(total_sweeps=total, sweeps_per_swap=sps, seed=seed, rule=rule, engine=engine,
                    store_states=False, digest=True)
    eng.run(cfg, sink)
    grid = eng.grid()
    ap, cp, ab, cb = eng.counters()
    info = eng.info()
    eng.close()
    return recs, grid, (ap, cp, ab, cb), info


def compare(pr, betas, pens, total, sps, seed, rule, engine, exact=True):
    rng_mode = "plane" if engine == "plane" else "slot"
    o = O.run(pr, betas, pens, total, sps, seed=seed, rule=rule, rng=rng_mode)
    recs, grid, (ap, cp, ab, cb), info = engine_run(pr, betas, pens, total, sps, seed, rule, engine)
    assert info["engine"] == {"slot": 1, "plane": 2}[engine]
    f = np.array([r[1] for r in recs])
    g = np.array([r[2] for r in recs])
    feas = np.array([bool(r[3]) for r in recs])
    dig = np.array([r[4] for r in recs], dtype=np.uint64)
    assert len(recs) == total // sps
    if exact:
        np.testing.assert_array_equal(f, o.f)
    else:
        np.testing.assert_allclose(f, o.f, rtol=1e-9, atol=1e-9)
    np.testing.assert_array_equal(g, o.g)
    np.testing.assert_array_equal(feas, o.feasible)
    np.testing.assert_array_equal(dig, o.digest)
    np.testing.assert_array_equal(grid, o.final_grid)
    np.testing.assert_array_equal(cp, o.accepts_p)
    np.testing.assert_array_equal(cb, o.accepts_b)
    np.testing.assert_array_equal(ap, o.attempts_p)
    np.testing.assert_array_equal(ab, o.attempts_b)
    return o


K10 = I.k10_pm1(1)
C5S = I.bipartite_3regular(512, seed=3)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
@pytest.mark.parametrize("sps", [1, 3])
def test_plane_k10_config1(rule, sps):
    b, p = I.config_schedule("c1")
    compare(K10, b, p, 300 * sps, sps, seed=5, rule=rule, engine="plane")


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_plane_bipartite_16x16(rule):
    b, p = I.config_schedule("c5")
    compare(C5S, b, p, 40, 1, seed=11, rule=rule, engine="plane")


def test_plane_ragged_grid():
    # 3 x 5 = 15 replicas: a partial 32-lane word and odd pair counts
    compare(K10, [0.3, 0.9, 2.0], [0.0, 0.25, 0.5, 1.0, 2.0], 120, 2, seed=9,
            rule="metropolis", engine="plane")


def test_plane_single_row_and_column():
    compare(K10, [1.0], [0.0, 0.5, 1.0, 1.5], 50, 1, seed=2, rule="metropolis", engine="plane")
    compare(K10, [0.2, 0.5, 1.0, 3.0], [1.0], 50, 1, seed=2, rule="heat_bath", engine="plane")
    compare(K10, [1.0], [2.0], 30, 1, seed=2, rule="metropolis", engine="plane")


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_slot_k10(rule):
    b, p = I.config_schedule("c1")
    compare(K10, b, p, 200, 1, seed=5, rule=rule, engine="slot")


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_slot_five_node_dyadic(rule):
    five = I.five_node_complete()
    pr = I.to_canonical(I.sparsify(5, list(zip(five.ci.tolist(), five.cj.tolist(), five.cw.tolist())),
                                   five.fields.tolist(), 2, 3))
    compare(pr, [0.5, 1.0, 1.5], [2.0, 4.0, 6.0, 8.0], 400, 5, seed=77, rule=rule, engine="slot")


def test_slot_float_instance():
    pr = I.to_canonical(I.sparsify(3, [(0, 1, 1.2), (0, 2, -1.5), (1, 2, 0.9)], [0.4, -0.3, 0.5], 3, 3))
    compare(pr, [0.8, 1.0, 1.25], [1.0, 2.0, 4.0], 300, 10, seed=11, rule="metropolis",
            engine="slot", exact=False)


def test_slot_wishart_float():
    pr = I.wishart_planted(8, 0.5, seed=4)
    b, p = I.wishart_schedule(pr, 4, 4)
    compare(pr, b, p, 100, 1, seed=3, rule="metropolis", engine="slot", exact=False)


@pytest.mark.skipif(not O.ref_available("philox"), reason="oracle/_ref not built")
def test_against_reference_build_directly():
    b, p = I.config_schedule("c1")
    r = O.run(K10, b, p, 100, 1, seed=13, impl="ref:philox")
    recs, grid, _, _ = engine_run(K10, b, p, 100, 1, 13, "metropolis", "slot")
    np.testing.assert_array_equal(np.array([x[1] for x in recs]), r.f)
    np.testing.assert_array_equal(np.array([x[4] for x in recs], dtype=np.uint64), r.digest)
    np.testing.assert_array_equal(grid, r.final_grid)
    r = O.run(K10, b, p, 100, 1, seed=13, impl="ref:plane")
    recs, grid, _, _ = engine_run(K10, b, p, 100, 1, 13, "metropolis", "plane")
    np.testing.assert_array_equal(np.array([x[4] for x in recs], dtype=np.uint64), r.digest)
    np.testing.assert_array_equal(grid, r.final_grid)


def test_resume_equals_single_run():
    b, p = I.config_schedule("c1")
    eng = Engine(0)
    eng.set_problem(K10)
    eng.set_schedule(b, p)
    cfg = RunConfig(total_sweeps=100, sweeps_per_swap=1, seed=21, engine="plane", store_states=False)
    eng.init(cfg)
    eng.advance(40)
    eng.advance(60)
    g1 = eng.grid()
    eng.close()
    o = O.run(K10, b, p, 100, 1, seed=21, rng="plane")
    np.testing.assert_array_equal(g1, o.final_grid)


def test_run_2dpt_api_trace():
    from paper_2506_14781_b200 import Schedule, run_2dpt
    b, p = I.config_schedule("c1")
    tr = run_2dpt(K10, Schedule(b, p), RunConfig(total_sweeps=60, sweeps_per_swap=2, seed=4,
                                                 engine="slot"))
    o = O.run(K10, b, p, 60, 2, seed=4, rng="slot", states=True, round_counters=True)
    assert len(tr.records) == 30
    for k, rec in enumerate(tr.records):
        assert rec.round == k + 1 and rec.sweep_count == 2 * (k + 1)
        assert rec.f == o.f[k] and rec.g == o.g[k]
        np.testing.assert_array_equal(rec.state, o.states[k])
