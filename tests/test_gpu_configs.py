"""GPU parity at the BASELINE.json configurations' real sizes (VERDICT r1,
"next round" item 1).  Each case runs the B200 engine through the C ABI and
the C port of the reference hot path (oracle/tg_oracle.c, pinned to the
reference sources in tests/test_oracle_ref.py) on the same instance, schedule
and seed, and compares every round's target record:

* config 2 (Wishart N=32 -> 928 spins, 16x8 grid), float32 couplings;
* config 3 (64 Wishart N=64 -> 3904 spins, 16x16 grids each, one batch);
* config 4 (Wishart N=256 -> 64768 spins, 32x32 grid);
* config 5 (bipartite 3-regular, N = 2^18, 16x16 grid), bit-plane engine.

Float instances: f within 1e-9 relative (the FP64 bookkeeping of both sides
sums the same float32 couplings in different orders), g / feasibility /
state digests / final configurations exact.  The trajectories themselves are
exact because both sides take the same decisions (reference.cpp
mc.cpp:21-35 with Philox draws).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig, Schedule, batch_state, run_2dpt_batch

pytestmark = pytest.mark.gpu

THREADS = max(1, min(os.cpu_count() or 1, 64))


def engine_trace(pr, betas, pens, total, sps, seed, rule="metropolis", engine="slot"):
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(betas, pens)
    recs = []

    def sink(r, n, states, ap, ab):
        for k in range(n):
            recs.append((r[k].f, r[k].g, r[k].feasible, r[k].digest))
        return 0

    eng.run(RunConfig(total_sweeps=total, sweeps_per_swap=sps, seed=seed, rule=rule, engine=engine,
                      store_states=False, digest=True), sink)
    grid = eng.grid()
    ctr = eng.counters()
    eng.close()
    f = np.array([r[0] for r in recs])
    g = np.array([r[1] for r in recs])
    fe = np.array([bool(r[2]) for r in recs])
    dg = np.array([r[3] for r in recs], dtype=np.uint64)
    return f, g, fe, dg, grid, ctr


def check(o, f, g, fe, dg, grid=None, ctr=None, exact_f=False):
    if exact_f:
        np.testing.assert_array_equal(f, o.f)
    else:
        np.testing.assert_allclose(f, o.f, rtol=1e-9, atol=1e-9)
    np.testing.assert_array_equal(g, o.g)
    np.testing.assert_array_equal(fe, o.feasible)
    np.testing.assert_array_equal(dg, o.digest)
    if grid is not None:
        np.testing.assert_array_equal(grid, o.final_grid)
    if ctr is not None:
        ap, cp, ab, cb = ctr
        np.testing.assert_array_equal(ap, o.attempts_p)
        np.testing.assert_array_equal(cp, o.accepts_p)
        np.testing.assert_array_equal(ab, o.attempts_b)
        np.testing.assert_array_equal(cb, o.accepts_b)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_config2_full_size(rule):
    pr = I.wishart_planted(32, 0.5, seed=1)
    assert pr.n == 928
    b, p = I.wishart_schedule(pr, 16, 8)
    o = O.run(pr, b, p, 200, 1, seed=21, rule=rule, rng="slot", threads=THREADS)
    check(o, *engine_trace(pr, b, p, 200, 1, 21, rule))


def test_config2_full_size_sps50():
    pr = I.wishart_planted(32, 0.5, seed=2)
    b, p = I.wishart_schedule(pr, 16, 8)
    o = O.run(pr, b, p, 50 * 12, 50, seed=4, rng="slot", threads=THREADS)
    check(o, *engine_trace(pr, b, p, 50 * 12, 50, 4))


def test_config3_full_batch():
    """64 instances x 3904 spins x 16x16 grids, 20 rounds, one batch launch:
    every instance's digests / f / g against its own oracle run, the full
    target trajectories of four instances, and their final grids."""
    prs = [I.wishart_planted(64, 0.75, seed=s) for s in range(1, 65)]
    assert all(p.n == 3904 for p in prs)
    scheds = [Schedule(*I.wishart_schedule(p, 16, 16)) for p in prs]
    seeds = [100 + s for s in range(64)]
    full = {0, 17, 42, 63}
    eng = Engine(0)
    traces = run_2dpt_batch(prs, scheds, RunConfig(total_sweeps=20, store_states=True), seeds,
                            engine=eng)

    def oracle(b):
        return O.run(prs[b], scheds[b].betas, scheds[b].penalties, 20, 1, seed=seeds[b],
                     rng="slot", states=b in full, final_grid=b in full)

    with ThreadPoolExecutor(THREADS) as ex:
        outs = list(ex.map(oracle, range(64)))
    for b, o in enumerate(outs):
        tr = traces[b]
        f = np.array([r.f for r in tr.records])
        g = np.array([r.g for r in tr.records])
        fe = np.array([r.feasible for r in tr.records])
        dg = np.array([r.digest for r in tr.records], dtype=np.uint64)
        check(o, f, g, fe, dg)
        if b in full:
            np.testing.assert_array_equal(np.stack([r.state for r in tr.records]), o.states)
            grid = np.stack([batch_state(eng, b, s, prs[b].n) for s in range(256)])
            np.testing.assert_array_equal(grid, o.final_grid)
    eng.close()


def test_config4_full_size():
    pr = I.wishart_planted(256, 0.5, seed=1)
    assert pr.n == 64768
    b, p = I.wishart_schedule(pr, 32, 32)
    o = O.run(pr, b, p, 10, 1, seed=8, rng="slot", threads=THREADS)
    check(o, *engine_trace(pr, b, p, 10, 1, 8))


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_config5_2p18_exact(rule):
    """The bench kernel's path (fused bit-plane rounds) at N = 2^18, 20 rounds:
    f / g / digests / counters / final grid bit for bit."""
    pr = I.bipartite_3regular(1 << 18, seed=1)
    b, p = I.config_schedule("c5")
    o = O.run(pr, b, p, 20, 1, seed=13, rule=rule, rng="plane", threads=THREADS)
    check(o, *engine_trace(pr, b, p, 20, 1, 13, rule, engine="plane"), exact_f=True)
