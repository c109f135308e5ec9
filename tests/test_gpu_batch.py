"""Batched instances (config 3, SURVEY.md §8b run_2dpt_batch): one launch over
several independent instances must equal independent runs instance by
instance -- here checked against the oracle's per-instance trajectories
(the reference's run_2dpt semantics with Philox draws)."""
import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig, Schedule, batch_state, run_2dpt_batch

pytestmark = pytest.mark.gpu


def small_batch():
    prs = [I.k10_pm1(1), I.k10_pm1(2), I.wishart_planted(6, 0.5, seed=3),
           I.to_canonical(I.sparsify(3, [(0, 1, 1.2), (0, 2, -1.5), (1, 2, 0.9)], [0.4, -0.3, 0.5], 3, 3))]
    scheds = [Schedule([0.3, 1.0, 3.0], [0.0, 0.5, 1.0]), Schedule([0.2, 0.7, 2.0], [0.0, 0.25, 0.5]),
              Schedule([0.2, 1.0, 5.0], [0.0, 0.1, 0.3]), Schedule([0.8, 1.0, 1.25], [1.0, 2.0, 4.0])]
    return prs, scheds, [5, 6, 7, 8]


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_batch_equals_independent_runs(rule):
    prs, scheds, seeds = small_batch()
    eng = Engine(0)
    traces = run_2dpt_batch(prs, scheds, RunConfig(total_sweeps=120, sweeps_per_swap=2, rule=rule,
                                                   store_states=True), seeds, engine=eng)
    for b, (pr, sc, sd) in enumerate(zip(prs, scheds, seeds)):
        o = O.run(pr, sc.betas, sc.penalties, 120, 2, seed=sd, rule=rule, rng="slot", states=True)
        tr = traces[b]
        assert len(tr.records) == 60
        exact = np.all(np.abs(pr.cw) == np.round(np.abs(pr.cw)))
        f = np.array([r.f for r in tr.records])
        if exact:
            np.testing.assert_array_equal(f, o.f)
        else:
            np.testing.assert_allclose(f, o.f, rtol=1e-9, atol=1e-9)
        np.testing.assert_array_equal([r.g for r in tr.records], o.g)
        np.testing.assert_array_equal(np.array([r.digest for r in tr.records], dtype=np.uint64), o.digest)
        np.testing.assert_array_equal(np.stack([r.state for r in tr.records]), o.states)
        grid = np.stack([batch_state(eng, b, s, pr.n) for s in range(9)])
        np.testing.assert_array_equal(grid, o.final_grid)
    eng.close()


def test_batch_rejects_mixed_grid_shapes():
    prs, scheds, seeds = small_batch()
    scheds[1] = Schedule([0.2, 2.0], [0.0, 0.25, 0.5])
    with pytest.raises(I.ConfigError):
        run_2dpt_batch(prs, scheds, RunConfig(total_sweeps=10), seeds)


def test_config3_shape_batch_runs():
    # 8 Wishart N=16 instances (config-3 style, reduced), 16x16 grids each
    prs = [I.wishart_planted(16, 0.75, seed=s) for s in range(1, 9)]
    scheds = [Schedule(*I.wishart_schedule(p, 16, 16)) for p in prs]
    counts = {}

    def sink(b, recs, n, states, ap, ab):
        counts[b] = counts.get(b, 0) + n
        return 0

    run_2dpt_batch(prs, scheds, RunConfig(total_sweeps=20, store_states=False, digest=False),
                   list(range(8)), sink=sink)
    assert counts == {b: 20 for b in range(8)}


def test_batch_duplicate_graph_other_schedule():
    """Two consecutive instances with the same graph but different schedules
    (the second with larger beta and P): the duplicate's preparation is
    reused, its FP32 error bands must follow its own schedule."""
    pr = I.wishart_planted(12, 0.5, seed=9)
    scheds = [Schedule([0.2, 0.5, 1.0], [0.0, 0.1, 0.2]), Schedule([0.5, 3.0, 9.0], [0.5, 2.0, 6.0])]
    seeds = [3, 4]
    traces = run_2dpt_batch([pr, pr], scheds, RunConfig(total_sweeps=150, sweeps_per_swap=1,
                                                        store_states=True), seeds)
    for b in range(2):
        o = O.run(pr, scheds[b].betas, scheds[b].penalties, 150, 1, seed=seeds[b], rng="slot",
                  states=True)
        np.testing.assert_allclose([r.f for r in traces[b].records], o.f, rtol=1e-9, atol=1e-9)
        np.testing.assert_array_equal(np.stack([r.state for r in traces[b].records]), o.states)
