"""Checkpoint / resume (tg_checkpoint, tg_restore; the reference has no resume,
engine.hpp:39-56): a run stopped after k rounds, snapshotted, restored into a
fresh context (same problem, schedule, config) and advanced to the end gives
the uninterrupted run's records and final grid bit for bit -- on every
single-GPU engine (fused PLANE kernels, SLOT v2, FLOAT) -- and a checkpoint of
another problem or seed is refused."""
import numpy as np
import pytest

from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, EngineError, RunConfig

pytestmark = pytest.mark.gpu

CASES = {
    "plane_c5": (lambda: I.bipartite_3regular(4096, seed=3), lambda pr: I.config_schedule("c5"), "plane"),
    "plane_k10": (lambda: I.k10_pm1(1), lambda pr: I.config_schedule("c1"), "plane"),
    "slot": (lambda: I.wishart_planted(12, 0.5, seed=2), lambda pr: I.wishart_schedule(pr, 4, 4), "slot"),
    "float": (lambda: I.wishart_planted(12, 0.5, seed=2), lambda pr: I.wishart_schedule(pr, 4, 4), "float"),
}


def make(pr, b, p, engine, total, rule="metropolis"):
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(b, p)
    eng.init(RunConfig(total_sweeps=total, sweeps_per_swap=1, seed=11, rule=rule, engine=engine,
                       store_states=False, digest=True))
    return eng


def records(eng, n):
    out = []

    def sink(r, k, st, ap, ab):
        for q in range(k):
            out.append((r[q].round, r[q].f, r[q].g, r[q].digest, r[q].target_state))
        return 0

    eng.advance(n, sink)
    return out


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
@pytest.mark.parametrize("name", list(CASES))
def test_restore_continues_bit_for_bit(name, rule):
    mk, sch, engine = CASES[name]
    pr = mk()
    b, p = sch(pr)
    full = make(pr, b, p, engine, 40, rule)
    ref = records(full, 40)
    ref_grid = full.grid()
    ref_ctr = full.counters()
    full.close()
    first = make(pr, b, p, engine, 40, rule)
    head = records(first, 17)
    blob = first.checkpoint()
    first.close()
    second = make(pr, b, p, engine, 40, rule)
    second.restore(blob)
    tail = records(second, 23)
    assert head + tail == ref
    np.testing.assert_array_equal(second.grid(), ref_grid)
    for x, y in zip(second.counters(), ref_ctr):
        np.testing.assert_array_equal(x, y)
    second.close()


def test_restore_refuses_another_run():
    pr = I.k10_pm1(1)
    b, p = I.config_schedule("c1")
    e1 = make(pr, b, p, "plane", 10)
    records(e1, 5)
    blob = e1.checkpoint()
    e1.close()
    e2 = Engine(0)
    e2.set_problem(pr)
    e2.set_schedule(b, p)
    e2.init(RunConfig(total_sweeps=10, seed=12, engine="plane"))
    with pytest.raises(Exception):
        e2.restore(blob)
    with pytest.raises(Exception):
        e2.restore(blob[:100])
    e2.close()
