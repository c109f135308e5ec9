"""Config-5 parity at the bench's own size (N = 2^20, 16x16 grid) through
size-independent properties -- the oracle cannot replay 2.7e8 updates per
sweep in test time -- plus exact oracle parity at N = 2^14 (the smallest
config-5 size) on both update rules.

Properties at 2^20: (1) every record's (f, g) equals the energy and
constraint value recomputed on the host from the reported state of the target
replica; (2) two runs with the same seed are identical (state digests), a
different seed differs; (3) resuming in pieces equals one run; (4) every slot's
final state has the (f, g) the engine reports for it."""
import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig

pytestmark = pytest.mark.gpu


def energy(pr, s):
    s = s.astype(np.int64)
    f = -np.sum(pr.cw * s[pr.ci] * s[pr.cj]) - np.sum(pr.fields * s)
    g = np.sum((s[pr.pa] - s[pr.pb]) ** 2)
    return float(f), float(g)


@pytest.fixture(scope="module")
def big():
    return I.bipartite_3regular(1 << 20, seed=1), I.config_schedule("c5")


def records(eng, cfg, n_rounds=None):
    out = []

    def sink(r, n, states, ap, ab):
        st = np.ctypeslib.as_array(states, shape=(n * eng.problem.n,)).reshape(n, -1) if states else None
        for k in range(n):
            out.append((r[k].round, r[k].f, r[k].g, r[k].digest, None if st is None else st[k].copy()))
        return 0

    if n_rounds is None:
        eng.run(cfg, sink)
    else:
        eng.advance(n_rounds, sink)
    return out


def test_records_match_reported_states_at_full_size(big):
    pr, (betas, pens) = big
    with Engine(0) as eng:
        eng.set_problem(pr)
        eng.set_schedule(betas, pens)
        recs = records(eng, RunConfig(total_sweeps=6, seed=11, engine="plane", store_states=True))
        assert len(recs) == 6
        for rnd, f, g, dig, st in recs:
            assert (f, g) == energy(pr, st)
            assert dig == O.digest(st)
        # every slot's final state carries the (f, g) of the last round's energies
        fs, gs = eng.energies()
        grid = eng.grid()
        for slot in range(0, 256, 37):
            assert (fs[slot], gs[slot]) == energy(pr, grid[slot])


def test_determinism_and_resume_at_full_size(big):
    pr, (betas, pens) = big

    def digests(seed, pieces):
        with Engine(0) as eng:
            eng.set_problem(pr)
            eng.set_schedule(betas, pens)
            cfg = RunConfig(total_sweeps=8, seed=seed, engine="plane", store_states=False, digest=True)
            if pieces == 1:
                return [r[3] for r in records(eng, cfg)]
            eng.init(cfg)
            return [r[3] for k in (3, 5) for r in records(eng, cfg, k)]

    a = digests(21, 1)
    assert a == digests(21, 1)
    assert a == digests(21, 2)
    assert a != digests(22, 1)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_oracle_parity_config5_smallest_size(rule):
    pr = I.bipartite_3regular(1 << 14, seed=1)
    betas, pens = I.config_schedule("c5")
    o = O.run(pr, betas, pens, 4, 1, seed=5, rule=rule, rng="plane")
    with Engine(0) as eng:
        eng.set_problem(pr)
        eng.set_schedule(betas, pens)
        recs = records(eng, RunConfig(total_sweeps=4, seed=5, rule=rule, engine="plane",
                                      store_states=False, digest=True))
        grid = eng.grid()
        _, cp, _, cb = eng.counters()
    np.testing.assert_array_equal([r[1] for r in recs], o.f)
    np.testing.assert_array_equal([r[2] for r in recs], o.g)
    np.testing.assert_array_equal(np.array([r[3] for r in recs], np.uint64), o.digest)
    np.testing.assert_array_equal(grid, o.final_grid)
    np.testing.assert_array_equal(cp, o.accepts_p)
    np.testing.assert_array_equal(cb, o.accepts_b)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_bond_counters_beyond_one_flush_period(rule):
    """2^21 sites x 1024 hot replicas: a warp of the config-5 kernel walks ~200
    two-site items per colour phase, each adding up to 3 unsatisfied bonds
    (~1.5 on average at beta = 0.01) to its 8-plane vertical counters, i.e.
    past 255 without the periodic flush.  Every record's (f, g) must equal the
    energy recomputed from the reported target state."""
    pr = I.bipartite_3regular(1 << 21, seed=3)
    betas = I.linear(0.01, 0.02, 32)
    pens = I.dyadic(I.linear(0.0, 1.0, 32))
    with Engine(0) as eng:
        eng.set_problem(pr)
        eng.set_schedule(betas, pens)
        recs = records(eng, RunConfig(total_sweeps=3, seed=4, rule=rule, engine="plane", store_states=True))
        assert eng.info()["sweep_kernel"] == "plane_c5_rounds_kernel"
        assert len(recs) == 3
        for rnd, f, g, dig, st in recs:
            assert (f, g) == energy(pr, st)
            assert dig == O.digest(st)
