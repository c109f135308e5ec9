"""GPU coverage of the less-travelled paths: the device instance preprocessing
(prep.cu) on inputs that force its host fallbacks, the reference's validation
messages raised through it, and the SLOT v1 engine (the multi-GPU slot path)
on one GPU.  Every run is checked against the oracle."""
import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig
from paper_2506_14781_b200.instances import ConfigError, Problem

pytestmark = pytest.mark.gpu


def run(pr, betas, pens, total, seed, engine, rule="metropolis"):
    with Engine(0) as eng:
        eng.set_problem(pr)
        eng.set_schedule(betas, pens)
        recs = []
        eng.run(RunConfig(total_sweeps=total, seed=seed, engine=engine, rule=rule, store_states=False,
                          digest=False),
                lambda r, n, s, a, b: [recs.append((r[k].f, r[k].g)) for k in range(n)] and 0, flags=0)
        grid = eng.grid()
        _, cp, _, cb = eng.counters()
    return np.array(recs), grid, cp, cb


def check(pr, betas, pens, total, seed, engine, rule="metropolis"):
    """Engine on `pr` (caller order) vs the oracle on the canonical relabel of `pr`
    (the engine equals the reference run on the relabelled instance)."""
    order, _, _ = I.canonical_order(pr)
    o = O.run(pr.permuted(order), betas, pens, total, 1, seed=seed, rule=rule,
              rng="plane" if engine == "plane" else "slot")
    recs, grid, cp, cb = run(pr, betas, pens, total, seed, engine, rule)
    np.testing.assert_array_equal(recs[:, 0], o.f)
    np.testing.assert_array_equal(recs[:, 1], o.g)
    np.testing.assert_array_equal(grid[:, np.asarray(order)], o.final_grid)
    np.testing.assert_array_equal(cp, o.accepts_p)
    np.testing.assert_array_equal(cb, o.accepts_b)


def path_graph(n, seed):
    rng = np.random.default_rng(seed)
    w = rng.choice([-1.0, 1.0], size=n - 1)
    return Problem.make(n, [(i, i + 1, float(w[i])) for i in range(n - 1)], [0.0] * n,
                        [(i, i + 3) for i in range(0, n - 3, 97)])


def test_long_dependency_chain_falls_back_to_host_colouring():
    # a path in index order: the colouring fixpoint needs ~n rounds (> the 4096
    # device budget), so set_problem finishes the canonical order on the host
    pr = path_graph(6000, 3)
    check(pr, [0.3, 1.0, 3.0], [0.0, 0.25, 0.5, 1.0] + [1.5, 2.0, 2.5, 3.0], 30, 5, "plane")


def test_short_chain_path_on_device():
    pr = path_graph(600, 4)   # within the device round budget, non-identity relabel
    check(pr, [0.3, 1.0, 3.0], [0.0, 0.5], 40, 6, "plane")
    check(pr, [0.3, 1.0, 3.0], [0.0, 0.5], 20, 6, "slot")


def test_many_colours_fall_back_to_host(monkeypatch):
    # K_70: 70 colours exceed the device colouring's 63-colour word; degree 69
    # is beyond SLOT v2's padded rows, so the CSR kernels of SLOT v1 run it
    monkeypatch.setenv("TG_SLOT_V1", "1")
    rng = np.random.default_rng(7)
    cpl = [(i, j, float(rng.choice([-1.0, 1.0]))) for i in range(70) for j in range(i + 1, 70)]
    pr = Problem.make(70, cpl, [0.0] * 70)
    check(pr, [0.05, 0.1], [0.0], 10, 3, "slot")


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_slot_v1_engine_on_one_gpu(monkeypatch, rule):
    monkeypatch.setenv("TG_SLOT_V1", "1")   # the multi-GPU SLOT kernels, single rank
    pr = I.k10_pm1(2)
    check(pr, *I.config_schedule("c1"), 60, 9, "slot", rule)
    f = I.five_node_complete()
    five = I.to_canonical(I.sparsify(5, list(zip(f.ci.tolist(), f.cj.tolist(), f.cw.tolist())),
                                     f.fields.tolist(), 2, 3))
    check(five, [0.5, 1.0, 1.5], [2.0, 4.0, 6.0], 60, 3, "slot", rule)


BAD = [
    ("self loop", Problem.make(4, [(0, 1, 1.0), (2, 2, 1.0)], [0.0] * 4)),
    ("index out of range", Problem.make(4, [(0, 1, 1.0), (1, 7, 1.0)], [0.0] * 4)),
    ("duplicate", Problem.make(4, [(0, 1, 1.0), (2, 3, 1.0), (1, 0, -1.0)], [0.0] * 4)),
    ("non-finite weight", Problem.make(4, [(0, 1, float("nan"))], [0.0] * 4)),
    ("non-finite field", Problem.make(4, [(0, 1, 1.0)], [0.0, float("inf"), 0.0, 0.0])),
    ("pair on one spin", Problem.make(4, [(0, 1, 1.0)], [0.0] * 4, [(2, 2)])),
    ("pair out of range", Problem.make(4, [(0, 1, 1.0)], [0.0] * 4, [(0, 9)])),
]


@pytest.mark.parametrize("name,pr", BAD, ids=[b[0] for b in BAD])
def test_device_validation_raises_reference_messages(name, pr):
    with Engine(0) as eng:
        with pytest.raises(ConfigError) as got:
            eng.set_problem(pr)
    if "non-finite" in name:
        # the reference accepts NaN/inf and runs into NaN energies; the engine
        # refuses them up front (its FP32 certificate needs finite fields)
        assert "must be finite" in str(got.value)
        return
    with pytest.raises(O.OracleError) as want:
        O.run(pr, [1.0], [0.5], 2, 1)
    assert str(got.value) == want.value.msg


@pytest.mark.parametrize("engine", ["slot", "plane"])
def test_degenerate_instances(engine):
    # a free spin (test_engine.cpp:23-25), isolated spins, and chains without couplings
    free = Problem.make(1, [], [0.0])
    lone = Problem.make(5, [], [0.0] * 5)
    pairs_only = Problem.make(6, [], [0.0] * 6, [(0, 3), (1, 4), (2, 5)])
    for pr in (free, lone, pairs_only):
        check(pr, [0.5, 1.0], [1.0, 2.0], 12, 4, engine)


def test_plane_full_word_budget_32x32():
    # 1024 replicas = 32 words per site row (the PLANE engine's maximum)
    pr = I.bipartite_3regular(256, seed=5)
    betas = list(np.geomspace(0.2, 5.0, 32))
    pens = [k / 64.0 for k in range(32)]
    check(pr, betas, pens, 12, 7, "plane")


def test_slot_32x32_grid():
    pr = I.wishart_planted(8, 0.5, seed=2)
    betas, pens = I.wishart_schedule(pr, 32, 32)
    order, _, _ = I.canonical_order(pr)
    o = O.run(pr.permuted(order), betas, pens, 8, 1, seed=3)
    recs, grid, cp, cb = run(pr, betas, pens, 8, 3, "slot")
    np.testing.assert_allclose(recs[:, 0], o.f, rtol=1e-9, atol=1e-9)
    np.testing.assert_array_equal(recs[:, 1], o.g)
    np.testing.assert_array_equal(grid[:, np.asarray(order)], o.final_grid)
    np.testing.assert_array_equal(cp, o.accepts_p)
    np.testing.assert_array_equal(cb, o.accepts_b)


@pytest.mark.parametrize("engine", ["slot", "plane"])
def test_record_every_decimates(engine):
    pr = I.k10_pm1(3)
    betas, pens = I.config_schedule("c1")
    o = O.run(pr, betas, pens, 30, 1, seed=4, states=True)
    if engine == "plane":
        o = O.run(pr, betas, pens, 30, 1, seed=4, states=True, rng="plane")
    with Engine(0) as eng:
        eng.set_problem(pr)
        eng.set_schedule(betas, pens)
        got = []

        def sink(r, n, states, ap, ab):
            st = np.ctypeslib.as_array(states, shape=(n * pr.n,)).reshape(n, pr.n)
            for k in range(n):
                got.append((r[k].round, r[k].f, r[k].g, st[k].copy()))
            return 0

        eng.run(RunConfig(total_sweeps=30, seed=4, engine=engine, record_every=3, store_states=True,
                          digest=False), sink)
    assert [g[0] for g in got] == list(range(3, 31, 3))
    for rnd, f, g, st in got:
        assert f == o.f[rnd - 1] and g == o.g[rnd - 1]
        np.testing.assert_array_equal(st, o.states[rnd - 1])


@pytest.mark.parametrize("engine", ["slot", "plane"])
def test_context_reuse_equals_fresh_contexts(engine):
    # one context: problem A, run, problem B, run, schedule change, run -- each
    # result must equal a fresh context's (buffers are pooled and re-sized)
    a, b = I.k10_pm1(1), I.bipartite_3regular(64, seed=2)
    sa, sb = I.config_schedule("c1"), ([0.3, 1.0, 2.0], [0.0, 0.25])
    runs = [(a, sa, 20, 1), (b, sb, 16, 2), (b, ([0.5, 1.5], [0.0, 0.5, 1.0]), 10, 3), (a, sa, 20, 1)]

    def once(eng, pr, sc, total, seed):
        eng.set_problem(pr)
        eng.set_schedule(*sc)
        recs = []
        eng.run(RunConfig(total_sweeps=total, seed=seed, engine=engine, store_states=False, digest=True),
                lambda r, n, s, x, y: [recs.append((r[k].f, r[k].g, r[k].digest)) for k in range(n)] and 0)
        return recs, eng.grid()

    with Engine(0) as eng:
        shared = [once(eng, *r) for r in runs]
    for r, (recs, grid) in zip(runs, shared):
        with Engine(0) as eng:
            fresh_recs, fresh_grid = once(eng, *r)
        assert recs == fresh_recs
        np.testing.assert_array_equal(grid, fresh_grid)


def test_large_key_range_run_list_read_back_in_two_steps(monkeypatch):
    # a hub of cost degree 34 and chain degree 31 on n = 70000 sites: the
    # (colour, dq, dc) key range 64*32*35 and n both exceed kPrepEagerRuns, so
    # device prep reads the run count before the run list (prep.cu); the
    # merged degree needs the CSR kernels of SLOT v1
    monkeypatch.setenv("TG_SLOT_V1", "1")
    n = 70000
    rng = np.random.default_rng(12)
    perm = rng.permutation(n)
    w = rng.choice([-1.0, 1.0], size=n + 32)
    cpl = [(int(perm[k]), int(perm[k + 1]), float(w[k])) for k in range(n - 1)]
    hub = int(perm[n // 2])
    others = [int(v) for v in rng.choice(n, size=200, replace=False) if int(v) != hub]
    path_nb = {int(perm[n // 2 - 1]), int(perm[n // 2 + 1])}
    others = [v for v in others if v not in path_nb]
    cpl += [(hub, v, float(w[n + k])) for k, v in enumerate(others[:32])]
    pairs = [(hub, v) for v in others[32:63]]
    pr = Problem.make(n, cpl, [0.0] * n, pairs)
    check(pr, [0.3, 2.0], [0.0, 0.5], 4, 9, "slot")
