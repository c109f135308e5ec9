"""The unfused round loop (full-grid records on one GPU; every multi-GPU run)
keeps its round counters on the device, so a chunk of rounds is one fixed
launch sequence: launched directly by default, replayed as a captured CUDA
graph with TG_GRAPHS=1.  Both must give the oracle's trajectories, including
across record-ring drains (chunks) and for the slot engine's multi-GPU
kernel path (TG_SLOT_V1)."""
import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _graphs_on(monkeypatch):
    monkeypatch.setenv("TG_GRAPHS", "1")  # the graph replay; TG_NO_GRAPHS=1 below overrides it


def unfused(pr, b, p, rounds, rule, seed, engine, grid=True, sps=1):
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(b, p)
    recs, states = [], []
    R = len(b) * len(p)

    def sink(r, n, st, ap, ab):
        for k in range(n):
            recs.append((r[k].round, r[k].f, r[k].g, r[k].digest, r[k].target_state))
        if st:
            per = R * pr.n if grid else pr.n
            states.append(np.ctypeslib.as_array(st, shape=(n * per,)).copy())
        return 0

    eng.run(RunConfig(total_sweeps=rounds * sps, sweeps_per_swap=sps, seed=seed, rule=rule, engine=engine,
                      store_states=not grid, store_target_only=not grid, digest=True), sink)
    fin = eng.grid()
    kern = eng.info()["sweep_kernel"]
    eng.close()
    return recs, np.concatenate(states) if states else None, fin, kern


@pytest.mark.parametrize("sweep", ["plane_c5_sweep_kernel", "plane_tpw_sweep_kernel"])
@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_graph_rounds_match_oracle_and_direct_launches(monkeypatch, rule, sweep):
    pr = I.bipartite_3regular(512, seed=3)
    b, p = I.config_schedule("c5")
    o = O.run(pr, b, p, 30, 1, seed=4, rule=rule, rng="plane")
    if sweep == "plane_tpw_sweep_kernel":
        monkeypatch.setenv("TG_PLANE_C5", "0")  # the thread-per-(site, word) sweep kernel
    g = unfused(pr, b, p, 30, rule, 4, "plane")
    assert g[3] == sweep
    np.testing.assert_array_equal([r[1] for r in g[0]], o.f)
    np.testing.assert_array_equal(np.array([r[3] for r in g[0]], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(g[2], o.final_grid)
    monkeypatch.setenv("TG_NO_GRAPHS", "1")
    d = unfused(pr, b, p, 30, rule, 4, "plane")
    assert g[0] == d[0]
    np.testing.assert_array_equal(g[1], d[1])
    np.testing.assert_array_equal(g[2], d[2])


def test_graph_rounds_across_ring_drains():
    # full-grid records of 16 x 16 x 512 int8 = 128 KB per round: the ring holds
    # 1024 rounds, so 1100 rounds span two chunks (two graph lengths)
    pr = I.bipartite_3regular(512, seed=5)
    b, p = I.config_schedule("c5")
    o = O.run(pr, b, p, 1100, 1, seed=9, rng="plane", final_grid=True)
    g = unfused(pr, b, p, 1100, "metropolis", 9, "plane")
    assert len(g[0]) == 1100
    np.testing.assert_array_equal([r[1] for r in g[0]], o.f)
    np.testing.assert_array_equal(np.array([r[3] for r in g[0]], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(g[2], o.final_grid)


def test_graph_rounds_slot_v1_kernels(monkeypatch):
    monkeypatch.setenv("TG_SLOT_V1", "1")
    pr = I.k10_pm1(1)
    b, p = I.config_schedule("c1")
    o = O.run(pr, b, p, 60, 1, seed=2, rng="slot")
    g = unfused(pr, b, p, 60, "metropolis", 2, "slot", grid=False)
    assert g[3].startswith("slot_sweep_kernel")
    np.testing.assert_array_equal([r[1] for r in g[0]], o.f)
    np.testing.assert_array_equal(np.array([r[3] for r in g[0]], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(g[2], o.final_grid)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_sweep_only_config5_kernel_several_sweeps_per_round(monkeypatch, rule):
    # three sweeps per launch of plane_c5_sweep_kernel (only the last one counts bonds),
    # direct launches, chain sites included
    monkeypatch.setenv("TG_GRAPHS", "0")
    pr = I.bipartite_3regular(2048, seed=8)
    b, p = I.config_schedule("c5")
    o = O.run(pr, b, p, 36, 3, seed=6, rule=rule, rng="plane")
    g = unfused(pr, b, p, 12, rule, 6, "plane", sps=3)
    assert g[3] == "plane_c5_sweep_kernel"
    np.testing.assert_array_equal([r[1] for r in g[0]], o.f)
    np.testing.assert_array_equal([r[2] for r in g[0]], o.g)
    np.testing.assert_array_equal(np.array([r[3] for r in g[0]], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(g[2], o.final_grid)
