"""GPU parity of the FLOAT engine (slot_fast.cu): float-coupling instances
with packed draws keyed by physical replica (oracle/philox_ref.h
tgo_pack_u53), certified FP32 decisions with an FP64 fallback, fixed-point
energies.  Compared with the oracle's "float" RNG association (itself pinned
to the reference sources compiled with the same draws, tests/test_oracle_ref.py):
decisions, g, feasibility, state digests, final grids and swap counters
exactly; f within 1e-9 relative (2^-40 fixed-point energy sums versus the
reference's FP64 merged-model sums)."""
import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig, Schedule, batch_state, run_2dpt_batch

pytestmark = pytest.mark.gpu


def run_float(pr, betas, pens, total, sps, seed, rule="metropolis"):
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(betas, pens)
    recs = []

    def sink(r, n, states, ap, ab):
        for k in range(n):
            recs.append((r[k].f, r[k].g, r[k].feasible, r[k].digest))
        return 0

    eng.run(RunConfig(total_sweeps=total, sweeps_per_swap=sps, seed=seed, rule=rule, engine="float",
                      store_states=False, digest=True), sink)
    info = eng.info()
    grid = eng.grid()
    ctr = eng.counters()
    eng.close()
    return recs, grid, ctr, info


def check(pr, betas, pens, total, sps, seed, rule="metropolis"):
    o = O.run(pr, betas, pens, total, sps, seed=seed, rule=rule, rng="float")
    recs, grid, (ap, cp, ab, cb), info = run_float(pr, betas, pens, total, sps, seed, rule)
    assert info["sweep_kernel"] == "slotf_sweep_kernel"
    assert len(recs) == total // sps
    np.testing.assert_allclose([r[0] for r in recs], o.f, rtol=1e-9, atol=1e-9)
    np.testing.assert_array_equal([r[1] for r in recs], o.g)
    np.testing.assert_array_equal([bool(r[2]) for r in recs], o.feasible)
    np.testing.assert_array_equal(np.array([r[3] for r in recs], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(grid, o.final_grid)
    np.testing.assert_array_equal(cp, o.accepts_p)
    np.testing.assert_array_equal(cb, o.accepts_b)
    np.testing.assert_array_equal(ap, o.attempts_p)
    np.testing.assert_array_equal(ab, o.attempts_b)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_float_wishart_small(rule):
    pr = I.wishart_planted(8, 0.5, seed=4)
    b, p = I.wishart_schedule(pr, 4, 4)
    check(pr, b, p, 100, 1, seed=3, rule=rule)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_float_config2_full_size(rule):
    pr = I.wishart_planted(32, 0.5, seed=1)  # 928 spins, 16 x 8 (Rp = 128: two sites per warp item)
    b, p = I.wishart_schedule(pr, 16, 8)
    check(pr, b, p, 200, 1, seed=21, rule=rule)


def test_float_config2_sps50():
    pr = I.wishart_planted(32, 0.5, seed=2)
    b, p = I.wishart_schedule(pr, 16, 8)
    check(pr, b, p, 50 * 6, 50, seed=4)


@pytest.mark.parametrize("grid", [(3, 5), (4, 8), (16, 16), (32, 32)])
def test_float_replica_layouts(grid):
    # Rp = 32 (8 sites per warp item), 32, 256 (one site), 1024 (4 group sets)
    pr = I.wishart_planted(16, 0.5, seed=7)
    b, p = I.wishart_schedule(pr, *grid)
    check(pr, b, p, 30, 1, seed=5)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_float_fields_and_dyadic_instance(rule):
    five = I.five_node_complete()
    pr = I.to_canonical(I.sparsify(5, list(zip(five.ci.tolist(), five.cj.tolist(), five.cw.tolist())),
                                   five.fields.tolist(), 2, 3))
    check(pr, [0.5, 1.0, 1.5], [2.0, 4.0, 6.0, 8.0], 400, 5, seed=77, rule=rule)


def test_float_higher_degree():
    # K10 sparsified with degree <= 6: the padded degree-8 kernel
    check(I.k10_pm1(1), *I.config_schedule("c1"), 200, 1, seed=5)


def test_float_config4_full_size():
    pr = I.wishart_planted(256, 0.5, seed=1)
    b, p = I.wishart_schedule(pr, 32, 32)
    o = O.run(pr, b, p, 6, 1, seed=8, rng="float", threads=16)
    recs, grid, (ap, cp, ab, cb), info = run_float(pr, b, p, 6, 1, 8)
    np.testing.assert_allclose([r[0] for r in recs], o.f, rtol=1e-9)
    np.testing.assert_array_equal(np.array([r[3] for r in recs], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(grid, o.final_grid)


def test_float_batch_config3_subset():
    prs = [I.wishart_planted(64, 0.75, seed=s) for s in range(1, 9)]
    scheds = [Schedule(*I.wishart_schedule(p, 16, 16)) for p in prs]
    seeds = [40 + s for s in range(8)]
    eng = Engine(0)
    traces = run_2dpt_batch(prs, scheds, RunConfig(total_sweeps=12, engine="float", store_states=True),
                            seeds, engine=eng)
    for b in range(8):
        o = O.run(prs[b], scheds[b].betas, scheds[b].penalties, 12, 1, seed=seeds[b], rng="float",
                  states=True)
        tr = traces[b]
        np.testing.assert_allclose([r.f for r in tr.records], o.f, rtol=1e-9)
        np.testing.assert_array_equal([r.g for r in tr.records], o.g)
        np.testing.assert_array_equal(np.stack([r.state for r in tr.records]), o.states)
        if b in (0, 7):
            grid = np.stack([batch_state(eng, b, s, prs[b].n) for s in range(256)])
            np.testing.assert_array_equal(grid, o.final_grid)
    eng.close()
