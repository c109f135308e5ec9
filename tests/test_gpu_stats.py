"""Statistical parity on the B200 engine: every replica's stationary marginal
against exact enumeration (test_engine.cpp:180-212; acceptance criterion 1,
acceptance.cpp:46-90), TV <= 0.02 as in the reference, for both engines and
both update rules."""
import numpy as np
import pytest

from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig

pytestmark = pytest.mark.gpu


def exact(pr, beta, penalty):
    n = pr.n
    states = ((np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1) * 2 - 1
    e = np.zeros(1 << n)
    for i, j, w in zip(pr.ci, pr.cj, pr.cw):
        e -= w * states[:, i] * states[:, j]
    e -= states @ pr.fields
    g = np.zeros(1 << n)
    for a, b in zip(pr.pa, pr.pb):
        g += (states[:, a] - states[:, b]) ** 2
    t = e + penalty * g
    w = np.exp(-beta * (t - t.min()))
    return w / w.sum()


def grid_run(pr, betas, pens, total, sps, seed, rule, engine):
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(betas, pens)
    R = len(betas) * len(pens)
    chunks = []

    def sink(recs, cnt, states, ap, ab):
        chunks.append(np.ctypeslib.as_array(states, shape=(cnt * R * pr.n,)).copy())
        return 0

    cfg = RunConfig(total_sweeps=total, sweeps_per_swap=sps, seed=seed, rule=rule, engine=engine,
                    store_target_only=False, store_states=False, digest=False)
    eng.run(cfg, sink)
    eng.close()
    return np.concatenate(chunks).reshape(-1, R, pr.n)


def max_tv(pr, betas, pens, grid, burn):
    weights = 1 << np.arange(pr.n)
    enc = ((grid[burn:] > 0).astype(np.int64) * weights).sum(axis=2)
    tvs = []
    for i, b in enumerate(betas):
        for j, p in enumerate(pens):
            h = np.bincount(enc[:, i * len(pens) + j], minlength=1 << pr.n) / enc.shape[0]
            tvs.append(0.5 * np.abs(h - exact(pr, b, p)).sum())
    return max(tvs)


def crit1_problem():
    return I.to_canonical(I.sparsify(3, [(0, 1, 1.2), (0, 2, -1.5), (1, 2, 0.9)],
                                     [0.4, -0.3, 0.5], 3, 3))


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_slot_engine_criterion1_marginals(rule):
    pr = crit1_problem()
    betas, pens = [0.8, 1.0, 1.25], [1.0, 2.0, 4.0]
    grid = grid_run(pr, betas, pens, 2_000_000, 10, 11, rule, "slot")  # acceptance.cpp:57-60
    assert max_tv(pr, betas, pens, grid, grid.shape[0] // 10) <= 0.02


def pm1_problem():
    # 5 spins, J = +-1 frustrated couplings and two copy-chain pairs: plane-engine
    # eligible, 32 states (the reference's own fixture has 4, test_engine.cpp:27-30)
    cpl = [(0, 1, 1.0), (1, 2, -1.0), (2, 3, 1.0), (3, 0, 1.0), (1, 4, -1.0)]
    pr = I.Problem.make(5, cpl, [0.0] * 5, [(0, 2), (3, 4)])
    return I.to_canonical(pr)


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_plane_engine_replica_marginals(rule):
    pr = pm1_problem()
    betas, pens = [0.4, 0.9], [0.25, 0.75]
    grid = grid_run(pr, betas, pens, 400_000, 5, 31, rule, "plane")  # test_engine.cpp:184-187
    assert max_tv(pr, betas, pens, grid, grid.shape[0] // 10) <= 0.02


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_float_engine_criterion1_marginals(rule):
    # the FLOAT engine (packed draws, certified FP32 decisions) on the
    # reference's float criterion-1 instance: every replica's marginal, TV <= 0.02
    pr = crit1_problem()
    betas, pens = [0.8, 1.0, 1.25], [1.0, 2.0, 4.0]
    grid = grid_run(pr, betas, pens, 2_000_000, 10, 13, rule, "float")
    assert max_tv(pr, betas, pens, grid, grid.shape[0] // 10) <= 0.02


def test_float_engine_energy_histograms_match_reference():
    """Float Wishart instance: the target replica's energy and feasibility
    statistics of the FLOAT engine and of the unmodified reference (O1:
    mt19937_64, oracle/_ref) are statistically indistinguishable (the
    float-instance contract of BASELINE.json north_star)."""
    import pyoracle as O
    from scipy import stats
    if not O.ref_available("mt"):
        pytest.skip("reference build (oracle/_ref) not present")
    pr = I.wishart_planted(8, 0.5, seed=4)
    betas, pens = I.wishart_schedule(pr, 4, 4)
    total, burn = 60_000, 5_000
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(betas, pens)
    rec = []

    def sink(r, n, states, ap, ab):
        for k in range(n):
            rec.append((r[k].f, r[k].feasible))
        return 0

    eng.run(RunConfig(total_sweeps=total, sweeps_per_swap=1, seed=5, engine="float",
                      store_states=False, digest=False), sink)
    eng.close()
    f_gpu = np.array([x[0] for x in rec])[burn:]
    fe_gpu = np.array([x[1] for x in rec], dtype=float)[burn:]
    o = O.run(pr, betas, pens, total, 1, seed=6, impl="ref:mt", final_grid=False)
    f_ref, fe_ref = o.f[burn:], o.feasible[burn:].astype(float)
    # observables: feasibility, energy moments and the occupancy of the pooled
    # energy distribution's quantile bins; each compared by a Welch t test on
    # 50 batch means per trajectory (batches much longer than the
    # autocorrelation time, so the batch means are nearly independent)
    edges = np.quantile(np.concatenate([f_gpu, f_ref]), [0.125 * k for k in range(1, 8)])

    def observables(f, fe):
        obs = [fe, f, f * f]
        bins = np.searchsorted(edges, f, side="right")
        obs += [(bins == k).astype(float) for k in range(8)]
        return np.stack(obs)

    def batch_means(x, nb=50):
        m = x.shape[1] // nb
        return x[:, :m * nb].reshape(x.shape[0], nb, m).mean(axis=2)

    bg = batch_means(observables(f_gpu, fe_gpu))
    br = batch_means(observables(f_ref, fe_ref))
    t = stats.ttest_ind(bg, br, axis=1, equal_var=False)
    tstat = np.nan_to_num(t.statistic, nan=0.0)  # constant observables (e.g. always feasible)
    names = ["feasible", "f", "f^2"] + [f"bin{k}" for k in range(8)]
    assert np.all(np.abs(tstat) < 4.5), dict(zip(names, np.round(tstat, 2)))
