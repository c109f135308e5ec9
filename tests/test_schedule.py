"""Schedule probes and the adaptive (beta, P) ladder (schedule.cpp:18-163;
SURVEY.md §8f row 2).  Golden vectors come from the reference's own
probe_population / build_schedule (tools/gen_golden_schedule.py ->
tests/golden/schedule.json, canonical-order instances); the C port replays
them on the CPU, the B200 engine (all chains of a probe in one cooperative
launch, moments pooled on the device) on the GPU."""
import itertools
import json
import os

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200.instances import Problem

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedule.json")))
STAT_KEYS = ("row", "column", "beta", "penalty", "sigma_e", "sigma_g", "mean_g")


def inst(name):
    i = FIX["instances"][name]
    return Problem(i["n"], np.array(i["ci"], np.int32), np.array(i["cj"], np.int32),
                   np.array(i["cw"]), np.array(i["fields"]), np.array(i["pa"], np.int32),
                   np.array(i["pb"], np.int32))


def dyadic(name):
    i = FIX["instances"][name]
    return all((64 * float(x)).is_integer() for x in i["cw"] + i["fields"])


def same_stats(got, want, exact):
    for k in STAT_KEYS:
        g, w = float(got[k]), float(want[k])
        if exact:
            assert g == w, (k, g, w)
        else:
            assert g == pytest.approx(w, rel=1e-9, abs=1e-12), (k, g, w)


def dyadic_value(x):
    return (1024 * float(x)).is_integer()


PIDS = [f"{p['instance']}-{p['rule']}-b{p['beta']}" for p in FIX["probes"]]
LIDS = [f"{l['instance']}-{l['rule']}-{k}" for k, l in enumerate(FIX["ladders"])]


@pytest.mark.parametrize("p", FIX["probes"], ids=PIDS)
def test_port_replays_reference_probes(p):
    st = O.probe_population(inst(p["instance"]), p["beta"], p["penalty"], p["n_chains"], p["sweeps"],
                            p["seed"], rule=p["rule"])
    same_stats(st, p["stats"], exact=True)  # the port sweeps in index order like the reference


@pytest.mark.parametrize("lad", FIX["ladders"], ids=LIDS)
def test_port_replays_reference_ladders(lad):
    b, pens, stats, ex = O.build_schedule(inst(lad["instance"]), rule=lad["rule"], **lad["config"])
    assert b.tolist() == lad["betas"] and pens.tolist() == lad["penalties"]
    assert ex == lad["budget_exhausted"] and len(stats) == len(lad["probe_stats"])
    for s, w in zip(stats, lad["probe_stats"]):
        same_stats(s, w, exact=True)


def test_port_reference_contracts():
    # test_schedule.cpp:58-74 and :146-157 on the port
    flat = Problem(4, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(4),
                   np.zeros(0, np.int32), np.zeros(0, np.int32))
    st = O.probe_population(flat, 1.0, 1.0, 8, 100, 1)
    assert st["sigma_e"] == 0.0 and st["sigma_g"] == 0.0 and st["mean_g"] == 0.0
    five = inst("five_spin")
    with pytest.raises(O.OracleError, match="2 chains"):
        O.probe_population(five, 1.0, 1.0, 1, 100, 1)
    with pytest.raises(O.OracleError, match="2 sweeps"):
        O.probe_population(five, 1.0, 1.0, 8, 1, 1)
    for bad, msg in ((dict(beta0=0.0), "beta0"), (dict(alpha_p=0.0), "learning rates"),
                     (dict(i_max=50, j_max=50), "replica budget")):
        with pytest.raises(O.OracleError, match=msg):
            O.build_schedule(five, **bad)


def test_ladder_invariants_on_port():
    # test_schedule.cpp:76-144: monotone ladders, budget, stopping rule
    lad = FIX["ladders"][2]
    b, p, stats, ex = O.build_schedule(inst(lad["instance"]), **lad["config"])
    assert len(p) >= 2 and np.all(np.diff(p) > 0) and np.all(np.diff(b) > 0)
    assert len(b) * len(p) <= 400
    if not ex:
        assert stats[-1]["column"] == len(p) - 1 and stats[-1]["mean_g"] < 0.5
    chain = FIX["ladders"][0]
    b, p, stats, ex = O.build_schedule(inst("chain6"), **chain["config"])
    assert p.tolist() == [0.5] and not ex and len(b) >= 2 and b[0] == 0.3
    assert stats[-1]["sigma_e"] <= 0.5 * np.sqrt(6.0) + 1e-12


# ------------------------------------------------------------------- GPU


def exact_moments(pr, beta, penalty):
    """Exact <E>, var E, <g>, var g at (beta, P) by enumeration (test_schedule.cpp:44-56)."""
    n = pr.n
    S = np.array(list(itertools.product([-1, 1], repeat=n)), dtype=np.float64)
    f = -(S @ pr.fields) - np.sum(pr.cw * S[:, pr.ci] * S[:, pr.cj], axis=1)
    g = np.sum((S[:, pr.pa] - S[:, pr.pb]) ** 2, axis=1)
    E = f + penalty * g
    w = np.exp(-beta * (E - E.min()))
    w /= w.sum()
    mE, mg = w @ E, w @ g
    return mE, w @ (E - mE) ** 2, mg, w @ (g - mg) ** 2


@pytest.mark.gpu
@pytest.mark.parametrize("p", FIX["probes"], ids=PIDS)
def test_engine_replays_reference_probes(p):
    from paper_2506_14781_b200.api import probe_population
    st = probe_population(inst(p["instance"]), p["beta"], p["penalty"], p["n_chains"], p["sweeps"],
                          p["seed"], rule=p["rule"])
    # exact where the reference's incremental f (mc.cpp:32) is exact: dyadic
    # couplings, fields and penalty; otherwise FP64 rounding-level agreement
    same_stats(st.__dict__, p["stats"], exact=dyadic(p["instance"]) and dyadic_value(p["penalty"]))


@pytest.mark.gpu
@pytest.mark.parametrize("lad", FIX["ladders"], ids=LIDS)
def test_engine_replays_reference_ladders(lad):
    from paper_2506_14781_b200.api import ScheduleConfig, build_schedule
    cfg = ScheduleConfig(rule=lad["rule"], **lad["config"])
    s = build_schedule(inst(lad["instance"]), cfg)
    # the ladder's penalties (P0 + alpha_P / (beta sigma_g)) are not dyadic, so
    # the reference's incremental f carries rounding: the ladder SHAPE (rows,
    # columns, stopping, budget flag) must match exactly, the values to 1e-9
    assert len(s.betas) == len(lad["betas"]) and len(s.penalties) == len(lad["penalties"])
    np.testing.assert_allclose(s.betas, lad["betas"], rtol=1e-9)
    np.testing.assert_allclose(s.penalties, lad["penalties"], rtol=1e-9)
    assert s.budget_exhausted == lad["budget_exhausted"]
    assert len(s.probe_stats) == len(lad["probe_stats"])
    for got, want in zip(s.probe_stats, lad["probe_stats"]):
        same_stats(got.__dict__, want, exact=False)
        assert (got.row, got.column) == (want["row"], want["column"])


@pytest.mark.gpu
def test_engine_probe_matches_exact_moments():
    # test_schedule.cpp:44-56: 64 chains x 2000 sweeps within 7 % of the exact moments
    from paper_2506_14781_b200.api import probe_population
    pr = inst("five_spin")
    st = probe_population(pr, 1.0, 2.0, 64, 2000, 99)
    _, vE, mg, vg = exact_moments(pr, 1.0, 2.0)
    assert st.sigma_e == pytest.approx(np.sqrt(vE), rel=0.07)
    assert st.sigma_g == pytest.approx(np.sqrt(vg), rel=0.07)
    assert abs(st.mean_g - mg) <= 0.07 * max(1.0, mg)


@pytest.mark.gpu
def test_engine_probe_errors_and_reuse():
    from paper_2506_14781_b200.api import Engine, probe_population
    from paper_2506_14781_b200.instances import ConfigError
    pr = inst("five_spin_dyadic")
    with Engine(0) as eng:
        with pytest.raises(ConfigError, match="2 chains"):
            probe_population(pr, 1.0, 1.0, 1, 100, 1, engine=eng)
        with pytest.raises(ConfigError, match="2 sweeps"):
            probe_population(pr, 1.0, 1.0, 8, 1, 1, engine=eng)
        a = probe_population(pr, 1.0, 2.0, 64, 500, 99, engine=eng)
        b = probe_population(pr, 3.0, 0.5, 64, 500, 7, engine=eng)   # rebinds beta, P, keys
        c = probe_population(pr, 1.0, 2.0, 64, 500, 99, engine=eng)  # same as a
        assert a == c and a != b
