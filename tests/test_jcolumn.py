"""Resource-matched J-column baseline, ``run_jcolumn_pt`` (engine.cpp:221-270;
SURVEY.md §8f row 3).  Golden vectors come from the reference's own
run_jcolumn_pt (tools/gen_golden_jcolumn.py -> tests/golden/jcolumn.json);
the C port replays them on the CPU, the B200 engine (one batched launch of all
repeats, ``tg_run_jcolumn``) on the GPU."""
import json
import os

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200.instances import ConfigError, Problem

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "jcolumn.json")))
CASES = FIX["cases"]
IDS = [c["name"] for c in CASES]


def problem(c):
    i = c["instance"]
    return Problem(i["n"], np.array(i["ci"], np.int32), np.array(i["cj"], np.int32),
                   np.array(i["cw"]), np.array(i["fields"]), np.array(i["pa"], np.int32),
                   np.array(i["pb"], np.int32))


def exact(c):
    return all(float(w).is_integer() or (4 * float(w)).is_integer() for w in c["instance"]["cw"] +
               c["instance"]["fields"])


def golden_best(c):
    return np.array([np.nan if x is None else x for x in c["best_f"]])


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_port_replays_reference_jcolumn(c):
    r = O.run_jcolumn(problem(c), c["betas"], c["p_fixed"], c["repeats"], c["total_sweeps"],
                      c["sweeps_per_swap"], seed=c["seed"])
    np.testing.assert_array_equal(r.best_f, golden_best(c))
    assert r.n_feasible.tolist() == c["n_feasible"] and r.n_total.tolist() == c["n_total"]
    assert r.feasible_fraction == c["feasible_fraction"]
    rounds = c["total_sweeps"] // c["sweeps_per_swap"]
    assert r.round.tolist() == list(range(1, rounds + 1))
    assert r.sweep_count.tolist() == [k * c["sweeps_per_swap"] for k in range(1, rounds + 1)]


def test_reference_contract_constrained_pair():
    # test_engine.cpp:252-274 on the port: 100 rounds, n_total == 3, best_f >= ground energy
    c = CASES[0]
    r = O.run_jcolumn(problem(c), [0.5, 1.0], 2.0, 3, 1000, 10, seed=5)
    assert len(r.round) == 100 and np.all(r.n_total == 3)
    assert np.all((r.n_feasible >= 0) & (r.n_feasible <= 3))
    assert np.array_equal(r.any_feasible, r.n_feasible > 0)
    ground = min(0.6 * a * b + 0.3 * a - 0.2 * b for a in (-1, 1) for b in (-1, 1))
    assert np.all(r.best_f[r.any_feasible] >= ground - 1e-12)
    assert 0.0 <= r.feasible_fraction <= 1.0
    for pf, reps, msg in ((0.0, 3, "P must be positive"), (2.0, 0, "repeats must be >= 1")):
        with pytest.raises(O.OracleError, match=msg):
            O.run_jcolumn(problem(c), [0.5, 1.0], pf, reps, 1000, 10, seed=5)


def test_api_validates_before_touching_the_device():
    from paper_2506_14781_b200.api import RunConfig, run_jcolumn_pt
    c = CASES[0]
    with pytest.raises(ConfigError, match="P must be positive"):
        run_jcolumn_pt(problem(c), [0.5, 1.0], -1.0, 3, RunConfig(total_sweeps=10))
    with pytest.raises(ConfigError, match="repeats must be >= 1"):
        run_jcolumn_pt(problem(c), [0.5, 1.0], 1.0, 0, RunConfig(total_sweeps=10))


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_engine_replays_reference_jcolumn(c):
    from paper_2506_14781_b200.api import RunConfig, run_jcolumn_pt
    t = run_jcolumn_pt(problem(c), c["betas"], c["p_fixed"], c["repeats"],
                       RunConfig(total_sweeps=c["total_sweeps"], sweeps_per_swap=c["sweeps_per_swap"],
                                 seed=c["seed"]))
    rounds = c["total_sweeps"] // c["sweeps_per_swap"]
    assert [r.round for r in t.records] == list(range(1, rounds + 1))
    assert [r.sweep_count for r in t.records] == [k * c["sweeps_per_swap"] for k in range(1, rounds + 1)]
    assert [r.n_feasible for r in t.records] == c["n_feasible"]
    assert [r.n_total for r in t.records] == c["n_total"]
    assert [r.any_feasible for r in t.records] == [x > 0 for x in c["n_feasible"]]
    got = np.array([r.best_f for r in t.records])
    if exact(c):
        np.testing.assert_array_equal(got, golden_best(c))
    else:
        np.testing.assert_allclose(got, golden_best(c), rtol=1e-9, atol=1e-12)
    assert t.feasible_fraction == c["feasible_fraction"]
    assert t.penalty == c["p_fixed"] and t.sweeps_per_swap == c["sweeps_per_swap"]


@pytest.mark.gpu
def test_engine_jcolumn_errors():
    from paper_2506_14781_b200.api import Engine, RunConfig, run_jcolumn_pt
    c = CASES[1]
    with Engine(0) as eng:
        with pytest.raises(ConfigError):
            run_jcolumn_pt(problem(c), [1.0, 0.5], 1.0, 2, RunConfig(total_sweeps=10), engine=eng)
        with pytest.raises(ConfigError):
            run_jcolumn_pt(problem(c), [0.5, 1.0], 1.0, 2, RunConfig(total_sweeps=10, engine="plane"),
                           engine=eng)
        # the context stays usable for a normal run afterwards
        t = run_jcolumn_pt(problem(c), [0.5, 1.0], 1.0, 2, RunConfig(total_sweeps=10), engine=eng)
        assert len(t.records) == 10
