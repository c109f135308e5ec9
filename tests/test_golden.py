"""Golden trajectories generated from the reference's own sources
(tools/gen_golden.py -> tests/golden/trajectories.json).  The C port replays
them on the CPU; the B200 engine replays them on the GPU (no oracle involved
at run time, /root/reference not needed)."""
import json
import os

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200.instances import Problem

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "trajectories.json")))
CASES = FIX["cases"]
IDS = [f"{c['name']}-{c['variant']}" for c in CASES]


def problem(c):
    i = c["instance"]
    return Problem(i["n"], np.array(i["ci"], np.int32), np.array(i["cj"], np.int32),
                   np.array(i["cw"]), np.array(i["fields"]), np.array(i["pa"], np.int32),
                   np.array(i["pb"], np.int32))


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_port_replays_reference_golden(c):
    r = O.run(problem(c), c["betas"], c["penalties"], c["total_sweeps"], c["sweeps_per_swap"],
              seed=c["seed"], rule=c["rule"], rng=c["rng"])
    np.testing.assert_array_equal(r.f, c["f"])
    np.testing.assert_array_equal(r.g, c["g"])
    assert [format(int(d), "016x") for d in r.digest] == c["digest"]
    assert [format(O.digest(s), "016x") for s in r.final_grid] == c["final_grid_digest"]
    assert r.accepts_p.tolist() == c["accepts_p"] and r.accepts_b.tolist() == c["accepts_b"]


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_engine_replays_reference_golden(c):
    from paper_2506_14781_b200.api import Engine, RunConfig
    eng = Engine(0)
    eng.set_problem(problem(c))
    eng.set_schedule(c["betas"], c["penalties"])
    got = []

    def sink(r, n, st, ap, ab):
        for k in range(n):
            got.append((r[k].f, r[k].g, r[k].digest))
        return 0

    engine = "plane" if c["rng"] == "plane" else "slot"
    cw, h = np.array(c["instance"]["cw"]), np.array(c["instance"]["fields"])
    if engine == "plane" and not (np.all(np.abs(cw) == 1.0) and np.all(h == 0.0)):
        pytest.skip("plane engine needs J = +-1, h = 0 (checked on the CPU port only)")
    eng.run(RunConfig(total_sweeps=c["total_sweeps"], sweeps_per_swap=c["sweeps_per_swap"],
                      seed=c["seed"], rule=c["rule"], engine=engine, store_states=False), sink)
    grid = eng.grid()
    _, cp, _, cb = eng.counters()
    eng.close()
    assert [x[0] for x in got] == c["f"]
    assert [x[1] for x in got] == c["g"]
    assert [format(int(x[2]), "016x") for x in got] == c["digest"]
    assert [format(O.digest(s), "016x") for s in grid] == c["final_grid_digest"]
    assert cp.tolist() == c["accepts_p"] and cb.tolist() == c["accepts_b"]
