"""Generate tests/golden/schedule.json from the REFERENCE's own
probe_population / build_schedule (schedule.cpp:18-163) built with the Philox
shadow rng.hpp (oracle/_ref/libtgref_philox.so, heat bath: _philox_hb).  Run
in the build container, where /root/reference exists:
    python tools/gen_golden_schedule.py
Instances are stored in canonical order (the engine's chromatic sweep equals
the reference's index-order sweep there); tests/test_schedule.py replays the
fixture on the C port (CPU) and on the B200 engine (GPU)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import pyoracle as O  # noqa: E402
from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.instances import Problem  # noqa: E402


def five_spin(dyadic=False):  # test_schedule.cpp:22-31 (dyadic: exact arithmetic variant)
    w = [0.75, -0.5, 0.5, -1.0, 0.25] if dyadic else [0.8, -0.6, 0.5, -0.9, 0.3]
    h = [0.25, -0.125, 0.0, 0.125, -0.25] if dyadic else [0.2, -0.1, 0.0, 0.1, -0.2]
    pr = Problem(5, np.array([0, 1, 2, 3, 0], np.int32), np.array([1, 2, 3, 4, 4], np.int32),
                 np.array(w), np.array(h), np.array([0, 1], np.int32), np.array([2, 3], np.int32))
    return I.to_canonical(pr)


def chain6():  # test_schedule.cpp:33-39
    pr = Problem(6, np.arange(5, dtype=np.int32), np.arange(1, 6, dtype=np.int32), np.ones(5),
                 np.zeros(6), np.zeros(0, np.int32), np.zeros(0, np.int32))
    return I.to_canonical(pr)


def five_sparse():
    f = I.five_node_complete()
    return I.to_canonical(I.sparsify(5, list(zip(f.ci.tolist(), f.cj.tolist(), f.cw.tolist())),
                                     f.fields.tolist(), 2, 3))


INST = {"five_spin": five_spin(), "five_spin_dyadic": five_spin(True), "chain6": chain6(),
        "five_sparse": five_sparse(), "k10_pm1": I.k10_pm1(1)}

PROBES = [  # instance, beta, P, chains, sweeps, seed, rule
    ("five_spin", 1.0, 2.0, 64, 2000, 99, "metropolis"),
    ("five_spin_dyadic", 1.0, 2.0, 64, 500, 99, "metropolis"),
    ("five_spin_dyadic", 0.7, 1.5, 16, 300, 5, "heat_bath"),
    ("chain6", 2.0, 1.0, 8, 100, 1, "metropolis"),
    ("k10_pm1", 0.5, 0.25, 32, 400, 3, "metropolis"),
    ("five_sparse", 1.3, 2.0, 48, 600, 12, "metropolis"),
]

LADDERS = [  # instance, rule, ScheduleConfig overrides (test_schedule.cpp:76-180)
    ("chain6", "metropolis", dict(n_chains=16, sweeps_per_probe=400, seed=7)),
    ("chain6", "metropolis", dict(sigma_min=1e6, n_chains=8, sweeps_per_probe=100)),
    ("five_spin_dyadic", "metropolis", dict(beta0=0.1, alpha_p=0.6, n_chains=16, sweeps_per_probe=400, seed=3)),
    ("five_spin_dyadic", "metropolis", dict(beta0=0.1, p0=0.1, j_max=1, i_max=10, replica_budget=10,
                                            n_chains=8, sweeps_per_probe=200)),
    ("five_sparse", "metropolis", dict(alpha_beta=1.3, alpha_p=1.5, i_max=2, n_chains=48,
                                       sweeps_per_probe=2000, seed=12)),
    ("five_spin", "metropolis", dict(beta0=0.1, alpha_p=0.6, n_chains=16, sweeps_per_probe=400, seed=3)),
    ("five_spin_dyadic", "heat_bath", dict(beta0=0.2, alpha_p=0.8, n_chains=16, sweeps_per_probe=300, seed=4)),
]

VARIANT = {"metropolis": "ref:philox", "heat_bath": "ref:philox_hb"}


def inst_json(pr):
    return {"n": pr.n, "ci": pr.ci.tolist(), "cj": pr.cj.tolist(), "cw": pr.cw.tolist(),
            "fields": pr.fields.tolist(), "pa": pr.pa.tolist(), "pb": pr.pb.tolist()}


def main():
    out = {"generator": "tools/gen_golden_schedule.py (reference schedule.cpp via oracle/_ref)",
           "instances": {k: inst_json(v) for k, v in INST.items()}, "probes": [], "ladders": []}
    for name, beta, pen, ch, sw, seed, rule in PROBES:
        st = O.probe_population(INST[name], beta, pen, ch, sw, seed, rule=rule, impl=VARIANT[rule])
        out["probes"].append({"instance": name, "beta": beta, "penalty": pen, "n_chains": ch,
                              "sweeps": sw, "seed": seed, "rule": rule, "stats": st})
    for name, rule, cfg in LADDERS:
        b, p, stats, ex = O.build_schedule(INST[name], rule=rule, impl=VARIANT[rule], **cfg)
        out["ladders"].append({"instance": name, "rule": rule, "config": cfg, "betas": b.tolist(),
                               "penalties": p.tolist(), "probe_stats": stats, "budget_exhausted": ex})
    path = os.path.join(ROOT, "tests", "golden", "schedule.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes,", len(out["probes"]), "probes,", len(out["ladders"]),
          "ladders")


if __name__ == "__main__":
    main()
