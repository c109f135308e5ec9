"""Generate tests/golden/jcolumn.json from the REFERENCE's own
run_jcolumn_pt (engine.cpp:221-270) built with the Philox shadow rng.hpp
(oracle/_ref/libtgref_philox.so).  Run in the build container, where
/root/reference exists:   python tools/gen_golden_jcolumn.py
The fixture carries the instances; tests/test_jcolumn.py replays it on the C
port (CPU) and on the B200 engine (GPU)."""
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


def constrained_pair():  # test_engine.cpp:27-30
    return Problem(2, np.array([0], np.int32), np.array([1], np.int32), np.array([0.6]),
                   np.array([0.3, -0.2]), np.array([0], np.int32), np.array([1], np.int32))


def five_sparse():
    f = I.five_node_complete()
    return I.to_canonical(I.sparsify(5, list(zip(f.ci.tolist(), f.cj.tolist(), f.cw.tolist())),
                                     f.fields.tolist(), 2, 3))


def c1_column():
    betas, pens = I.config_schedule("c1")
    return betas, float(np.mean(pens)), len(pens)  # acceptance.cpp:385-393: mean P, J repeats


CASES = [
    # name, problem, betas, p_fixed, repeats, total, sps, seed
    ("constrained_pair", constrained_pair(), [0.5, 1.0], 2.0, 3, 1000, 10, 5),  # test_engine.cpp:252-258
    ("c1_k10_pm1", I.k10_pm1(1), *c1_column(), 400, 2, 11),
    ("five_node_sparse", five_sparse(), [0.5, 1.0, 1.5, 2.5], 3.0, 5, 300, 3, 7000),
    ("wishart_n6", I.wishart_planted(6, 0.5, seed=3), [0.2, 1.0, 5.0], 0.75, 4, 200, 1, 7001),
]


def main():
    out = {"generator": "tools/gen_golden_jcolumn.py (reference run_jcolumn_pt via oracle/_ref)",
           "cases": []}
    for name, pr, betas, pf, reps, total, sps, seed in CASES:
        r = O.run_jcolumn(pr, betas, pf, reps, total, sps, seed=seed, impl="ref:philox")
        out["cases"].append({
            "name": name,
            "instance": {"n": pr.n, "ci": pr.ci.tolist(), "cj": pr.cj.tolist(), "cw": pr.cw.tolist(),
                         "fields": pr.fields.tolist(), "pa": pr.pa.tolist(), "pb": pr.pb.tolist()},
            "betas": list(map(float, betas)), "p_fixed": pf, "repeats": reps,
            "total_sweeps": total, "sweeps_per_swap": sps, "seed": seed,
            "best_f": [None if np.isnan(x) else float(x) for x in r.best_f],
            "n_feasible": r.n_feasible.tolist(), "n_total": r.n_total.tolist(),
            "feasible_fraction": r.feasible_fraction,
        })
    path = os.path.join(ROOT, "tests", "golden", "jcolumn.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes,", len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
