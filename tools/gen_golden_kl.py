"""Generate tests/golden/kl.json from the REFERENCE's own kl_curve
(analysis.cpp:215-241) over its run_2dpt with the Philox shadow rng.hpp
(oracle/_ref/libtgref_philox.so).  Run in the build container:
    python tools/gen_golden_kl.py
tests/test_kl.py replays the fixture on the C port (CPU) and on the B200
engine's on-device decode / histogram / KL (GPU)."""
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


def logical_of(pr):
    n, cpl, h = pr.meta["logical"]
    return Problem.make(n, cpl, h)


def main():
    pr = I.k10_pm1(1)
    lp = logical_of(pr)
    betas, pens = I.config_schedule("c1")
    cases = []
    for seed in (1, 2, 3, 4):
        for discard in (False, True):
            t, smp, kl = O.kl_curve(pr, betas, pens, 1500, 1, seed, lp, pr.copies, 3.0, discard,
                                    impl="ref:philox")
            cases.append({"seed": seed, "discard": discard, "total_sweeps": 1500, "sps": 1,
                          "samples": smp.tolist(),
                          "kl": [None if np.isnan(x) else float(x) for x in kl]})
    out = {"generator": "tools/gen_golden_kl.py (reference kl_curve via oracle/_ref)",
           "instance": {"n": pr.n, "ci": pr.ci.tolist(), "cj": pr.cj.tolist(), "cw": pr.cw.tolist(),
                        "fields": pr.fields.tolist(), "pa": pr.pa.tolist(), "pb": pr.pb.tolist()},
           "logical": {"n": lp.n, "ci": lp.ci.tolist(), "cj": lp.cj.tolist(), "cw": lp.cw.tolist(),
                       "fields": lp.fields.tolist()},
           "copies": [list(map(int, c)) for c in pr.copies], "betas": list(map(float, betas)),
           "penalties": list(map(float, pens)), "beta_kl": 3.0, "cases": cases}
    path = os.path.join(ROOT, "tests", "golden", "kl.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes,", len(cases), "cases")


if __name__ == "__main__":
    main()
