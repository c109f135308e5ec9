"""Generate tests/golden/trajectories.json from the REFERENCE's own sources
(oracle/_ref builds: reference engine + Philox shadow rng.hpp, and the
alt_sweep heat-bath / bit-plane variants).  Run in the build container, where
/root/reference exists:   python tools/gen_golden.py
The fixture carries the instances themselves, so the tests do not depend on
the generators; tests/test_golden.py replays it on the C port (CPU) and on the
B200 engine (GPU)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import pyoracle as O  # noqa: E402
from paper_2506_14781_b200 import instances as I  # noqa: E402


def five_sparse():
    f = I.five_node_complete()
    return I.to_canonical(I.sparsify(5, list(zip(f.ci.tolist(), f.cj.tolist(), f.cw.tolist())),
                                     f.fields.tolist(), 2, 3))


CASES = [
    ("c1_k10_pm1", I.k10_pm1(1), *I.config_schedule("c1"), 80, 1, 5),
    ("five_node_sparse", five_sparse(), [0.5, 1.0, 1.5], [2.0, 4.0, 6.0, 8.0], 120, 3, 77),
    ("c5_bipartite_128", I.bipartite_3regular(128, seed=4), *I.config_schedule("c5"), 30, 1, 9),
]
VARIANTS = [("metropolis", "slot", "philox"), ("heat_bath", "slot", "philox_hb"),
            ("metropolis", "plane", "plane"), ("heat_bath", "plane", "plane_hb")]


def main():
    out = {"generator": "tools/gen_golden.py (reference sources via oracle/_ref)", "cases": []}
    for name, pr, betas, pens, total, sps, seed in CASES:
        inst = {"n": pr.n, "ci": pr.ci.tolist(), "cj": pr.cj.tolist(), "cw": pr.cw.tolist(),
                "fields": pr.fields.tolist(), "pa": pr.pa.tolist(), "pb": pr.pb.tolist()}
        for rule, rng, variant in VARIANTS:
            r = O.run(pr, betas, pens, total, sps, seed=seed, rule=rule, rng=rng,
                      impl="ref:" + variant, round_counters=False)
            out["cases"].append({
                "name": name, "rule": rule, "rng": rng, "variant": variant,
                "instance": inst, "betas": list(map(float, betas)), "penalties": list(map(float, pens)),
                "total_sweeps": total, "sweeps_per_swap": sps, "seed": seed,
                "f": r.f.tolist(), "g": r.g.tolist(),
                "digest": [format(int(d), "016x") for d in r.digest],
                "final_grid_digest": [format(O.digest(s), "016x") for s in r.final_grid],
                "accepts_p": r.accepts_p.tolist(), "accepts_b": r.accepts_b.tolist(),
            })
    path = os.path.join(ROOT, "tests", "golden", "trajectories.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes,", len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
