"""Long-run soak of the config-5 fused kernel on a B200: `rounds` rounds at N spins (default 20000 x 2^20,
256 replicas = 5.4e12 updates per run), twice with the same seed and once resumed in pieces.  Checks that every
round's (f, g, digest) is identical across the three runs and that the final grid's (f, g) of sampled slots
equal the energies recomputed on the host from the reported states -- rare paths (deep lazy planes in the
drains, chain-site deferral, counter flushes) get ~1e4 times the exposure of the unit tests.

    python tools/soak_c5.py [n] [rounds] [rule]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401

from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.api import Engine, RunConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
rule = sys.argv[3] if len(sys.argv) > 3 else "metropolis"
pr = I.bipartite_3regular(n, seed=1)
betas, pens = I.config_schedule("c5")


def energy(s):
    s = s.astype(np.int64)
    return (float(-np.sum(pr.cw * s[pr.ci] * s[pr.cj]) - np.sum(pr.fields * s)),
            float(np.sum((s[pr.pa] - s[pr.pb]) ** 2)))


def run(pieces):
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(betas, pens)
    out = []

    def sink(r, k, st, ap, ab):
        for q in range(k):
            out.append((r[q].f, r[q].g, r[q].digest, r[q].target_state))
        return 0

    cfg = RunConfig(total_sweeps=rounds, sweeps_per_swap=1, seed=7, rule=rule, engine="plane",
                    store_states=False, digest=True)
    t0 = time.time()
    if pieces == 1:
        eng.run(cfg, sink)
    else:
        eng.init(cfg)
        left = rounds
        step = max(1, rounds // pieces + 3)
        while left > 0:
            k = min(step, left)
            eng.advance(k, sink)
            left -= k
    wall = time.time() - t0
    fs, gs = eng.energies()
    grid = eng.grid()
    kern = eng.info()["sweep_kernel"]
    eng.close()
    return out, fs, gs, grid, wall, kern


a = run(1)
b = run(1)
c = run(7)
assert len(a[0]) == rounds
assert a[0] == b[0], "two runs with one seed differ"
assert a[0] == c[0], "resumed run differs"
assert np.array_equal(a[3], b[3]) and np.array_equal(a[3], c[3])
for slot in range(0, len(betas) * len(pens), 29):
    assert (a[1][slot], a[2][slot]) == energy(a[3][slot]), slot
print(f"soak ok: N={n} rounds={rounds} rule={rule} kernel={a[5]} updates/run={n * 256 * rounds:.3e} "
      f"wall={a[4]:.1f}s ({n * 256 * rounds / a[4]:.3e} flips/s incl. records), "
      f"final target f={a[0][-1][0]} g={a[0][-1][1]} digest={a[0][-1][2]:#x}")
