"""Long exact-parity runs against the oracle (C port, sweep threads) on a B200: every round's (f, g,
digest), the accept counters and the final grid of the fused PLANE kernels must equal the oracle's over
`rounds` rounds -- ~100x the rounds of the unit tests, so the rare paths (lazy planes beyond the second tail
block, chain-site deferral, counter flushes) are hit many times.

    python tools/soak_oracle.py [n] [rounds]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401

import pyoracle as O  # noqa: E402
from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.api import Engine, RunConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
betas, pens = I.config_schedule("c5")
for rule in ("metropolis", "heat_bath"):
    for env, kname in ((None, None), ("TG_PLANE_CL", "0")):
        if env:
            os.environ[env] = kname
        pr = I.bipartite_3regular(n, seed=11, chain_frac=0.25)
        t0 = time.time()
        o = O.run(pr, betas, pens, rounds, 1, seed=13, rule=rule, rng="plane", threads=os.cpu_count() or 1)
        t_or = time.time() - t0
        eng = Engine(0)
        eng.set_problem(pr)
        eng.set_schedule(betas, pens)
        recs = []

        def sink(r, k, st, ap, ab):
            for q in range(k):
                recs.append((r[q].f, r[q].g, r[q].digest))
            return 0

        eng.run(RunConfig(total_sweeps=rounds, sweeps_per_swap=1, seed=13, rule=rule, engine="plane",
                          store_states=False, digest=True), sink)
        grid = eng.grid()
        _, cp, _, cb = eng.counters()
        kern = eng.info()["sweep_kernel"]
        eng.close()
        assert np.array_equal(np.array([r[0] for r in recs]), o.f), (rule, kern)
        assert np.array_equal(np.array([r[1] for r in recs]), o.g), (rule, kern)
        assert np.array_equal(np.array([r[2] for r in recs], dtype=np.uint64), o.digest), (rule, kern)
        assert np.array_equal(grid, o.final_grid), (rule, kern)
        assert np.array_equal(cp, o.accepts_p) and np.array_equal(cb, o.accepts_b), (rule, kern)
        print(f"oracle soak ok: N={n} chains 25% rounds={rounds} rule={rule} kernel={kern} "
              f"({n * 256 * rounds:.2e} updates, oracle {t_or:.0f} s)", flush=True)
        if env:
            del os.environ[env]

# FLOAT engine (one-comparison certified decisions): config-2 shape, Wishart N = 32 -> 928 spins, 16 x 8 grid
frounds = max(rounds * 3, 1000)
prw = I.wishart_planted(32, 0.5, seed=3)
bw, pw = I.wishart_schedule(prw, 16, 8)
for rule in ("metropolis", "heat_bath"):
    t0 = time.time()
    o = O.run(prw, bw, pw, frounds, 1, seed=5, rule=rule, rng="float", threads=os.cpu_count() or 1)
    t_or = time.time() - t0
    eng = Engine(0)
    eng.set_problem(prw)
    eng.set_schedule(bw, pw)
    recs = []

    def fsink(r, k, st, ap, ab):
        for q in range(k):
            recs.append((r[q].f, r[q].g, r[q].digest))
        return 0

    eng.run(RunConfig(total_sweeps=frounds, sweeps_per_swap=1, seed=5, rule=rule, engine="float",
                      store_states=False, digest=True), fsink)
    grid = eng.grid()
    _, cp, _, cb = eng.counters()
    kern = eng.info()["sweep_kernel"]
    eng.close()
    np.testing.assert_allclose([r[0] for r in recs], o.f, rtol=1e-9, atol=1e-9)
    assert np.array_equal(np.array([r[1] for r in recs]), o.g), rule
    assert np.array_equal(np.array([r[2] for r in recs], dtype=np.uint64), o.digest), rule
    assert np.array_equal(grid, o.final_grid), rule
    assert np.array_equal(cp, o.accepts_p) and np.array_equal(cb, o.accepts_b), rule
    print(f"oracle soak ok: FLOAT engine, Wishart N=32 (928 spins, 16x8) rounds={frounds} rule={rule} kernel={kern} "
          f"({prw.n * 128 * frounds:.2e} updates, oracle {t_or:.0f} s)", flush=True)
