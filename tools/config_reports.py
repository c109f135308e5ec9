"""The report column of BASELINE configs 2 and 3 on one B200:

  config 2: sweeps until the target replica holds the planted ground state
            (g = 0 and f <= E_planted + 1e-6 |E_planted|), 32 Wishart N=32
            instances (seeds 1..32), 16x8 grid, sps = 1 -- time_to_residual
            (analysis.cpp:260-270) per seed;
  config 3: residual energy rho_E(t) with bootstrap CI over the 64-instance
            Wishart N=64 batch (16x16 grids) -- residual_curve
            (analysis.cpp:38-96), on a truncated sweep budget.

All instances of a config run as ONE batch launch (run_2dpt_batch, SLOT
engine); records are streamed.  Writes profiles-style JSON/CSV to
gpurun_out/ (copy the ones to keep into profiles/).

    python tools/config_reports.py [--c2-sweeps 100000] [--c3-sweeps 10000] [--c3-every 100]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401  (CUDA runtime / NCCL first, as bench.py)

from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200 import reports as RP  # noqa: E402
from paper_2506_14781_b200.api import RunConfig, Schedule, run_2dpt_batch  # noqa: E402


def c2(sweeps, out_dir):
    prs = [I.wishart_planted(32, 0.5, seed=s) for s in range(1, 33)]
    scheds = [Schedule(*map(list, I.wishart_schedule(p, 16, 8))) for p in prs]
    e_gs = [p.meta["planted_energy"] for p in prs]
    n_log = prs[0].meta["n_logical"]
    out = {"config": "C2 Wishart N=32 logical (alpha 0.5) -> %d physical, 16x8 grid, metropolis" % prs[0].n,
           "instances": "seeds 1..32 (instance seed = run seed), planted all-ones ground state",
           "schedule": "beta geometric 0.2-5 (16), P_ref linear 0..Pmax/4 (8) (SURVEY.md 8d)",
           "criterion": "g = 0 and f <= E_planted + 1e-6 |E_planted| (time_to_residual, analysis.cpp:260-270)",
           "sweeps_budget": sweeps, "runs": {}}
    for sps in (1, 50):
        best = [np.inf] * len(prs)
        tts = [None] * len(prs)

        def sink(b, recs, n, states, ap, ab):
            # time_to_residual restated incrementally over the streamed records
            for k in range(n):
                r = recs[k]
                if not r.feasible:
                    continue
                best[b] = min(best[b], r.f)
                if tts[b] is None and (best[b] - e_gs[b]) / n_log <= 1e-6 * abs(e_gs[b]) / n_log:
                    tts[b] = int(r.sweep_count)
            return 0

        cfg = RunConfig(total_sweeps=sweeps, sweeps_per_swap=sps, seed=1, store_states=False,
                        digest=False, engine="slot")
        t0 = time.perf_counter()
        run_2dpt_batch(prs, scheds, cfg, seeds=list(range(1, 33)), sink=sink)
        wall = time.perf_counter() - t0
        solved = [t for t in tts if t is not None]
        rho = [(bb - e) / n_log if np.isfinite(bb) else None for bb, e in zip(best, e_gs)]
        out["runs"]["sps=%d" % sps] = {
            "time_to_solution_sweeps": tts, "solved": len(solved),
            "median_sweeps_solved": float(np.median(solved)) if solved else None,
            "best_feasible_rho_per_instance": rho,
            "median_best_rho": float(np.median([r for r in rho if r is not None])),
            "wall_s_all_32_in_one_batch": wall,
            "spin_updates": float(prs[0].n) * 128 * sweeps * 32}
        print(json.dumps({"sps": sps, "solved": len(solved),
                          "median_best_rho": out["runs"]["sps=%d" % sps]["median_best_rho"],
                          "wall_s": wall}))
    with open(os.path.join(out_dir, "c2_time_to_solution.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def c3(sweeps, every, out_dir):
    prs = [I.wishart_planted(64, 0.75, seed=s) for s in range(1, 65)]
    scheds = [Schedule(*map(list, I.wishart_schedule(p, 16, 16))) for p in prs]
    recs = [[] for _ in prs]

    class Rec:
        __slots__ = ("sweep_count", "f", "feasible", "state")

    n = prs[0].n

    def sink(b, rr, k, states, ap, ab):
        st = np.ctypeslib.as_array(states, shape=(k * n,)) if states else None
        for q in range(k):
            r = Rec()
            r.sweep_count, r.f, r.feasible = int(rr[q].sweep_count), float(rr[q].f), bool(rr[q].feasible)
            r.state = st[q * n:(q + 1) * n].copy() if (st is not None and not r.feasible) else None
            recs[b].append(r)
        return 0

    cfg = RunConfig(total_sweeps=sweeps, sweeps_per_swap=1, seed=1, store_states=True, digest=False,
                    record_every=every, engine="slot")
    t0 = time.perf_counter()
    run_2dpt_batch(prs, scheds, cfg, seeds=list(range(1, 65)), sink=sink)
    wall = time.perf_counter() - t0
    runs = [(recs[b], prs[b].meta["planted_energy"], b, prs[b].copies, prs[b].meta["logical"])
            for b in range(len(prs))]
    curve = RP.residual_curve(runs, None, None, 64)
    with open(os.path.join(out_dir, "c3_residual.csv"), "w") as fh:
        fh.write("t,rho_E,ci95\n")
        for p in curve.points:
            fh.write(f"{p.t},{p.rho_e!r},{p.ci95!r}\n")
    print(json.dumps({"c3_points": len(curve.points), "rho_E_first": curve.points[0].rho_e,
                      "rho_E_last": curve.points[-1].rho_e, "wall_s": wall,
                      "spin_updates": float(n) * 256 * sweeps * 64}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2-sweeps", type=int, default=100000)
    ap.add_argument("--c3-sweeps", type=int, default=10000)
    ap.add_argument("--c3-every", type=int, default=100)
    ap.add_argument("--out", default="gpurun_out")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    c2(a.c2_sweeps, a.out)
    c3(a.c3_sweeps, a.c3_every, a.out)


if __name__ == "__main__":
    main()
