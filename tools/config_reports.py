"""The report column of the BASELINE configs on one B200:

  config 1: mean KL(decoded target samples || logical Boltzmann at beta = 3)
            over 100 chains of the K10 +-1 instance (8x8 grid, 1e5 sweeps),
            KL evaluated on the device every round (kl_curve,
            analysis.cpp:215-241; mean over chains as acceptance.cpp:96-121),
            and its final-decade log-log slope (analysis.cpp:272-288);
  config 2: sweeps until the target replica holds the planted ground state
            (g = 0 and f <= E_planted + 1e-6 |E_planted|), 32 Wishart N=32
            instances (seeds 1..32), sps = 1 and 50 -- time_to_residual
            (analysis.cpp:260-270) per seed, on the fixed 16x8 grid and on the
            adaptive ladder of build_schedule (schedule.cpp:77-163);
  config 3: residual energy rho_E(t) with bootstrap CI over the 64-instance
            Wishart N=64 batch (16x16 grids) -- residual_curve
            (analysis.cpp:38-96), 1e6 sweeps;
  config 4: the N=256 Wishart instance (64768 spins, 32x32), 1e6 sweeps:
            best feasible residual energy over time.

Instances of a config run as batches (run_2dpt_batch); records are streamed.
Float configs run on the FLOAT engine (--engine slot: SLOT v2).  Writes
JSON/CSV to --out (copy the ones to keep into profiles/).

    python tools/config_reports.py [--only c1,c2,c3,c4] [--c3-sweeps 1000000] ...
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
from paper_2506_14781_b200.api import (Engine, RunConfig, Schedule, ScheduleConfig,  # noqa: E402
                                       build_schedule, run_2dpt_batch)

ENGINE = "float"


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
                        digest=False, engine=ENGINE)
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
                    record_every=every, engine=ENGINE)
    t0 = time.perf_counter()
    run_2dpt_batch(prs, scheds, cfg, seeds=list(range(1, 65)), sink=sink)
    wall = time.perf_counter() - t0
    runs = [(recs[b], prs[b].meta["planted_energy"], b, prs[b].copies, prs[b].meta["logical"])
            for b in range(len(prs))]
    curve = RP.residual_curve(runs, None, None, 64)
    with open(os.path.join(out_dir, "c3_residual_%d.csv" % sweeps), "w") as fh:
        fh.write("t,rho_E,ci95\n")
        for p in curve.points:
            fh.write(f"{p.t},{p.rho_e!r},{p.ci95!r}\n")
    print(json.dumps({"c3_points": len(curve.points), "rho_E_first": curve.points[0].rho_e,
                      "rho_E_last": curve.points[-1].rho_e, "wall_s": wall,
                      "spin_updates": float(n) * 256 * sweeps * 64}))


def loglog_slope(points, t_lo, t_hi):
    """Least-squares slope of log KL against log t over [t_lo, t_hi]
    (analysis.cpp:272-288)."""
    xs = [np.log(t) for t, y in points if t_lo <= t <= t_hi and y > 0]
    ys = [np.log(y) for t, y in points if t_lo <= t <= t_hi and y > 0]
    if len(xs) < 2:
        return float("nan")
    return float(np.polyfit(xs, ys, 1)[0])


def c1(sweeps, chains, out_dir):
    """Mean KL of the target replica's decoded samples over `chains` chains."""
    pr = I.k10_pm1(1)
    betas, pens = I.config_schedule("c1")
    n_log, cpl, h = pr.meta["logical"]
    logical = I.Problem.make(n_log, cpl, h)
    eng = Engine(0)
    eng.set_kl_decoder(logical, pr.copies, float(betas[-1]))
    scheds = [Schedule(list(betas), list(pens))] * chains
    t0 = time.perf_counter()
    run_2dpt_batch([pr] * chains, scheds, RunConfig(total_sweeps=sweeps, sweeps_per_swap=1, store_states=False,
                                                    digest=False, engine="slot"),
                   seeds=list(range(1, chains + 1)), engine=eng, sink=lambda *a: 0)
    wall = time.perf_counter() - t0
    curves = [eng.kl_curve(b, sweeps, 1) for b in range(chains)]
    eng.close()
    t = np.array([p.t for p in curves[0]])
    mean = np.mean([[p.kl for p in c] for c in curves], axis=0)
    iid = np.array([p.iid_reference for p in curves[0]])
    pts = list(zip(t.tolist(), mean.tolist()))
    slope = loglog_slope(pts, sweeps / 10.0, sweeps)
    keep = sorted(set([int(x) for x in np.unique(np.geomspace(1, sweeps, 60).astype(int))]))
    out = {"config": "C1 K10 +-1 -> %d physical (copies 2, degree <= 6), 8x8 grid, metropolis, sps=1" % pr.n,
           "chains": chains, "sweeps": sweeps, "beta_target": float(betas[-1]),
           "kl_final": float(mean[-1]), "kl_at_1e4": float(mean[min(len(mean), 10000) - 1]),
           "iid_reference_final": float(iid[-1]),
           "final_decade_loglog_slope": slope, "wall_s": wall,
           "curve": [[int(t[k - 1]), float(mean[k - 1])] for k in keep if k <= len(mean)]}
    with open(os.path.join(out_dir, "c1_kl.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("kl_final", "kl_at_1e4", "iid_reference_final",
                                          "final_decade_loglog_slope", "wall_s")}))


def c2_adaptive(sweeps, out_dir):
    """Config 2 on each instance's adaptive (beta, P) ladder (build_schedule)."""
    prs = [I.wishart_planted(32, 0.5, seed=s) for s in range(1, 33)]
    e_gs = [p.meta["planted_energy"] for p in prs]
    n_log = prs[0].meta["n_logical"]
    res = {}
    t_all = time.perf_counter()
    scheds = []
    for b, pr in enumerate(prs):
        bs = build_schedule(pr, ScheduleConfig(seed=b + 1, i_max=16, j_max=8, replica_budget=128))
        scheds.append(bs)
    # batches need one grid shape: group the instances by their ladder's shape
    groups = {}
    for b, sc in enumerate(scheds):
        groups.setdefault((len(sc.betas), len(sc.penalties)), []).append(b)
    for sps in (1, 50):
        best = [np.inf] * len(prs)
        tts = [None] * len(prs)
        for shape, members in groups.items():
            def sink(k, recs, n, states, ap, ab, members=members):
                b = members[k]
                for q in range(n):
                    r = recs[q]
                    if not r.feasible:
                        continue
                    best[b] = min(best[b], r.f)
                    if tts[b] is None and (best[b] - e_gs[b]) / n_log <= 1e-6 * abs(e_gs[b]) / n_log:
                        tts[b] = int(r.sweep_count)
                return 0
            run_2dpt_batch([prs[b] for b in members], [Schedule(scheds[b].betas, scheds[b].penalties)
                                                        for b in members],
                           RunConfig(total_sweeps=sweeps, sweeps_per_swap=sps, store_states=False,
                                     digest=False, engine=ENGINE),
                           seeds=[b + 1 for b in members], sink=sink)
        solved = [x for x in tts if x is not None]
        rho = [(bb - e) / n_log if np.isfinite(bb) else None for bb, e in zip(best, e_gs)]
        res["sps=%d" % sps] = {"time_to_solution_sweeps": tts, "solved": len(solved),
                               "median_sweeps_solved": float(np.median(solved)) if solved else None,
                               "best_feasible_rho_per_instance": rho}
        print(json.dumps({"c2_adaptive_sps": sps, "solved": len(solved)}))
    out = {"config": "C2 Wishart N=32 logical -> %d physical, adaptive ladder (build_schedule, "
                     "i_max 16, j_max 8, replica budget 128)" % prs[0].n,
           "ladders": [[len(sc.betas), len(sc.penalties)] for sc in scheds],
           "sweeps_budget": sweeps, "wall_s": time.perf_counter() - t_all, "runs": res}
    with open(os.path.join(out_dir, "c2_adaptive_time_to_solution.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def c4(sweeps, every, out_dir):
    """Config 4: best feasible residual energy of the target replica over time."""
    pr = I.wishart_planted(256, 0.5, seed=1)
    betas, pens = I.wishart_schedule(pr, 32, 32)
    e_gs = pr.meta["planted_energy"]
    n_log = pr.meta["n_logical"]
    pts, best = [], [np.inf]
    feas = [0, 0]

    def sink(b, recs, n, states, ap, ab):
        for q in range(n):
            r = recs[q]
            feas[1] += 1
            if r.feasible:
                feas[0] += 1
                best[0] = min(best[0], r.f)
            pts.append((int(r.sweep_count), (best[0] - e_gs) / n_log if np.isfinite(best[0]) else None,
                        bool(r.feasible), float(r.f)))
        return 0

    t0 = time.perf_counter()
    run_2dpt_batch([pr], [Schedule(list(betas), list(pens))],
                   RunConfig(total_sweeps=sweeps, sweeps_per_swap=1, store_states=False, digest=False,
                             record_every=every, engine=ENGINE), seeds=[1], sink=sink)
    wall = time.perf_counter() - t0
    out = {"config": "C4 Wishart N=256 logical (alpha 0.5) -> %d physical, 32x32 grid, sps=1" % pr.n,
           "sweeps": sweeps, "record_every": every, "wall_s": wall,
           "spin_updates": float(pr.n) * 1024 * sweeps,
           "flips_per_s_incl_records": float(pr.n) * 1024 * sweeps / wall,
           "feasible_fraction_of_records": feas[0] / max(feas[1], 1),
           "final_best_feasible_rho": pts[-1][1] if pts else None,
           "series": pts}
    with open(os.path.join(out_dir, "c4_residual_%d.json" % sweeps), "w") as fh:
        json.dump(out, fh)
    print(json.dumps({k: out[k] for k in ("wall_s", "flips_per_s_incl_records", "feasible_fraction_of_records",
                                          "final_best_feasible_rho")}))


def main():
    global ENGINE
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c3,c4")
    ap.add_argument("--engine", default="float", choices=["float", "slot"])
    ap.add_argument("--c1-sweeps", type=int, default=100000)
    ap.add_argument("--c1-chains", type=int, default=100)
    ap.add_argument("--c2-sweeps", type=int, default=100000)
    ap.add_argument("--c3-sweeps", type=int, default=1000000)
    ap.add_argument("--c3-every", type=int, default=1000)
    ap.add_argument("--c4-sweeps", type=int, default=1000000)
    ap.add_argument("--c4-every", type=int, default=1000)
    ap.add_argument("--out", default="gpurun_out")
    a = ap.parse_args()
    ENGINE = a.engine
    os.makedirs(a.out, exist_ok=True)
    only = set(a.only.split(","))
    if "c1" in only:
        c1(a.c1_sweeps, a.c1_chains, a.out)
    if "c2" in only:
        c2(a.c2_sweeps, a.out)
        c2_adaptive(a.c2_sweeps, a.out)
    if "c3" in only:
        c3(a.c3_sweeps, a.c3_every, a.out)
    if "c4" in only:
        c4(a.c4_sweeps, a.c4_every, a.out)


if __name__ == "__main__":
    main()
