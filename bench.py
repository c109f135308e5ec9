#!/usr/bin/env python
"""bench.py -- spin-flips/s of the 2D-PT hot path on B200 (BASELINE.json metric).

Workload (BASELINE.json config 5, the configuration the metric is quoted on):
random bipartite 3-regular Ising graph, J = +-1, h = 0, copy-constraint chain
pairs on 10% of the nodes, N = 2^20 physical spins, 16 x 16 (beta, P) grid
(beta geometric 0.2-5, P_cfg linear 0-4 -> P_ref = P_cfg/4 rounded to 1/64),
one sweep per swap round, Metropolis.  Synthetic instance, seed 1 (there is no
public benchmark suite).

A "step" = ROUNDS rounds of (one chromatic sweep of all 256 replicas, one
swap phase, one trace record).  spin-flips/s = N x replicas x sweeps / time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints ONE JSON line.  Under torchrun each rank sweeps 256/N replicas
(column blocks of the grid) and the per-round (f, g) all-gather runs over
NCCL inside the engine; timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spin-flips/s (whole box) at 1/2/4/8 B200 and % of sweep roofline vs CPU ref"
UNIT = "spin-flips/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1 << 20, help="physical spins")
    ap.add_argument("--rounds", type=int, default=None,
                    help="rounds per step (default: 1000 for c5 -- one launch, one record ring; 20 for the "
                         "float workloads)")
    ap.add_argument("--sps", type=int, default=1, help="sweeps per swap")
    ap.add_argument("--rule", default="metropolis")
    ap.add_argument("--engine", default="plane")
    ap.add_argument("--workload", default="c5", choices=["c5", "c2", "c3", "c4"],
                    help="c5: config 5 (the metric's config, default); c2/c4: Wishart float32 "
                         "configs on the slot engine; c3: the 64-instance Wishart batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-heat-bath", action="store_true", help="skip the heat-bath sub-record")
    ap.add_argument("--cpu-sweeps", type=int, default=16, help="marginal sweeps of the CPU sample")
    args = ap.parse_args()
    if args.rounds is None:
        args.rounds = 1000 if args.workload == "c5" else 20
    return args


def workload(n, kind="c5"):
    from paper_2506_14781_b200 import instances as I
    if kind == "c2":   # N=32 logical, alpha=0.5, degree <= 3 chains (928 spins), 16x8 grid
        pr = I.wishart_planted(32, 0.5, seed=1)
        betas, pens = I.wishart_schedule(pr, 16, 8)
        return pr, betas, pens
    if kind == "c3":   # one instance of the config-3 batch (the CPU legs time one instance)
        prs, scheds = c3_instances()
        return prs[0], scheds[0][0], scheds[0][1]
    if kind == "c4":   # N=256 logical, alpha=0.5 (64768 spins), 32x32 grid
        pr = I.wishart_planted(256, 0.5, seed=1)
        betas, pens = I.wishart_schedule(pr, 32, 32)
        return pr, betas, pens
    pr = I.bipartite_3regular(n, seed=1)
    betas, pens = I.config_schedule("c5")
    return pr, betas, pens


def workload_name(args, pr, R, rule):
    if args.workload == "c5":
        return f"C5 bipartite 3-regular N=2^{pr.n.bit_length() - 1} 16x16 sps={args.sps} {rule}"
    nl = pr.meta.get("n_logical")
    return (f"{args.workload.upper()} Wishart N={nl} logical -> {pr.n} physical (deg<=3), "
            f"{R} replicas sps={args.sps} {rule}")


def b_alg(pr):
    """Algorithmic bytes per spin update: (mean degree + 1) int8."""
    deg = 2.0 * (pr.n_couplings + pr.n_pairs) / pr.n
    return deg + 1.0


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:  # noqa: BLE001
        return {}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup(gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def reduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------- CPU legs

def cpu_reference_rate(pr, betas, pens, sweeps, threads):
    """Marginal updates/s of the unmodified reference run_2dpt (oracle/_ref O1
    when built here, else the C port) from two run lengths."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    kind = "reference" if O.ref_available("mt") else "port"
    R = len(betas) * len(pens)

    def run(S):
        t = time.perf_counter()
        if kind == "reference":
            O.ref_timed("mt", pr, betas, pens, S, 1, seed=1, threads=threads)
        else:
            O.run(pr, betas, pens, S, 1, seed=1, final_grid=False)
        return time.perf_counter() - t

    t1 = run(1)
    t2 = run(1 + sweeps)
    dt = max(t2 - t1, 1e-9)
    rate = pr.n * R * sweeps / dt
    return rate, kind, dt


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline_record(pr, betas, pens, sweeps, what):
    """The reference on the host cores: all threads (the reported value) and
    one thread, with the CPU model (BASELINE.md CPU-baseline plan)."""
    nproc = os.cpu_count() or 1
    rate_n, kind, dt_n = cpu_reference_rate(pr, betas, pens, sweeps, nproc)
    s1 = max(1, sweeps // 8)
    rate_1, _, dt_1 = cpu_reference_rate(pr, betas, pens, s1, 1)
    return {"value": rate_n, "unit": UNIT, "cores": nproc if kind == "reference" else 1,
            "kind": kind, "cpu_model": cpu_model(), "nproc": nproc,
            "value_1thread": rate_1,
            "sample": f"{what}; marginal rate of {1 + sweeps} vs 1 sweeps at RunConfig.threads="
                      f"{nproc} ({dt_n:.1f} s of sweeping) and {1 + s1} vs 1 sweeps at threads=1 "
                      f"({dt_1:.1f} s)"}


def repo_libraries():
    """Shared objects of this repo mapped into the process (/proc/self/maps)."""
    libs = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                path = line.split()[-1]
                if path.startswith(ROOT) and ".so" in path:
                    libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


def bench_config(args, pr, R, world):
    """The workload description both arms print (identical dicts)."""
    return {"workload": workload_name(args, pr, R, args.rule), "n_spins": int(pr.n),
            "replicas": R, "sweeps_per_swap": args.sps, "rule": args.rule,
            "rounds_per_step": args.rounds, "parallelism": f"replica-split x{world}",
            "l2": "flushed between timed GPU steps (256 MB write)"}


def run_reference_arm(args, rank, world):
    """The unmodified reference run_2dpt (oracle/_ref/libtgref_mt.so: the
    reference's own engine/mc/ising/constraints sources, mt19937_64,
    Metropolis, FP64) on all host threads.  Rank 0 only; the engine library
    is never loaded in this process."""
    if rank != 0:
        return
    if args.rule != "metropolis":
        print(json.dumps({"impl": "reference", "unavailable": "the reference implements Metropolis only"}))
        return
    pr, betas, pens = workload(args.n, args.workload)
    R = len(betas) * len(pens)
    threads = os.cpu_count() or 1
    vals, dts = [], []
    kind = "reference"
    for k in range(args.warmup + args.steps):
        rate, kind, dt = cpu_reference_rate(pr, betas, pens, args.cpu_sweeps, threads)
        if k >= args.warmup:
            vals.append(rate)
            dts.append(dt)
    value = statistics.median(vals)
    sample = (f"reference run_2dpt on the full workload (N={pr.n}, {R} replicas), marginal rate of "
              f"{1 + args.cpu_sweeps} vs 1 sweeps per step, RunConfig.threads={threads}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(dts), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, pr, R, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "libraries_mapped": repo_libraries(),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg

def c3_instances():
    """Config 3: 64 Wishart instances, N=64 logical, alpha=0.75, float32 J, degree <= 3
    chains (3904 physical spins each), each on its own 16x16 grid (schedule rule of C2)."""
    from paper_2506_14781_b200 import instances as I
    prs = [I.wishart_planted(64, 0.75, seed=s) for s in range(1, 65)]
    scheds = [I.wishart_schedule(p, 16, 16) for p in prs]
    return prs, scheds


def run_ours_batch(args, rank, world, local):
    """Config 3 through the batch engine (tg_batch_*): one launch sweeps every
    instance's 256 replicas.  Under torchrun each rank takes instances
    rank::world (no collective: the instances are independent)."""
    import ctypes as C
    import numpy as np
    import torch
    from paper_2506_14781_b200 import _lib
    from paper_2506_14781_b200.api import Engine, RunConfig, Schedule, run_2dpt_batch

    torch.cuda.set_device(local)
    prs_all, scheds_all = c3_instances()
    mine = list(range(rank, len(prs_all), world))
    prs = [prs_all[b] for b in mine]
    scheds = [Schedule(*scheds_all[b]) for b in mine]
    seeds = [1 + b for b in mine]
    R = 256
    eng = Engine(local)
    L = eng._L
    keep = []
    L.tg_batch_clear(eng._h)
    for pr, sc, sd in zip(prs, scheds, seeds):
        arrs = [np.ascontiguousarray(x, dtype=t) for x, t in (
            (pr.ci, np.int32), (pr.cj, np.int32), (pr.cw, np.float64), (pr.fields, np.float64),
            (pr.pa, np.int32), (pr.pb, np.int32), (sc.betas, np.float64), (sc.penalties, np.float64))]
        keep.append(arrs)
        P = [a.ctypes.data_as(C.c_void_p) for a in arrs]
        eng._check(L.tg_batch_add(eng._h, pr.n, len(arrs[0]), P[0], P[1], P[2], P[3], len(arrs[4]),
                                  P[4], P[5], len(arrs[6]), P[6], len(arrs[7]), P[7], sd, None))
    total = args.rounds * args.sps * (args.warmup + args.steps + 1)
    cfg = RunConfig(total_sweeps=total, sweeps_per_swap=args.sps, seed=1, rule=args.rule,
                    engine=args.engine, store_states=False, digest=False)
    c = eng._cfg(cfg)
    c.record_flags = 0
    eng._check(L.tg_batch_init(eng._h, C.byref(c)))
    eng.set_profiling(True)
    stream = torch.cuda.ExternalStream(eng.stream_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    nosink = C.cast(None, _lib.BATCH_SINK)

    def step():
        eng._check(L.tg_batch_advance(eng._h, args.rounds, nosink, None))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    info0 = eng.info()
    step_ms, sweep_ms = [], 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            sweep_ms += eng.info()["last_sweep_ms"]
    torch.cuda.synchronize()
    barrier(world)
    info1 = eng.info()
    eng.close()
    total_ms = reduce_max(sum(step_ms), world)
    sweeps = args.steps * args.rounds * args.sps
    n_spins = sum(p.n for p in prs_all)
    value = float(n_spins) * R * sweeps / (total_ms / 1e3)
    n_sweep = info1["sweep_launches"] - info0["sweep_launches"]
    launches = n_sweep + info1["other_launches"] - info0["other_launches"]
    mean_sweep_s = reduce_max(sweep_ms, world) / 1e3 / max(n_sweep, 1)
    bal = b_alg(prs[0])
    my_spins = sum(p.n for p in prs)
    achieved = bal * my_spins * R * sweeps / max(n_sweep, 1) / mean_sweep_s / 1e9
    peaks = load_peaks()
    smem_peak = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e9
    clocks = clk.summary()

    # e2e: run_2dpt_batch from pinned host arrays (instances up, build, rounds, records down)
    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    from paper_2506_14781_b200.instances import Problem
    pprs = [Problem(p.n, pinned(p.ci), pinned(p.cj), pinned(p.cw), pinned(p.fields), pinned(p.pa),
                    pinned(p.pb)) for p in prs]
    cfg2 = RunConfig(total_sweeps=args.rounds * args.sps, sweeps_per_swap=args.sps, seed=2,
                     rule=args.rule, engine=args.engine, store_states=False, digest=False)
    times = []
    for k in range(args.warmup + args.steps):
        barrier(world)
        t = time.perf_counter()
        run_2dpt_batch(pprs, scheds, cfg2, seeds, device=local, sink=lambda *a: 0)
        dt = time.perf_counter() - t
        if k >= args.warmup:
            times.append(dt)
    t_e2e = reduce_max(statistics.median(times) * 1e3, world) / 1e3
    h2d = sum(a.nbytes for p in pprs for a in (p.ci, p.cj, p.cw, p.fields, p.pa, p.pb))
    e2e = {"value": float(n_spins) * R * args.rounds * args.sps / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(48 * args.rounds * len(prs)),
           "ms_per_step": 1e3 * t_e2e, "inputs": "pinned host arrays"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, kind, dt = cpu_reference_rate(prs[0], *scheds_all[0], args.cpu_sweeps, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads if kind == "reference" else 1,
               "kind": kind, "sample": f"unmodified reference run_2dpt on instance 1 of 64 "
                                       f"(N={prs[0].n}, 16x16); marginal rate of "
                                       f"{1 + args.cpu_sweeps} vs 1 sweeps ({dt:.1f} s)"}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C3 batch: 64 Wishart N=64 logical (alpha 0.75) -> "
                                   f"{prs_all[0].n} physical each, 16x16 grids, sps={args.sps} "
                                   f"{args.rule}",
                       "instances": len(prs_all), "n_spins_total": n_spins, "replicas": R,
                       "rounds_per_step": args.rounds, "engine": f"{args.engine} (batch)",
                       "parallelism": f"instances x{world}",
                       "l2": "flushed between timed steps (256 MB write)"},
            "roofline": {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                         "frac": achieved / smem_peak, "traffic": None,
                         "kernel": info1.get("sweep_kernel") or "slot2_sweep_kernel",
                         "bytes_per_update": bal, "mean_launch_ms": mean_sweep_s * 1e3},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks}),
            flush=True)


def device_leg(args, pr, betas, pens, rank, world, local, rule):
    """Device-timed throughput: inputs resident in HBM, K steps of
    args.rounds rounds (sweeps + swap phase + per-round digest record), L2
    flushed between steps, CUDA events on the engine's stream, max over
    ranks.  Returns the numbers of the line (and of the heat-bath record)."""
    import torch
    from paper_2506_14781_b200 import _lib
    from paper_2506_14781_b200.api import Engine, RunConfig

    R = len(betas) * len(pens)
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    eng = Engine(local, rank, world, nccl_id)
    eng.set_problem(pr)
    eng.set_schedule(betas, pens)
    total = args.rounds * args.sps * (args.warmup + args.steps + 1)
    cfg = RunConfig(total_sweeps=total, sweeps_per_swap=args.sps, seed=1, rule=rule,
                    engine=args.engine, store_states=False, digest=True)
    eng.init(cfg, flags=_lib.REC_DIGEST)  # per-round (f, g, feasible, target digest) records
    eng.set_profiling(True)
    stream = torch.cuda.ExternalStream(eng.stream_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    nrec = [0]

    def sink(r, n, s, a, b):
        nrec[0] += n
        return 0

    def step():
        eng.advance(args.rounds, sink)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    info0 = eng.info()
    sweep_ms = 0.0
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed steps (not timed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            sweep_ms += eng.info()["last_sweep_ms"]
    torch.cuda.synchronize()
    barrier(world)
    info1 = eng.info()
    eng.close()
    total_ms = reduce_max(sum(step_ms), world)
    sweeps = args.steps * args.rounds * args.sps
    value = float(pr.n) * R * sweeps / (total_ms / 1e3)  # all ranks together
    launches = (info1["sweep_launches"] - info0["sweep_launches"]) + \
               (info1["other_launches"] - info0["other_launches"])
    n_sweep_launches = info1["sweep_launches"] - info0["sweep_launches"]
    mean_sweep_s = reduce_max(sweep_ms, world) / 1e3 / max(n_sweep_launches, 1)
    bal = b_alg(pr)
    # algorithmic bytes of this rank per launch of the dominant kernel
    bytes_per_launch = bal * pr.n * (R / world) * sweeps / max(n_sweep_launches, 1)
    peaks = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    smem_peak_gbs = 148 * 128 * sm_max * 1e6 / 1e9  # SURVEY.md §8d official smem roofline
    achieved_gbs = bytes_per_launch / mean_sweep_s / 1e9
    kname = info1.get("sweep_kernel") or dominant_kernel(args, world)
    return {"value": value, "total_ms": total_ms, "launches": launches, "bal": bal,
            "mean_sweep_s": mean_sweep_s, "achieved_gbs": achieved_gbs, "peak_gbs": smem_peak_gbs,
            "sm_max": sm_max, "kernel": kname, "clocks": clk.summary(), "sweeps": sweeps,
            "sweeps_per_launch": sweeps / max(n_sweep_launches, 1), "records": nrec[0]}


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    from paper_2506_14781_b200 import _lib
    from paper_2506_14781_b200.api import Engine, RunConfig

    torch.cuda.set_device(local)
    pr, betas, pens = workload(args.n, args.workload)
    R = len(betas) * len(pens)
    d = device_leg(args, pr, betas, pens, rank, world, local, args.rule)
    traffic = ncu_traffic(d["kernel"], args, pr, R, d["sweeps_per_launch"])
    hb = None
    if args.workload == "c5" and args.rule == "metropolis" and not args.no_heat_bath:
        # the north star's p-bit rule s = sign(tanh(beta h) - u) on the same workload
        h = device_leg(args, pr, betas, pens, rank, world, local, "heat_bath")
        hb = {"value": h["value"], "unit": UNIT, "ms_per_step": h["total_ms"] / args.steps,
              "kernel": h["kernel"], "roofline_frac": h["achieved_gbs"] / h["peak_gbs"],
              "achieved_gbs": h["achieved_gbs"], "clocks": h["clocks"], "gpu_launches": h["launches"]}

    # e2e: the public API with host buffers -- H2D of the instance (from pinned
    # host memory), device preprocessing, init, the same rounds, per-round
    # digest records to a host sink, D2H of the target configuration.  N = 1:
    # a fresh Engine per step (run_2dpt as a user calls it); N > 1: the Engine
    # (its NCCL communicator) is the session, each step re-sends the instance.
    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    from paper_2506_14781_b200.instances import Problem
    prp = Problem(pr.n, pinned(pr.ci), pinned(pr.cj), pinned(pr.cw), pinned(pr.fields),
                  pinned(pr.pa), pinned(pr.pb))
    cfg2 = RunConfig(total_sweeps=args.rounds * args.sps, sweeps_per_swap=args.sps, seed=2,
                     rule=args.rule, engine=args.engine, store_states=False, digest=True)
    h2d = sum(a.nbytes for a in (prp.ci, prp.cj, prp.cw, prp.fields, prp.pa, prp.pb)) + 8 * (
        len(betas) + len(pens))
    sess = None
    if world > 1:
        import torch.distributed as dist
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        sess = Engine(local, rank, world, obj[0])
    times = []
    tgt = None
    for k in range(args.warmup + args.steps):
        barrier(world)
        t = time.perf_counter()
        e = sess or Engine(local)
        e.set_problem(prp)
        e.set_schedule(betas, pens)
        recs = []
        e.run(cfg2, lambda r, n, s, a, b: recs.append(n) or 0, flags=_lib.REC_DIGEST)
        tgt = e.state(R - 1)
        if sess is None:
            e.close()
        dt = time.perf_counter() - t
        if k >= args.warmup:
            times.append(dt)
    if sess is not None:
        sess.close()
    t_e2e = reduce_max(statistics.median(times) * 1e3, world) / 1e3  # slowest rank
    d2h = tgt.nbytes + 48 * args.rounds
    e2e = {"value": float(pr.n) * R * args.rounds * args.sps / t_e2e,
           "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "ms_per_step": 1e3 * t_e2e, "inputs": "pinned host arrays"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_record(pr, betas, pens, args.cpu_sweeps,
                                  f"unmodified reference run_2dpt (mt19937_64, Metropolis, FP64) on "
                                  f"the same N={pr.n} instance and {R}-replica grid")

    if rank == 0:
        line = {
            "metric": METRIC, "value": d["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": d["total_ms"] / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": bench_config(args, pr, R, world),
            "engine": args.engine,
            "roofline": {"bound": "smem", "achieved": d["achieved_gbs"], "peak": d["peak_gbs"],
                         "unit": "GB/s", "frac": d["achieved_gbs"] / d["peak_gbs"],
                         "traffic": traffic["bytes_per_launch"] if traffic else None,
                         "traffic_source": traffic["source"] if traffic else None,
                         "issue": issue_roofline(traffic, d["value"] / world, d["sm_max"]),
                         "kernel": d["kernel"],
                         "bytes_per_update": d["bal"],
                         "mean_launch_ms": d["mean_sweep_s"] * 1e3,
                         "peak_note": "148 SM x 128 B/clk x sm_max_mhz (MEASURED_PEAKS.json), "
                                      "SURVEY.md §8d"},
            "heat_bath": hb,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(d["launches"]),
            "records_per_step": d["records"] // max(args.steps + args.warmup, 1),
            "clocks": d["clocks"],
        }
        print(json.dumps(line), flush=True)


def dominant_kernel(args, world):
    if args.engine == "slot":
        return "slot2_sweep_kernel" if world == 1 else "slot_sweep_kernel"
    return "plane_tpw_rounds_kernel" if world == 1 else "plane_sweep_kernel"


def issue_roofline(traffic, updates_per_s_per_gpu, sm_max_mhz):
    """The bound the integer-issue kernels actually meet: lane-instructions per
    spin update (committed ncu capture, smsp__inst_executed x 32 / updates)
    against the SM issue peak (148 SMs x 4 schedulers x 32 lanes x clock)."""
    ipu = traffic.get("lane_instr_per_update") if traffic else None
    if not ipu:
        return None
    peak = 148 * 4 * 32 * sm_max_mhz * 1e6
    bound = peak / ipu
    return {"lane_instr_per_update": ipu, "peak_lane_instr_per_s": peak,
            "issue_bound_updates_per_s": bound, "frac": updates_per_s_per_gpu / bound,
            "note": "issue-slot roofline of the dominant kernel; instructions/update from profiles/traffic.json"}


def ncu_traffic(kname, args, pr, R, sweeps_per_launch):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel from the
    committed `ncu --set full` capture (profiles/traffic.json), rescaled from the
    captured launch to this run's launch size (the kernel's DRAM traffic is per
    sweep of the same instance); None when no capture matches this workload."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as fh:
            caps = json.load(fh)
    except (OSError, ValueError):
        return None
    for c in caps:
        if c.get("kernel") == kname and c.get("workload") == args.workload and \
                c.get("n_spins") == pr.n and c.get("replicas") == R and c.get("rule") == args.rule:
            per_sweep = c["dram_bytes"] / c["sweeps_per_launch"]
            return {"bytes_per_launch": per_sweep * sweeps_per_launch,
                    "source": f"profiles/traffic.json: {c['source']}",
                    "lane_instr_per_update": c.get("lane_instr_per_update")}
    return None


def spawn_or_check(args):
    """--gpus N > 1 without torchrun: re-launch this command as N ranks (one
    process per GPU over NCCL); under torchrun WORLD_SIZE must equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                   "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
            sys.exit(subprocess.call(cmd))
        return
    if int(world) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)


def main():
    args = parse()
    spawn_or_check(args)
    if args.workload != "c5" and args.engine == "plane":
        args.engine = "float"  # float32 Wishart couplings: the FLOAT engine (--engine slot: SLOT v2)
    if args.impl == "reference":
        # the reference arm never maps the engine library: instances are built
        # with the pure-Python host helpers, the timed code is oracle/_ref
        from paper_2506_14781_b200 import instances as I
        I.use_native_helpers(False)
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, rank, int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, world, local = dist_setup(args.gpus)
    if args.workload == "c3":
        run_ours_batch(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
