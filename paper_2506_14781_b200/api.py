"""Python mirror of the reference's run_2dpt API over the C ABI.

Same names, argument meaning and error behaviour as
``tempergrid::run_2dpt`` (/root/reference/proj/include/tempergrid/engine.hpp:26-63)
-- ``RunConfig``, ``Schedule``, ``TraceRecord``, ``Trace`` -- with the
reference's exceptions mapped from the C status codes (config_error -> 2,
resource_error -> 3).  Extra ``RunConfig`` fields select the update rule and
the engine; their defaults keep the reference's Metropolis rule.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from .instances import ConfigError, Problem, ResourceError


class EngineError(RuntimeError):
    pass


def _raise(code: int, msg: str):
    if code == _lib.TG_ERR_CONFIG:
        raise ConfigError(msg)
    if code == _lib.TG_ERR_RESOURCE:
        raise ResourceError(msg)
    raise EngineError(f"[{code}] {msg}")


@dataclass
class Schedule:
    """schedule.hpp:35-42 (betas per row, penalties per column)."""
    betas: Sequence[float]
    penalties: Sequence[float]


@dataclass
class RunConfig:
    """engine.hpp:26-32 plus engine options."""
    total_sweeps: int = 0
    sweeps_per_swap: int = 1
    seed: int = 1
    store_target_only: bool = True
    threads: int = 1                 # accepted for API parity; results never depend on it
    rule: str = "metropolis"         # or "heat_bath"
    engine: str = "auto"             # "slot" | "plane" | "float" | "auto"
    record_every: int = 1
    store_states: bool = True        # TraceRecord.state for every record
    digest: bool = True


@dataclass
class TraceRecord:
    """engine.hpp:39-50"""
    round: int
    sweep_count: int
    f: float
    g: float
    feasible: bool
    state: Optional[np.ndarray]
    acceptance_rates_p: List[float]
    acceptance_rates_beta: List[float]
    grid: Optional[np.ndarray] = None
    digest: int = 0
    target_state: int = -1


@dataclass
class Trace:
    """engine.hpp:52-56"""
    betas: List[float]
    penalties: List[float]
    sweeps_per_swap: int
    records: List[TraceRecord] = field(default_factory=list)


def p_swap_probability(beta: float, d_penalty: float, dg: float) -> float:
    return _lib.lib().tg_p_swap_probability(beta, d_penalty, dg)


def beta_swap_probability(d_beta: float, d_energy: float) -> float:
    return _lib.lib().tg_beta_swap_probability(d_beta, d_energy)


def general_swap_probability(beta_a: float, beta_b: float, de_a: float, de_b: float) -> float:
    return _lib.lib().tg_general_swap_probability(beta_a, beta_b, de_a, de_b)


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def attempts_per_round(I: int, J: int, rnd: int):
    """Deterministic attempt counts of round `rnd` (engine.cpp:121-187)."""
    even = 1 if rnd % 2 == 0 else 0
    direction = 1 if ((rnd - 1) // 2) % 2 == 0 else -1
    if I == 1 and J == 1:
        dp = db = False
    elif I == 1:
        dp, db = True, False
    elif J == 1:
        dp, db = False, True
    else:
        dp, db = direction == 1, direction != 1
    ap = np.zeros(I * max(J - 1, 0), np.int64)
    ab = np.zeros(max(I - 1, 0) * J, np.int64)
    if dp:
        for i in range(I):
            for p in range(even, J - 1, 2):
                ap[i * (J - 1) + p] += 1
    if db:
        for j in range(J):
            for b in range(even, I - 1, 2):
                ab[b * J + j] += 1
    return ap, ab


class Engine:
    """One engine context (one GPU).  Thin owner of a ``tg_ctx``."""

    def __init__(self, device: int = 0, rank: int = 0, world_size: int = 1,
                 nccl_id: Optional[bytes] = None):
        self._L = _lib.lib()
        h = C.c_void_p()
        if world_size == 1 and nccl_id is None:
            rc = self._L.tg_create(device, C.byref(h))
        else:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            rc = self._L.tg_create_distributed(device, rank, world_size, buf, C.byref(h))
        if rc != 0:
            _raise(rc, self._err(None))
        self._h = h
        self.problem: Optional[Problem] = None
        self.schedule: Optional[Schedule] = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        rc = _lib.lib().tg_nccl_unique_id(buf)
        if rc != 0:
            raise EngineError("ncclGetUniqueId failed")
        return buf.raw

    def _err(self, h) -> str:
        buf = C.create_string_buffer(1024)
        self._L.tg_last_error(h, buf, 1024)
        return buf.value.decode()

    def _check(self, rc: int):
        if rc != 0:
            _raise(rc, self._err(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._L.tg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------ setup
    def set_problem(self, pr: Problem):
        self._keep_p = [_arr(pr.ci, np.int32), _arr(pr.cj, np.int32), _arr(pr.cw, np.float64),
                        _arr(pr.fields, np.float64), _arr(pr.pa, np.int32), _arr(pr.pb, np.int32)]
        ci, cj, cw, h, pa, pb = self._keep_p
        self._check(self._L.tg_set_problem(self._h, pr.n, len(ci), _p(ci), _p(cj), _p(cw), _p(h),
                                           len(pa), _p(pa), _p(pb)))
        self.problem = pr

    def set_schedule(self, betas, penalties):
        b, p = _arr(betas, np.float64), _arr(penalties, np.float64)
        self._check(self._L.tg_set_schedule(self._h, len(b), _p(b), len(p), _p(p)))
        self.schedule = Schedule(list(b), list(p))

    def _cfg(self, cfg: RunConfig) -> _lib.RunConfigC:
        flags = 0
        if cfg.digest:
            flags |= _lib.REC_DIGEST
        if cfg.store_states:
            flags |= _lib.REC_STATE
        if not cfg.store_target_only:
            flags |= _lib.REC_GRID
        flags |= _lib.REC_COUNTERS
        if cfg.rule not in _lib.RULES:
            raise ConfigError(f"run: unknown rule {cfg.rule}")
        if cfg.engine not in _lib.ENGINES:
            raise ConfigError(f"run: unknown engine {cfg.engine}")
        return _lib.RunConfigC(int(cfg.total_sweeps), int(cfg.sweeps_per_swap),
                               int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, _lib.RULES[cfg.rule],
                               _lib.ENGINES[cfg.engine], flags, max(int(cfg.record_every), 1))

    def init(self, cfg: RunConfig, flags: Optional[int] = None):
        c = self._cfg(cfg)
        if flags is not None:
            c.record_flags = flags
        self._check(self._L.tg_init(self._h, C.byref(c)))
        self._cfg_py = cfg

    def advance(self, n_rounds: int, sink: Optional[Callable] = None):
        cb = _make_sink(sink) if sink else C.cast(None, _lib.SINK)
        self._check(self._L.tg_advance(self._h, int(n_rounds), cb, None))

    def run(self, cfg: RunConfig, sink: Optional[Callable] = None, flags: Optional[int] = None):
        c = self._cfg(cfg)
        if flags is not None:
            c.record_flags = flags
        cb = _make_sink(sink) if sink else C.cast(None, _lib.SINK)
        self._check(self._L.tg_run(self._h, C.byref(c), cb, None))

    # ------------------------------------------------------------ queries
    def state(self, slot: int) -> np.ndarray:
        out = np.zeros(self.problem.n, np.int8)
        self._check(self._L.tg_get_state(self._h, int(slot), _p(out)))
        return out

    def grid(self) -> np.ndarray:
        R = len(self.schedule.betas) * len(self.schedule.penalties)
        return np.stack([self.state(r) for r in range(R)])

    def counters(self):
        I, J = len(self.schedule.betas), len(self.schedule.penalties)
        ap, cp = np.zeros(I * max(J - 1, 0), np.int64), np.zeros(I * max(J - 1, 0), np.int64)
        ab, cb = np.zeros(max(I - 1, 0) * J, np.int64), np.zeros(max(I - 1, 0) * J, np.int64)
        self._check(self._L.tg_get_counters(self._h, _p(ap), _p(cp), _p(ab), _p(cb)))
        return ap, cp, ab, cb

    def energies(self):
        R = len(self.schedule.betas) * len(self.schedule.penalties)
        f, g = np.zeros(R), np.zeros(R)
        self._check(self._L.tg_get_energies(self._h, _p(f), _p(g)))
        return f, g

    def info(self) -> dict:
        i = _lib.InfoC()
        self._check(self._L.tg_get_info(self._h, C.byref(i)))
        d = {k: getattr(i, k) for k, _ in _lib.InfoC._fields_}
        d["sweep_kernel"] = d["sweep_kernel"].decode()
        return d

    def stream_ptr(self) -> int:
        return int(self._L.tg_stream(self._h) or 0)

    def set_kl_decoder(self, logical: Problem, copies, beta: float, discard_infeasible: bool = False):
        """Decoded-sample KL observer for the following SLOT-engine runs
        (``tg_set_kl_decoder``; kl_curve, analysis.cpp:215-241)."""
        li, lj = _arr(logical.ci, np.int32), _arr(logical.cj, np.int32)
        lw, lh = _arr(logical.cw, np.float64), _arr(logical.fields, np.float64)
        off = np.zeros(len(copies) + 1, np.int32)
        off[1:] = np.cumsum([len(c) for c in copies])
        flat = _arr(np.concatenate([np.asarray(c, np.int64) for c in copies]) if len(copies) else
                    np.zeros(0), np.int32)
        self._check(self._L.tg_set_kl_decoder(self._h, logical.n, len(li), _p(li), _p(lj), _p(lw),
                                              _p(lh), float(beta), _p(off), _p(flat),
                                              1 if discard_infeasible else 0))
        self._kl_k = 1 << logical.n

    def clear_kl_decoder(self):
        self._check(self._L.tg_clear_kl_decoder(self._h))

    def kl_curve(self, instance: int = 0, rounds: Optional[int] = None,
                 sweeps_per_swap: int = 1) -> List["KlPoint"]:
        """The device KL curve of the last decoded run (KlPoint, analysis.hpp:74-79)."""
        if rounds is None:
            rounds = int(self.info()["rounds_done"])
        kl = np.zeros(rounds)
        smp = np.zeros(rounds, np.int64)
        self._check(self._L.tg_get_kl_curve(self._h, int(instance), 1, int(rounds), _p(kl), _p(smp)))
        k = self._kl_k
        return [KlPoint(int((r + 1) * sweeps_per_swap), int(smp[r]), float(kl[r]),
                        (k - 1) / (2.0 * smp[r]) if smp[r] > 0 else float("nan"))
                for r in range(rounds)]

    def checkpoint(self) -> bytes:
        """Snapshot of the run (``tg_checkpoint``): spins of every physical
        state, slot labels, accept counters, round counter, swap-stream
        position.  The reference has no resume (engine.hpp:39-56)."""
        n = C.c_size_t()
        self._check(self._L.tg_checkpoint_size(self._h, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self._check(self._L.tg_checkpoint(self._h, buf, n.value))
        return buf.raw

    def restore(self, blob: bytes):
        """Continue from a checkpoint (``tg_restore``) on a context initialised
        with the same problem, schedule and config."""
        buf = C.create_string_buffer(bytes(blob), len(blob))
        self._check(self._L.tg_restore(self._h, buf, len(blob)))

    def set_profiling(self, on: bool):
        self._check(self._L.tg_set_profiling(self._h, 1 if on else 0))


def _make_sink(fn: Callable):
    def _cb(user, recs, n, states, acc_p, acc_b):
        try:
            return int(fn(recs, int(n), states, acc_p, acc_b) or 0)
        except Exception:  # noqa: BLE001 - report through the C status
            import traceback
            traceback.print_exc()
            return 1
    return _lib.SINK(_cb)


def run_2dpt(problem: Problem, schedule: Schedule, cfg: RunConfig, device: int = 0,
             engine: Optional[Engine] = None) -> Trace:
    """Drop-in for ``tempergrid::run_2dpt`` (engine.cpp:83-219) on a B200."""
    I, J = len(schedule.betas), len(schedule.penalties)
    R, n = I * J, problem.n
    trace = Trace(list(map(float, schedule.betas)), list(map(float, schedule.penalties)),
                  int(cfg.sweeps_per_swap))
    eng = engine or Engine(device)
    try:
        eng.set_problem(problem)
        eng.set_schedule(schedule.betas, schedule.penalties)
        np_, nb_ = I * max(J - 1, 0), max(I - 1, 0) * J
        att_p = np.zeros(np_, np.int64)
        att_b = np.zeros(nb_, np.int64)
        last_round = [0]

        def sink(recs, cnt, states, acc_p, acc_b):
            per = (R * n) if not cfg.store_target_only else (n if cfg.store_states else 0)
            st = (np.ctypeslib.as_array(states, shape=(cnt * per,)).copy() if per and states
                  else None)
            ap = np.ctypeslib.as_array(acc_p, shape=(cnt * np_,)).copy() if np_ else np.zeros(0, np.int64)
            ab = np.ctypeslib.as_array(acc_b, shape=(cnt * nb_,)).copy() if nb_ else np.zeros(0, np.int64)
            for k in range(cnt):
                r = recs[k]
                # cumulative attempts up to this round (deterministic)
                while last_round[0] < r.round:
                    last_round[0] += 1
                    a1, a2 = attempts_per_round(I, J, last_round[0])
                    att_p[:] += a1
                    att_b[:] += a2
                cp = ap[k * np_:(k + 1) * np_]
                cb = ab[k * nb_:(k + 1) * nb_]
                rp = [float(c) / a if a else 0.0 for c, a in zip(cp, att_p)]
                rb = [float(c) / a if a else 0.0 for c, a in zip(cb, att_b)]
                state = grid = None
                if st is not None:
                    chunk = st[k * per:(k + 1) * per]
                    if cfg.store_target_only:
                        state = chunk.copy()
                    else:
                        grid = chunk.reshape(R, n).copy()
                        state = grid[R - 1].copy()
                trace.records.append(TraceRecord(int(r.round), int(r.sweep_count), float(r.f),
                                                 float(r.g), bool(r.feasible), state, rp, rb, grid,
                                                 int(r.digest), int(r.target_state)))
            return 0

        eng.run(cfg, sink)
    finally:
        if engine is None:
            eng.close()
    return trace


def run_2dpt_batch(problems: Sequence[Problem], schedules: Sequence[Schedule], cfg: RunConfig,
                   seeds: Sequence[int], device: int = 0, engine: Optional[Engine] = None,
                   sink: Optional[Callable] = None) -> List[Trace]:
    """Independent instances in one launch (SURVEY.md §8b ``run_2dpt_batch``,
    config 3).  Result b equals ``run_2dpt(problems[b], schedules[b], cfg with
    seed=seeds[b])`` under the SLOT engine.  With ``sink`` set, records are
    streamed to ``sink(instance, records, n, states, acc_p, acc_b)`` instead of
    being collected into Traces."""
    if not (len(problems) == len(schedules) == len(seeds)):
        raise ConfigError("batch: problems, schedules and seeds differ in length")
    eng = engine or Engine(device)
    L = eng._L
    try:
        L.tg_batch_clear(eng._h)
        keep = []
        for pr, sc, sd in zip(problems, schedules, seeds):
            arrs = [_arr(pr.ci, np.int32), _arr(pr.cj, np.int32), _arr(pr.cw, np.float64),
                    _arr(pr.fields, np.float64), _arr(pr.pa, np.int32), _arr(pr.pb, np.int32),
                    _arr(sc.betas, np.float64), _arr(sc.penalties, np.float64)]
            keep.append(arrs)
            ci, cj, cw, h, pa, pb, b, p = arrs
            eng._check(L.tg_batch_add(eng._h, pr.n, len(ci), _p(ci), _p(cj), _p(cw), _p(h), len(pa),
                                      _p(pa), _p(pb), len(b), _p(b), len(p), _p(p),
                                      int(sd) & 0xFFFFFFFFFFFFFFFF, None))
        c = eng._cfg(cfg)
        c.engine = _lib.ENGINES["slot"] if cfg.engine == "auto" else c.engine
        traces = [Trace(list(map(float, sc.betas)), list(map(float, sc.penalties)),
                        int(cfg.sweeps_per_swap)) for sc in schedules]
        I, J = len(schedules[0].betas), len(schedules[0].penalties)
        R = I * J
        np_, nb_ = I * max(J - 1, 0), max(I - 1, 0) * J
        att = [[np.zeros(np_, np.int64), np.zeros(nb_, np.int64), 0] for _ in problems]

        def _cb(user, b, recs, n, states, acc_p, acc_b):
            try:
                if sink is not None:
                    return int(sink(b, recs, int(n), states, acc_p, acc_b) or 0)
                pr = problems[b]
                per = (R * pr.n) if not cfg.store_target_only else (pr.n if cfg.store_states else 0)
                st = (np.ctypeslib.as_array(states, shape=(n * per,)).copy() if per and states else None)
                ap = np.ctypeslib.as_array(acc_p, shape=(n * np_,)).copy() if np_ else np.zeros(0, np.int64)
                ab = np.ctypeslib.as_array(acc_b, shape=(n * nb_,)).copy() if nb_ else np.zeros(0, np.int64)
                a = att[b]
                for k in range(n):
                    r = recs[k]
                    while a[2] < r.round:
                        a[2] += 1
                        x1, x2 = attempts_per_round(I, J, a[2])
                        a[0][:] += x1
                        a[1][:] += x2
                    cp, cb_ = ap[k * np_:(k + 1) * np_], ab[k * nb_:(k + 1) * nb_]
                    rp = [float(v) / q if q else 0.0 for v, q in zip(cp, a[0])]
                    rb = [float(v) / q if q else 0.0 for v, q in zip(cb_, a[1])]
                    state = grid = None
                    if st is not None:
                        chunk = st[k * per:(k + 1) * per]
                        if cfg.store_target_only:
                            state = chunk.copy()
                        else:
                            grid = chunk.reshape(R, pr.n).copy()
                            state = grid[R - 1].copy()
                    traces[b].records.append(TraceRecord(int(r.round), int(r.sweep_count), float(r.f),
                                                         float(r.g), bool(r.feasible), state, rp, rb,
                                                         grid, int(r.digest), int(r.target_state)))
                return 0
            except Exception:  # noqa: BLE001
                import traceback
                traceback.print_exc()
                return 1

        cb = _lib.BATCH_SINK(_cb)
        eng._check(L.tg_batch_run(eng._h, C.byref(c), cb, None))
        eng._batch_problems = problems
        return traces
    finally:
        if engine is None:
            eng.close()


@dataclass
class KlPoint:
    """``tempergrid::KlPoint`` (analysis.hpp:74-79)."""
    t: int
    samples: int
    kl: float
    iid_reference: float


def run_2dpt_kl(problem: Problem, schedule: Schedule, cfg: RunConfig, logical: Problem, copies,
                beta: float, discard_infeasible: bool = False, device: int = 0,
                engine: Optional[Engine] = None) -> List[KlPoint]:
    """``kl_curve(run_2dpt(...), map, logical, beta, discard)`` (analysis.cpp:215-241)
    with the decode, histogram and KL evaluated on the device every round."""
    eng = engine or Engine(device)
    try:
        eng.set_kl_decoder(logical, copies, beta, discard_infeasible)
        eng.set_problem(problem)
        eng.set_schedule(schedule.betas, schedule.penalties)
        c = RunConfig(**{**cfg.__dict__, "engine": "slot", "store_states": False, "digest": False})
        eng.run(c, None, flags=0)
        rounds = int(cfg.total_sweeps) // max(int(cfg.sweeps_per_swap), 1)
        return eng.kl_curve(0, rounds, int(cfg.sweeps_per_swap))
    finally:
        if engine is None:
            eng.close()


@dataclass
class BaselineRecord:
    """``tempergrid::BaselineRecord`` (engine.hpp:67-74)."""
    round: int
    sweep_count: int
    best_f: float
    any_feasible: bool
    n_feasible: int
    n_total: int


@dataclass
class BaselineTrace:
    """``tempergrid::BaselineTrace`` (engine.hpp:76-82)."""
    betas: List[float]
    penalty: float
    sweeps_per_swap: int
    records: List[BaselineRecord] = field(default_factory=list)
    feasible_fraction: float = 0.0


def run_jcolumn_pt(problem: Problem, betas, p_fixed: float, j_repeats: int, cfg: RunConfig,
                   device: int = 0, engine: Optional[Engine] = None) -> BaselineTrace:
    """Drop-in for ``tempergrid::run_jcolumn_pt`` (engine.cpp:221-270): the
    resource-matched baseline of J independent standard-PT columns at a fixed
    penalty, run as one device batch (``tg_run_jcolumn``) and merged per round."""
    if not p_fixed > 0.0:  # engine.cpp:224-225, checked before anything else
        raise ConfigError("baseline: P must be positive")
    if j_repeats < 1:
        raise ConfigError("baseline: repeats must be >= 1")
    b = _arr(betas, np.float64)
    eng = engine or Engine(device)
    try:
        eng.set_problem(problem)
        rounds = int(cfg.total_sweeps) // max(int(cfg.sweeps_per_swap), 1)
        recs = (_lib.BaselineRecordC * max(rounds, 1))()
        ff = C.c_double(0.0)
        c = eng._cfg(cfg)
        eng._check(eng._L.tg_run_jcolumn(eng._h, len(b), _p(b), float(p_fixed), int(j_repeats),
                                         C.byref(c), recs, rounds, C.byref(ff)))
        out = BaselineTrace(list(map(float, b)), float(p_fixed), int(cfg.sweeps_per_swap))
        out.records = [BaselineRecord(int(r.round), int(r.sweep_count), float(r.best_f),
                                      bool(r.any_feasible), int(r.n_feasible), int(r.n_total))
                       for r in recs[:rounds]]
        out.feasible_fraction = float(ff.value)
        return out
    finally:
        if engine is None:
            eng.close()


@dataclass
class ProbeStats:
    """``tempergrid::ProbeStats`` (schedule.hpp:24-32)."""
    row: int = 0
    column: int = 0
    beta: float = 0.0
    penalty: float = 0.0
    sigma_e: float = 0.0
    sigma_g: float = 0.0
    mean_g: float = 0.0


@dataclass
class ScheduleConfig:
    """``tempergrid::ScheduleConfig`` (schedule.hpp:10-22) plus the probe sweep rule."""
    beta0: float = 0.3
    p0: float = 0.5
    i_max: int = 20
    j_max: int = 20
    sigma_min: float = 0.0
    alpha_beta: float = 1.0
    alpha_p: float = 1.2
    n_chains: int = 32
    sweeps_per_probe: int = 1000
    replica_budget: int = 400
    seed: int = 1
    rule: str = "metropolis"


@dataclass
class BuiltSchedule(Schedule):
    """``tempergrid::Schedule`` as build_schedule returns it (schedule.hpp:34-42)."""
    probe_stats: List[ProbeStats] = field(default_factory=list)
    budget_exhausted: bool = False


def _stats(s) -> ProbeStats:
    return ProbeStats(int(s.row), int(s.column), float(s.beta), float(s.penalty), float(s.sigma_e),
                      float(s.sigma_g), float(s.mean_g))


def probe_population(problem: Problem, beta: float, penalty: float, n_chains: int, sweeps: int,
                     seed: int, rule: str = "metropolis", device: int = 0,
                     engine: Optional[Engine] = None) -> ProbeStats:
    """Drop-in for ``tempergrid::probe_population`` (schedule.cpp:18-52): all
    chains in one device launch (``tg_probe_population``)."""
    eng = engine or Engine(device)
    try:
        eng.set_problem(problem)
        out = _lib.ProbeStatsC()
        eng._check(eng._L.tg_probe_population(eng._h, float(beta), float(penalty), int(n_chains),
                                              int(sweeps), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                              _lib.RULES[rule], C.byref(out)))
        return _stats(out)
    finally:
        if engine is None:
            eng.close()


def build_schedule(problem: Problem, cfg: Optional[ScheduleConfig] = None, device: int = 0,
                   engine: Optional[Engine] = None) -> BuiltSchedule:
    """Drop-in for ``tempergrid::build_schedule`` (schedule.cpp:77-163): the
    adaptive (beta, P) ladder, every probe on the device (``tg_build_schedule``)."""
    cfg = cfg or ScheduleConfig()
    c = _lib.ScheduleConfigC(float(cfg.beta0), float(cfg.p0), int(cfg.i_max), int(cfg.j_max),
                             float(cfg.sigma_min), float(cfg.alpha_beta), float(cfg.alpha_p),
                             int(cfg.n_chains), int(cfg.sweeps_per_probe), int(cfg.replica_budget),
                             _lib.RULES[cfg.rule], int(cfg.seed) & 0xFFFFFFFFFFFFFFFF)
    im, jm = max(int(cfg.i_max), 1), max(int(cfg.j_max), 1)
    betas, pens = np.zeros(im), np.zeros(jm + 1)
    cap = im * (jm + 1) + 1
    stats = (_lib.ProbeStatsC * cap)()
    nb, npn, ns, ex = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    eng = engine or Engine(device)
    try:
        eng.set_problem(problem)
        eng._check(eng._L.tg_build_schedule(eng._h, C.byref(c), _p(betas), im, C.byref(nb), _p(pens),
                                            jm + 1, C.byref(npn), stats, cap, C.byref(ns),
                                            C.byref(ex)))
    finally:
        if engine is None:
            eng.close()
    out = BuiltSchedule(list(map(float, betas[:nb.value])), list(map(float, pens[:npn.value])))
    out.probe_stats = [_stats(stats[k]) for k in range(min(ns.value, cap))]
    out.budget_exhausted = bool(ex.value)
    return out


def batch_state(engine: Engine, instance: int, slot: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.int8)
    engine._check(engine._L.tg_batch_get_state(engine._h, int(instance), int(slot), _p(out)))
    return out
