"""oracle/pyoracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the parity checkers: the C restatement
(``build/libtg_oracle.so``, tg_oracle.c) and the reference's own sources built
into ``_ref/libtgref_*.so`` (ref_harness.cpp).  Imported only by tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference legs.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "build", "libtg_oracle.so")
REF_LIBS = {
    "mt": "libtgref_mt.so",            # O1: unmodified reference
    "philox": "libtgref_philox.so",    # O2: reference + Philox streams
    "philox_hb": "libtgref_philox_hb.so",
    "plane": "libtgref_plane.so",
    "plane_hb": "libtgref_plane_hb.so",
    "pack": "libtgref_pack.so",        # O2: reference + packed draws (FLOAT engine)
    "pack_hb": "libtgref_pack_hb.so",
}

RULE = {"metropolis": 0, "heat_bath": 1}
RNG = {"slot": 0, "plane": 1, "float": 2}


class _Problem(C.Structure):
    _fields_ = [("n", C.c_int), ("n_couplings", C.c_int), ("ci", C.c_void_p), ("cj", C.c_void_p),
                ("cw", C.c_void_p), ("fields", C.c_void_p), ("n_pairs", C.c_int),
                ("pa", C.c_void_p), ("pb", C.c_void_p)]


class _RunCfg(C.Structure):
    _fields_ = [("n_betas", C.c_int), ("betas", C.c_void_p), ("n_penalties", C.c_int),
                ("penalties", C.c_void_p), ("total_sweeps", C.c_int64),
                ("sweeps_per_swap", C.c_int64), ("seed", C.c_uint64), ("rule", C.c_int),
                ("rng_mode", C.c_int)]


class _Outputs(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in (
        "f", "g", "feasible", "digest", "states", "grid_states", "round_acc_p", "round_acc_b",
        "attempts_p", "accepts_p", "attempts_b", "accepts_b", "final_grid", "final_f",
        "final_g", "final_state_id")]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_port = None
_refs = {}


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_LIB):
            raise RuntimeError(f"oracle port not built: {PORT_LIB} (run `make -C oracle port`)")
        _port = C.CDLL(PORT_LIB)
        _port.tgo_run_2dpt.restype = C.c_int
        _port.tgo_digest.restype = C.c_uint64
        _port.tgo_encode_state.restype = C.c_uint64
        _port.tgo_derive.restype = C.c_uint64
        _port.tgo_derive.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        _port.tgo_bits.restype = C.c_uint64
        _port.tgo_bits.argtypes = [C.c_uint64, C.c_uint64]
        _port.tgo_plane.restype = C.c_uint64
        _port.tgo_plane.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int]
        for fn in ("tgo_p_swap_probability", "tgo_beta_swap_probability",
                   "tgo_general_swap_probability"):
            getattr(_port, fn).restype = C.c_double
        _port.tgo_p_swap_probability.argtypes = [C.c_double] * 3
        _port.tgo_beta_swap_probability.argtypes = [C.c_double] * 2
        _port.tgo_general_swap_probability.argtypes = [C.c_double] * 4
    return _port


def ref_available(variant: str = "philox") -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", REF_LIBS[variant]))


def ref_lib(variant: str):
    if variant not in _refs:
        path = os.path.join(HERE, "_ref", REF_LIBS[variant])
        if not os.path.exists(path):
            raise RuntimeError(f"reference oracle not built: {path} (run `make -C oracle ref`)")
        lib = C.CDLL(path)
        lib.tgr_run_2dpt.restype = C.c_int
        lib.tgr_run_2dpt_timed.restype = C.c_int
        _refs[variant] = lib
    return _refs[variant]


@dataclass
class OracleResult:
    f: np.ndarray
    g: np.ndarray
    feasible: np.ndarray
    digest: np.ndarray
    states: Optional[np.ndarray]
    attempts_p: np.ndarray
    accepts_p: np.ndarray
    attempts_b: np.ndarray
    accepts_b: np.ndarray
    round_acc_p: Optional[np.ndarray]
    round_acc_b: Optional[np.ndarray]
    final_grid: Optional[np.ndarray]
    grid_states: Optional[np.ndarray] = None


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _marshal(pr, betas, penalties, total_sweeps, sps, seed, rule, rng_mode):
    keep = {
        "ci": np.ascontiguousarray(pr.ci, dtype=np.int32),
        "cj": np.ascontiguousarray(pr.cj, dtype=np.int32),
        "cw": np.ascontiguousarray(pr.cw, dtype=np.float64),
        "h": np.ascontiguousarray(pr.fields, dtype=np.float64),
        "pa": np.ascontiguousarray(pr.pa, dtype=np.int32),
        "pb": np.ascontiguousarray(pr.pb, dtype=np.int32),
        "betas": np.ascontiguousarray(betas, dtype=np.float64),
        "pens": np.ascontiguousarray(penalties, dtype=np.float64),
    }
    p = _Problem(pr.n, len(keep["ci"]), _ptr(keep["ci"]), _ptr(keep["cj"]), _ptr(keep["cw"]),
                 _ptr(keep["h"]), len(keep["pa"]), _ptr(keep["pa"]), _ptr(keep["pb"]))
    c = _RunCfg(len(keep["betas"]), _ptr(keep["betas"]), len(keep["pens"]), _ptr(keep["pens"]),
                int(total_sweeps), int(sps), int(seed) & 0xFFFFFFFFFFFFFFFF, RULE[rule], RNG[rng_mode])
    return p, c, keep


def run(pr, betas, penalties, total_sweeps, sps=1, seed=1, rule="metropolis", rng="slot",
        impl="port", states=False, grid=False, round_counters=False, threads=1,
        final_grid=True) -> OracleResult:
    """Run one 2D-PT trajectory on the C port (impl='port') or on a reference
    build (impl='ref:<variant>')."""
    p, c, keep = _marshal(pr, betas, penalties, total_sweeps, sps, seed, rule, rng)
    I, J = len(keep["betas"]), len(keep["pens"])
    R = I * J
    rounds = int(total_sweeps) // max(int(sps), 1)
    npp, nbb = I * max(J - 1, 0), max(I - 1, 0) * J
    o = dict(
        f=np.zeros(rounds), g=np.zeros(rounds), feasible=np.zeros(rounds, np.uint8),
        digest=np.zeros(rounds, np.uint64),
        states=np.zeros((rounds, pr.n), np.int8) if states else None,
        grid_states=np.zeros((rounds, R, pr.n), np.int8) if grid else None,
        round_acc_p=np.zeros((rounds, npp), np.int64) if round_counters else None,
        round_acc_b=np.zeros((rounds, nbb), np.int64) if round_counters else None,
        attempts_p=np.zeros(npp, np.int64), accepts_p=np.zeros(npp, np.int64),
        attempts_b=np.zeros(nbb, np.int64), accepts_b=np.zeros(nbb, np.int64),
        final_grid=np.zeros((R, pr.n), np.int8) if final_grid else None,
    )
    out = _Outputs(*[_ptr(o.get(k)) for k, _ in _Outputs._fields_])
    err = C.create_string_buffer(512)
    if impl == "port":
        if threads > 1:  # sweep threads of the port (result independent of the count)
            os.environ["TGO_THREADS"] = str(int(threads))
        try:
            rc = port_lib().tgo_run_2dpt(C.byref(p), C.byref(c), C.byref(out), err, 512)
        finally:
            if threads > 1:
                os.environ.pop("TGO_THREADS", None)
    else:
        variant = impl.split(":", 1)[1]
        rc = ref_lib(variant).tgr_run_2dpt(C.byref(p), C.byref(c), C.byref(out), int(threads),
                                           0, err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return OracleResult(o["f"], o["g"], o["feasible"].astype(bool), o["digest"], o["states"],
                        o["attempts_p"], o["accepts_p"], o["attempts_b"], o["accepts_b"],
                        o["round_acc_p"], o["round_acc_b"], o["final_grid"], o["grid_states"])


class _BaselineOut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in (
        "round", "sweep_count", "best_f", "any_feasible", "n_feasible", "n_total",
        "feasible_fraction")]


@dataclass
class BaselineResult:
    round: np.ndarray
    sweep_count: np.ndarray
    best_f: np.ndarray
    any_feasible: np.ndarray
    n_feasible: np.ndarray
    n_total: np.ndarray
    feasible_fraction: float


def run_jcolumn(pr, betas, p_fixed, j_repeats, total_sweeps, sps=1, seed=1, rule="metropolis",
                impl="port", threads=1) -> BaselineResult:
    """run_jcolumn_pt (engine.cpp:221-270) on the C port or a reference build."""
    p, c, keep = _marshal(pr, betas, [max(float(p_fixed), 0.0)], total_sweeps, sps, seed, rule, "slot")
    rounds = int(total_sweeps) // max(int(sps), 1)
    o = dict(round=np.zeros(rounds, np.int64), sweep_count=np.zeros(rounds, np.int64),
             best_f=np.zeros(rounds), any_feasible=np.zeros(rounds, np.uint8),
             n_feasible=np.zeros(rounds, np.int32), n_total=np.zeros(rounds, np.int32),
             feasible_fraction=np.zeros(1))
    out = _BaselineOut(*[_ptr(o[k]) for k, _ in _BaselineOut._fields_])
    err = C.create_string_buffer(512)
    if impl == "port":
        rc = port_lib().tgo_run_jcolumn(C.byref(p), C.byref(c), C.c_double(p_fixed), int(j_repeats),
                                        C.byref(out), err, 512)
    else:
        rc = ref_lib(impl.split(":", 1)[1]).tgr_run_jcolumn(
            C.byref(p), C.byref(c), C.c_double(p_fixed), int(j_repeats), int(threads), C.byref(out),
            err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return BaselineResult(o["round"], o["sweep_count"], o["best_f"], o["any_feasible"].astype(bool),
                          o["n_feasible"], o["n_total"], float(o["feasible_fraction"][0]))


class _ProbeStats(C.Structure):
    _fields_ = [("row", C.c_int), ("column", C.c_int), ("beta", C.c_double),
                ("penalty", C.c_double), ("sigma_e", C.c_double), ("sigma_g", C.c_double),
                ("mean_g", C.c_double)]


class _ScheduleCfg(C.Structure):
    _fields_ = [("beta0", C.c_double), ("p0", C.c_double), ("i_max", C.c_int), ("j_max", C.c_int),
                ("sigma_min", C.c_double), ("alpha_beta", C.c_double), ("alpha_p", C.c_double),
                ("n_chains", C.c_int), ("sweeps_per_probe", C.c_int), ("replica_budget", C.c_int),
                ("seed", C.c_uint64)]


SCHEDULE_DEFAULTS = dict(beta0=0.3, p0=0.5, i_max=20, j_max=20, sigma_min=0.0, alpha_beta=1.0,
                         alpha_p=1.2, n_chains=32, sweeps_per_probe=1000, replica_budget=400,
                         seed=1)  # schedule.hpp:10-22


def _stats_dict(s):
    return {k: getattr(s, k) for k, _ in _ProbeStats._fields_}


def probe_population(pr, beta, penalty, n_chains, sweeps, seed, rule="metropolis", impl="port"):
    """probe_population (schedule.cpp:18-52) on the C port or a reference build
    ('ref:philox' / 'ref:philox_hb'); returns the ProbeStats fields as a dict."""
    p, _, keep = _marshal(pr, [1.0], [0.0], 1, 1, 1, rule, "slot")
    out = _ProbeStats()
    err = C.create_string_buffer(512)
    if impl == "port":
        rc = port_lib().tgo_probe_population(C.byref(p), C.c_double(beta), C.c_double(penalty),
                                             int(n_chains), int(sweeps), C.c_uint64(seed),
                                             RULE[rule], C.byref(out), err, 512)
    else:
        rc = ref_lib(impl.split(":", 1)[1]).tgr_probe_population(
            C.byref(p), C.c_double(beta), C.c_double(penalty), int(n_chains), int(sweeps),
            C.c_uint64(seed), C.byref(out), err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return _stats_dict(out)


def build_schedule(pr, rule="metropolis", impl="port", **cfg):
    """build_schedule (schedule.cpp:77-163); returns (betas, penalties, probe_stats,
    budget_exhausted)."""
    c = dict(SCHEDULE_DEFAULTS)
    c.update(cfg)
    sc = _ScheduleCfg(**c)
    p, _, keep = _marshal(pr, [1.0], [0.0], 1, 1, 1, rule, "slot")
    im, jm = max(int(c["i_max"]), 1), max(int(c["j_max"]), 1)
    betas, pens = np.zeros(im), np.zeros(jm + 1)
    cap = im * (jm + 1) + 1
    stats = (_ProbeStats * cap)()
    nb, npn, ns, be = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    err = C.create_string_buffer(512)
    args = (C.byref(p), C.byref(sc))
    tail = (_ptr(betas), C.byref(nb), _ptr(pens), C.byref(npn), stats, cap, C.byref(ns), C.byref(be),
            err, 512)
    if impl == "port":
        rc = port_lib().tgo_build_schedule(*args, RULE[rule], *tail)
    else:
        rc = ref_lib(impl.split(":", 1)[1]).tgr_build_schedule(*args, *tail)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return (betas[:nb.value].copy(), pens[:npn.value].copy(),
            [_stats_dict(stats[k]) for k in range(min(ns.value, cap))], bool(be.value))


class _Decoder(C.Structure):
    _fields_ = [("logical", C.c_void_p), ("copy_off", C.c_void_p), ("copies", C.c_void_p)]


def _decoder(logical_pr, copies):
    lp, _, keep = _marshal(logical_pr, [1.0], [0.0], 1, 1, 1, "metropolis", "slot")
    off = np.zeros(len(copies) + 1, np.int32)
    off[1:] = np.cumsum([len(c) for c in copies])
    flat = np.ascontiguousarray(np.concatenate([np.asarray(c, np.int32) for c in copies]), np.int32)
    keep.update(lp=lp, off=off, flat=flat)
    return _Decoder(C.cast(C.pointer(lp), C.c_void_p), _ptr(off), _ptr(flat)), keep


def enumerate_boltzmann(logical_pr, beta):
    p, _, keep = _marshal(logical_pr, [1.0], [0.0], 1, 1, 1, "metropolis", "slot")
    probs = np.zeros(1 << logical_pr.n)
    err = C.create_string_buffer(512)
    rc = port_lib().tgo_enumerate_boltzmann(C.byref(p), C.c_double(beta), _ptr(probs), None, err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return probs


def kl_curve(pr, betas, penalties, total_sweeps, sps, seed, logical_pr, copies, beta,
             discard_infeasible=False, rule="metropolis", impl="port", threads=1):
    """run_2dpt + kl_curve (analysis.cpp:215-241) on the port or a reference build;
    returns (t, samples, kl) per round."""
    p, c, keep = _marshal(pr, betas, penalties, total_sweeps, sps, seed, rule, "slot")
    dec, keep2 = _decoder(logical_pr, copies)
    rounds = int(total_sweeps) // max(int(sps), 1)
    t, smp, kl = np.zeros(rounds, np.int64), np.zeros(rounds, np.int64), np.zeros(rounds)
    err = C.create_string_buffer(512)
    if impl == "port":
        rc = port_lib().tgo_kl_curve(C.byref(p), C.byref(c), C.byref(dec), C.c_double(beta),
                                     int(discard_infeasible), _ptr(t), _ptr(smp), _ptr(kl), err, 512)
    else:
        rc = ref_lib(impl.split(":", 1)[1]).tgr_kl_curve(
            C.byref(p), C.byref(c), C.byref(dec), C.c_double(beta), int(discard_infeasible),
            int(threads), _ptr(t), _ptr(smp), _ptr(kl), err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return t, smp, kl


def ref_timed(variant, pr, betas, penalties, total_sweeps, sps=1, seed=1, threads=1) -> float:
    """Run the reference build once; returns the last target f (for timing legs)."""
    p, c, keep = _marshal(pr, betas, penalties, total_sweeps, sps, seed, "metropolis", "slot")
    err = C.create_string_buffer(512)
    f = C.c_double(0.0)
    rc = ref_lib(variant).tgr_run_2dpt_timed(C.byref(p), C.byref(c), int(threads), C.byref(f), err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return f.value


def energy(pr, penalty: float, state: np.ndarray):
    p, _, keep = _marshal(pr, [1.0], [penalty], 1, 1, 1, "metropolis", "slot")
    s = np.ascontiguousarray(state, dtype=np.int8)
    f, g = C.c_double(), C.c_double()
    rc = port_lib().tgo_energy_breakdown(C.byref(p), C.c_double(penalty), _ptr(s), C.byref(f), C.byref(g))
    if rc:
        raise OracleError(rc, "energy")
    return f.value, g.value


def digest(state: np.ndarray) -> int:
    s = np.ascontiguousarray(state, dtype=np.int8)
    return int(port_lib().tgo_digest(_ptr(s), int(s.size)))


def canonical_order(pr):
    p, _, keep = _marshal(pr, [1.0], [0.0], 1, 1, 1, "metropolis", "slot")
    color = np.zeros(pr.n, np.int32)
    order = np.zeros(pr.n, np.int32)
    nc = C.c_int32()
    port_lib().tgo_canonical_order(C.byref(p), _ptr(color), _ptr(order), C.byref(nc))
    return order, color, nc.value


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, np.uint32)
    port_lib().tgo_philox(_ptr(c), _ptr(k), _ptr(o))
    return o


def derive_seed(master, purpose, index) -> int:
    return int(port_lib().tgo_derive(master, purpose, index))


def stream_bits(seed, n) -> int:
    return int(port_lib().tgo_bits(seed, n))


def plane_u53(pkey, grp, t, site, lane) -> int:
    return int(port_lib().tgo_plane(pkey, grp, t, site, lane))


def p_swap_probability(beta, dp, dg):
    return port_lib().tgo_p_swap_probability(beta, dp, dg)


def beta_swap_probability(db, de):
    return port_lib().tgo_beta_swap_probability(db, de)


def general_swap_probability(ba, bb, dea, deb):
    return port_lib().tgo_general_swap_probability(ba, bb, dea, deb)


def ref_sparsify(n, couplings, fields, copies, max_degree, variant="mt"):
    """The reference's own sparsify (constraints.cpp:50-120) via oracle/_ref."""
    lib = ref_lib(variant)
    c = np.asarray(couplings, dtype=np.float64).reshape(-1, 3)
    ci = np.ascontiguousarray(c[:, 0], dtype=np.int32)
    cj = np.ascontiguousarray(c[:, 1], dtype=np.int32)
    cw = np.ascontiguousarray(c[:, 2])
    h = np.ascontiguousarray(fields, dtype=np.float64)
    cap_n = n * copies
    cap_e = len(ci) + 1
    oci, ocj = np.zeros(cap_e, np.int32), np.zeros(cap_e, np.int32)
    ow = np.zeros(cap_e)
    oh = np.zeros(cap_n)
    opa, opb = np.zeros(cap_n, np.int32), np.zeros(cap_n, np.int32)
    nc, npp = C.c_int(), C.c_int()
    err = C.create_string_buffer(512)
    lib.tgr_sparsify.restype = C.c_int
    rc = lib.tgr_sparsify(n, len(ci), _ptr(ci), _ptr(cj), _ptr(cw), _ptr(h), copies, max_degree,
                          _ptr(oci), _ptr(ocj), _ptr(ow), C.byref(nc), _ptr(oh), _ptr(opa),
                          _ptr(opb), C.byref(npp), err, 512)
    if rc < 0:
        raise OracleError(-rc, err.value.decode())
    return (rc, oci[:nc.value].copy(), ocj[:nc.value].copy(), ow[:nc.value].copy(), oh[:rc].copy(),
            opa[:npp.value].copy(), opb[:npp.value].copy())
