"""ctypes binding of the C ABI (include/tempergrid_b200.h).

The engine library must be built in-tree (``python -m paper_2506_14781_b200.build``);
importing this module without it raises immediately -- there is no CPU
fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TG_ENGINE_LIB") or os.path.join(PKG, "libtempergrid_b200.so")  # override: A/B builds

TG_OK, TG_ERR_INTERNAL, TG_ERR_CONFIG, TG_ERR_RESOURCE, TG_ERR_CUDA, TG_ERR_SINK = range(6)
RULES = {"metropolis": 0, "heat_bath": 1}
ENGINES = {"auto": 0, "slot": 1, "plane": 2, "float": 3}
REC_DIGEST, REC_STATE, REC_GRID, REC_COUNTERS = 1, 2, 4, 8


class RunConfigC(C.Structure):
    _fields_ = [("total_sweeps", C.c_int64), ("sweeps_per_swap", C.c_int64), ("seed", C.c_uint64),
                ("rule", C.c_int32), ("engine", C.c_int32), ("record_flags", C.c_int32),
                ("record_every", C.c_int32)]


class BaselineRecordC(C.Structure):
    _fields_ = [("round", C.c_int64), ("sweep_count", C.c_int64), ("best_f", C.c_double),
                ("any_feasible", C.c_int32), ("n_feasible", C.c_int32), ("n_total", C.c_int32),
                ("reserved", C.c_int32)]


class ProbeStatsC(C.Structure):
    _fields_ = [("row", C.c_int32), ("column", C.c_int32), ("beta", C.c_double),
                ("penalty", C.c_double), ("sigma_e", C.c_double), ("sigma_g", C.c_double),
                ("mean_g", C.c_double)]


class ScheduleConfigC(C.Structure):
    _fields_ = [("beta0", C.c_double), ("p0", C.c_double), ("i_max", C.c_int32),
                ("j_max", C.c_int32), ("sigma_min", C.c_double), ("alpha_beta", C.c_double),
                ("alpha_p", C.c_double), ("n_chains", C.c_int32), ("sweeps_per_probe", C.c_int32),
                ("replica_budget", C.c_int32), ("rule", C.c_int32), ("seed", C.c_uint64)]


class RecordC(C.Structure):
    _fields_ = [("round", C.c_int64), ("sweep_count", C.c_int64), ("f", C.c_double),
                ("g", C.c_double), ("feasible", C.c_int32), ("target_state", C.c_int32),
                ("digest", C.c_uint64)]


class InfoC(C.Structure):
    _fields_ = [("engine", C.c_int32), ("n_colors", C.c_int32), ("n_replicas", C.c_int32),
                ("local_replicas", C.c_int32), ("words", C.c_int32), ("device_sms", C.c_int32),
                ("rounds_done", C.c_int64), ("last_sweep_ms", C.c_double),
                ("last_swap_ms", C.c_double), ("sweep_launches", C.c_int64),
                ("other_launches", C.c_int64), ("sweep_kernel", C.c_char * 48)]


BATCH_SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(RecordC), C.c_int64,
                         C.POINTER(C.c_int8), C.POINTER(C.c_int64), C.POINTER(C.c_int64))
SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(RecordC), C.c_int64, C.POINTER(C.c_int8),
                   C.POINTER(C.c_int64), C.POINTER(C.c_int64))

_lib = None


def lib() -> C.CDLL:
    """Load the engine library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"tempergrid B200 engine not built ({LIB_PATH} missing); run "
            "`python -m paper_2506_14781_b200.build` -- there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, i32p, f64p = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_double)
    L.tg_abi_version.restype = C.c_int
    L.tg_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.tg_create_distributed.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(vp)]
    L.tg_nccl_unique_id.argtypes = [C.c_void_p]
    L.tg_destroy.argtypes = [vp]
    L.tg_destroy.restype = None
    L.tg_last_error.argtypes = [vp, C.c_char_p, C.c_size_t]
    L.tg_last_error.restype = C.c_size_t
    L.tg_checkpoint_size.argtypes = [vp, C.POINTER(C.c_size_t)]
    L.tg_checkpoint.argtypes = [vp, C.c_void_p, C.c_size_t]
    L.tg_restore.argtypes = [vp, C.c_void_p, C.c_size_t]
    L.tg_set_problem.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, vp, vp]
    L.tg_set_schedule.argtypes = [vp, C.c_int, vp, C.c_int, vp]
    L.tg_run.argtypes = [vp, C.POINTER(RunConfigC), SINK, C.c_void_p]
    L.tg_init.argtypes = [vp, C.POINTER(RunConfigC)]
    L.tg_advance.argtypes = [vp, C.c_int64, SINK, C.c_void_p]
    L.tg_get_state.argtypes = [vp, C.c_int, vp]
    L.tg_get_counters.argtypes = [vp, vp, vp, vp, vp]
    L.tg_get_energies.argtypes = [vp, vp, vp]
    L.tg_get_info.argtypes = [vp, C.POINTER(InfoC)]
    L.tg_stream.argtypes = [vp]
    L.tg_stream.restype = C.c_void_p
    L.tg_set_profiling.argtypes = [vp, C.c_int]
    L.tg_canonical_order.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, vp, vp, vp, vp, vp]
    for fn, n in (("tg_p_swap_probability", 3), ("tg_beta_swap_probability", 2),
                  ("tg_general_swap_probability", 4)):
        getattr(L, fn).restype = C.c_double
        getattr(L, fn).argtypes = [C.c_double] * n
    L.tg_batch_clear.argtypes = [vp]
    L.tg_batch_add.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, vp, vp, C.c_int, vp,
                               C.c_int, vp, C.c_uint64, vp]
    L.tg_batch_run.argtypes = [vp, C.POINTER(RunConfigC), BATCH_SINK, C.c_void_p]
    L.tg_batch_get_state.argtypes = [vp, C.c_int, C.c_int, vp]
    L.tg_batch_get_counters.argtypes = [vp, C.c_int, vp, vp, vp, vp]
    L.tg_batch_init.argtypes = [vp, vp]
    L.tg_batch_advance.argtypes = [vp, C.c_int64, BATCH_SINK, vp]
    L.tg_run_jcolumn.argtypes = [vp, C.c_int, vp, C.c_double, C.c_int, vp, vp, C.c_int64, vp]
    L.tg_set_kl_decoder.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_double, vp, vp, C.c_int]
    L.tg_clear_kl_decoder.argtypes = [vp]
    L.tg_get_kl_curve.argtypes = [vp, C.c_int, C.c_int64, C.c_int64, vp, vp]
    L.tg_probe_population.argtypes = [vp, C.c_double, C.c_double, C.c_int, C.c_int, C.c_uint64,
                                      C.c_int, vp]
    L.tg_build_schedule.argtypes = [vp, vp, vp, C.c_int, vp, vp, C.c_int, vp, vp, C.c_int, vp, vp]
    L.tg_partition.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]
    L.tg_swap_phase_host.argtypes = [C.c_int, vp, C.c_int, vp, C.c_int64, C.c_int, C.c_uint64,
                                     C.c_uint64, vp, vp, vp, vp, vp]
    _lib = L
    return L


EXPORTED = [
    "tg_abi_version", "tg_create", "tg_create_distributed", "tg_nccl_unique_id", "tg_destroy",
    "tg_last_error", "tg_set_problem", "tg_set_schedule", "tg_run", "tg_init", "tg_advance",
    "tg_get_state", "tg_get_counters", "tg_get_energies", "tg_get_info", "tg_stream",
    "tg_set_profiling", "tg_canonical_order", "tg_p_swap_probability", "tg_beta_swap_probability",
    "tg_general_swap_probability", "tg_swap_phase_host", "tg_partition", "tg_batch_clear",
    "tg_batch_add", "tg_batch_run", "tg_batch_get_state", "tg_batch_get_counters",
    "tg_batch_init", "tg_batch_advance", "tg_run_jcolumn", "tg_probe_population", "tg_build_schedule", "tg_set_kl_decoder",
    "tg_clear_kl_decoder", "tg_get_kl_curve", "tg_checkpoint_size", "tg_checkpoint", "tg_restore",
]
