"""B200-native 2D parallel tempering hot path (arXiv 2506.14781, reference ``tempergrid``).

The sweep / swap / RNG / observable machinery under ``tempergrid::run_2dpt``
runs as hand-written sm_100a CUDA kernels behind a C ABI
(``include/tempergrid_b200.h``); this package holds the kernels (``csrc/``),
the build recipe, the ctypes binding, the reference-mirroring Python API and
the host-side instance generators.
"""
from .instances import (ConfigError, Problem, ResourceError, bipartite_3regular, canonical_order,
                        config_schedule, five_node_complete, k10_pm1, sparsify, to_canonical,
                        wishart_planted, wishart_schedule)
from .api import (Engine, EngineError, RunConfig, Schedule, Trace, TraceRecord,
                  beta_swap_probability, general_swap_probability, p_swap_probability, run_2dpt,
                  run_2dpt_batch)

__all__ = [
    "ConfigError", "ResourceError", "EngineError", "Problem", "Engine", "RunConfig", "Schedule",
    "Trace", "TraceRecord", "run_2dpt", "run_2dpt_batch", "p_swap_probability", "beta_swap_probability",
    "general_swap_probability", "sparsify", "canonical_order", "to_canonical",
    "five_node_complete", "k10_pm1", "wishart_planted", "bipartite_3regular", "config_schedule",
    "wishart_schedule",
]
