"""GPU parity of the PLANE engine's fused kernels across their dispatch space.

The single-GPU fused round loop has three device paths with one contract
(plane_tpw.cu, plane_sweep.cu): the thread-per-(site, word) kernel's config-5
path (cost degree 3, chain degree 0/1; the default where it applies), its generic path (any site type, both rules; TG_PLANE_TPW=2) and
the thread-per-site kernel (everything else by default, TG_PLANE_TPW=0).
The config-5 path serves both rules (heat bath: four classes per chain-free
site, staged per colour phase in shared memory).  Every case is compared bit
for bit with the oracle (f, g, feasibility, digests, final grid, counters)
and the test checks which kernel the engine reports it launched.
"""
import numpy as np
import pytest

from paper_2506_14781_b200 import instances as I
from test_gpu_parity import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _no_c5_kernel(monkeypatch):
    # these cases pin the tpw / thread-per-site kernels: keep the config-5
    # kernel (plane_c5.cu, tests/test_gpu_c5.py) out of the dispatch
    monkeypatch.setenv("TG_PLANE_C5", "0")
    monkeypatch.setenv("TG_PLANE_CL", "0")

C5S = I.bipartite_3regular(512, seed=3)      # cost degree 3, chain degree 0/1, 2 colours
K10 = I.k10_pm1(1)                           # non-bipartite, larger degrees: generic path


def sched(n_b, n_p, b0=0.2, b1=5.0):
    betas = np.geomspace(b0, b1, n_b) if b0 > 0 else np.linspace(b0, b1, n_b)
    pens = np.round(np.linspace(0.0, 1.0, n_p) * 64) / 64  # dyadic: exact thresholds
    return list(betas), list(pens)


def run_and_kernel(pr, b, p, rounds, rule, seed=7):
    o = compare(pr, b, p, rounds, 1, seed=seed, rule=rule, engine="plane")
    return o


def kernel_of(pr, b, p, rule):
    from paper_2506_14781_b200.api import Engine, RunConfig
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(b, p)
    eng.run(RunConfig(total_sweeps=2, sweeps_per_swap=1, seed=1, rule=rule, engine="plane",
                      store_states=False), None)
    k = eng.info()["sweep_kernel"]
    eng.close()
    return k


# (I, J) -> words per site: 32 -> 1, 64 -> 2, 96 -> 4 (one padded word), 128 -> 4,
# 256 -> 8, 512 -> 16, 1024 -> 32
@pytest.mark.parametrize("grid", [(4, 8), (8, 8), (8, 12), (16, 8), (16, 16), (16, 32), (32, 32)])
def test_tpw_config5_path_word_counts(grid):
    b, p = sched(*grid)
    run_and_kernel(C5S, b, p, 12, "metropolis")
    assert kernel_of(C5S, b, p, "metropolis") == "plane_tpw_rounds_kernel"


@pytest.mark.parametrize("grid", [(4, 8), (16, 16), (32, 32)])
def test_tpw_generic_path_heat_bath(monkeypatch, grid):
    monkeypatch.setenv("TG_PLANE_TPW", "2")
    b, p = sched(*grid)
    run_and_kernel(C5S, b, p, 12, "heat_bath")
    assert kernel_of(C5S, b, p, "heat_bath") == "plane_tpw_rounds_kernel"


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_tpw_generic_path_non_bipartite(monkeypatch, rule):
    monkeypatch.setenv("TG_PLANE_TPW", "2")
    b, p = sched(8, 8, 0.1, 3.0)
    run_and_kernel(K10, b, p, 40, rule)


@pytest.mark.parametrize("mode", ["1", "2"])
def test_tpw_negative_betas_disable_the_class_shortcut(monkeypatch, mode):
    # beta < 0 makes classes 2 and 3 "always" for some labels: the config-5
    # path's single-select compare must not be taken (flag bit 0 off)
    monkeypatch.setenv("TG_PLANE_TPW", mode)
    b, p = sched(16, 16, -1.0, 2.0)
    run_and_kernel(C5S, b, p, 12, "metropolis")


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_default_dispatch(rule):
    # config-5 site types: the tpw kernel for both rules; other types: thread per site
    b, p = sched(8, 8, 0.1, 3.0)
    assert kernel_of(K10, b, p, rule) == "plane_rounds_kernel"
    b, p = sched(16, 16)
    assert kernel_of(C5S, b, p, rule) == "plane_tpw_rounds_kernel"


@pytest.mark.parametrize("grid", [(4, 8), (16, 16), (32, 32)])
def test_tpw_config5_path_heat_bath(grid):
    b, p = sched(*grid)
    run_and_kernel(C5S, b, p, 12, "heat_bath")
    run_and_kernel(C5S, *sched(grid[0], grid[1], 0.05, 2.0), 12, "heat_bath", seed=9)


def test_non_power_of_two_rows_use_the_thread_per_site_kernel():
    b, p = sched(16, 24)   # 384 replicas -> 12 words per site
    run_and_kernel(C5S, b, p, 12, "metropolis")
    assert kernel_of(C5S, b, p, "metropolis") == "plane_rounds_kernel"


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_thread_per_site_kernel_on_request(monkeypatch, rule):
    monkeypatch.setenv("TG_PLANE_TPW", "0")
    b, p = sched(16, 16)
    run_and_kernel(C5S, b, p, 12, rule)
    assert kernel_of(C5S, b, p, rule) == "plane_rounds_kernel"


def test_large_instance_many_items_per_warp():
    # 2^16 sites: several deferred-tail drains and counter flushes per warp and phase
    pr = I.bipartite_3regular(1 << 16, seed=5)
    b, p = sched(16, 16)
    run_and_kernel(pr, b, p, 6, "metropolis", seed=3)


@pytest.mark.parametrize("every", [1, 2])
def test_vertical_counter_flush_mid_phase(monkeypatch, every):
    # flushing after every item / every second item must give the same energies
    monkeypatch.setenv("TG_TPW_FLUSH_EVERY", str(every))
    monkeypatch.setenv("TG_PLANE_TPW", "2")
    pr = I.bipartite_3regular(1 << 14, seed=9)
    b, p = sched(16, 16)
    run_and_kernel(pr, b, p, 6, "metropolis", seed=2)
    run_and_kernel(K10, *sched(8, 8, 0.1, 3.0), 20, "heat_bath")


def run_grid_records(pr, b, p, rounds, rule, seed):
    """Full-grid records force the unfused round loop (sweep kernel, swap
    kernel, extract): the multi-GPU path's kernels on one GPU."""
    import pyoracle as O
    from paper_2506_14781_b200.api import Engine, RunConfig
    o = O.run(pr, b, p, rounds, 1, seed=seed, rule=rule, rng="plane")
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(b, p)
    recs = []

    def sink(r, n, states, ap, ab):
        for k in range(n):
            recs.append((r[k].f, r[k].g, r[k].digest))
        return 0

    eng.run(RunConfig(total_sweeps=rounds, sweeps_per_swap=1, seed=seed, rule=rule, engine="plane",
                      store_states=False, store_target_only=False), sink)
    grid = eng.grid()
    kern = eng.info()["sweep_kernel"]
    eng.close()
    np.testing.assert_array_equal(np.array([x[0] for x in recs]), o.f)
    np.testing.assert_array_equal(np.array([x[1] for x in recs]), o.g)
    np.testing.assert_array_equal(np.array([x[2] for x in recs], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(grid, o.final_grid)
    return kern


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_unfused_round_loop_uses_the_tpw_sweep_kernel(rule):
    b, p = sched(16, 16)
    assert run_grid_records(C5S, b, p, 10, rule, 4) == "plane_tpw_sweep_kernel"


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_unfused_round_loop_tpw_generic(monkeypatch, rule):
    monkeypatch.setenv("TG_PLANE_TPW", "2")
    b, p = sched(16, 16)
    assert run_grid_records(C5S, b, p, 10, rule, 4) == "plane_tpw_sweep_kernel"
    b, p = sched(8, 8, 0.1, 3.0)
    assert run_grid_records(K10, b, p, 20, rule, 6) == "plane_tpw_sweep_kernel"


def test_unfused_round_loop_thread_per_site_kernel(monkeypatch):
    monkeypatch.setenv("TG_PLANE_TPW", "0")
    b, p = sched(16, 16)
    assert run_grid_records(C5S, b, p, 10, "metropolis", 4) == "plane_sweep_kernel"


@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_config5_path_several_sweeps_per_round(rule):
    # the dynamic-tail counters are per (parity, colour, sweep of the round)
    pr = I.bipartite_3regular(1 << 14, seed=12)
    b, p = sched(16, 16)
    compare(pr, b, p, 3 * 8, 3, seed=5, rule=rule, engine="plane")
    assert kernel_of(pr, b, p, rule) == "plane_tpw_rounds_kernel"


@pytest.mark.parametrize("n,chain_frac", [(1002, 0.1), (30, 0.1), (4096, 0.0), (4096, 0.5)])
@pytest.mark.parametrize("rule", ["metropolis", "heat_bath"])
def test_config5_path_shapes(n, chain_frac, rule):
    # partial last items (colour sizes not a multiple of the item's sites),
    # no chain sites at all, and many chain sites
    pr = I.bipartite_3regular(n, seed=21, chain_frac=chain_frac)
    b, p = sched(16, 16)
    compare(pr, b, p, 10, 1, seed=8, rule=rule, engine="plane")
    assert kernel_of(pr, b, p, rule) == "plane_tpw_rounds_kernel"
