"""GPU parity of the word-local fused round kernel (plane_cl.cu): the CTAs are
partitioned by 32-replica word (or word pair), a colour phase ends with a
barrier among the word's CTAs only, one tagged-word (f, g) exchange per round,
neighbour entries staged by TMA bulk copies, threshold planes per CTA in
shared memory.  Three variants share the code: hardware thread-block clusters
(cluster barrier, word counts reduced through distributed shared memory), and
the "group" launch (software word barrier on all SMs) with one word or a word
pair per thread.  It is the default single-GPU path of both rules for config-5
instances (cost degree 3, chain degree 0/1, 2 colours) up to 2^18 sites; every
case is compared bit for bit with the oracle (f, g, feasibility, digests,
final grid, counters) and checks which kernel ran."""
import numpy as np
import pytest

from paper_2506_14781_b200 import instances as I
from test_gpu_parity import compare
from test_gpu_tpw import kernel_of, sched

pytestmark = pytest.mark.gpu

C5S = I.bipartite_3regular(512, seed=3)
RULES = ["metropolis", "heat_bath"]
KERNEL = "plane_cl_rounds_kernel"


@pytest.fixture(autouse=True, params=["cluster", "group", "pair"])
def _mode(request, monkeypatch):
    # cluster: hardware clusters (cluster barrier, DSMEM totals); group: the same
    # kernel as an ordinary cooperative launch, G CTAs per word behind a
    # software word barrier, totals by global atomics (the default up to 2^15
    # sites); pair: group mode with two words per thread (2^15 .. 2^18)
    monkeypatch.setenv("TG_PLANE_CL_MODE", "cluster" if request.param == "cluster" else "group")
    monkeypatch.setenv("TG_PLANE_CL_PAIR", "1" if request.param == "pair" else "0")


# (I, J) -> words per site = clusters: 32 -> 1, 64 -> 2, 96 -> 4 (one padded
# word), 128 -> 4, 256 -> 8, 512 -> 16, 1024 -> 32
@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("grid", [(4, 8), (8, 8), (8, 12), (16, 8), (16, 16), (16, 32), (32, 32)])
def test_cl_word_counts(grid, rule):
    b, p = sched(*grid)
    compare(C5S, b, p, 12, 1, seed=7, rule=rule, engine="plane")
    assert kernel_of(C5S, b, p, rule) == KERNEL


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("n,chain_frac", [(1002, 0.1), (30, 0.1), (4096, 0.0), (4096, 0.5),
                                          (1 << 14, 0.1)])
def test_cl_shapes(n, chain_frac, rule):
    # slices that are not multiples of 32 sites, CTAs without any site (n = 30),
    # no chain sites at all, many chain sites
    pr = I.bipartite_3regular(n, seed=21, chain_frac=chain_frac)
    b, p = sched(16, 16)
    compare(pr, b, p, 10, 1, seed=8, rule=rule, engine="plane")
    assert kernel_of(pr, b, p, rule) == KERNEL


@pytest.mark.parametrize("rule", RULES)
def test_cl_several_sweeps_per_round(rule):
    pr = I.bipartite_3regular(1 << 14, seed=12)
    b, p = sched(16, 16)
    compare(pr, b, p, 3 * 8, 3, seed=5, rule=rule, engine="plane")


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("csize", [16, 8, 2, 1])
def test_cl_cluster_sizes(monkeypatch, csize, rule):
    # smaller clusters: more sites per CTA, several items per thread
    monkeypatch.setenv("TG_PLANE_CL_SIZE", str(csize))
    pr = I.bipartite_3regular(1 << 13, seed=4)
    b, p = sched(16, 16)
    compare(pr, b, p, 8, 1, seed=2, rule=rule, engine="plane")
    assert kernel_of(pr, b, p, rule) == KERNEL


@pytest.mark.parametrize("rule", RULES)
def test_cl_entries_from_global_memory(monkeypatch, rule):
    # the un-staged path (slices that exceed shared memory)
    monkeypatch.setenv("TG_PLANE_CL_NOSTAGE", "1")
    pr = I.bipartite_3regular(1 << 14, seed=9)
    compare(pr, *sched(16, 16), 8, 1, seed=6, rule=rule, engine="plane")


@pytest.mark.parametrize("rule", RULES)
def test_cl_large_instance_many_drains(rule):
    # 2^16 sites: several deferred-tail drains per warp and phase; cold (beta
    # up to 8) labels leave few undecided lanes
    pr = I.bipartite_3regular(1 << 16, seed=5)
    compare(pr, *sched(16, 16), 6, 1, seed=3, rule=rule, engine="plane")
    compare(pr, *sched(16, 16, 0.5, 8.0), 6, 1, seed=4, rule=rule, engine="plane")
    assert kernel_of(pr, *sched(16, 16), rule) == KERNEL


@pytest.mark.parametrize("rule", RULES)
def test_cl_counter_flush_bound(monkeypatch, rule):
    # one CTA per word at 2^16 sites: 64 items per thread and phase, > 85 with
    # the chain sites' second counter -- the mid-phase flush of the 8-bit
    # vertical counters
    monkeypatch.setenv("TG_PLANE_CL_SIZE", "1")
    monkeypatch.setenv("TG_PLANE_CL", "1")
    pr = I.bipartite_3regular(1 << 17, seed=15)
    compare(pr, *sched(16, 8), 4, 1, seed=3, rule=rule, engine="plane")


def test_cl_resume_and_relaunch():
    # several launches of the kernel in one run (record chunks) and init+advance
    from paper_2506_14781_b200 import _lib
    from paper_2506_14781_b200.api import Engine, RunConfig
    import pyoracle as O
    pr = I.bipartite_3regular(2048, seed=2)
    b, p = sched(16, 16)
    o = O.run(pr, b, p, 30, 1, seed=4, rule="metropolis", rng="plane")
    eng = Engine(0)
    eng.set_problem(pr)
    eng.set_schedule(b, p)
    got = []

    def sink(r, n, st, ap, ab):
        for k in range(n):
            got.append((r[k].f, r[k].g, r[k].digest))
        return 0

    eng.init(RunConfig(total_sweeps=30, sweeps_per_swap=1, seed=4, engine="plane", store_states=False),
             flags=_lib.REC_DIGEST)
    for n in (7, 1, 12, 10):
        eng.advance(n, sink)
    assert eng.info()["sweep_kernel"] == KERNEL
    grid = eng.grid()
    eng.close()
    np.testing.assert_array_equal(np.array([x[0] for x in got]), o.f)
    np.testing.assert_array_equal(np.array([x[2] for x in got], dtype=np.uint64), o.digest)
    np.testing.assert_array_equal(grid, o.final_grid)


def test_cl_negative_betas_fall_back():
    b, p = sched(16, 16, -1.0, 2.0)
    compare(C5S, b, p, 12, 1, seed=7, rule="metropolis", engine="plane")
    assert kernel_of(C5S, b, p, "metropolis") != KERNEL
