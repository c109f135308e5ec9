"""GPU parity of the config-5 fused round kernel (plane_c5.cu): two words per
thread, chain-free and chain sites in separate loops, per-warp deferred tail.
It is the default single-GPU path of both rules for config-5 instances (cost
degree 3, chain degree 0/1, 2 colours) with at least two words per site row;
every case is compared bit for bit with the oracle (f, g, feasibility,
digests, final grid, counters) and checks which kernel ran."""
import numpy as np
import pytest

from paper_2506_14781_b200 import instances as I
from test_gpu_parity import compare
from test_gpu_tpw import kernel_of, sched

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _no_cluster_kernel(monkeypatch):
    # these cases pin plane_c5_rounds_kernel: keep the cluster-per-word kernel
    # (plane_cl.cu, tests/test_gpu_cl.py; the default up to 2^16 sites) out
    monkeypatch.setenv("TG_PLANE_CL", "0")

C5S = I.bipartite_3regular(512, seed=3)


# (I, J) -> words per site: 64 -> 2, 96 -> 4 (one padded word), 128 -> 4, 256 -> 8,
# 512 -> 16, 1024 -> 32
RULES = ["metropolis", "heat_bath"]


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("grid", [(8, 8), (8, 12), (16, 8), (16, 16), (16, 32), (32, 32)])
def test_c5_word_counts(grid, rule):
    b, p = sched(*grid)
    compare(C5S, b, p, 12, 1, seed=7, rule=rule, engine="plane")
    assert kernel_of(C5S, b, p, rule) == "plane_c5_rounds_kernel"


def test_c5_dispatch():
    b1, p1 = sched(4, 8)  # one word per row: the tpw kernel
    assert kernel_of(C5S, b1, p1, "metropolis") == "plane_tpw_rounds_kernel"
    assert kernel_of(C5S, b1, p1, "heat_bath") == "plane_tpw_rounds_kernel"


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("n,chain_frac", [(1002, 0.1), (30, 0.1), (4096, 0.0), (4096, 0.5),
                                          (1 << 14, 0.1)])
def test_c5_shapes(n, chain_frac, rule):
    # partial items (colour and chain-free counts not multiples of the item's
    # sites), no chain sites at all, many chain sites
    pr = I.bipartite_3regular(n, seed=21, chain_frac=chain_frac)
    b, p = sched(16, 16)
    compare(pr, b, p, 10, 1, seed=8, rule=rule, engine="plane")
    assert kernel_of(pr, b, p, rule) == "plane_c5_rounds_kernel"


@pytest.mark.parametrize("rule", RULES)
def test_c5_several_sweeps_per_round(rule):
    pr = I.bipartite_3regular(1 << 14, seed=12)
    b, p = sched(16, 16)
    compare(pr, b, p, 3 * 8, 3, seed=5, rule=rule, engine="plane")


@pytest.mark.parametrize("rule", RULES)
def test_c5_large_instance_many_drains(rule):
    # 2^16 sites: many deferred-tail drains per warp and phase, counters near
    # their flush bound; cold (beta up to 8) labels leave few undecided lanes
    pr = I.bipartite_3regular(1 << 16, seed=5)
    compare(pr, *sched(16, 16), 6, 1, seed=3, rule=rule, engine="plane")
    compare(pr, *sched(16, 16, 0.5, 8.0), 6, 1, seed=4, rule=rule, engine="plane")


def test_c5_negative_betas_fall_back():
    # beta < 0 makes classes 2, 3 "always" for some labels: not the c5 path
    b, p = sched(16, 16, -1.0, 2.0)
    compare(C5S, b, p, 12, 1, seed=7, rule="metropolis", engine="plane")
    assert kernel_of(C5S, b, p, "metropolis") != "plane_c5_rounds_kernel"
