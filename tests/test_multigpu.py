"""GPU-count invariance on real GPUs (the B200 analogue of the reference's
thread-count invariance, test_engine.cpp:214-227, acceptance criterion 8):
the same run on 2 GPUs -- replicas split over the ranks, per-round (f, g)
all-gathered over NCCL, the swap phase replayed on every rank, target digests
and snapshots all-reduced per record chunk -- gives the 1-GPU records and
final grid bit for bit.  Needs >= 2 GPUs (skipped otherwise; the exchange
logic itself is covered on CPU by tests/test_multirank.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


needs2 = pytest.mark.skipif(n_gpus() < 2, reason="needs 2 GPUs")


def _case(name):
    from paper_2506_14781_b200 import instances as I
    if name == "plane":
        return I.bipartite_3regular(4096, seed=2), *I.config_schedule("c5"), "plane"
    pr = I.k10_pm1(1)
    return pr, *I.config_schedule("c1"), "slot"


def _run(pr, b, p, engine, rank=0, world=1, nccl_id=None, device=0):
    from paper_2506_14781_b200.api import Engine, RunConfig
    eng = Engine(device, rank, world, nccl_id)
    eng.set_problem(pr)
    eng.set_schedule(b, p)
    recs = []

    def sink(r, n, st, ap, ab):
        for k in range(n):
            recs.append((r[k].round, r[k].f, r[k].g, r[k].digest, r[k].target_state))
        return 0

    eng.run(RunConfig(total_sweeps=40, sweeps_per_swap=1, seed=17, engine=engine, store_states=False,
                      digest=True), sink)
    grid = eng.grid()
    eng.close()
    return recs, grid


def _worker(rank, world, port, name, nccl_id, q):
    import torch
    torch.cuda.set_device(rank)
    pr, b, p, engine = _case(name)
    recs, grid = _run(pr, b, p, engine, rank, world, nccl_id, device=rank)
    q.put((rank, recs, grid))


@needs2
@pytest.mark.parametrize("name", ["plane", "slot"])
def test_two_gpus_equal_one_gpu(name):
    import torch.multiprocessing as mp
    from paper_2506_14781_b200.api import Engine
    pr, b, p, engine = _case(name)
    ref_recs, ref_grid = _run(pr, b, p, engine)
    nid = Engine.nccl_unique_id()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, nid, q)) for r in range(2)]
    for pr_ in procs:
        pr_.start()
    out = [q.get(timeout=600) for _ in procs]
    for pr_ in procs:
        pr_.join(timeout=60)
    for rank, recs, grid in out:
        assert recs == ref_recs, rank
        np.testing.assert_array_equal(grid, ref_grid)


@pytest.mark.parametrize("name", ["plane", "slot"])
def test_one_rank_nccl_round_loop_equals_fused(name, monkeypatch):
    """The multi-GPU round loop on one GPU: with TG_DIST_SELFTEST=1 a world-size-1
    context initialises a one-rank NCCL communicator and takes the unfused path
    (sweep launches, ncclAllGather of (f, g) per round and the per-chunk
    ncclAllReduce of digests inside the captured CUDA graph).  Its records and
    final grid must equal the fused single-GPU run's."""
    from paper_2506_14781_b200.api import Engine
    pr, b, p, engine = _case(name)
    ref_recs, ref_grid = _run(pr, b, p, engine)
    monkeypatch.setenv("TG_DIST_SELFTEST", "1")
    for graphs in ("0", "1"):  # direct launches (default) and the captured-graph replay
        monkeypatch.setenv("TG_GRAPHS", graphs)
        recs, grid = _run(pr, b, p, engine, 0, 1, Engine.nccl_unique_id())
        assert recs == ref_recs, graphs
        np.testing.assert_array_equal(grid, ref_grid)
