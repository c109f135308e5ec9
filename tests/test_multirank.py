"""Multi-rank exchange logic on CPU (gloo, world_size 2): the replica
partition of tg_partition, the all-gather of per-replica (f, g) and the
identical swap-phase replay every rank performs (tg_swap_phase_host, the same
routine the device swap kernel runs).  Every rank must reach the same labels
and counters as a single-process run."""
import ctypes as C
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_14781_b200 import _lib

I_, J_ = 4, 16        # 64 replicas: two 32-replica words, one per rank
ROUNDS = 60
SEED = 23


def P(a):
    return a.ctypes.data_as(C.c_void_p)


def energies(rnd, R):
    rng = np.random.default_rng(1000 + rnd)
    return rng.normal(size=R) * 5.0, 4.0 * rng.integers(0, 5, size=R).astype(np.float64)


def replay(L, slices):
    betas = np.geomspace(0.2, 5.0, I_)
    pens = np.linspace(0.0, 1.0, J_)
    R = I_ * J_
    ss = np.arange(R, dtype=np.int32)
    ap = np.zeros(I_ * (J_ - 1), np.int64)
    ab = np.zeros((I_ - 1) * J_, np.int64)
    base = 0
    for rnd in range(1, ROUNDS + 1):
        f, g = slices(rnd)
        assert L.tg_swap_phase_host(I_, P(betas), J_, P(pens), rnd, 0, SEED, base, P(f), P(g),
                                    P(ss), P(ap), P(ab)) == 0
        even = rnd % 2 == 0
        direction = 1 if ((rnd - 1) // 2) % 2 == 0 else -1
        base += I_ * ((J_ - even) // 2) if direction == 1 else J_ * ((I_ - even) // 2)
    return ss, ap, ab


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = _lib.lib()
    R = I_ * J_
    s0, cnt = C.c_int32(), C.c_int32()
    assert L.tg_partition(R, rank, world, 2, C.byref(s0), C.byref(cnt)) == 0

    def gathered(rnd):
        f, g = energies(rnd, R)
        local = torch.from_numpy(np.stack([f, g])[:, s0.value:s0.value + cnt.value].copy())
        out = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(out, local)
        full = torch.cat(out, dim=1).numpy()
        assert np.array_equal(full[0], f) and np.array_equal(full[1], g)
        return np.ascontiguousarray(full[0]), np.ascontiguousarray(full[1])

    ss, ap, ab = replay(L, gathered)
    res = [None] * world
    dist.all_gather_object(res, (ss.tolist(), ap.tolist(), ab.tolist(), s0.value, cnt.value))
    if rank == 0:
        q.put(res)
    dist.destroy_process_group()


def test_two_rank_exchange_matches_single_process():
    L = _lib.lib()
    single = replay(L, lambda rnd: energies(rnd, I_ * J_))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][3:] == (0, 32) and res[1][3:] == (32, 32)
    for r in res:
        assert r[0] == single[0].tolist()
        assert r[1] == single[1].tolist() and r[2] == single[2].tolist()
    assert single[1].sum() + single[2].sum() > 0  # swaps actually happened


def test_partition_rules():
    L = _lib.lib()
    s0, cnt = C.c_int32(), C.c_int32()
    assert L.tg_partition(256, 3, 8, 2, C.byref(s0), C.byref(cnt)) == 0 and (s0.value, cnt.value) == (96, 32)
    assert L.tg_partition(256, 0, 16, 2, C.byref(s0), C.byref(cnt)) == _lib.TG_ERR_CONFIG  # 16 per rank
    assert L.tg_partition(256, 0, 16, 1, C.byref(s0), C.byref(cnt)) == 0  # slot engine: any split
    assert L.tg_partition(100, 0, 3, 1, C.byref(s0), C.byref(cnt)) == _lib.TG_ERR_CONFIG
