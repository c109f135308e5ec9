"""Per-round time of the multi-GPU round loop on ONE GPU (TG_DIST_SELFTEST=1: one-rank NCCL
communicator, sweep launches + ncclAllGather + swap + per-chunk ncclAllReduce inside the captured
graph) next to the fused single-GPU kernel, config 5.   python tools/dist_selftest_rate.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.api import Engine, RunConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
pr = I.bipartite_3regular(n, seed=1)
betas, pens = I.config_schedule("c5")
for name in ("fused", "dist-selftest", "dist-selftest graphs"):
    if name.startswith("dist"):
        os.environ["TG_DIST_SELFTEST"] = "1"
        if "graphs" in name:
            os.environ["TG_GRAPHS"] = "1"
        e = Engine(0, 0, 1, Engine.nccl_unique_id())
    else:
        e = Engine(0)
    e.set_problem(pr)
    e.set_schedule(betas, pens)
    e.init(RunConfig(total_sweeps=1, sweeps_per_swap=1, seed=2, store_states=False, digest=True))
    st = torch.cuda.ExternalStream(e.stream_ptr())
    e.advance(100)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rounds = 400
    a.record(st)
    e.advance(rounds)
    b.record(st)
    b.synchronize()
    us = 1e3 * a.elapsed_time(b) / rounds
    print(f"N={n} {name:<26s} {us:8.2f} us/round  {n * 256 / us * 1e6:.3e} flips/s  kernel={e.info()['sweep_kernel']}", flush=True)
    e.close()
