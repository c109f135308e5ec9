"""Fixed per-round cost of the fused PLANE round loop: device time per round
at small N (where the sweep work is negligible) for record-flag variants.
Run on a GPU box:  python tools/round_overhead.py [n] [chain_frac]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_14781_b200 import _lib  # noqa: E402
from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.api import Engine, RunConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
chain_frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
pr = I.bipartite_3regular(n, seed=1, chain_frac=chain_frac)
betas, pens = I.config_schedule("c5")
for name, flags in (("digest+counters", _lib.REC_DIGEST | _lib.REC_COUNTERS),
                    ("digest", _lib.REC_DIGEST), ("none", 0)):
    e = Engine(0)
    e.set_problem(pr)
    e.set_schedule(betas, pens)
    e.init(RunConfig(total_sweeps=1, sweeps_per_swap=1, seed=2, store_states=False), flags=flags)
    st = torch.cuda.ExternalStream(e.stream_ptr())
    e.advance(200)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rounds = 2000
    a.record(st)
    e.advance(rounds)
    b.record(st)
    b.synchronize()
    print(f"N={n} chains={chain_frac} {name:<16s} {1e3 * a.elapsed_time(b) / rounds:7.2f} us/round  kernel={e.info()['sweep_kernel']}",
          flush=True)
    e.close()
