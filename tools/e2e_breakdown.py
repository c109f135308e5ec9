"""Where the e2e (public API, host buffers) time of bench.py's default workload
goes: run with TG_HOST_TIMING=1 on a GPU box; prints the library's host phase
timers plus Python-side wall times of each API call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TG_HOST_TIMING", "1")
import torch  # noqa: E402,F401  (NCCL / CUDA runtime first, as bench.py)

from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.api import Engine, RunConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1 << 20
t = time.perf_counter()
pr = I.bipartite_3regular(n, seed=1)
if "--pinned" in sys.argv:  # as bench.py's e2e leg
    import numpy as np
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    pr = I.Problem(pr.n, pin(pr.ci), pin(pr.cj), pin(pr.cw), pin(pr.fields), pin(pr.pa), pin(pr.pb))
betas, pens = I.config_schedule("c5")
print(f"generate {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
for rep in range(3):
    print(f"--- rep {rep}", flush=True)
    T = {}
    t = time.perf_counter(); e = Engine(0); T["Engine()"] = time.perf_counter() - t
    t = time.perf_counter(); e.set_problem(pr); T["set_problem"] = time.perf_counter() - t
    t = time.perf_counter(); e.set_schedule(betas, pens); T["set_schedule"] = time.perf_counter() - t
    t = time.perf_counter()
    e.run(RunConfig(total_sweeps=100, sweeps_per_swap=1, seed=2, store_states=False, digest=False),
          lambda r, k, s, a, b: 0, flags=0)
    T["run(100 rounds)"] = time.perf_counter() - t
    t = time.perf_counter(); e.state(255); T["state"] = time.perf_counter() - t
    t = time.perf_counter(); e.close(); T["close"] = time.perf_counter() - t
    for k, v in T.items():
        print(f"  {k:<20s} {1e3 * v:9.2f} ms", flush=True)
