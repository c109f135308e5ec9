"""Stage timeline of the cluster-per-word round kernel (profiling variant build):
    tools/variant.sh CP "-DTG_CL_PROF=1"
    TG_ENGINE_LIB=$PWD/paper_2506_14781_b200/libtempergrid_b200_CP.so python tools/cl_stages.py [n]
Prints mean microseconds of each stage (block 0) over rounds 8..63 of one 64-round launch."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401

from paper_2506_14781_b200 import _lib  # noqa: E402
from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.api import Engine, RunConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
L = _lib.lib()
pr = I.bipartite_3regular(n, seed=1)
betas, pens = I.config_schedule("c5")
e = Engine(0)
e.set_problem(pr)
e.set_schedule(betas, pens)
e.init(RunConfig(total_sweeps=1, sweeps_per_swap=1, seed=2, store_states=False),
       flags=_lib.REC_DIGEST)
e.advance(64)
torch.cuda.synchronize()
e.advance(64)
torch.cuda.synchronize()
assert e.info()["sweep_kernel"] == "plane_cl_rounds_kernel", e.info()["sweep_kernel"]
buf = np.zeros((64, 16), dtype=np.uint64)
L.tg_debug_cl_prof(buf.ctypes.data_as(C.c_void_p))
t = buf[8:64].astype(np.float64)
names = [(0, 1, "phase 0 items"), (1, 2, "phase 0 cluster barrier"), (2, 3, "phase 1 items + flush"),
         (3, 4, "DSMEM totals + cluster barrier"), (4, 5, "publish + flag wait"),
         (2, 9, "  phase 1: chain-free loop"), (9, 10, "  phase 1: final drain"),
         (10, 11, "  phase 1: chain loop"), (11, 3, "  phase 1: counter flush"),
         (4, 13, "  publish + swap uniform"), (13, 5, "  poll + CTA barrier"),
         (5, 12, "  swap attempts (thread 0)"), (12, 6, "  CTA barrier after swaps"),
         (5, 6, "energies + swap replay"), (6, 7, "records + threshold planes"), (7, 8, "digest")]
for a, b, name in names:
    print(f"N={n} {name:<34s} {np.mean(t[:, b] - t[:, a]) / 1e3:8.2f} us")
print(f"N={n} {'round':<34s} {np.mean(np.diff(t[:, 0])) / 1e3:8.2f} us")
e.close()
