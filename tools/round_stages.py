"""Stage timeline of the fused tpw round loop (profiling variant build):
    tools/variant.sh P "-DTG_TPW_PROF=1"
    TG_ENGINE_LIB=$PWD/paper_2506_14781_b200/libtempergrid_b200_P.so python tools/round_stages.py [n]
Prints mean microseconds of each stage over rounds 8..63 of one 64-round launch."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401

from paper_2506_14781_b200 import _lib  # noqa: E402
from paper_2506_14781_b200 import instances as I  # noqa: E402
from paper_2506_14781_b200.api import Engine, RunConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = _lib.lib()
pr = I.bipartite_3regular(n, seed=1)
betas, pens = I.config_schedule("c5")
e = Engine(0)
e.set_problem(pr)
e.set_schedule(betas, pens)
e.init(RunConfig(total_sweeps=1, sweeps_per_swap=1, seed=2, store_states=False),
       flags=_lib.REC_DIGEST | _lib.REC_COUNTERS)
e.advance(64)
torch.cuda.synchronize()
L.tg_debug_tpw_prof_reset()
e.advance(64)
torch.cuda.synchronize()
buf = np.zeros((64, 16), dtype=np.uint64)
L.tg_debug_tpw_prof(buf.ctypes.data_as(C.c_void_p))
t = buf[8:64].astype(np.float64)
names = [(0, 1, "phase 0 items (block 0)"), (0, 2, "phase 0 items (last block)"),
         (2, 3, "phase 0 flush + barrier"), (3, 4, "phase 1 items (block 0)"),
         (3, 5, "phase 1 items (last block)"), (5, 6, "phase 1 flush + barrier"),
         (6, 8, "epilogue: energies + swap replay"), (8, 9, "epilogue: thresholds"),
         (9, 10, "epilogue: digest"), (10, 7, "epilogue barrier")]
for a, b, name in names:
    print(f"N={n} {name:<34s} {np.mean(t[:, b] - t[:, a]) / 1e3:8.2f} us")
print(f"N={n} {'round':<34s} {np.mean(np.diff(t[:, 0])) / 1e3:8.2f} us")
e.close()
