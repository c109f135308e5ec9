"""Small config-5 run on the c5 kernel (debugging / sanitizer target)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200.api import Engine, RunConfig

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
npen = int(sys.argv[3]) if len(sys.argv) > 3 else 8
pr = I.bipartite_3regular(n, seed=3)
b = list(np.geomspace(0.2, 5.0, nb))
p = list(np.round(np.linspace(0.0, 1.0, npen) * 64) / 64)
eng = Engine(0)
eng.set_problem(pr)
eng.set_schedule(b, p)
eng.run(RunConfig(total_sweeps=4, sweeps_per_swap=1, seed=1, engine="plane", store_states=False), None)
print(eng.info()["sweep_kernel"])
eng.close()
