import os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2208_02995_b200 import Emin
from workloads.problems import make_config, sgs_key
prob = make_config("3")
key = sgs_key(prob, "color")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = Emin.from_problem(prob, device="cuda", stagnation_rel=0.0, precond="sgs", sgs_key=key,
                          debug_flags=8 if rep == 2 else 0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("setup ms", round(1e3 * (t1 - t0), 2), flush=True)
    g.close()
