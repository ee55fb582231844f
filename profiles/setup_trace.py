"""EMIN_DBG_TRACE phases of emin_setup (device inputs) for a config, after a
warm-up setup, plus the host-timed iterate/energy/get_P/destroy of one step."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_02995_b200 import Emin  # noqa: E402
from workloads.problems import make_config  # noqa: E402

prob = make_config(sys.argv[1] if len(sys.argv) > 1 else "3")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = Emin.from_problem(prob, device="cuda", stagnation_rel=0.0, debug_flags=8 if rep == 2 else 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    g.iterate(prob.iters, want=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    g.energy()
    t3 = time.perf_counter()
    g.get_P()
    t4 = time.perf_counter()
    g.close()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"rep {rep}: setup {1e3*(t1-t0):.2f} ms (incl. H2D of the torch copies), iterate {1e3*(t2-t1):.2f}, "
          f"energy {1e3*(t3-t2):.2f}, get_P(+D2H) {1e3*(t4-t3):.2f}, destroy {1e3*(t5-t4):.2f}", flush=True)
