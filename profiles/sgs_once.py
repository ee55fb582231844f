"""One SGS-preconditioned context (colouring key) of a config: warm-up
emin_iterate(k), reset, emin_iterate(k) again -- for launch lists of the SGS
iteration (ncu --metrics gpu__time_duration.sum).

  python profiles/sgs_once.py config [k] [size]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_02995_b200 import Emin  # noqa: E402
from workloads.problems import make_config, sgs_key  # noqa: E402

cfg = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
size = int(sys.argv[3]) if len(sys.argv) > 3 else None
prob = make_config(cfg, size=size) if size else make_config(cfg)
key = torch.from_numpy(np.ascontiguousarray(sgs_key(prob, "color"))).cuda()
g = Emin.from_problem(prob, precond="sgs", sgs_key=key, stagnation_rel=0.0)
g.iterate(k, want=False)
g.reset()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.iterate(k, want=False)
e1.record()
torch.cuda.synchronize()
print(f"config {cfg} sgs: {e0.elapsed_time(e1) / k:.3f} ms per iteration, levels {g.report()['sgs_levels']}", flush=True)
