"""A/B variant check: the same config with debug_flags 0 and the given flags
must give bitwise-identical P, energy and step count (kernel variants change
only the schedule, never the arithmetic).

  python profiles/ab_bitwise.py config flags [k] [size]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_02995_b200 import Emin  # noqa: E402
from workloads.problems import make_config  # noqa: E402

cfg = sys.argv[1]
dbg = int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 10
size = int(sys.argv[4]) if len(sys.argv) > 4 else None
prob = make_config(cfg, size=size) if size else make_config(cfg)
res = []
for f in (0, dbg):
    g = Emin.from_problem(prob, stagnation_rel=0.0, debug_flags=f)
    kd, dE = g.iterate(k)
    res.append((kd, np.asarray(dE), g.energy(), g.get_P()))
    g.close()
torch.cuda.synchronize()
a, b = res
ok = a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2] and np.array_equal(a[3], b[3])
print(f"config {cfg} flags {dbg}: k {a[0]}/{b[0]} E {a[2]!r}/{b[2]!r} bitwise={'OK' if ok else 'DIFF'}", flush=True)
sys.exit(0 if ok else 1)
