"""SGS A/B: the same config with the colouring key, debug_flags 0 and the
given flags: bitwise comparison of dE, P, E after k steps, and ms per
iteration of each.

  python profiles/sgs_ab.py config flags [k] [size]
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
dbg = int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 10
size = int(sys.argv[4]) if len(sys.argv) > 4 else None
prob = make_config(cfg, size=size) if size else make_config(cfg)
key = torch.from_numpy(np.ascontiguousarray(sgs_key(prob, "color"))).cuda()
res = []
for f in (0, dbg):
    g = Emin.from_problem(prob, precond="sgs", sgs_key=key, stagnation_rel=0.0, debug_flags=f)
    g.iterate(k, want=False)
    g.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    kd, dE = g.iterate(k)
    e1.record()
    torch.cuda.synchronize()
    res.append((kd, np.asarray(dE), g.energy(), g.get_P(), e0.elapsed_time(e1) / max(kd, 1)))
    g.close()
a, b = res
ok = a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2] and np.array_equal(a[3], b[3])
print(f"config {cfg} sgs flags 0 vs {dbg}: {a[4]:.3f} vs {b[4]:.3f} ms/iter, k {a[0]}/{b[0]}, "
      f"bitwise={'OK' if ok else 'DIFF'}", flush=True)
