"""Device time per CG iteration of emin_iterate(k) (CUDA events around the
call, after a warm-up call), for the given debug_flags.

  python profiles/iter_time.py config flags [k] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2208_02995_b200 import Emin  # noqa: E402
from workloads.problems import make_config  # noqa: E402

cfg = sys.argv[1]
dbg = int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
prob = make_config(cfg)
g = Emin.from_problem(prob, stagnation_rel=0.0, debug_flags=dbg)
s = torch.cuda.current_stream()
ts = []
for r in range(reps + 1):
    g.reset()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.iterate(k, want=False)
    e1.record(s)
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1) / k)
ts.sort()
print(f"config {cfg} flags {dbg}: {1e3 * ts[len(ts) // 2]:.1f} us per iteration (median of {reps}, k={k}), "
      f"launches {g.report().get('launches')}", flush=True)
