"""Per-step device times of the bench step loop (emin_setup from device
inputs on a side stream, iterate, energy, get_P, report, destroy), to look
for drift over many steps.

  python profiles/step_series.py config steps flags
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_02995_b200 import emin as E  # noqa: E402
from workloads.problems import make_config  # noqa: E402

cfg = sys.argv[1]
steps = int(sys.argv[2])
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
prob = make_config(cfg)
keys = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]
dev = {k: (None if getattr(prob, k) is None else torch.from_numpy(np.ascontiguousarray(getattr(prob, k))).cuda())
       for k in keys}
out = torch.empty(int(prob.P_rowptr[-1]), dtype=torch.float64, device="cuda")
stream = torch.cuda.Stream()
ts = []
with torch.cuda.stream(stream):
    for it in range(steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h = E.emin_setup(prob.n, prob.nc, dev["A_rowptr"], dev["A_col"], dev["A_val"], dev["is_coarse"],
                         dev["P_rowptr"], dev["P_col"], dev["P_val"], prob.nv, dev["B"], dev["Bc"],
                         block_size=prob.block_size, stagnation_rel=0.0, stream=stream.cuda_stream,
                         debug_flags=flags)
        E.emin_iterate(h, prob.iters)
        E.emin_energy(h)
        E.emin_get_P(h, out)
        E.emin_report(h)
        E.emin_destroy(h)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
print("per-step ms:", " ".join(f"{t:.2f}" for t in ts))
print(f"median {sorted(ts)[len(ts) // 2]:.3f} ms, first {ts[0]:.2f}, last {ts[-1]:.2f}")
