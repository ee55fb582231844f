"""Device-timed bench step (emin_setup from device inputs + emin_iterate(k) +
emin_energy + emin_get_P + emin_destroy) for two debug_flags values, median
of reps (CUDA events around the whole step, after warm-up steps).

  python profiles/step_ab.py config flagsA flagsB [reps]
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
flags = [int(sys.argv[2]), int(sys.argv[3])]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 7
prob = make_config(cfg)
keys = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]
dev = {k: (None if getattr(prob, k) is None else torch.from_numpy(np.ascontiguousarray(getattr(prob, k))).cuda())
       for k in keys}
out = torch.empty(int(prob.P_rowptr[-1]), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()


def step(f):
    h = E.emin_setup(prob.n, prob.nc, dev["A_rowptr"], dev["A_col"], dev["A_val"], dev["is_coarse"],
                     dev["P_rowptr"], dev["P_col"], dev["P_val"], prob.nv, dev["B"], dev["Bc"],
                     block_size=prob.block_size, stagnation_rel=0.0, debug_flags=f)
    E.emin_iterate(h, prob.iters)
    E.emin_energy(h)
    E.emin_get_P(h, out)
    E.emin_destroy(h)


res = {f: [] for f in flags}
for r in range(reps + 2):
    for f in flags:
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        step(f)
        e1.record(s)
        torch.cuda.synchronize()
        if r >= 2:
            res[f].append(e0.elapsed_time(e1))
for f in flags:
    v = sorted(res[f])
    print(f"config {cfg} flags {f}: step {v[len(v) // 2]:.3f} ms (median of {reps}; min {v[0]:.3f})", flush=True)
