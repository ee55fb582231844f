"""Host-timed breakdown of one bench step (setup / iterate / energy / get_P /
destroy) with the EMIN_DBG_TRACE phase timing of emin_setup.

  python profiles/step_breakdown.py [config]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_02995_b200 import emin as E  # noqa: E402
from workloads.problems import make_config  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
    prob = make_config(cfg)
    keys = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]
    dev = {k: (None if getattr(prob, k) is None else torch.from_numpy(np.ascontiguousarray(getattr(prob, k))).cuda())
           for k in keys}
    out = torch.empty(int(prob.P_rowptr[-1]), dtype=torch.float64, device="cuda")
    res = []
    for rep in range(4):
        t = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = E.emin_setup(prob.n, prob.nc, dev["A_rowptr"], dev["A_col"], dev["A_val"], dev["is_coarse"],
                         dev["P_rowptr"], dev["P_col"], dev["P_val"], prob.nv, dev["B"], dev["Bc"],
                         block_size=prob.block_size, stagnation_rel=0.0, debug_flags=8 if rep == 3 else 0)
        torch.cuda.synchronize()
        t["setup"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        E.emin_iterate(h, prob.iters)
        torch.cuda.synchronize()
        t["iterate"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        E.emin_energy(h)
        t["energy"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        E.emin_get_P(h, out)
        torch.cuda.synchronize()
        t["get_P"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        E.emin_destroy(h)
        torch.cuda.synchronize()
        t["destroy"] = time.perf_counter() - t0
        res.append({k: round(v * 1e3, 3) for k, v in t.items()})
        print(json.dumps(res[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"config": cfg, "ms": res[-1]}))


if __name__ == "__main__":
    main()
