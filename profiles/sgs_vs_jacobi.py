"""Jacobi M_1 vs projected SGS M_2 on the GPU path: energy
after k steps and device time per step, per config.

  python profiles/sgs_vs_jacobi.py [config] [k]

Prints one JSON line per preconditioner: ms per iteration (CUDA events
around emin_iterate(k) after a warm-up call and emin_reset), the energy
decrease ratios dE_k / dE_1 and the final energy, so the time to reach a
given energy can be compared (the paper's point: SGS reduces the energy
'more than twice as fast' per iteration but was slower per unit time in
their MPI code)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_02995_b200 import emin as E  # noqa: E402
from workloads.problems import make_config, sgs_key  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
    prob = make_config(cfg)
    k = int(sys.argv[2]) if len(sys.argv) > 2 else prob.iters
    keys = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]
    dev = {n: (None if getattr(prob, n) is None else torch.from_numpy(np.ascontiguousarray(getattr(prob, n))).cuda())
           for n in keys}
    for pc, kind in (("jacobi", None), ("sgs", "color"), ("sgs", "natural")):
        only = os.environ.get("SGS_ONLY")          # e.g. "sgs:color" (profiling runs)
        if only and only != f"{pc}:{kind}":
            continue
        key = None if kind is None else sgs_key(prob, kind)
        h = E.emin_setup(prob.n, prob.nc, dev["A_rowptr"], dev["A_col"], dev["A_val"], dev["is_coarse"],
                         dev["P_rowptr"], dev["P_col"], dev["P_val"], prob.nv, dev["B"], dev["Bc"],
                         block_size=prob.block_size, stagnation_rel=0.0, precond=pc,
                         sgs_key=None if key is None else torch.from_numpy(key).cuda())
        E.emin_iterate(h, k)
        E.emin_reset(h)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        kd, dE = E.emin_iterate(h, k, want=True)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        rep = E.emin_report(h)
        En = E.emin_energy(h)
        E.emin_destroy(h)
        print(json.dumps({"config": cfg, "precond": pc, "order": kind, "levels": rep["sgs_levels"], "k": kd,
                          "ms_per_iter": ms / max(kd, 1), "E0": rep["E0"], "E_k": En,
                          "dE_ratio": [float(dE[j] / dE[0]) for j in (1, 3, 9, kd - 1) if j < kd]}), flush=True)


if __name__ == "__main__":
    main()
