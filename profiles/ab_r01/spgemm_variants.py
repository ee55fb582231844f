"""A/B of the per-iteration masked-SpGEMM variants on one config (GPU).

  python profiles/spgemm_variants.py [config] [variants...]   (win2 | EMIN_NODAL=s ...)

Times every kernel class with CUDA events (emin_kernel_times) over
emin_iterate(k) after a warm-up call, for each EMIN_SPGEMM variant, and
checks that all variants give the same energy (to 1e-12 relative).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_02995_b200 import emin as E  # noqa: E402
from workloads.problems import make_config  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
    variants = sys.argv[2:] or ["hdr", "win", "tile", "pipe"]
    prob = make_config(cfg)
    keys = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]
    dev = {k: (None if getattr(prob, k) is None else torch.from_numpy(np.ascontiguousarray(getattr(prob, k))).cuda())
           for k in keys}
    k = prob.iters
    res = {}
    for var in variants:
        # "win2" sets EMIN_SPGEMM; "EMIN_NODAL=s" sets that variable
        ek, ev = var.split("=", 1) if "=" in var else ("EMIN_SPGEMM", var)
        saved = os.environ.get(ek)
        os.environ[ek] = ev
        h = E.emin_setup(prob.n, prob.nc, dev["A_rowptr"], dev["A_col"], dev["A_val"], dev["is_coarse"],
                         dev["P_rowptr"], dev["P_col"], dev["P_val"], prob.nv, dev["B"], dev["Bc"],
                         block_size=prob.block_size, stagnation_rel=0.0)
        E.emin_iterate(h, k)
        E.emin_reset(h)
        E.emin_set_profiling(h, 1)
        E.emin_iterate(h, k)
        kt = E.emin_kernel_times(h)
        en = E.emin_energy(h)
        E.emin_destroy(h)
        if saved is None:
            os.environ.pop(ek)
        else:
            os.environ[ek] = saved
        res[var] = {n: round(ms / max(c, 1) * 1e3, 2) for n, (ms, c) in kt.items()}
        res[var]["energy"] = en
        print(var, json.dumps(res[var]), flush=True)
    es = [r["energy"] for r in res.values()]
    assert max(es) - min(es) <= 1e-12 * abs(es[0]), es
    print(json.dumps({"config": cfg, "us_per_launch": res}))


if __name__ == "__main__":
    main()
