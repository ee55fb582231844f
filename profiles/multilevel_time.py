"""Time the multilevel hierarchy on one GPU: per level
the device milliseconds of the pattern growth, emin_setup, emin_iterate(k)
and emin_galerkin, with CUDA events on the current stream (after one
untimed warm-up build of the same hierarchy).

usage: python profiles/multilevel_time.py CONFIG [LEVELS] [ITERS]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_02995_b200.build import build  # noqa: E402
from paper_2208_02995_b200.multilevel import emin_multilevel  # noqa: E402
from workloads.problems import coarse_split, make_config  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
    nlev = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    t0 = time.time()
    prob = make_config(cfg)
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else prob.iters
    build()
    dims, zlo = prob.meta["dims"], prob.meta.get("zlo", 0)
    iscs = []
    for _ in range(nlev):
        isc, dims, zlo = coarse_split(dims, zlo)
        iscs.append(torch.from_numpy(np.repeat(isc, prob.block_size).astype(np.uint8)).cuda())
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    args = (t(prob.A_rowptr), t(prob.A_col), t(prob.A_val), iscs, t(prob.B))
    kw = dict(block_size=prob.block_size, P_rowptr=t(prob.P_rowptr), P_col=t(prob.P_col),
              P_val=t(prob.P_val), iters=iters)
    print(f"# inputs {time.time() - t0:.1f}s", file=sys.stderr)
    emin_multilevel(*args, **kw)                      # warm-up
    torch.cuda.synchronize()
    levels = emin_multilevel(*args, timing=True, **kw)
    tot = dict(pattern=0.0, setup=0.0, iterate=0.0, galerkin=0.0)
    for lv in levels:
        for k in tot:
            tot[k] += lv["ms"][k]
        nnzAc = int(lv["A_c"][1].numel())
        print(json.dumps(dict(config=cfg, level=lv["level"], n=lv["n"], nc=lv["nc"], nnz_A=lv["nnz_A"],
                              nnz_W=lv["nnz_W"], nnz_Ac=nnzAc, k=lv["k_done"], E0=lv["E0"], E=lv["E"],
                              kernel_path=lv["kernel_path"], ms=lv["ms"],
                              updates_per_s=lv["nnz_W"] * lv["k_done"] / (lv["ms"]["iterate"] * 1e-3))))
    print(json.dumps(dict(config=cfg, levels=nlev, total_ms=tot, sum_ms=sum(tot.values()))))


if __name__ == "__main__":
    main()
