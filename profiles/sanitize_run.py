"""Small end-to-end runs of every kernel path for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per gpurun call):
setup (Alg. 2, r0, E0) -> iterate -> energy -> get_P on configs 1, 1b, 2b
(10^3), 3 (12^3), 4 (3 elements) and 5 (8^3), the scalar, nodal and generic
paths, the SGS preconditioner, the max-vol start, the pattern and Galerkin
calls, and a 2-rank loopback run (halo exchange).

  compute-sanitizer --tool memcheck python profiles/sanitize_run.py
"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_02995_b200 import Emin  # noqa: E402
from paper_2208_02995_b200 import emin as E  # noqa: E402
from paper_2208_02995_b200.partition import partition_rows, plane_rows, rank_slice  # noqa: E402
from workloads.problems import make_config, sgs_key  # noqa: E402


def run(prob, k, **kw):
    g = Emin.from_problem(prob, **kw)
    kd, _ = g.iterate(k)
    e = g.energy()
    P = g.get_P()
    rep = g.report()
    g.close()
    return kd, e, P, rep


def loopback(prob, R, k):
    ranges = partition_rows(prob.P_rowptr, prob.is_coarse, R, plane=plane_rows(prob))
    lb = E.emin_loopback_create(R)
    out = [None] * R

    def work(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        rb, re_ = ranges[r]
        a = rank_slice(prob, rb, re_)
        h = E.emin_setup(prob.n, prob.nc, a["A_rowptr"], a["A_col"], a["A_val"], a["is_coarse"], a["P_rowptr"],
                         a["P_col"], a["P_val"], prob.nv, a["B"], a["Bc"], block_size=prob.block_size,
                         stream=st.cuda_stream, row_begin=rb, row_end=re_, loopback=lb, loopback_rank=r)
        kd, _ = E.emin_iterate(h, k, want=True)
        out[r] = (kd, E.emin_energy(h), E.emin_report(h)["n_halo_rows"])
        E.emin_destroy(h)

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    E.emin_loopback_destroy(lb)
    return out


def main():
    torch.cuda.set_device(0)
    cases = [("1", None, 20, {}), ("1b", None, 20, {}), ("2b", 10, 30, {}), ("3", 12, 40, {}), ("4", 3, 30, {}),
             ("5", 8, 10, {}), ("4", 3, 10, dict(debug_flags=1)), ("3", 12, 10, dict(debug_flags=1)),
             ("1b", None, 10, dict(project_after_jacobi=1)), ("4", 3, 10, dict(start="maxvol")),
             ("1b", None, 10, dict(device="host"))]
    for name, size, k, kw in cases:
        prob = make_config(name, size=size)
        kd, e, _, rep = run(prob, k, **kw)
        print(f"{name}({size}) {kw}: k {kd} E {e:.12e} path {rep['kernel_path']}", flush=True)
    for name, size, kind in [("3", 12, "color"), ("4", 3, "color"), ("1b", None, "natural")]:
        prob = make_config(name, size=size)
        kd, e, _, rep = run(prob, 10, precond="sgs", sgs_key=sgs_key(prob, kind))
        print(f"sgs {name}({size}) {kind}: k {kd} E {e:.12e} levels {rep['sgs_levels']}", flush=True)
    for name, size in [("3", 12), ("4", 3)]:
        prob = make_config(name, size=size)
        rp, col = E.emin_pattern(prob.n, prob.A_rowptr, prob.A_col, prob.is_coarse, prob.block_size, prob.nv,
                                 prob.Bc, prob.nc)
        assert np.array_equal(rp, prob.P_rowptr)
        Pv = Emin.from_problem(prob).get_P()
        rpc, colc, valc = E.emin_galerkin(prob.n, prob.nc, prob.A_rowptr, prob.A_col, prob.A_val, prob.P_rowptr,
                                          prob.P_col, Pv)
        print(f"pattern + galerkin {name}({size}): nnz(A_c) {len(colc)}", flush=True)
    for name, size in [("3", 12), ("4", 4)]:
        print(f"loopback 2 ranks {name}({size}):", loopback(make_config(name, size=size), 2, 10), flush=True)
    torch.cuda.synchronize()
    print("sanitize_run OK", flush=True)


if __name__ == "__main__":
    main()
