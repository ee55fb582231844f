"""Multilevel driver (reading A26): the paper's real use
of the method -- the prolongation of every level of the hierarchy is built
by Alg. 1's pattern + Alg. 2 + Alg. 3 (T_i sums over the levels),
and the next level's operator is the Galerkin product A_c = P^T A P formed
by the coarse grid construction.

Every step is one C-ABI call of libemin (emin_pattern, emin_setup,
emin_iterate, emin_energy, emin_get_P, emin_galerkin); this module only
sequences them and keeps the arrays on the device.  The C/F splitting of
each level is an input (the paper takes it from PMIS, out of scope;
the configs use geometric 2x coarsening, ``workloads.problems.coarse_split``).
"""
from __future__ import annotations

from .emin import (emin_destroy, emin_energy, emin_galerkin, emin_get_P, emin_iterate, emin_pattern,
                   emin_report, emin_setup)


def emin_multilevel(A_rowptr, A_col, A_val, is_coarse_levels, B, *, block_size=1, P_rowptr=None,
                    P_col=None, P_val=None, iters=30, l0=2, l0_coarse=1, lmax=4, galerkin_last=True,
                    timing=False, **setup_opts):
    """Build the prolongations of len(is_coarse_levels) levels on the GPU.

    A_*        level-1 operator, CSR, CUDA tensors (int64 / int32 / float64).
    is_coarse_levels  one uint8 CUDA tensor per level (C/F of that level's
               unknowns; level l + 1 has sum(is_coarse_levels[l]) unknowns).
    B          level-1 near kernel [n, nv] float64 CUDA tensor; level l + 1
               uses B_c of level l (its injection).
    P_rowptr / P_col   level-1 pattern (else Alg. 1's growth from distance
               l0); coarser levels grow from distance l0_coarse (A26).
    P_val      level-1 start values or None (least-norm start).
    Returns a list of dicts per level: n, nc, nnz_A, nnz_W, E0, E, k_done,
    the level's P (rowptr, col, val) and its operator, plus the next
    operator A_c when galerkin_last or not the last level; with timing=True
    also the device milliseconds of pattern / setup / iterate / galerkin.
    """
    import torch
    levels = []
    A = (A_rowptr, A_col, A_val)
    Bl = B
    nv = int(B.shape[1])
    for lev, isc in enumerate(is_coarse_levels):
        isc = isc.to(torch.uint8).contiguous()
        n = int(A[0].numel() - 1)
        if int(isc.numel()) != n:
            raise ValueError(f"level {lev + 1}: is_coarse has {isc.numel()} entries, the operator {n} rows")
        cmask = isc.bool()
        nc = int(cmask.sum().item())
        Bc = Bl[cmask].contiguous()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timing else None
        if ev:
            ev[0].record()
        if lev == 0 and P_rowptr is not None:
            prp, pcol = P_rowptr, P_col
            pval = P_val
        else:
            prp, pcol = emin_pattern(n, A[0], A[1], isc, block_size, nv, Bc, nc,
                                     l0=l0 if lev == 0 else l0_coarse, lmax=max(lmax, l0_coarse + 1))
            pval = None
        if ev:
            ev[1].record()
        ctx = emin_setup(n, nc, A[0], A[1], A[2], isc, prp, pcol, pval, nv, Bl, Bc,
                         block_size=block_size, **setup_opts)
        try:
            if ev:
                ev[2].record()
            kd, dE = emin_iterate(ctx, iters, want=True)
            if ev:
                ev[3].record()
            E = emin_energy(ctx)
            rep = emin_report(ctx)
            Pv = torch.empty(int(pcol.numel()), dtype=torch.float64, device=A[2].device)
            emin_get_P(ctx, Pv)
        finally:
            emin_destroy(ctx)
        info = dict(level=lev + 1, n=n, nc=nc, nnz_A=int(A[1].numel()), nnz_W=int(rep["nnz_W"]),
                    E0=rep["E0"], E=E, k_done=kd, dE=dE, P=(prp, pcol, Pv), A=A,
                    kernel_path=rep.get("kernel_path"))
        if galerkin_last or lev + 1 < len(is_coarse_levels):
            Ac = emin_galerkin(n, nc, A[0], A[1], A[2], prp, pcol, Pv)
            info["A_c"] = Ac
            A = Ac
            Bl = Bc
        if ev:
            ev[4].record()
            ev[4].synchronize()
            info["ms"] = dict(pattern=ev[0].elapsed_time(ev[1]), setup=ev[1].elapsed_time(ev[2]),
                              iterate=ev[2].elapsed_time(ev[3]), galerkin=ev[3].elapsed_time(ev[4]))
        levels.append(info)
    return levels
