"""CPU oracle for the restricted-PCG energy minimisation (arXiv 2208.02995).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2208_02995_b200``) never imports it, and
this package never imports the product path: the two share no code.

The arithmetic lives in ``emin_oracle.c`` (plain C, fp64; OpenMP threads only
on loops whose iterations are independent, every global sum serial);
this file is ctypes marshalling only.  See the C file's header for the
paper passages each step follows and DESIGN.md §3 for the readings of the
garbled passages.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "emin_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

STOP_REASONS = {0: "running", 1: "gamma<=0", 2: "y'Ky==0", 3: "tau", 4: "stagnation"}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no -ffast-math, IEEE fp64)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-fopenmp",
                               "-ffp-contract=off", "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, i32, dbl = C.c_int64, C.c_int, C.c_double
        lib.oracle_create.argtypes = [C.POINTER(P), i64, i64, P, P, P, P, P, P, P, i32, P, P,
                                      dbl, dbl, dbl, i32, i32, P, i32]
        lib.oracle_create.restype = i32
        lib.oracle_iterate.argtypes = [P, i32, C.POINTER(i32), P]
        lib.oracle_iterate.restype = i32
        for name, rt in [("oracle_nF", i64), ("oracle_nnzW", i64), ("oracle_E0", dbl),
                         ("oracle_dE1", dbl), ("oracle_k_total", i64), ("oracle_stopped", i32),
                         ("oracle_n_svd", i64), ("oracle_n_frozen", i64),
                         ("oracle_sum_diag_cc", dbl), ("oracle_energy", dbl),
                         ("oracle_n_maxvol_fail", i64)]:
            getattr(lib, name).argtypes = [P]
            getattr(lib, name).restype = rt
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_set_threads.restype = None
        lib.oracle_max_threads.argtypes = []
        lib.oracle_max_threads.restype = i32
        lib.oracle_energy_of.argtypes = [P, P]
        lib.oracle_energy_of.restype = dbl
        lib.oracle_destroy.argtypes = [P]
        lib.oracle_reset.argtypes = [P]
        lib.oracle_get_W.argtypes = [P, P]
        lib.oracle_get_P.argtypes = [P, P]
        lib.oracle_copy_layout.argtypes = [P, P, P, P]
        lib.oracle_copy_vec.argtypes = [P, i32, P]
        lib.oracle_copy_Q.argtypes = [P, P, P]
        lib.oracle_project.argtypes = [P, P, P]
        lib.oracle_apply_prec.argtypes = [P, P, P]
        lib.oracle_masked_AX.argtypes = [P, P, i32, P]
        lib.oracle_setup_row.argtypes = [i32, i32, P, P, dbl, P, P, C.POINTER(i32)]
        lib.oracle_setup_row.restype = i32
        lib.oracle_maxvol.argtypes = [i32, i32, P, P]
        lib.oracle_maxvol.restype = i32
        lib.oracle_pattern.argtypes = [i64, P, P, P, i32, i32, P, i32, i32, P, P, P]
        lib.oracle_pattern.restype = i64
        lib.oracle_gram_full_rank.argtypes = [i32, P]
        lib.oracle_gram_full_rank.restype = i32
        lib.oracle_galerkin.argtypes = [i64, i64, P, P, P, P, P, P, P, P, P]
        lib.oracle_galerkin.restype = i64
        _lib = lib
    return _lib


def set_threads(n: int) -> None:
    """Threads of the oracle's parallel loops (1 = everything serial)."""
    _load().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"oracle {where} failed with status {code}")
        self.code = code


class Oracle:
    """Oracle state for one problem (see workloads.problems.Problem)."""

    def __init__(self, prob, rank_tol=1e-10, tau=0.0, stagnation_rel=1e-30, project_z=True,
                 P_val="from_problem", precond="jacobi", sgs_key=None, start="given"):
        """precond: "jacobi" (M_1) or "sgs" (projected SGS M_2,
        P:916-938); sgs_key (per global row, optional): SGS visits the rows
        of each K block in ascending (key, row) order (reading A23).
        start: "given" (P_val, or the least-norm start if None) or "maxvol"
        (Alg. 1's tentative start on the prescribed pattern, reading A24)."""
        lib = _load()
        self._keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a
        Pv = prob.P_val if isinstance(P_val, str) else P_val
        h = C.c_void_p()
        st = lib.oracle_create(C.byref(h), prob.n, prob.nc,
                               _p(arr(prob.A_rowptr, np.int64)), _p(arr(prob.A_col, np.int32)),
                               _p(arr(prob.A_val, np.float64)), _p(arr(prob.is_coarse, np.uint8)),
                               _p(arr(prob.P_rowptr, np.int64)), _p(arr(prob.P_col, np.int32)),
                               _p(None if Pv is None else arr(Pv, np.float64)),
                               prob.nv, _p(arr(prob.B, np.float64)), _p(arr(prob.Bc, np.float64)),
                               rank_tol, tau, stagnation_rel, 1 if project_z else 0,
                               {"jacobi": 0, "sgs": 1}[precond],
                               _p(None if sgs_key is None else arr(sgs_key, np.int64)),
                               {"given": 0, "maxvol": 1}[start])
        self._keep = []
        if st != 0:
            raise OracleError(st, "create")
        self._h = h
        self._lib = lib
        self.nv = prob.nv
        self.nF = lib.oracle_nF(h)
        self.nnzW = lib.oracle_nnzW(h)
        self.nnzP = int(prob.P_rowptr[-1])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.oracle_destroy(h)
            self._h = None

    # -- Alg. 3 -----------------------------------------------------------
    def iterate(self, k):
        dE = np.zeros(max(k, 1))
        kd = C.c_int(0)
        st = self._lib.oracle_iterate(self._h, k, C.byref(kd), _p(dE))
        if st != 0:
            raise OracleError(st, "iterate")
        return kd.value, dE[:kd.value].copy()

    def reset(self):
        self._lib.oracle_reset(self._h)

    # -- results -----------------------------------------------------------
    @property
    def E0(self):
        return self._lib.oracle_E0(self._h)

    @property
    def dE1(self):
        return self._lib.oracle_dE1(self._h)

    @property
    def k_total(self):
        return self._lib.oracle_k_total(self._h)

    @property
    def stop_reason(self):
        return STOP_REASONS[self._lib.oracle_stopped(self._h)]

    @property
    def n_svd(self):
        return self._lib.oracle_n_svd(self._h)

    @property
    def n_frozen(self):
        return self._lib.oracle_n_frozen(self._h)

    @property
    def n_maxvol_fail(self):
        return self._lib.oracle_n_maxvol_fail(self._h)

    def energy(self):
        return self._lib.oracle_energy(self._h)

    def energy_of(self, W):
        W = np.ascontiguousarray(W, dtype=np.float64)
        return self._lib.oracle_energy_of(self._h, _p(W))

    def get_W(self):
        out = np.empty(self.nnzW)
        self._lib.oracle_get_W(self._h, _p(out))
        return out

    def get_P(self):
        out = np.empty(self.nnzP)
        self._lib.oracle_get_P(self._h, _p(out))
        return out

    def layout(self):
        wptr = np.empty(self.nF + 1, np.int64)
        wcol = np.empty(self.nnzW, np.int32)
        frow = np.empty(self.nF, np.int64)
        self._lib.oracle_copy_layout(self._h, _p(wptr), _p(wcol), _p(frow))
        return wptr, wcol, frow

    def vec(self, name):
        which = {"w0": 0, "dw": 1, "r": 2, "y": 3, "yb": 4, "d": 5}[name]
        out = np.empty(self.nF if which == 5 else self.nnzW)
        self._lib.oracle_copy_vec(self._h, which, _p(out))
        return out

    def Q(self):
        Q = np.empty((self.nnzW, self.nv))
        k = np.empty(self.nF, np.int32)
        self._lib.oracle_copy_Q(self._h, _p(Q), _p(k))
        return Q, k

    # -- the pieces --------------------------------------------------------
    def project(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._lib.oracle_project(self._h, _p(x), _p(out))
        return out

    def apply_prec(self, x):
        """z = Pi M^{-1} x with the oracle's preconditioner (Alg. 3 line P:840)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._lib.oracle_apply_prec(self._h, _p(x), _p(out))
        return out

    def masked_AX(self, X, with_fc=False):
        X = np.ascontiguousarray(X, dtype=np.float64)
        out = np.empty_like(X)
        self._lib.oracle_masked_AX(self._h, _p(X), 1 if with_fc else 0, _p(out))
        return out


def maxvol(M):
    """Max-vol selection of nv rows of the tall M (m x nv) as the oracle's
    Alg. 1 start does it (reading A24).  Returns the row indices (or None if
    no nonsingular selection exists)."""
    lib = _load()
    M = np.asarray(M, dtype=np.float64)
    m, nv = M.shape
    Mc = np.ascontiguousarray(M.T)            # column-major m x nv
    S = np.zeros(nv, np.int32)
    ok = lib.oracle_maxvol(m, nv, _p(Mc), _p(S))
    return S.copy() if ok else None


def pattern(prob, l0=2, lmax=4):
    """Alg. 1's pattern growth from the graph of A (reading A25): returns
    (P_rowptr, P_col, hist) for all rows of prob (C rows identity)."""
    lib = _load()
    n = prob.n
    rp = np.zeros(n + 1, np.int64)
    hist = np.zeros(lmax + 1, np.int64)
    args = [np.ascontiguousarray(prob.A_rowptr, np.int64), np.ascontiguousarray(prob.A_col, np.int32),
            np.ascontiguousarray(prob.is_coarse, np.uint8)]
    Bc = np.ascontiguousarray(prob.Bc, np.float64)
    nnz = lib.oracle_pattern(n, _p(args[0]), _p(args[1]), _p(args[2]), prob.block_size, prob.nv, _p(Bc),
                             l0, lmax, _p(rp), None, None)
    col = np.zeros(max(nnz, 1), np.int32)
    lib.oracle_pattern(n, _p(args[0]), _p(args[1]), _p(args[2]), prob.block_size, prob.nv, _p(Bc),
                       l0, lmax, _p(rp), _p(col), _p(hist))
    return rp, col[:nnz], hist


def galerkin(n, nc, A_rowptr, A_col, A_val, P_rowptr, P_col, P_val):
    """A_c = P^T A P (reading A26, NEXT-4): returns (rowptr, col, val) of the
    nc x nc coarse operator, columns ascending, structural pattern."""
    lib = _load()
    a = [np.ascontiguousarray(A_rowptr, np.int64), np.ascontiguousarray(A_col, np.int32),
         np.ascontiguousarray(A_val, np.float64), np.ascontiguousarray(P_rowptr, np.int64),
         np.ascontiguousarray(P_col, np.int32), np.ascontiguousarray(P_val, np.float64)]
    rp = np.zeros(nc + 1, np.int64)
    nnz = lib.oracle_galerkin(n, nc, *[_p(x) for x in a], _p(rp), None, None)
    col = np.zeros(max(nnz, 1), np.int32)
    val = np.zeros(max(nnz, 1), np.float64)
    lib.oracle_galerkin(n, nc, *[_p(x) for x in a], _p(rp), _p(col), _p(val))
    return rp, col[:nnz], val[:nnz]


def gram_full_rank(G):
    G = np.ascontiguousarray(G, np.float64)
    return bool(_load().oracle_gram_full_rank(G.shape[0], _p(G)))


def setup_row(M, r, tol=1e-10):
    """Alg. 2 on one row: M = B_c(J,:) (nj x nv), r = v - M^T w^.
    Returns (Q [nj, nv] zero-padded, delta [nj], k, used_svd)."""
    lib = _load()
    M = np.asarray(M, dtype=np.float64)
    nj, nv = M.shape
    Mc = np.ascontiguousarray(M.T)            # column-major nj x nv
    rv = np.ascontiguousarray(r, dtype=np.float64)
    Q = np.zeros((nj, nv))
    delta = np.zeros(nj)
    used = C.c_int(0)
    k = lib.oracle_setup_row(nj, nv, _p(Mc), _p(rv), tol, _p(Q), _p(delta), C.byref(used))
    return Q, delta, k, bool(used.value)
