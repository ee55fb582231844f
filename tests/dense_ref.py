"""Dense, from-the-definition references used to PIN the oracle.

Nothing here re-types the oracle's formulas: every quantity is derived from
the problem statement of the paper itself,

  minimise   E(P) = tr(P^T A P)            (Eq. trace)
  subject to P B_c = B,  P = [W; I]        (Eq. inKern/TSP)
  with W on the fixed pattern

by building the dense linear map  w -> vec(P(w))  and differentiating the
dense trace.  numpy/scipy library routines (solve, lstsq, svd, null_space)
serve as steps.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def dense_A(prob):
    A = np.zeros((prob.n, prob.n))
    rows = np.repeat(np.arange(prob.n), np.diff(prob.A_rowptr))
    A[rows, prob.A_col] = prob.A_val
    return A


def w_entries(prob):
    """(row, coarse col) of every F-pattern entry in W-layout order."""
    f = prob.fine_rows
    rows, cols = [], []
    for r in f:
        s, e = prob.P_rowptr[r], prob.P_rowptr[r + 1]
        rows.extend([r] * (e - s))
        cols.extend(prob.P_col[s:e].tolist())
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)


def P_of(prob, w):
    """Dense P = [W; I] (in global row order) for W-layout values w."""
    P = np.zeros((prob.n, prob.nc))
    c = np.flatnonzero(prob.is_coarse)
    P[c, np.arange(c.size)] = 1.0
    r, j = w_entries(prob)
    P[r, j] = w
    return P


def energy(prob, w, A=None):
    A = dense_A(prob) if A is None else A
    P = P_of(prob, w)
    return float(np.trace(P.T @ A @ P))


def quadratic_form(prob, A=None):
    """E(w) = w^T H w / 2 + g^T w + e0, derived from the dense trace:
    vec(P) = Phi w + c0  =>  H = 2 Phi^T (I (x) A) Phi,  g = 2 Phi^T (I (x) A) c0."""
    A = dense_A(prob) if A is None else A
    r, j = w_entries(prob)
    m = r.size
    # (I (x) A) applied column-block-wise: column j of P lives in block j
    # Phi e_e = unit at (r_e, j_e).  H_ef = 2 * [j_e == j_f] * A[r_e, r_f]
    # computed as 2 * (Phi^T (I (x) A) Phi) without forming the kron:
    PhiT_APhi = np.zeros((m, m))
    c0 = P_of(prob, np.zeros(m))
    AC0 = A @ c0
    for col in np.unique(j):
        idx = np.flatnonzero(j == col)
        PhiT_APhi[np.ix_(idx, idx)] = A[np.ix_(r[idx], r[idx])]
    H = 2.0 * PhiT_APhi
    g = 2.0 * AC0[r, j]
    e0 = float(np.trace(c0.T @ A @ c0))
    return H, g, e0


def constraint_matrix(prob):
    """C w = b  <=>  (P(w) B_c - B)|_F = 0  (linear in w)."""
    r, j = w_entries(prob)
    f = prob.fine_rows
    fpos = {int(x): t for t, x in enumerate(f)}
    nv = prob.nv
    Cm = np.zeros((f.size * nv, r.size))
    for e in range(r.size):
        for mm in range(nv):
            Cm[fpos[int(r[e])] * nv + mm, e] = prob.Bc[j[e], mm]
    b = prob.B[f].reshape(-1)
    return Cm, b


def kkt_solution(prob):
    """Solve [H C^T; C 0][w; mu] = [-g; b] (saddle point system, Eq. sadsys
    P:355-370) densely."""
    H, g, _ = quadratic_form(prob)
    Cm, b = constraint_matrix(prob)
    # symmetric diagonal equilibration w = S v (exact change of variables;
    # keeps high-contrast operators solvable to ~1e-12)
    s = 1.0 / np.sqrt(np.diag(H))
    Hs = H * s[:, None] * s[None, :]
    Cs = Cm * s[None, :]
    m, q = H.shape[0], Cm.shape[0]
    K = np.zeros((m + q, m + q))
    K[:m, :m] = Hs
    K[:m, m:] = Cs.T
    K[m:, :m] = Cs
    rhs = np.concatenate([-g * s, b])
    sol = np.linalg.solve(K, rhs)
    return sol[:m] * s


def nullspace_solution(prob, w0):
    """Null-space method: w = w0 + Z u, (Z^T H Z) u = -Z^T (H w0 + g)."""
    H, g, _ = quadratic_form(prob)
    Cm, _ = constraint_matrix(prob)
    s = 1.0 / np.sqrt(np.diag(H))
    Z = s[:, None] * sla.null_space(Cm * s[None, :])   # basis of ker(C), scaled
    u = np.linalg.solve(Z.T @ H @ Z, -Z.T @ (H @ w0 + g))
    return w0 + Z @ u


def dense_projected_pcg(prob, w0, k):
    """Alg. 3 written densely from the quadratic form alone, as
    a step-by-step reference for the oracle's recurrence.  With
    E(w) = w^T H w / 2 + g^T w + e0 the paper's K = H / 2 and f = -g / 2
    (E = w^T K w - 2 f^T w + e0); Pi = I - C^T (C C^T)^+ C is the orthogonal
    projector onto ker C built from the dense constraint matrix (not from
    per-row bases); M = diag(K) (Jacobi).  Returns the list of
    (dE_k, w_k) for k = 1..steps taken (stops, like Alg. 3, when gamma or
    y^T yb is not positive)."""
    H, g, _ = quadratic_form(prob)
    K = H / 2.0
    f = -g / 2.0
    Cm, _ = constraint_matrix(prob)
    Pi = np.eye(K.shape[0]) - Cm.T @ np.linalg.pinv(Cm @ Cm.T) @ Cm
    dK = np.diag(K)
    w = w0.copy()
    r = Pi @ (f - K @ w)                                   # P:838 (readings A1, A2)
    y = None
    gamma_old = None
    out = []
    for it in range(k):
        z = Pi @ (r / dK)
        gamma = float(r @ z)
        if not gamma > 0.0:
            break
        y = z.copy() if it == 0 else z + (gamma / gamma_old) * y
        gamma_old = gamma
        yb = Pi @ (K @ y)
        den = float(y @ yb)
        if not den > 0.0:
            break
        alpha = gamma / den
        w = w + alpha * y
        r = r - alpha * yb
        out.append((gamma * alpha, w.copy()))              # dE_k = gamma alpha
    return out
