"""Pins of the CPU oracle against what the paper and the mathematics fix
(not against itself).  CPU only (-m "not gpu").

Each test names the passage it pins (P:n = PAPER.md, S:n = SPEC.md lines).
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

import dense_ref as D
from oracle import Oracle, OracleError, setup_row
from workloads.problems import make_config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# --------------------------------------------------------------------------
# Alg. 2 per row: QR branch, SVD branch, least-norm delta
# --------------------------------------------------------------------------

def test_setup_row_least_norm_S288():
    g = GOLD["least_norm_S288"]
    Q, delta, k, svd = setup_row(np.array(g["M"]), np.array(g["r"]))
    assert k == g["k"] and not svd
    assert np.allclose(delta, g["delta"], atol=1e-15, rtol=0)
    assert np.allclose(np.abs(Q[:, 0]), [2 ** -0.5] * 2, atol=1e-15)


def test_setup_row_qr_S80():
    g = GOLD["qr_S80"]
    Q, delta, k, svd = setup_row(np.array(g["M"]), np.array(g["r"]))
    assert k == 1 and not svd
    assert np.allclose(np.abs(Q[:, 0]), g["Q_abs"], atol=1e-15)
    assert np.allclose(delta, g["delta"], atol=1e-15)


def test_setup_row_rank_deficient_routes_to_svd():
    g = GOLD["rank_deficient_S289"]
    M = np.array(g["M"])
    r = np.array(g["r"])
    Q, delta, k, svd = setup_row(M, r)
    assert svd and k == g["k"]
    # least-squares / least-norm solution of M^T delta = r (library pinv)
    assert np.allclose(delta, np.linalg.pinv(M.T, rcond=1e-10) @ r, atol=1e-13)
    # Q spans range(M)
    U = np.linalg.svd(M, full_matrices=False)[0][:, :1]
    assert np.allclose(Q[:, :1] @ Q[:, :1].T, U @ U.T, atol=1e-13)
    assert np.all(Q[:, 1:] == 0.0)


@pytest.mark.parametrize("nj,nv,seed", [(5, 1, 0), (12, 6, 1), (41, 6, 2), (54, 6, 3), (6, 6, 4)])
def test_setup_row_matches_lstsq_and_projector(nj, nv, seed):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((nj, nv))
    r = rng.standard_normal(nv)
    Q, delta, k, svd = setup_row(M, r)
    assert k == nv and not svd
    # least-norm solution of M^T delta = r
    ref = np.linalg.lstsq(M.T, r, rcond=None)[0]
    assert np.allclose(delta, ref, atol=1e-12 * max(1, np.abs(ref).max()))
    assert np.allclose(M.T @ delta, r, atol=1e-12)
    # Q orthonormal basis of range(M): Q Q^T equals the SVD projector
    assert np.allclose(Q.T @ Q, np.eye(nv), atol=1e-13)
    U = np.linalg.svd(M, full_matrices=False)[0]
    assert np.allclose(Q @ Q.T, U @ U.T, atol=1e-13)


def test_setup_row_skinny_uses_svd():
    # |J| < nv: SVD branch, k = |J|, delta = least-squares solution
    rng = np.random.default_rng(7)
    M = rng.standard_normal((3, 6))
    r = rng.standard_normal(6)
    Q, delta, k, svd = setup_row(M, r)
    assert svd and k == 3
    assert np.allclose(delta, np.linalg.pinv(M.T) @ r, atol=1e-12)


# --------------------------------------------------------------------------
# masked product, projection, energy vs dense definitions
# --------------------------------------------------------------------------

def _integer_problem(seed=0):
    """Tiny SPD-agnostic problem with integer values so that dense and
    sparse sums are exact in fp64 regardless of order."""
    p = make_config("1b", size=8)
    rng = np.random.default_rng(seed)
    p.A_val = rng.integers(-4, 5, p.A_val.size).astype(np.float64)
    rows = np.repeat(np.arange(p.n), np.diff(p.A_rowptr))
    p.A_val[rows == p.A_col] = rng.integers(1, 9, p.n)   # positive diagonal
    return p


def test_masked_product_equals_gather_of_dense_product():
    p = _integer_problem()
    o = Oracle(p)
    A = D.dense_A(p)
    rng = np.random.default_rng(1)
    X = rng.integers(-3, 4, o.nnzW).astype(np.float64)
    r, j = D.w_entries(p)
    PX = D.P_of(p, X)
    # without the C-identity term: A_FF-part only
    PF = PX.copy()
    PF[p.is_coarse == 1] = 0.0
    full = A @ PF
    assert np.array_equal(o.masked_AX(X, with_fc=False), full[r, j])
    # with the C-identity term: (A P)|F-pattern
    assert np.array_equal(o.masked_AX(X, with_fc=True), (A @ PX)[r, j])


def test_masked_product_identity_S71():
    p = make_config("1b", size=8)
    rows = np.repeat(np.arange(p.n), np.diff(p.A_rowptr))
    keep = rows == p.A_col
    p.A_rowptr = np.r_[0, np.cumsum(np.bincount(rows[keep], minlength=p.n))].astype(np.int64)
    p.A_col = p.A_col[keep]
    p.A_val = np.ones(keep.sum())
    o = Oracle(p)
    X = np.random.default_rng(0).standard_normal(o.nnzW)
    assert np.array_equal(o.masked_AX(X), X)


def test_energy_equals_dense_trace():
    p = _integer_problem(3)
    o = Oracle(p)
    W = np.random.default_rng(5).integers(-3, 4, o.nnzW).astype(np.float64)
    assert o.energy_of(W) == D.energy(p, W)


def test_projection_nv1_closed_form_and_idempotent():
    p = make_config("2b", size=6)
    o = Oracle(p)
    wptr, _, _ = o.layout()
    x = np.random.default_rng(2).standard_normal(o.nnzW)
    px = o.project(x)
    # nv = 1, B = 1: Q_i = 1/sqrt|J_i| -> Pi subtracts the row mean
    ref = x.copy()
    for i in range(o.nF):
        s, e = wptr[i], wptr[i + 1]
        ref[s:e] -= x[s:e].mean()
    assert np.allclose(px, ref, atol=1e-15)
    assert np.allclose(o.project(px), px, atol=1e-15)


def test_projection_annihilates_range_and_is_idempotent_elasticity():
    p = make_config("4", size=3)
    o = Oracle(p)
    wptr, wcol, frow = o.layout()
    rng = np.random.default_rng(3)
    x = rng.standard_normal(o.nnzW)
    px = o.project(x)
    assert np.allclose(o.project(px), px, atol=1e-13)
    # B~^T (Pi x) = 0 row by row and Pi(M_i c) = 0
    for i in range(o.nF):
        s, e = wptr[i], wptr[i + 1]
        M = p.Bc[wcol[s:e]]
        assert np.abs(M.T @ px[s:e]).max() <= 1e-12 * np.linalg.norm(x[s:e])
        y = np.zeros(o.nnzW)
        y[s:e] = M @ rng.standard_normal(p.nv)
        assert np.abs(o.project(y)[s:e]).max() <= 1e-12 * np.abs(y).max()


# --------------------------------------------------------------------------
# the whole path against the dense problem statement
# --------------------------------------------------------------------------

SMALL = [("1b", 8), ("2b", 6), ("3", 6), ("4", 2), ("4", 3)]


@pytest.mark.parametrize("name,size", SMALL)
def test_setup_satisfies_constraint_and_r0_is_projected_negative_gradient(name, size):
    p = make_config(name, size=size)
    o = Oracle(p)
    w0 = o.vec("w0")
    Cm, b = D.constraint_matrix(p)
    assert np.abs(Cm @ w0 - b).max() <= 1e-12 * max(1.0, np.abs(b).max())
    # r0 = Pi(f - K w0) = -Pi grad E(w0)/2 with grad from the dense trace (A1, A2)
    H, g, _ = D.quadratic_form(p)
    grad = H @ w0 + g
    r0 = o.vec("r")
    ref = -o.project(grad / 2.0)
    assert np.allclose(r0, ref, atol=1e-12 * np.abs(ref).max())
    # and E0 is the dense trace
    assert abs(o.E0 - D.energy(p, w0)) <= 1e-12 * abs(o.E0)


@pytest.mark.parametrize("name,size", SMALL)
def test_converged_pcg_matches_dense_kkt(name, size):
    p = make_config(name, size=size)
    o = Oracle(p)
    o.iterate(400)
    W = o.get_W()
    w_kkt = D.kkt_solution(p)
    w_ns = D.nullspace_solution(p, o.vec("w0"))
    scale = np.abs(w_kkt).max()
    assert np.abs(W - w_kkt).max() <= 1e-9 * scale
    assert np.abs(W - w_ns).max() <= 1e-9 * scale
    Eref = D.energy(p, w_kkt)
    assert abs(o.energy() - Eref) <= 1e-11 * abs(Eref)


@pytest.mark.parametrize("name,size,k", [("1b", 8, 12), ("3", 6, 20), ("4", 3, 15), ("2b", 6, 15)])
def test_every_iterate_constraint_monotone_telescoping(name, size, k):
    p = make_config(name, size=size)
    o = Oracle(p)
    A = D.dense_A(p)
    Cm, b = D.constraint_matrix(p)
    E_prev = o.E0
    tele = o.E0
    for it in range(k):
        kd, dE = o.iterate(1)
        if kd == 0:
            break
        W = o.get_W()
        E = D.energy(p, W, A)
        assert np.abs(Cm @ W - b).max() <= 1e-12 * max(1.0, np.abs(b).max())
        assert E <= E_prev + 1e-12 * abs(E_prev)            # monotone (Eq. CG_dE)
        tele -= dE[0]
        assert abs(E - tele) <= 1e-10 * abs(o.E0)           # E_k = E_0 - sum dE_j
        assert abs((E_prev - E) - dE[0]) <= 1e-9 * abs(o.E0)
        E_prev = E


def test_1d_closed_form():
    g = GOLD["closed_form_1d"]
    p = make_config("1d", size=g["n"])
    assert p.nc == g["n_C"]
    o = Oracle(p)
    assert o.E0 > g["E_star"] + 1e-3          # least-norm start is not optimal
    o.iterate(200)
    W = o.get_W()
    wptr, wcol, frow = o.layout()
    cid_glob = np.flatnonzero(p.is_coarse)
    for i in range(o.nF):
        for t in range(wptr[i], wptr[i + 1]):
            adjacent = abs(int(cid_glob[wcol[t]]) - int(frow[i])) == 1
            assert abs(W[t] - (0.5 if adjacent else 0.0)) <= 1e-13
    assert abs(o.energy() - g["E_star"]) <= 1e-12 * g["E_star"]


def test_config1_degenerate_and_1b_converges_to_symmetric_P():
    g = GOLD["config1_symmetric_limit"]
    p1 = make_config("1")
    o1 = Oracle(p1)
    W1 = o1.vec("w0")
    assert D.energy(p1, W1) == g["E_star"]
    # degenerate start: first energy decrease is round-off (finding 4)
    o1n = Oracle(p1, stagnation_rel=0.0)
    kd, dE = o1n.iterate(1)
    assert kd == 1 and dE[0] <= 1e-20 * o1n.E0
    # the guard (A18) stops it without any update
    kd, _ = o1.iterate(20)
    assert kd == 0 and o1.stop_reason in ("stagnation", "gamma<=0")
    p1b = make_config("1b")
    o = Oracle(p1b)
    kd, dE = o.iterate(60)
    assert np.abs(o.get_W() - W1).max() <= 1e-10
    assert abs(o.energy() - g["E_star"]) <= 1e-10 * g["E_star"]


def test_theorem1_and_corollary():
    """diag(Z^T K Z) = A(i,i) per row block, Z^T D_K Z diagonal, Z^T D_K Q = 0
    (Theorem 1 / Corollary) on K = H/2 from the dense trace."""
    p = make_config("4", size=2)
    o = Oracle(p)
    H, _, _ = D.quadratic_form(p)
    K = H / 2.0
    Q, krank = o.Q()
    wptr, wcol, frow = o.layout()
    m = o.nnzW
    Zb, Qb = [], []
    for i in range(o.nF):
        s, e = wptr[i], wptr[i + 1]
        Qi = Q[s:e, :krank[i]]
        Zi = sla.null_space(Qi.T)
        Zfull = np.zeros((m, Zi.shape[1]))
        Zfull[s:e] = Zi
        Qfull = np.zeros((m, Qi.shape[1]))
        Qfull[s:e] = Qi
        Zb.append((i, Zfull))
        Qb.append(Qfull)
    Z = np.hstack([z for _, z in Zb])
    Qm = np.hstack(Qb)
    DK = np.diag(np.diag(K))
    dz = np.diag(Z.T @ K @ Z)
    expect = np.concatenate([[p.A_val[p.A_rowptr[frow[i]]:p.A_rowptr[frow[i] + 1]]
                              [p.A_col[p.A_rowptr[frow[i]]:p.A_rowptr[frow[i] + 1]] == frow[i]][0]]
                             * z.shape[1] for i, z in Zb])
    assert np.allclose(dz, expect, rtol=1e-12, atol=0)
    ZDZ = Z.T @ DK @ Z
    assert np.abs(ZDZ - np.diag(np.diag(ZDZ))).max() <= 1e-12 * np.abs(DK).max()
    assert np.abs(Z.T @ DK @ Qm).max() <= 1e-12 * np.abs(DK).max()
    # the oracle's Jacobi diagonal is diag(K) row by row
    d = o.vec("d")
    assert np.allclose(np.repeat(d, np.diff(wptr)), np.diag(K), rtol=0, atol=0)


@pytest.mark.parametrize("name,size", [("4", 3), ("3", 6)])
def test_jacobi_needs_no_post_projection(name, size):
    """P:911-914 / reading A7: with M_J the post-projection changes nothing
    beyond round-off."""
    p = make_config(name, size=size)
    a = Oracle(p, project_z=True)
    b = Oracle(p, project_z=False)
    a.iterate(15)
    b.iterate(15)
    Wa, Wb = a.get_W(), b.get_W()
    assert np.abs(Wa - Wb).max() <= 1e-12 * np.abs(Wa).max()


def test_basis_invariance():
    """P is invariant under B -> B M (A17): same constraint set."""
    p = make_config("4", size=3)
    a = Oracle(p)
    a.iterate(10)
    rng = np.random.default_rng(11)
    Mx = rng.standard_normal((6, 6)) + 3 * np.eye(6)
    p.B = p.B @ Mx
    p.Bc = p.Bc @ Mx
    b = Oracle(p)
    b.iterate(10)
    assert np.abs(a.get_W() - b.get_W()).max() <= 1e-10 * np.abs(a.get_W()).max()


def test_tau_one_runs_exactly_one_update():
    """tau = 1: dE_2 < dE_1 stops at k = 2 without its update (S:334, P:852 + A4)."""
    p = make_config("1b", size=8)
    o = Oracle(p, tau=1.0)
    kd, dE = o.iterate(20)
    assert kd == 1 and o.stop_reason == "tau"


def test_iterate_composes():
    p = make_config("3", size=6)
    a = Oracle(p)
    b = Oracle(p)
    a.iterate(7)
    a.iterate(5)
    b.iterate(12)
    assert np.array_equal(a.get_W(), b.get_W())


def test_reset_restores_start():
    p = make_config("1b", size=8)
    o = Oracle(p)
    _, dE1 = o.iterate(5)
    o.reset()
    _, dE2 = o.iterate(5)
    assert np.array_equal(dE1, dE2)


# --------------------------------------------------------------------------
# input validation (error contract of the ABI)
# --------------------------------------------------------------------------

def test_validation_errors():
    p = make_config("1b", size=8)
    bad = make_config("1b", size=8)
    bad.Bc = bad.Bc.copy()
    bad.Bc[0, 0] = 2.0
    with pytest.raises(OracleError) as e:
        Oracle(bad)
    assert e.value.code == 4
    bad = make_config("1b", size=8)
    c = int(np.flatnonzero(bad.is_coarse)[0])
    bad.P_col = bad.P_col.copy()
    bad.P_col[bad.P_rowptr[c]] = 1
    with pytest.raises(OracleError) as e:
        Oracle(bad)
    assert e.value.code == 3
    bad = make_config("1b", size=8)
    bad.A_val = bad.A_val.copy()
    rows = np.repeat(np.arange(bad.n), np.diff(bad.A_rowptr))
    f = int(np.flatnonzero(bad.is_coarse == 0)[0])
    bad.A_val[(rows == f) & (bad.A_col == f)] = -1.0
    with pytest.raises(OracleError) as e:
        Oracle(bad)
    assert e.value.code == 5
    bad = make_config("1b", size=8)
    bad.A_col = bad.A_col.copy()
    bad.A_col[[0, 1]] = bad.A_col[[1, 0]]
    with pytest.raises(OracleError) as e:
        Oracle(bad)
    assert e.value.code == 2
    Oracle(p)


# --------------------------------------------------------------------------
# Projected SGS preconditioner M_2
# --------------------------------------------------------------------------

def _dense_sgs_prec(prob, key):
    """Pi (L+D)^{-T} D (L+D)^{-1} from the dense K (= H/2 of the dense trace,
    block diagonal over coarse columns), L = the part of K below
    the diagonal when each column block's unknowns are ordered by (key, row)
    (reading A23), Pi = orthogonal projector onto ker(C) (the constraint
    matrix of P B_c = B).  Library solves only."""
    H, _, _ = D.quadratic_form(prob)
    K = H / 2.0
    r, j = D.w_entries(prob)
    kk = np.zeros(prob.n, np.int64) if key is None else np.asarray(key)
    rank = np.lexsort((r, kk[r]))            # position of each unknown in (key, row) order
    pos = np.empty_like(rank)
    pos[rank] = np.arange(rank.size)
    same_col = j[:, None] == j[None, :]
    before = pos[None, :] < pos[:, None]     # unknown f visited before unknown e
    Lm = np.where(same_col & before, K, 0.0)
    Dm = np.diag(np.diag(K))
    Cm, _ = D.constraint_matrix(prob)
    Rc = sla.orth(Cm.T)
    Pi = np.eye(K.shape[0]) - Rc @ Rc.T
    M = np.linalg.solve((Lm + Dm).T, Dm @ np.linalg.solve(Lm + Dm, np.eye(K.shape[0])))
    return Pi @ M


@pytest.mark.parametrize("name,size,kind", [("1b", 8, "natural"), ("1b", 8, "color"), ("3", 5, "natural"),
                                            ("3", 5, "color"), ("4", 2, "natural"), ("4", 2, "color")])
def test_sgs_apply_matches_dense_formula(name, size, kind):
    """P:917-920 / P:933: z = Pi M_SGS^{-1} x, M_SGS^{-1} = (L+D)^{-T} D (L+D)^{-1}."""
    from workloads.problems import sgs_key
    prob = make_config(name, size=size)
    key = sgs_key(prob, kind)
    o = Oracle(prob, precond="sgs", sgs_key=key)
    Md = _dense_sgs_prec(prob, key)
    rng = np.random.default_rng(3)
    for _ in range(3):
        x = rng.standard_normal(o.nnzW)
        z = o.apply_prec(x)
        ref = Md @ x
        assert np.abs(z - ref).max() <= 1e-11 * np.abs(ref).max()


def test_sgs_differs_from_jacobi_and_is_spd_on_range():
    """M_SGS^{-1} is symmetric positive definite (K SPD); restricted to
    range(Z) (Pi x = x) z^T x > 0, and it is not the Jacobi operator."""
    prob = make_config("3", size=5)
    o = Oracle(prob, precond="sgs")
    oj = Oracle(prob, precond="jacobi", project_z=True)
    rng = np.random.default_rng(5)
    for _ in range(4):
        x = o.project(rng.standard_normal(o.nnzW))
        z = o.apply_prec(x)
        assert z @ x > 0
        assert np.abs(z - oj.apply_prec(x)).max() > 1e-3 * np.abs(z).max()
    Md = _dense_sgs_prec(prob, None)
    Cm, _ = D.constraint_matrix(prob)
    Z = sla.null_space(Cm)
    S = Z.T @ Md @ Z
    assert np.allclose(S, S.T, atol=1e-12 * np.abs(S).max())
    assert np.linalg.eigvalsh((S + S.T) / 2).min() > 0


def test_sgs_reduces_to_jacobi_when_A_FF_is_diagonal():
    """1D Laplacian, C = even points: F points couple only to C points, so
    K's blocks are diagonal, L = 0 and M_SGS = D (= Jacobi M_1)."""
    prob = make_config("1d", size=33)
    oj = Oracle(prob, precond="jacobi", project_z=True, stagnation_rel=0.0)
    os_ = Oracle(prob, precond="sgs", stagnation_rel=0.0)
    kj, dEj = oj.iterate(10)
    ks, dEs = os_.iterate(10)
    assert kj == ks
    assert np.allclose(dEj, dEs, rtol=1e-12, atol=0)
    assert np.abs(oj.get_W() - os_.get_W()).max() <= 1e-13


@pytest.mark.parametrize("name,size,kind", [("1b", 10, "natural"), ("3", 6, "color"), ("4", 2, "color")])
def test_sgs_pcg_converges_to_kkt_monotone_constrained(name, size, kind):
    """Same constrained minimiser as the dense KKT solve --
    the preconditioner changes the path, not the solution; energy monotone
    and telescoping and P B_c = B at every iterate."""
    from workloads.problems import sgs_key
    prob = make_config(name, size=size)
    o = Oracle(prob, precond="sgs", sgs_key=sgs_key(prob, kind), stagnation_rel=1e-28)
    Cm, b = D.constraint_matrix(prob)
    E_prev = o.E0
    tel = o.E0
    for _ in range(200):
        k, dE = o.iterate(1)
        if k == 0:
            break
        w = o.get_W()
        E = D.energy(prob, w)
        assert E <= E_prev + 1e-12 * abs(E_prev)
        tel -= dE[0]
        assert abs(E - tel) <= 1e-10 * abs(o.E0)
        assert np.abs(Cm @ w - b).max() <= 1e-12
        E_prev = E
    w_kkt = D.kkt_solution(prob)
    assert np.abs(o.get_W() - w_kkt).max() <= 1e-8 * np.abs(w_kkt).max()


@pytest.mark.parametrize("name,size", [("3", 8), ("4", 3), ("1b", 16)])
def test_sgs_reduces_energy_faster_than_jacobi(name, size):
    """with SGS the energy drops 'more than twice as fast' as
    with Jacobi per iteration -- after 4 steps the remaining decrease
    dE_4 / dE_1 is smaller."""
    prob = make_config(name, size=size)
    oj = Oracle(prob, precond="jacobi", project_z=True, stagnation_rel=0.0)
    os_ = Oracle(prob, precond="sgs", stagnation_rel=0.0)
    _, dEj = oj.iterate(4)
    _, dEs = os_.iterate(4)
    assert oj.E0 - dEs.sum() < oj.E0 - dEj.sum() + 1e-12 * abs(oj.E0)
    assert dEs[3] / dEs[0] < 0.5 * dEj[3] / dEj[0]


# --------------------------------------------------------------------------
# Alg. 1 tentative start: max-vol selection (NEXT-3, reading A24)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("m,nv,seed", [(12, 6, 0), (41, 6, 1), (54, 6, 2), (7, 3, 3), (9, 1, 4), (6, 6, 5)])
def test_maxvol_selection_is_dominant(m, nv, seed):
    """[Gor08]: S is a dominant (locally maximum-volume) submatrix iff every
    entry of M M(S,:)^{-1} is at most 1 in modulus -- checked with numpy,
    and no single row swap increases |det M(S,:)|."""
    from oracle import maxvol
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((m, nv))
    S = maxvol(M)
    assert S is not None and len(set(S.tolist())) == nv
    C = np.linalg.solve(M[S].T, M.T).T
    assert np.abs(C).max() <= 1 + 1e-8
    v0 = abs(np.linalg.det(M[S]))
    for t in range(m):
        for c in range(nv):
            S2 = S.copy()
            S2[c] = t
            assert abs(np.linalg.det(M[S2])) <= v0 * (1 + 1e-8)


def test_maxvol_small_brute_force_ratio():
    """A dominant submatrix of an m x nv matrix has volume >= max volume /
    nv^(nv/2) (Goreinov-Tyrtyshnikov); here checked by brute force."""
    import itertools
    from oracle import maxvol
    rng = np.random.default_rng(7)
    for _ in range(5):
        M = rng.standard_normal((8, 3))
        S = maxvol(M)
        best = max(abs(np.linalg.det(M[list(c)])) for c in itertools.combinations(range(8), 3))
        assert abs(np.linalg.det(M[S])) >= best / 3 ** 1.5 - 1e-12


def test_maxvol_rank_deficient_returns_none():
    from oracle import maxvol
    M = np.ones((5, 2))
    assert maxvol(M) is None


@pytest.mark.parametrize("name,size", [("1b", 8), ("3", 6), ("4", 2)])
def test_maxvol_start_is_sparse_and_exact(name, size):
    """The Alg. 1 start satisfies each local constraint exactly (P:527-540:
    ||v - B w|| = 0) with at most nv nonzeros per row, so Alg. 2's correction
    delta vanishes and W0 is the tentative start itself."""
    prob = make_config(name, size=size)
    o = Oracle(prob, start="maxvol")
    assert o.n_maxvol_fail == 0
    w0 = o.vec("w0")
    wptr, wcol, frow = o.layout()
    Cm, b = D.constraint_matrix(prob)
    assert np.abs(Cm @ w0 - b).max() <= 1e-13 * max(1.0, np.abs(b).max())
    for i in range(len(wptr) - 1):
        row = w0[wptr[i]:wptr[i + 1]]
        assert np.count_nonzero(np.abs(row) > 1e-13 * np.abs(row).max()) <= prob.nv


def test_maxvol_start_scalar_B1_is_injection_from_first_column():
    """nv = 1, B = 1: all |V_c| equal, the tie goes to the first column of
    J_i, so the start injects from it: w = 1 there, 0 elsewhere."""
    prob = make_config("1b", size=8)
    o = Oracle(prob, start="maxvol")
    w0 = o.vec("w0")
    wptr, _, _ = o.layout()
    for i in range(len(wptr) - 1):
        row = w0[wptr[i]:wptr[i + 1]]
        assert abs(row[0] - 1.0) <= 1e-15 and np.all(np.abs(row[1:]) <= 1e-15)


@pytest.mark.parametrize("name,size", [("1b", 10), ("4", 2)])
def test_maxvol_start_converges_to_kkt(name, size):
    """The minimiser does not depend on the start."""
    prob = make_config(name, size=size)
    o = Oracle(prob, start="maxvol", stagnation_rel=1e-28)
    o.iterate(400)
    w = D.kkt_solution(prob)
    assert np.abs(o.get_W() - w).max() <= 1e-8 * np.abs(w).max()


# --------------------------------------------------------------------------
# Alg. 1 pattern growth from the graph of A (reading A25)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("name,size", [("1b", None), ("2", 10), ("2b", 12), ("3", 12), ("3", 17),
                                       ("4", 3), ("4", 6), ("5", 8), ("1v3", 16), ("1v3", 11)])
def test_pattern_from_graph_matches_generator(name, size):
    """The oracle's BFS over the graph of A reproduces, bit for bit, the input
    generator's pattern -- built independently from grid-box arithmetic
    (Manhattan balls for the 5/7-point stencils, Chebyshev balls of the
    27-point node graph, per-row growth until full rank)."""
    from oracle import pattern
    prob = make_config(name, size=size)
    rp, col, hist = pattern(prob)
    assert np.array_equal(rp, prob.P_rowptr) and np.array_equal(col, prob.P_col)
    nodes = prob.n_F // prob.block_size
    assert hist.sum() == nodes
    assert {l: int(c) for l, c in enumerate(hist) if c} == {int(k): int(v) for k, v in prob.meta["growth"].items()}


def test_gram_full_rank_matches_numpy():
    """The oracle's rank test of Alg. 1's growth loop (reading A25,
    lambda_min(M^T M) > 1e-10 lambda_max) by cyclic Jacobi with the
    trace-relative stopping rule of reading A27 decides as numpy's
    eigvalsh, also for conditions within 1e-4 (relative) of the threshold."""
    from oracle import gram_full_rank
    rng = np.random.default_rng(11)
    conds = [1e0, 1e3, 1e8, 1e12, 1e20] + list(np.geomspace(1e9, 1e11, 41)) + [1e10 * (1 + 1e-4), 1e10 * (1 - 1e-4)]
    for nv in (1, 3, 6):
        for cond in conds:
            U = np.linalg.qr(rng.standard_normal((nv, nv)))[0]
            ev = np.geomspace(1.0, 1.0 / cond, nv)
            G = (U * ev) @ U.T
            ref = np.linalg.eigvalsh(G)
            if nv > 1 and abs(np.log10(ref[0] / ref[-1]) + 10.0) < 1e-9:
                continue                      # exactly at the threshold: either answer
            assert gram_full_rank(G) == bool(ref[0] > 1e-10 * max(ref[-1], 0.0)), (nv, cond)


@pytest.mark.parametrize("precond,start", [("jacobi", "given"), ("sgs", "given"), ("jacobi", "maxvol")])
def test_linear_modes_nv3_converges_to_kkt(precond, start):
    """A scalar operator with the 3-mode near kernel {1, x, y} (nv = 3, point
    rows, pattern grown until rank 3): the converged CG equals the dense KKT
    solution for both preconditioners and both starts, and the
    constraint holds to 1e-12."""
    prob = make_config("1v3", size=8)
    o = Oracle(prob, precond=precond, start=start, project_z=True, stagnation_rel=1e-28)
    o.iterate(500)
    w = D.kkt_solution(prob)
    assert np.abs(o.get_W() - w).max() <= 1e-8 * np.abs(w).max()
    Cm, b = D.constraint_matrix(prob)
    assert np.abs(Cm @ o.get_W() - b).max() <= 1e-12 * max(1.0, np.abs(b).max())


# --------------------------------------------------------------------------
# Galerkin coarse operator A_c = P^T A P (reading A26;
# Eq. trace, coarse grid construction P:957-961)
# --------------------------------------------------------------------------

def _linear_interp_1d(prob):
    """1D linear interpolation on prob's (wider) pattern: W(i, c) = 1/2 for
    the two C neighbours of F point i, 0 on the other pattern entries."""
    P = np.zeros(prob.P_rowptr[-1])
    for i in range(prob.n):
        for q in range(prob.P_rowptr[i], prob.P_rowptr[i + 1]):
            c = prob.P_col[q]
            if prob.is_coarse[i]:
                P[q] = 1.0
            elif abs(2 * c - i) == 1:
                P[q] = 0.5
    return P


def test_galerkin_1d_linear_interpolation_closed_form():
    # textbook: P^T tridiag(-1, 2, -1) P with linear interpolation =
    # (1/2) tridiag(-1, 2, -1) on the coarse grid; at the Dirichlet ends
    # A_c(0, 0) = A00 + A01 + A11 / 4 = 3/2.  Exact in binary.
    from oracle import galerkin
    p = make_config("1d", 17)
    Pv = _linear_interp_1d(p)
    rp, col, val = galerkin(p.n, p.nc, p.A_rowptr, p.A_col, p.A_val, p.P_rowptr, p.P_col, Pv)
    Ac = np.zeros((p.nc, p.nc))
    for c in range(p.nc):
        assert np.all(np.diff(col[rp[c]:rp[c + 1]]) > 0)
        Ac[c, col[rp[c]:rp[c + 1]]] = val[rp[c]:rp[c + 1]]
    want = np.diag(np.full(p.nc, 1.0)) - 0.5 * (np.eye(p.nc, k=1) + np.eye(p.nc, k=-1))
    want[0, 0] = want[-1, -1] = 1.5
    assert np.array_equal(Ac, want)
    # structural pattern: distance-3 pattern of P, A tridiagonal -> |c - c'| <= 3
    # wherever a product chain exists (checked against boolean matrix products)
    Pb = np.zeros((p.n, p.nc), np.int64)
    for i in range(p.n):
        Pb[i, p.P_col[p.P_rowptr[i]:p.P_rowptr[i + 1]]] = 1
    Ab = (np.abs(np.eye(p.n, k=1)) + np.eye(p.n) + np.eye(p.n, k=-1)).astype(np.int64)
    S = (Pb.T @ Ab @ Pb) > 0
    got = np.zeros_like(S)
    for c in range(p.nc):
        got[c, col[rp[c]:rp[c + 1]]] = True
    assert np.array_equal(got, S)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_galerkin_matches_dense_product(seed):
    from oracle import galerkin
    rng = np.random.default_rng(seed)
    n, nc = 70, 17
    M = (rng.random((n, n)) < 0.08) * rng.standard_normal((n, n))
    A = M + M.T + np.diag(rng.random(n) + 1.0)
    Pd = (rng.random((n, nc)) < 0.2) * rng.standard_normal((n, nc))
    Pd[rng.integers(0, n, 5), :] = 0.0                       # a few empty rows of P
    def csr(D):
        rp = np.zeros(D.shape[0] + 1, np.int64)
        cols, vals = [], []
        for i in range(D.shape[0]):
            nz = np.flatnonzero(D[i])
            cols.append(nz); vals.append(D[i, nz]); rp[i + 1] = rp[i] + nz.size
        return rp, np.concatenate(cols).astype(np.int32), np.concatenate(vals)
    Arp, Acol, Aval = csr(A)
    Prp, Pcol, Pval = csr(Pd)
    rp, col, val = galerkin(n, nc, Arp, Acol, Aval, Prp, Pcol, Pval)
    Ac = np.zeros((nc, nc))
    got = np.zeros((nc, nc), bool)
    for c in range(nc):
        Ac[c, col[rp[c]:rp[c + 1]]] = val[rp[c]:rp[c + 1]]
        got[c, col[rp[c]:rp[c + 1]]] = True
    dense = Pd.T @ A @ Pd
    assert np.allclose(Ac, dense, rtol=0, atol=1e-13 * np.abs(dense).max())
    S = ((Pd != 0).astype(np.int64).T @ (A != 0).astype(np.int64) @ (Pd != 0).astype(np.int64)) > 0
    assert np.array_equal(got, S)


@pytest.mark.parametrize("name,size", [("3", 12), ("4", 4), ("1v3", 10)])
def test_galerkin_trace_is_energy_symmetric_and_keeps_near_kernel(name, size):
    # tr(P^T A P) is the energy (Eq. trace) computed by the
    # oracle's own energy routine; A_c symmetric; and because every iterate
    # keeps P B_c = B, A_c B_c = P^T A P B_c = P^T (A B)
    import scipy.sparse as sp
    from oracle import galerkin
    p = make_config(name, size)
    o = Oracle(p)
    o.iterate(6)
    Pv = o.get_P()
    rp, col, val = galerkin(p.n, p.nc, p.A_rowptr, p.A_col, p.A_val, p.P_rowptr, p.P_col, Pv)
    Ac = sp.csr_matrix((val, col, rp), shape=(p.nc, p.nc))
    assert abs(Ac.diagonal().sum() - o.energy()) <= 1e-12 * abs(o.energy())
    d = (Ac - Ac.T).tocoo()
    assert np.abs(d.data).max(initial=0.0) <= 1e-13 * np.abs(val).max()
    assert (Ac != 0).sum() <= Ac.nnz and np.array_equal(np.sort(Ac.indices), np.sort(Ac.T.tocsr().indices))
    A = sp.csr_matrix((p.A_val, p.A_col, p.A_rowptr), shape=(p.n, p.n))
    P = sp.csr_matrix((Pv, p.P_col, p.P_rowptr), shape=(p.n, p.nc))
    lhs = Ac @ p.Bc
    rhs = P.T @ (A @ p.B)
    assert np.abs(lhs - rhs).max() <= 1e-10 * max(np.abs(rhs).max(), np.abs(lhs).max(), 1.0)


@pytest.mark.parametrize("name,size,k", [("1b", None, 20), ("2b", 8, 30), ("3", 10, 40), ("4", 3, 30),
                                         ("5", 6, 10)])
def test_threaded_oracle_equals_serial_order(name, size, k):
    """The OpenMP loops of the oracle (per-row projection, masked product,
    Alg. 2, Jacobi scaling, vector updates, per-entry energy terms) leave
    every global sum serial in its order, so 1 thread and all threads give
    the same bits: E0, dE_k, E and P."""
    import oracle
    from oracle import Oracle
    from workloads.problems import make_config
    prob = make_config(name, size=size)
    out = []
    orig = oracle.max_threads()
    try:
        for nt in (1, max(2, orig)):
            oracle.set_threads(nt)
            o = Oracle(prob, project_z=True)
            kd, dE = o.iterate(k)
            out.append((o.E0, kd, dE, o.energy(), o.get_P(), o.n_svd, o.n_frozen))
    finally:
        oracle.set_threads(orig)
    a, b = out
    assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2]) and a[3] == b[3]
    assert np.array_equal(a[4], b[4]) and a[5:] == b[5:]


@pytest.mark.parametrize("name,size,k", [("1b", 8, 10), ("3", 6, 10), ("4", 2, 10), ("1v3", 6, 10), ("2b", 6, 10)])
def test_cg_trajectory_step_by_step_matches_dense_pcg(name, size, k):
    """Step-by-step pin of Alg. 3's recurrence (beta = gamma / gamma_old,
    the updates of w and r, dE_k = gamma alpha): the oracle's dE_k and W_k
    after every step k <= 10 equal a dense projected PCG written from the
    quadratic form with the dense orthogonal projector onto ker C
    (tests/dense_ref.py), not from the oracle's per-row Q_i."""
    prob = make_config(name, size=size)
    o = Oracle(prob, project_z=True, stagnation_rel=0.0)
    w0 = o.get_W()
    ref = D.dense_projected_pcg(prob, w0, k)
    assert len(ref) == k
    for step, (dE_ref, w_ref) in enumerate(ref, start=1):
        kd, dE = o.iterate(1)
        assert kd == 1
        assert abs(dE[0] - dE_ref) <= 1e-9 * abs(ref[0][0]), (step, dE[0], dE_ref)
        assert np.abs(o.get_W() - w_ref).max() <= 1e-9 * np.abs(w_ref).max(), step
