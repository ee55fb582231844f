"""Input generators: sizes of SURVEY §8d, graph-distance patterns, near kernel.
CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

from workloads.problems import make_config, q1_element_stiffness

# SURVEY §8d table (exact counts under the §8c readings)
COUNTS = {
    "1": dict(n=1024, n_F=768, nnz_A=4992, nnz_A_FF=2752, nnz_W=1953, hist={1: 33, 2: 510, 4: 225}),
    "2": dict(n=262144, n_F=229376, nnz_A=1810432, nnz_A_FF=1390592, nnz_W=824607,
              hist={1: 3169, 2: 101277, 4: 95139, 8: 29791}),
    "3": dict(n=2097152, n_F=1835008, nnz_A=14581760, nnz_A_FF=11198464, nnz_W=6705727),
    "4": dict(n=345744, n_F=300744, nnz_A=26869950, nnz_A_FF=20194488, nnz_W=12059703),
}


@pytest.mark.parametrize("name", ["1", "2", "3", "4"])
def test_config_counts(name):
    p = make_config(name)
    c = COUNTS[name]
    assert p.n == c["n"] and p.n_F == c["n_F"] and p.nnz_A == c["nnz_A"]
    assert p.nnz_A_FF() == c["nnz_A_FF"] and p.nnz_W == c["nnz_W"]
    if "hist" in c:
        assert p.J_hist() == c["hist"]


def _csr(p):
    return sp.csr_matrix((p.A_val, p.A_col, p.A_rowptr), shape=(p.n, p.n))


@pytest.mark.parametrize("name,size", [("1", 10), ("2", 7), ("3", 7)])
def test_scalar_pattern_is_graph_distance(name, size):
    """J_i = C points within graph distance l_i of i in the graph of A, with
    l_i the smallest l >= 2 giving a non-empty set (B = 1; A11/A12)."""
    p = make_config(name, size=size)
    A = _csr(p)
    G = (A != 0).astype(np.int32)
    I = sp.identity(p.n, dtype=np.int32, format="csr")
    reach = {1: ((G + I) > 0).astype(np.int32)}
    for l in range(2, 5):
        reach[l] = ((reach[l - 1] @ reach[1]) > 0).astype(np.int32)
    cid = np.cumsum(p.is_coarse) - 1
    for i in np.flatnonzero(p.is_coarse == 0):
        J = p.P_col[p.P_rowptr[i]:p.P_rowptr[i + 1]]
        for l in range(2, 5):
            nb = reach[l][i].indices
            cset = np.sort(cid[nb[p.is_coarse[nb] == 1]])
            if cset.size:
                assert np.array_equal(J, cset), (i, l)
                break


def test_elasticity_pattern_and_symmetry():
    p = make_config("4", size=4)
    A = _csr(p)
    assert abs(A - A.T).max() <= 1e-14 * abs(A).max()
    ev = np.linalg.eigvalsh(A.toarray())
    assert ev[0] > 0
    # the 3 dof rows of a node share J, J is blockwise (3c, 3c+1, 3c+2)
    for node in range(p.n // 3):
        rows = [3 * node + d for d in range(3)]
        Js = [p.P_col[p.P_rowptr[r]:p.P_rowptr[r + 1]] for r in rows]
        if not p.is_coarse[3 * node]:
            assert all(np.array_equal(Js[0], J) for J in Js)
            assert Js[0].size % 3 == 0
            assert np.array_equal(Js[0][1::3], Js[0][0::3] + 1)


def test_rigid_body_modes_in_kernel_away_from_clamp():
    p = make_config("4", size=4)
    A = _csr(p)
    R = A @ p.B
    # rows whose node does not touch the clamped layer (z = 1 nodes do)
    nx = 5
    z = (np.arange(p.n) // 3) // (nx * nx) + 1
    far = z >= 2
    assert np.abs(R[far]).max() <= 1e-12 * abs(A).max()
    assert np.abs(R[~far]).max() > 1e-6


def test_element_stiffness_has_six_zero_modes():
    K = q1_element_stiffness(0.3)
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == 6 and ev[6] > 1e-3


def test_full_rank_constraints_and_bc_injection():
    p = make_config("4", size=4)
    c = np.flatnonzero(p.is_coarse)
    assert np.array_equal(p.Bc, p.B[c])
    for i in np.flatnonzero(p.is_coarse == 0):
        J = p.P_col[p.P_rowptr[i]:p.P_rowptr[i + 1]]
        assert np.linalg.matrix_rank(p.Bc[J]) == 6


def test_perturbed_start_seeded():
    a = make_config("1b", size=8)
    b = make_config("1b", size=8)
    assert np.array_equal(a.P_val, b.P_val)
    c = np.flatnonzero(a.is_coarse)
    assert np.all(a.P_val[a.P_rowptr[c]] == 1.0)
