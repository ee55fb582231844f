"""NEXT-4 on the GPU: emin_galerkin (A_c = P^T A P) and the multilevel driver
against the CPU oracle (reading A26).

emin_galerkin is compared BITWISE with the oracle's two-product definition
on the same P (both sum every entry's product terms in the same order with
one rounding per operation).  The multilevel runs are compared level by
level with the north-star bars: pattern bit-exact, energy 1e-10 relative,
P within 1e-8 * max|P| (the coarse operators then agree to rounding).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

E_TOL = 1e-10
P_TOL = 1e-8


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_02995_b200.build import build
    build()


def _oracle_P(prob, k):
    from oracle import Oracle
    o = Oracle(prob)
    o.iterate(k)
    return o.get_P()


def _both(prob, Pv, device):
    import torch
    from oracle import galerkin
    from paper_2208_02995_b200.emin import emin_galerkin
    args = [prob.A_rowptr, prob.A_col, prob.A_val, prob.P_rowptr, prob.P_col, Pv]
    want = galerkin(prob.n, prob.nc, *args)
    if device == "cuda":
        targs = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in args]
        got = [t.cpu().numpy() for t in emin_galerkin(prob.n, prob.nc, *targs)]
    else:
        got = emin_galerkin(prob.n, prob.nc, *args)
    return got, want


def _assert_bitwise(got, want):
    for g, w in zip(got, want):
        assert g.shape == w.shape
        assert np.array_equal(g, w)


@pytest.mark.parametrize("name,size,k", [("1d", 17, 40), ("1b", 32, 5), ("3", 12, 5), ("3", 24, 3),
                                         ("4", 4, 5), ("4", 7, 3), ("1v3", 10, 4), ("5", 5, 3)])
@pytest.mark.parametrize("device", ["cuda", "host"])
def test_galerkin_bitwise_matches_oracle(name, size, k, device):
    from workloads.problems import make_config
    p = make_config(name, size)
    got, want = _both(p, _oracle_P(p, k), device)
    _assert_bitwise(got, want)


@pytest.mark.parametrize("name,size", [("4", 4), ("4", 7), ("5", 5)])
def test_galerkin_block_path_equals_point_path(name, size):
    # elasticity inputs take the 3x3-block product; it must give the point
    # path's (and the oracle's) bits
    import torch
    from paper_2208_02995_b200.emin import emin_galerkin, load_library
    from workloads.problems import make_config
    p = make_config(name, size)
    Pv = _oracle_P(p, 3)
    args = [torch.from_numpy(np.ascontiguousarray(a)).cuda()
            for a in (p.A_rowptr, p.A_col, p.A_val, p.P_rowptr, p.P_col, Pv)]
    blk = [t.cpu().numpy() for t in emin_galerkin(p.n, p.nc, *args)]
    assert load_library().emin_galerkin_path() == 1
    pt = [t.cpu().numpy() for t in emin_galerkin(p.n, p.nc, *args, point=True)]
    assert load_library().emin_galerkin_path() == 0
    _assert_bitwise(blk, pt)


def test_galerkin_block_path_falls_back_on_wide_node_rows():
    # one 3x3-block node whose P row spans 1100 C nodes (> 1024 node columns,
    # the block path's widest table): the point path takes over, same bits
    from oracle import galerkin
    from paper_2208_02995_b200.emin import emin_galerkin, load_library
    rng = np.random.default_rng(3)
    n, ncn = 3, 1100
    nc = 3 * ncn
    Arp = np.array([0, 3, 6, 9], np.int64)
    Acol = np.tile(np.arange(3), 3).astype(np.int32)
    Aval = rng.standard_normal(9) + 3.0 * np.eye(3).reshape(-1)
    Prp = np.array([0, nc, 2 * nc, 3 * nc], np.int64)
    Pcol = np.tile(np.arange(nc), 3).astype(np.int32)
    Pval = rng.standard_normal(3 * nc)
    want = galerkin(n, nc, Arp, Acol, Aval, Prp, Pcol, Pval)
    got = emin_galerkin(n, nc, Arp, Acol, Aval, Prp, Pcol, Pval)
    assert load_library().emin_galerkin_path() == 0
    _assert_bitwise(got, want)


def _csr(D):
    rp = np.zeros(D.shape[0] + 1, np.int64)
    cols, vals = [], []
    for i in range(D.shape[0]):
        nz = np.flatnonzero(D[i])
        cols.append(nz)
        vals.append(D[i, nz])
        rp[i + 1] = rp[i] + nz.size
    return rp, np.concatenate(cols).astype(np.int32), np.concatenate(vals)


@pytest.mark.parametrize("density,expect_tier", [(0.004, 1), (0.02, 2)])
def test_galerkin_wide_rows_all_table_tiers(density, expect_tier):
    # rows of T / A_c wider than 128 (and 1024) distinct columns go to the
    # 2048- (and 16384-) slot tables; still bitwise equal to the oracle
    from oracle import galerkin
    from paper_2208_02995_b200.emin import emin_galerkin
    rng = np.random.default_rng(7)
    n, nc = 1500, 3000
    M = (rng.random((n, n)) < 0.004) * rng.standard_normal((n, n))
    A = M + M.T + np.eye(n) * 4.0
    Pd = (rng.random((n, nc)) < density) * rng.standard_normal((n, nc))
    Arp, Acol, Aval = _csr(A)
    Prp, Pcol, Pval = _csr(Pd)
    want = galerkin(n, nc, Arp, Acol, Aval, Prp, Pcol, Pval)
    got = emin_galerkin(n, nc, Arp, Acol, Aval, Prp, Pcol, Pval)
    _assert_bitwise(got, want)
    widest = np.diff(want[0]).max()
    assert widest > (128 if expect_tier == 1 else 1024)


def test_galerkin_too_wide_row_and_bad_input_errors():
    from paper_2208_02995_b200.emin import EminError, emin_galerkin
    n, nc = 2, 9000
    Arp = np.array([0, 1, 2], np.int64)
    Acol = np.array([0, 1], np.int32)
    Aval = np.ones(2)
    Prp = np.array([0, nc, nc + 1], np.int64)
    Pcol = np.concatenate([np.arange(nc), [0]]).astype(np.int32)
    Pval = np.ones(nc + 1)
    with pytest.raises(EminError) as e:
        emin_galerkin(n, nc, Arp, Acol, Aval, Prp, Pcol, Pval)
    assert e.value.code == 1                        # EMIN_ERR_ARG
    bad = Pcol.copy()
    bad[5] = nc                                     # column id out of range
    with pytest.raises(EminError) as e:
        emin_galerkin(n, nc, Arp, Acol, Aval, Prp, bad, Pval)
    assert e.value.code == 2                        # EMIN_ERR_CSR


def _oracle_levels(prob, nlev, iters, l0_coarse=1, lmax=4):
    """The same hierarchy with the oracle only (pattern, Alg. 2/3, Galerkin)."""
    from oracle import Oracle, galerkin, pattern
    from workloads.problems import coarse_problem
    out = []
    p = prob
    for lev in range(nlev):
        if lev > 0:
            rp, col, _ = pattern(p, l0=l0_coarse, lmax=max(lmax, l0_coarse + 1))
            p.P_rowptr, p.P_col = rp, col
        o = Oracle(p)
        o.E0
        kd, _ = o.iterate(iters)
        Pv = o.get_P()
        Ac = galerkin(p.n, p.nc, p.A_rowptr, p.A_col, p.A_val, p.P_rowptr, p.P_col, Pv)
        out.append(dict(n=p.n, nc=p.nc, E0=o.E0, E=o.energy(), k=kd, P=(p.P_rowptr, p.P_col, Pv), A_c=Ac))
        p = coarse_problem(p, *Ac, iters=iters)
    return out


@pytest.mark.parametrize("name,size,nlev,iters", [("3", 16, 3, 8), ("1b", 32, 3, 10), ("4", 6, 2, 6),
                                                  ("2b", 16, 2, 8)])
def test_multilevel_matches_oracle(name, size, nlev, iters):
    import torch
    from paper_2208_02995_b200.multilevel import emin_multilevel
    from workloads.problems import coarse_split, make_config
    prob = make_config(name, size)
    want = _oracle_levels(make_config(name, size), nlev, iters)
    # the C/F splittings of the levels (geometric, A26)
    dims, zlo = prob.meta["dims"], prob.meta.get("zlo", 0)
    iscs = []
    for _ in range(nlev):
        isc, dims, zlo = coarse_split(dims, zlo)
        iscs.append(torch.from_numpy(np.repeat(isc, prob.block_size).astype(np.uint8)).cuda())
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    got = emin_multilevel(t(prob.A_rowptr), t(prob.A_col), t(prob.A_val), iscs, t(prob.B),
                          block_size=prob.block_size, P_rowptr=t(prob.P_rowptr), P_col=t(prob.P_col),
                          P_val=t(prob.P_val), iters=iters)
    assert len(got) == nlev
    for g, w in zip(got, want):
        assert g["n"] == w["n"] and g["nc"] == w["nc"]
        prp, pcol, pv = [x.cpu().numpy() for x in g["P"]]
        assert np.array_equal(prp, w["P"][0]) and np.array_equal(pcol, w["P"][1])
        assert g["k_done"] == w["k"]
        assert abs(g["E0"] - w["E0"]) <= E_TOL * abs(w["E0"])
        assert abs(g["E"] - w["E"]) <= E_TOL * abs(w["E"])
        assert np.abs(pv - w["P"][2]).max() <= P_TOL * np.abs(w["P"][2]).max()
        arp, acol, aval = [x.cpu().numpy() for x in g["A_c"]]
        assert np.array_equal(arp, w["A_c"][0]) and np.array_equal(acol, w["A_c"][1])
        assert np.abs(aval - w["A_c"][2]).max() <= 1e-9 * np.abs(w["A_c"][2]).max()
        assert g["E"] <= g["E0"] * (1 + 1e-12)
        if prob.block_size == 3:
            # Galerkin levels have > 27 blocks per node: still the nodal path
            # (v2 staged in chunks of 27 blocks)
            assert g["kernel_path"] == 2


def test_sgs_on_a_galerkin_level_matches_oracle():
    # projected SGS on the elasticity level-2 operator (up to 125 blocks per
    # node: the nodal sweeps stage them in chunks of 27)
    from oracle import Oracle, galerkin, pattern
    from paper_2208_02995_b200 import Emin
    from workloads.problems import coarse_problem, make_config, sgs_key
    p = make_config("4", 8)
    o = Oracle(p)
    o.iterate(5)
    Ac = galerkin(p.n, p.nc, p.A_rowptr, p.A_col, p.A_val, p.P_rowptr, p.P_col, o.get_P())
    p2 = coarse_problem(p, *Ac, iters=8)
    p2.P_rowptr, p2.P_col, _ = pattern(p2, l0=1, lmax=4)
    for kind in ("color", "natural"):
        key = sgs_key(p2, kind)
        g = Emin.from_problem(p2, device="cuda", precond="sgs", sgs_key=key)
        assert g.report()["kernel_path"] == 2
        o2 = Oracle(p2, precond="sgs", sgs_key=key)
        kd, _ = g.iterate(8)
        kdo, _ = o2.iterate(8)
        assert kd == kdo
        E, Eo = g.energy(), o2.energy()
        assert abs(E - Eo) <= E_TOL * abs(Eo)
        P, Po = g.get_P(), o2.get_P()
        assert np.abs(P - Po).max() <= P_TOL * np.abs(Po).max()
        g.close()


def test_galerkin_full_size_config3_bitwise():
    # BASELINE config 3 at full size (2.1M rows, 40 oracle iterations would
    # take minutes: 3 here) -- the production sizes of T and A_c
    from workloads.problems import make_config
    p = make_config("3")
    got, want = _both(p, _oracle_P(p, 3), "cuda")
    _assert_bitwise(got, want)
