"""The row-partitioned path with R > 1 ranks.

P:980-986 [§4]: the pattern of P is communicated once before PCG, then only
the entries of P (here: the search direction y, W0 and dW on the halo rows)
are exchanged; Pi_B needs no communication.  gpurun gives one GPU,
so the R ranks are R contexts on that device in one process, one host thread
each, joined by the in-process loopback transport (emin_loopback_create):
the halo plan (dist.cu: k_mark_halo, the request / answer exchange, the halo
tail of the W layout), the per-iteration halo exchange and the allreduced CG
scalars all run with real data (n_halo_rows > 0 on every rank); only the
transport under them differs from the NCCL path.  Every rank passes only its
own rows of A, P and B (partition.rank_slice).  The concatenated result is
compared with the single-process oracle: index structure bit-exact, energy
within 1e-10 relative, P within 1e-8 max|P|, the same k and dE_k.
"""
import threading

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


def run_ranks(prob, R, k, ranges=None, chunks=None, sgs_key_global=None, **kw):
    """R loopback ranks, one thread each: setup, report, iterate(k), energy,
    get_P, layout.  Returns the per-rank results (rank order).  With
    sgs_key_global every rank passes its owned rows' slice of the key."""
    import torch
    from paper_2208_02995_b200 import emin as E
    from paper_2208_02995_b200.partition import partition_rows, plane_rows, rank_slice
    if ranges is None:
        ranges = partition_rows(prob.P_rowptr, prob.is_coarse, R, plane=plane_rows(prob))
    lb = E.emin_loopback_create(R)
    out = [None] * R
    err = [None] * R

    def work(r):
        h = None
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            rb, re_ = ranges[r]
            a = rank_slice(prob, rb, re_)
            if sgs_key_global is not None:
                kw_r = dict(kw, sgs_key=np.ascontiguousarray(sgs_key_global[rb:re_]))
                if hasattr(a["A_val"], "is_cuda"):
                    kw_r["sgs_key"] = torch.from_numpy(kw_r["sgs_key"]).cuda()
            else:
                kw_r = kw
            h = E.emin_setup(prob.n, prob.nc, a["A_rowptr"], a["A_col"], a["A_val"], a["is_coarse"],
                             a["P_rowptr"], a["P_col"], a["P_val"], prob.nv, a["B"], a["Bc"],
                             block_size=prob.block_size, stream=stream.cuda_stream, row_begin=rb,
                             row_end=re_, loopback=lb, loopback_rank=r, **kw_r)
            rep0 = E.emin_report(h)
            kd, dE = 0, []
            for kk in (chunks or [k]):
                kd1, dE1 = E.emin_iterate(h, kk, want=True)
                kd += kd1
                dE.append(dE1)
            dE = np.concatenate(dE)
            En = E.emin_energy(h)
            P = np.empty(int(a["P_rowptr"][-1]))
            E.emin_get_P(h, P)
            wptr, wcol, pofs = E.emin_get_layout(h)
            out[r] = dict(rep0=rep0, rep=E.emin_report(h), kd=kd, dE=dE, E=En, P=P, wptr=wptr, wcol=wcol,
                          pofs=pofs, p0=int(prob.P_rowptr[rb]))
        except Exception as ex:  # noqa: BLE001
            err[r] = ex
        finally:
            if h is not None:
                E.emin_destroy(h)

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    E.emin_loopback_destroy(lb)
    for e in err:
        if e is not None:
            raise e
    return out, ranges


def _concat_layout(res):
    wptr, wcol, pofs = [np.zeros(1, np.int64)], [], []
    off = 0
    for r in res:
        wptr.append(r["wptr"][1:] + off)
        off += int(r["wptr"][-1])
        wcol.append(r["wcol"])
        pofs.append(r["pofs"] + r["p0"])
    return np.concatenate(wptr), np.concatenate(wcol), np.concatenate(pofs)


CASES = [("3", 17, 40, 2), ("3", 17, 40, 3), ("3", 17, 40, 4), ("2b", 10, 30, 2), ("2b", 10, 30, 3),
         ("4", 5, 30, 2), ("4", 5, 30, 3), ("5", 8, 40, 2), ("5", 8, 40, 4), ("1b", None, 20, 2)]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name,size,k,R", CASES)
def test_loopback_ranks_match_oracle(name, size, k, R):
    from oracle import Oracle
    from workloads.problems import make_config
    prob = make_config(name, size=size)
    res, ranges = run_ranks(prob, R, k)
    o = Oracle(prob, project_z=True)
    # every rank really exchanges halo rows with its neighbours
    for r in res:
        assert r["rep"]["nranks"] == R
        assert r["rep"]["n_halo_rows"] > 0 and r["rep"]["n_halo_entries"] > 0
        assert r["rep"]["n_send_entries"] > 0
    # the interior part of y^ overlaps the halo exchange on the thicker slabs
    if (name, size) in (("3", 17), ("5", 8), ("2b", 10)) and R == 2:
        assert all(r["rep"]["n_interior_units"] > 0 for r in res)
    # index structure, bit-exact
    wptr, wcol, pofs = _concat_layout(res)
    owptr, owcol, ofrow = o.layout()
    assert np.array_equal(wptr, owptr) and np.array_equal(wcol, owcol)
    assert np.array_equal(pofs, prob.P_rowptr[ofrow])
    # the global scalars agree on every rank
    for r in res:
        assert r["rep0"]["E0"] == res[0]["rep0"]["E0"] and r["E"] == res[0]["E"]
        assert r["kd"] == res[0]["kd"] and np.array_equal(r["dE"], res[0]["dE"])
    assert abs(res[0]["rep0"]["E0"] - o.E0) <= E_TOL * abs(o.E0)
    assert sum(r["rep"]["n_svd_rows"] for r in res) == o.n_svd
    assert sum(r["rep"]["n_frozen_rows"] for r in res) == o.n_frozen
    kdo, dEo = o.iterate(k)
    assert res[0]["kd"] == kdo
    if kdo:
        assert np.allclose(res[0]["dE"], dEo, rtol=1e-8, atol=1e-12 * abs(o.E0))
    Eo = o.energy()
    assert abs(res[0]["E"] - Eo) <= E_TOL * abs(Eo)
    P = np.concatenate([r["P"] for r in res])
    Po = o.get_P()
    assert np.abs(P - Po).max() <= P_TOL * np.abs(Po).max()
    assert res[0]["rep"]["k_total"] == o.k_total


@pytest.mark.timeout(600)
def test_loopback_uneven_ranges_and_composability():
    """A hand-made partition that cuts inside z-planes (uneven, not
    plane-aligned) gives the same P as the single context; iterate(7) +
    iterate(5) on the ranks equals iterate(12) on one context (loopback
    iterations are enqueued eagerly, the same kernels in the same order)."""
    from paper_2208_02995_b200 import Emin
    from workloads.problems import make_config
    prob = make_config("3", size=12)
    n = prob.n
    ranges = [(0, n // 5), (n // 5, n // 2 + 7), (n // 2 + 7, n)]
    res, _ = run_ranks(prob, 3, 12, ranges=ranges, chunks=[7, 5])
    one = Emin.from_problem(prob)
    one.iterate(12)
    P1 = one.get_P()
    P = np.concatenate([r["P"] for r in res])
    assert np.abs(P - P1).max() <= 1e-12 * np.abs(P1).max()
    assert abs(res[0]["E"] - one.energy()) <= 1e-13 * abs(one.energy())


SGS_MR_CASES = [("3", 12, 20, 2, "color"), ("3", 12, 12, 3, "natural"), ("2b", 10, 20, 2, "color"),
                ("2b", 10, 20, 3, "color"), ("4", 4, 15, 2, "color"), ("5", 8, 15, 2, "color"),
                ("5", 8, 10, 3, "color"), ("1b", None, 12, 2, "natural"), ("4", 3, 10, 2, "natural")]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name,size,k,R,kind", SGS_MR_CASES)
def test_loopback_sgs_matches_oracle(name, size, k, R, kind):
    """Projected SGS on R ranks: every rank sweeps all global
    levels and refreshes the halo rows' u / z after each level (P:995-1004:
    the sweep is matrix-free like the masked product, only values move).
    The dependency levels equal the single-GPU ones (the order is global:
    (key, global F id)); P, E, k and dE_k match the single-process oracle to
    the parity bars and the single-GPU context to round-off."""
    from oracle import Oracle
    from paper_2208_02995_b200 import Emin
    from workloads.problems import make_config, sgs_key
    prob = make_config(name, size=size)
    key = sgs_key(prob, kind)
    res, _ = run_ranks(prob, R, k, sgs_key_global=key, precond="sgs")
    one = Emin.from_problem(prob, precond="sgs", sgs_key=key)
    rep1 = one.report()
    for r in res:
        assert r["rep"]["nranks"] == R and r["rep"]["n_halo_rows"] > 0
        assert r["rep"]["precond"] == 1
        assert r["rep"]["sgs_levels"] == rep1["sgs_levels"]
        assert r["rep"]["kernel_path"] == rep1["kernel_path"]
        assert r["kd"] == res[0]["kd"] and np.array_equal(r["dE"], res[0]["dE"])
    k1, dE1 = one.iterate(k)
    P1 = one.get_P()
    o = Oracle(prob, precond="sgs", sgs_key=key)
    kdo, dEo = o.iterate(k)
    assert res[0]["kd"] == kdo == k1
    assert np.allclose(res[0]["dE"], dEo, rtol=1e-8, atol=1e-12 * abs(o.E0))
    assert np.allclose(res[0]["dE"], dE1, rtol=1e-10, atol=1e-14 * abs(o.E0))
    Eo = o.energy()
    assert abs(res[0]["E"] - Eo) <= E_TOL * abs(Eo)
    P = np.concatenate([r["P"] for r in res])
    Po = o.get_P()
    assert np.abs(P - Po).max() <= P_TOL * np.abs(Po).max()
    assert np.abs(P - P1).max() <= 1e-11 * np.abs(P1).max()
