"""Multi-rank host logic on CPU: world_size 2 (and 3) with the gloo backend.

Each rank takes its row range from partition_rows, derives its halo rows
with halo_plan (what dist.cu builds on the device), requests them from
their owners over torch.distributed (gloo), receives the halo rows' pattern
once and their values, and computes the masked product K x on its own rows
from owned + halo data only.  The concatenation over the ranks must equal
the single-process oracle's masked product, and every request must be
served by the rank that owns the row.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, size, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2208_02995_b200.partition import halo_plan, partition_rows, f_ids
        from workloads.problems import make_config
        prob = make_config(name, size=size)
        dims = prob.meta["dims"]
        plane = dims[0] * dims[1] * (3 if prob.nv == 6 else 1)
        ranges = partition_rows(prob.P_rowptr, prob.is_coarse, world, plane=plane)
        halo, owners, (fb, fe), franges = halo_plan(prob.A_rowptr, prob.A_col, prob.is_coarse, ranges, rank)
        isc = prob.is_coarse != 0
        fid = f_ids(prob.is_coarse)
        frow_of = np.flatnonzero(~isc)                       # global F id -> global row
        rng = np.random.default_rng(7)
        X_global = rng.standard_normal(prob.nnz_W)           # same seeded values on every rank
        wlen = np.diff(prob.P_rowptr)[~isc]
        wptr_g = np.r_[0, np.cumsum(wlen)]
        # ---- requests to owners (global F ids), answered with pattern + values
        req = {p: halo[owners == p].tolist() for p in range(world)}
        all_req = [None] * world
        dist.all_gather_object(all_req, req)
        answers = {}
        for p in range(world):
            if p == rank:
                continue
            rows = all_req[p].get(rank, [])
            assert all(fb <= g < fe for g in rows), "request sent to a non-owner"
            answers[p] = [(g, prob.P_col[prob.P_rowptr[frow_of[g]]:prob.P_rowptr[frow_of[g] + 1]].tolist(),
                           X_global[wptr_g[g]:wptr_g[g + 1]].tolist()) for g in rows]
        gathered = [None] * world
        dist.all_gather_object(gathered, answers)
        halo_rows = {}
        for p in range(world):
            if p != rank:
                for g, cols, vals in gathered[p].get(rank, []):
                    halo_rows[g] = (np.array(cols), np.array(vals))
        assert sorted(halo_rows) == halo.tolist()
        # ---- masked product on the owned rows from owned + halo data only
        def row_data(g):
            if fb <= g < fe:
                r = frow_of[g]
                return (prob.P_col[prob.P_rowptr[r]:prob.P_rowptr[r + 1]], X_global[wptr_g[g]:wptr_g[g + 1]])
            return halo_rows[g]
        out = []
        b, e = ranges[rank]
        for r in range(b, e):
            if isc[r]:
                continue
            Ji = prob.P_col[prob.P_rowptr[r]:prob.P_rowptr[r + 1]]
            acc = np.zeros(Ji.size)
            for q in range(prob.A_rowptr[r], prob.A_rowptr[r + 1]):
                c = prob.A_col[q]
                if isc[c]:
                    continue
                Jk, Xk = row_data(fid[c])
                for t, j in enumerate(Ji):
                    s = np.searchsorted(Jk, j)
                    if s < Jk.size and Jk[s] == j:
                        acc[t] += prob.A_val[q] * Xk[s]
            out.append(acc)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.concatenate(out) if out else np.zeros(0))
        np.save(os.path.join(out_dir, f"range{rank}.npy"), np.array(ranges[rank]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,size,world", [("3", 12, 2), ("2b", 10, 3), ("4", 4, 2)])
def test_partitioned_masked_product_matches_oracle(tmp_path, name, size, world):
    from oracle import Oracle
    from workloads.problems import make_config
    mp.spawn(_worker, args=(world, _free_port(), name, size, str(tmp_path)), nprocs=world, join=True)
    prob = make_config(name, size=size)
    o = Oracle(prob)
    rng = np.random.default_rng(7)
    X = rng.standard_normal(prob.nnz_W)
    ref = o.masked_AX(X)
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    assert got.shape == ref.shape
    assert np.allclose(got, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    ranges = [tuple(np.load(tmp_path / f"range{r}.npy")) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == prob.n
    assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))


def test_partition_balances_work():
    from paper_2208_02995_b200.partition import partition_rows
    from workloads.problems import make_config
    prob = make_config("3", size=32)
    for R in (2, 4, 8):
        ranges = partition_rows(prob.P_rowptr, prob.is_coarse, R, plane=32 * 32)
        w = np.where(prob.is_coarse == 0, np.diff(prob.P_rowptr), 0)
        loads = [w[b:e].sum() for b, e in ranges]
        assert max(loads) / (sum(loads) / R) < 1.2
        assert all(b % (32 * 32) == 0 for b, _ in ranges)
