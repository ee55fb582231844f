"""Seeded synthetic inputs for the energy-minimisation hot path.

This module holds NO arithmetic of the method (no projection, no QR, no
masked product, no CG).  It only builds the inputs that BASELINE.json's
``configs`` describe, following the readings in DESIGN.md §3 (SURVEY §8c
A9-A17):

* the SPD operator A (CSR: int64 rowptr, int32 cols, float64 vals),
* the C/F splitting (C <=> every grid/node coordinate even, A13),
* the fixed pattern of P (C columns within graph distance l of each F row,
  grown row by row l = 2, 3, ... until rank(B_c(J_i,:)) = nv, A11/A12),
* the near kernel B (constant vector, or the 6 rigid-body modes from centred
  node coordinates, A17) and its injection B_c,
* an optional starting ``P_val`` (equal weights, or the perturbed start of
  configs 1b/2b).

Both the CUDA path (through the C ABI) and the oracle consume these arrays;
neither is imported here.

Paper cross-references (PAPER.md line numbers, section in brackets):
  P:156-175 [§2 Eq. CFspl, prol]  C/F ordering, P = [W; I]
  P:259-279 [§3 Eq. enlPatt]      pattern = distance-k growth in the graph
  P:281-305 [§3 Eq. TSP, Constr]  W V_c = V_f row by row
  P:527-540 [§3.2 Alg. 1]         per-row distance growth until solvable
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "Problem", "make_config", "CONFIGS",
    "poisson2d", "poisson3d", "fv_diffusion", "elasticity_q1",
    "q1_element_stiffness",
]


@dataclass
class Problem:
    """All arrays are host numpy arrays in the layouts the C ABI expects."""
    name: str
    n: int
    nc: int
    A_rowptr: np.ndarray      # int64 [n+1]
    A_col: np.ndarray         # int32 [nnz]
    A_val: np.ndarray         # float64 [nnz]
    is_coarse: np.ndarray     # uint8 [n]
    P_rowptr: np.ndarray      # int64 [n+1]
    P_col: np.ndarray         # int32 [nnzP]   coarse ids, ascending per row
    P_val: Optional[np.ndarray]  # float64 [nnzP] or None (least-norm start)
    nv: int
    B: np.ndarray             # float64 [n, nv] row-major
    Bc: np.ndarray            # float64 [nc, nv] row-major
    iters: int
    block_size: int = 1
    meta: dict = field(default_factory=dict)

    # -- derived counts --------------------------------
    @property
    def nnz_A(self) -> int:
        return int(self.A_rowptr[-1])

    @property
    def fine_rows(self) -> np.ndarray:
        return np.flatnonzero(self.is_coarse == 0)

    @property
    def n_F(self) -> int:
        return int(self.n - self.nc)

    @property
    def nnz_W(self) -> int:
        f = self.fine_rows
        return int((self.P_rowptr[f + 1] - self.P_rowptr[f]).sum())

    def nnz_A_FF(self) -> int:
        rows = np.repeat(np.arange(self.n), np.diff(self.A_rowptr))
        return int(((self.is_coarse[rows] == 0) & (self.is_coarse[self.A_col] == 0)).sum())

    def J_hist(self) -> dict:
        f = self.fine_rows
        cnt = self.P_rowptr[f + 1] - self.P_rowptr[f]
        u, c = np.unique(cnt, return_counts=True)
        return {int(a): int(b) for a, b in zip(u, c)}


# ---------------------------------------------------------------------------
# CSR assembly from a box stencil table
# ---------------------------------------------------------------------------

def _csr_from_table(deltas, vals, mask):
    """Rows r, entries (r + deltas[o]) for each offset o with mask[r, o].

    ``deltas`` must be ascending so that columns come out sorted.
    vals, mask: [n, n_off].
    """
    n = mask.shape[0]
    cnt = mask.sum(axis=1, dtype=np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rowptr[1:])
    rows = np.arange(n, dtype=np.int64)[:, None]
    cols = (rows + np.asarray(deltas, dtype=np.int64)[None, :])[mask].astype(np.int32)
    v = vals[mask].astype(np.float64)
    return rowptr, cols, v


def _shifted(a, d, axis, fill=0.0):
    """out[i] = a[i + d] along axis (fill outside)."""
    out = np.full_like(a, fill)
    n = a.shape[axis]
    src = [slice(None)] * a.ndim
    dst = [slice(None)] * a.ndim
    if d >= 0:
        src[axis] = slice(d, n)
        dst[axis] = slice(0, n - d)
    else:
        src[axis] = slice(0, n + d)
        dst[axis] = slice(-d, n)
    out[tuple(dst)] = a[tuple(src)]
    return out


# ---------------------------------------------------------------------------
# Scalar operators (Dirichlet eliminated)
# ---------------------------------------------------------------------------

def _scalar_7pt(shape_zyx, coef_faces, diag):
    """Generic 5/7-point operator on a box.  coef_faces[(axis, sign)] is the
    positive coupling array (shape_zyx) to the neighbour in that direction;
    A(r, nb) = -coef.  ``diag`` array (shape_zyx)."""
    nz, ny, nx = shape_zyx
    strides = {2: 1, 1: nx, 0: nx * ny}     # numpy axis -> linear stride
    offs = []
    for (axis, sign), c in coef_faces.items():
        offs.append((sign * strides[axis], axis, sign, c))
    offs.append((0, None, 0, None))
    offs.sort(key=lambda t: t[0])
    n = nx * ny * nz
    vals = np.zeros((n, len(offs)))
    mask = np.zeros((n, len(offs)), dtype=bool)
    for o, (delta, axis, sign, c) in enumerate(offs):
        if axis is None:
            vals[:, o] = diag.reshape(-1)
            mask[:, o] = True
            continue
        ex = np.ones(shape_zyx, dtype=bool)
        idx = [slice(None)] * 3
        idx[axis] = slice(shape_zyx[axis] - 1, None) if sign > 0 else slice(0, 1)
        ex[tuple(idx)] = False
        vals[:, o] = -c.reshape(-1)
        mask[:, o] = ex.reshape(-1)
    return _csr_from_table([t[0] for t in offs], vals, mask)


def poisson2d(n):
    """5-point Dirichlet Laplacian on an n x n grid (diag 4, off -1)."""
    shape = (1, n, n)
    one = np.ones(shape)
    faces = {(2, -1): one, (2, 1): one, (1, -1): one, (1, 1): one}
    return _scalar_7pt(shape, faces, 4.0 * one), (n, n, 1)


def poisson3d(n, eps=(1.0, 1.0, 1e-3)):
    """7-point anisotropic Dirichlet Laplacian, coefficients (x, y, z)."""
    shape = (n, n, n)
    one = np.ones(shape)
    ex, ey, ez = eps
    faces = {(2, -1): ex * one, (2, 1): ex * one, (1, -1): ey * one,
             (1, 1): ey * one, (0, -1): ez * one, (0, 1): ez * one}
    return _scalar_7pt(shape, faces, 2.0 * (ex + ey + ez) * one), (n, n, n)


def lognormal_field(n, seed=0, corr=8.0, lo=-6.0, hi=6.0):
    """white N(0,1) (PCG64 seed) -> Gaussian filter with
    sigma = corr/sqrt(2), periodic wrap -> standardise -> log10 k = lo +
    (hi-lo) Phi(g): log-uniform marginal on [lo, hi]."""
    from scipy.ndimage import gaussian_filter
    from scipy.special import ndtr
    rng = np.random.Generator(np.random.PCG64(seed))
    g = rng.standard_normal((n, n, n))
    g = gaussian_filter(g, sigma=corr / math.sqrt(2.0), mode="wrap")
    g = (g - g.mean()) / g.std()
    return 10.0 ** (lo + (hi - lo) * ndtr(g))


def fv_diffusion(n, seed=0, corr=8.0):
    """Two-point-flux finite volumes, h = 1: face transmissibility is the
    harmonic mean 2 k1 k2/(k1+k2); Dirichlet faces use the half cell, 2k."""
    k = lognormal_field(n, seed=seed, corr=corr)
    shape = k.shape
    faces = {}
    diag = np.zeros(shape)
    for axis in (0, 1, 2):
        for sign in (-1, 1):
            kn = _shifted(k, sign, axis, fill=np.nan)
            t = 2.0 * k * kn / (k + kn)
            bnd = np.isnan(t)
            t_face = np.where(bnd, 0.0, t)
            faces[(axis, sign)] = t_face
            diag += np.where(bnd, 2.0 * k, t_face)
    return _scalar_7pt(shape, faces, diag), (n, n, n), k


# ---------------------------------------------------------------------------
# Q1 linear elasticity
# ---------------------------------------------------------------------------

def q1_element_stiffness(nu, E=1.0):
    """24x24 stiffness of the trilinear hex on the UNIT cube with 2x2x2
    Gauss points; local dof = 3*corner + d, corner = ax + 2 ay + 4 az.
    On a cube of side h the matrix scales by h."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2 * mu
    D[3, 3] = D[4, 4] = D[5, 5] = mu
    gp = np.array([0.5 - 0.5 / math.sqrt(3.0), 0.5 + 0.5 / math.sqrt(3.0)])
    corners = np.array([[a & 1, (a >> 1) & 1, (a >> 2) & 1] for a in range(8)], float)
    K = np.zeros((24, 24))
    for xi in gp:
        for eta in gp:
            for zeta in gp:
                p = np.array([xi, eta, zeta])
                # N_a = prod_d (c_d p_d + (1-c_d)(1-p_d)); dN/dp_d
                f = corners * p + (1 - corners) * (1 - p)          # [8,3]
                df = 2 * corners - 1                               # [8,3]
                dN = np.empty((8, 3))
                dN[:, 0] = df[:, 0] * f[:, 1] * f[:, 2]
                dN[:, 1] = f[:, 0] * df[:, 1] * f[:, 2]
                dN[:, 2] = f[:, 0] * f[:, 1] * df[:, 2]
                Bm = np.zeros((6, 24))
                for a in range(8):
                    gx, gy, gz = dN[a]
                    c = 3 * a
                    Bm[0, c] = gx
                    Bm[1, c + 1] = gy
                    Bm[2, c + 2] = gz
                    Bm[3, c] = gy; Bm[3, c + 1] = gx
                    Bm[4, c + 1] = gz; Bm[4, c + 2] = gy
                    Bm[5, c] = gz; Bm[5, c + 2] = gx
                K += Bm.T @ D @ Bm * 0.125
    return 0.5 * (K + K.T)


def _node_offsets27(nx, ny):
    offs = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dx + nx * (dy + ny * dz), dx, dy, dz))
    offs.sort(key=lambda t: t[0])
    return offs


def elasticity_q1(N, nu, E_elem):
    """Q1 hex mesh of N^3 elements on the unit cube (h = 1/N), nodes
    (N+1)^3, bottom face z = 0 clamped (nodes eliminated).  E_elem: array
    [N(z), N(y), N(x)] of Young's moduli.  Returns the point CSR with rows
    3*node + d, node = x + (N+1)(y + (N+1)(z-1)), z = 1..N."""
    h = 1.0 / N
    Kh = q1_element_stiffness(nu) * h
    nxn = N + 1
    nzn = N                           # z = 1..N remain
    Epad = np.zeros((N + 2, N + 2, N + 2))
    Epad[1:N + 1, 1:N + 1, 1:N + 1] = E_elem
    # node grid arrays (z index k -> physical z = k+1)
    zz = np.arange(1, N + 1)[:, None, None]
    yy = np.arange(nxn)[None, :, None]
    xx = np.arange(nxn)[None, None, :]
    nnode = nzn * nxn * nxn
    offs = _node_offsets27(nxn, nxn)
    blocks = np.zeros((nnode, 3, len(offs), 3))
    mask_node = np.zeros((nnode, len(offs)), dtype=bool)
    for o, (delta, dx, dy, dz) in enumerate(offs):
        exists = ((xx + dx >= 0) & (xx + dx <= N) & (yy + dy >= 0) & (yy + dy <= N)
                  & (zz + dz >= 1) & (zz + dz <= N))
        exists = np.broadcast_to(exists, (nzn, nxn, nxn))
        mask_node[:, o] = exists.reshape(-1)
        choices = []
        for off in (dx, dy, dz):
            if off == 0:
                choices.append([(0, 0), (1, 1)])
            elif off == 1:
                choices.append([(0, 1)])
            else:
                choices.append([(1, 0)])
        acc = np.zeros((nnode, 3, 3))
        for (ax, bx) in choices[0]:
            for (ay, by) in choices[1]:
                for (az, bz) in choices[2]:
                    a = ax + 2 * ay + 4 * az
                    b = bx + 2 * by + 4 * bz
                    # element origin o = node - a ; Epad index o + 1
                    Ee = Epad[(zz - az + 1), (yy - ay + 1), (xx - ax + 1)]
                    Ee = np.broadcast_to(Ee, (nzn, nxn, nxn)).reshape(-1)
                    acc += Ee[:, None, None] * Kh[3 * a:3 * a + 3, 3 * b:3 * b + 3][None]
        blocks[:, :, o, :] = acc
    # point CSR: row (node, d) has entries for each existing offset, 3 each
    n = 3 * nnode
    cnt = 3 * mask_node.sum(axis=1)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.repeat(cnt, 3), out=rowptr[1:])
    node = np.arange(nnode, dtype=np.int64)
    ncol_node = node[:, None] + np.array([t[0] for t in offs], dtype=np.int64)[None, :]
    colblk = 3 * ncol_node[:, None, :, None] + np.arange(3)[None, None, None, :]   # [nnode,1,27,3]
    colblk = np.broadcast_to(colblk, (nnode, 3, len(offs), 3))
    m4 = np.broadcast_to(mask_node[:, None, :, None], (nnode, 3, len(offs), 3))
    col = colblk[m4].astype(np.int32)
    val = blocks[m4]
    coords = np.stack(np.broadcast_arrays(xx, yy, zz), axis=-1).reshape(-1, 3).astype(np.float64) * h
    return (rowptr, col, val), (nxn, nxn, nzn), coords


# ---------------------------------------------------------------------------
# C/F splitting, pattern (distance-l in the graph of A), near kernel
# ---------------------------------------------------------------------------

def _ball_offsets(l, metric):
    offs = []
    r = range(-l, l + 1)
    for dz in r:
        for dy in r:
            for dx in r:
                d = (abs(dx) + abs(dy) + abs(dz)) if metric == "manhattan" else max(abs(dx), abs(dy), abs(dz))
                if d <= l:
                    offs.append((dx, dy, dz))
    return offs


def _box_pattern(dims, zlo, is_c_grid, cid_grid, l, metric, sel=None):
    """C targets within graph distance l of each node (box grid, x fastest).
    dims = (nx, ny, nz) node counts, z coordinate runs zlo..zlo+nz-1.
    Returns (counts[n_sel], cols) with cols ascending per row."""
    nx, ny, nz = dims
    offs = _ball_offsets(l, metric)
    offs.sort(key=lambda t: t[0] + nx * (t[1] + ny * t[2]))
    n = nx * ny * nz
    if sel is None:
        sel = np.arange(n)
    x = sel % nx
    y = (sel // nx) % ny
    z = sel // (nx * ny)
    cols = np.full((sel.size, len(offs)), -1, dtype=np.int64)
    for o, (dx, dy, dz) in enumerate(offs):
        tx, ty, tz = x + dx, y + dy, z + dz
        ok = (tx >= 0) & (tx < nx) & (ty >= 0) & (ty < ny) & (tz >= 0) & (tz < nz)
        t = np.where(ok, tx + nx * (ty + ny * tz), 0)
        ok &= is_c_grid[t]
        cols[:, o] = np.where(ok, cid_grid[t], -1)
    m = cols >= 0
    return m.sum(axis=1), cols[m]


def _rank_ok(Bc_node, counts, cols, nv, dofs):
    """rank(B_c(J,:)) == nv per row via the Gram matrix (generator-side
    decision only).  Bc_node: [n_cnode, dofs, nv]."""
    nrow = counts.size
    G = np.zeros((nrow, nv, nv))
    g_node = np.einsum("cdi,cdj->cij", Bc_node, Bc_node)
    rows = np.repeat(np.arange(nrow), counts)
    if rows.size:
        _add_grouped(G, rows, g_node[cols])
    ev = np.linalg.eigvalsh(G)
    top = np.maximum(ev[:, -1], 0.0)
    return (counts > 0) & (ev[:, 0] > 1e-10 * top)


def _add_grouped(G, rows, vals):
    # rows are sorted ascending: segment sums via reduceat
    starts = np.flatnonzero(np.r_[True, rows[1:] != rows[:-1]])
    sums = np.add.reduceat(vals, starts, axis=0)
    G[rows[starts]] += sums


def _grow_pattern(dims, zlo, is_c_node, cid_node, fine_nodes, metric, Bc_node, nv, dofs,
                  l0=2, lmax=4):
    """Per-row growth l = l0, l0+1, ... until full rank (Alg. 1 loop,
    P:527-540).  Returns counts/cols for fine_nodes (node level) and the
    histogram of distances used."""
    counts = np.zeros(fine_nodes.size, dtype=np.int64)
    cols_per = [None] * fine_nodes.size
    todo = np.arange(fine_nodes.size)
    used = {}
    result_counts = np.zeros(fine_nodes.size, dtype=np.int64)
    pieces = {}
    for l in range(l0, lmax + 1):
        if todo.size == 0:
            break
        c, cl = _box_pattern(dims, zlo, is_c_node, cid_node, l, metric, sel=fine_nodes[todo])
        ok = _rank_ok(Bc_node, c, cl, nv, dofs) if l < lmax else np.ones(todo.size, bool)
        starts = np.zeros(todo.size + 1, dtype=np.int64)
        np.cumsum(c, out=starts[1:])
        acc = todo[ok]
        for_rows_ok = np.flatnonzero(ok)
        pieces[l] = (acc, c[ok], _gather_segments(cl, starts, for_rows_ok))
        result_counts[acc] = c[ok]
        used[l] = int(acc.size)
        todo = todo[~ok]
    # assemble in row order
    rowptr = np.zeros(fine_nodes.size + 1, dtype=np.int64)
    np.cumsum(result_counts, out=rowptr[1:])
    cols = np.empty(int(rowptr[-1]), dtype=np.int64)
    for l, (acc, c, cl) in pieces.items():
        if acc.size == 0:
            continue
        dst = _segment_positions(rowptr, acc, c)
        cols[dst] = cl
    return rowptr, cols, used


def _gather_segments(flat, starts, rows):
    if rows.size == 0:
        return flat[:0]
    lens = starts[rows + 1] - starts[rows]
    idx = np.repeat(starts[rows] - np.r_[0, np.cumsum(lens)[:-1]], lens) + np.arange(lens.sum())
    return flat[idx]


def _segment_positions(rowptr, rows, lens):
    base = rowptr[rows]
    return np.repeat(base - np.r_[0, np.cumsum(lens)[:-1]], lens) + np.arange(lens.sum())


# ---------------------------------------------------------------------------
# Config assembly
# ---------------------------------------------------------------------------

def _scalar_problem(name, csr, dims, iters, start, seed_pert=1, meta=None, linear_modes=False):
    rowptr, col, val = csr
    nx, ny, nz = dims
    n = nx * ny * nz
    x = np.arange(n) % nx
    y = (np.arange(n) // nx) % ny
    z = np.arange(n) // (nx * ny)
    is_c = ((x % 2 == 0) & (y % 2 == 0) & (z % 2 == 0))
    cid = np.full(n, -1, dtype=np.int64)
    cid[is_c] = np.arange(int(is_c.sum()))
    nc = int(is_c.sum())
    if linear_modes:
        # near kernel {1, x, y} (centred grid coordinates): nv = 3 on a scalar
        # operator -- exercises the general (nv > 1, point) kernel path
        B = np.stack([np.ones(n), x - (nx - 1) / 2.0, y - (ny - 1) / 2.0], axis=1)
    else:
        B = np.ones((n, 1))
    nv = B.shape[1]
    Bc = B[is_c].copy()
    fine = np.flatnonzero(~is_c)
    wp, wc, used = _grow_pattern((nx, ny, nz), 0, is_c, cid, fine, "manhattan",
                                 Bc.reshape(nc, 1, nv), nv, 1)
    P_rowptr, P_col = _merge_pattern(n, is_c, cid, fine, wp, wc, 1)
    P_val = _start_values(start, n, is_c, fine, P_rowptr, seed_pert)
    m = dict(dims=dims, growth=used, **(meta or {}))
    return Problem(name, n, nc, rowptr, col, val, is_c.astype(np.uint8), P_rowptr, P_col,
                   P_val, nv, B, Bc, iters, 1, m)


def _merge_pattern(n, is_c, cid, fine, wp, wc, dofs):
    """Full P pattern over all rows: C rows identity, F rows from wp/wc.
    For dofs = 3 (elasticity) node-level lists expand blockwise."""
    cnt = np.zeros(n, dtype=np.int64)
    if dofs == 1:
        cnt[fine] = np.diff(wp)
        cnt[is_c] = 1
        rowptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(cnt, out=rowptr[1:])
        col = np.empty(int(rowptr[-1]), dtype=np.int32)
        cidx = np.flatnonzero(is_c)
        col[rowptr[cidx]] = cid[cidx]
        dst = _segment_positions(rowptr, fine, np.diff(wp))
        col[dst] = wc
        return rowptr, col
    raise AssertionError


def _start_values(start, n, is_c, fine_rows, P_rowptr, seed):
    """'leastnorm' -> None (Alg. 2 from w-hat = 0, A9); 'equal' -> 1/|J_i|;
    'perturbed' -> 1/|J_i| + 0.25 U(-1,1) per entry, PCG64(seed), rows
    ascending."""
    if start == "leastnorm":
        return None
    cnt = np.diff(P_rowptr)
    val = np.repeat(1.0 / np.maximum(cnt, 1), cnt)
    if start == "perturbed":
        fmask = np.repeat(is_c.astype(bool) == False, cnt)  # noqa: E712
        rng = np.random.Generator(np.random.PCG64(seed))
        val[fmask] += 0.25 * rng.uniform(-1.0, 1.0, int(fmask.sum()))
    crow = np.flatnonzero(is_c)
    val[P_rowptr[crow]] = 1.0
    return val


def _rbm(coords):
    """6 rigid-body modes from centred coordinates (A17); rows 3*node+d,
    columns [tx, ty, tz, rx=(0,-z,y), ry=(z,0,-x), rz=(-y,x,0)]."""
    c = coords - coords.mean(axis=0)
    nn = c.shape[0]
    B = np.zeros((nn, 3, 6))
    B[:, 0, 0] = 1.0
    B[:, 1, 1] = 1.0
    B[:, 2, 2] = 1.0
    x, y, z = c[:, 0], c[:, 1], c[:, 2]
    B[:, 1, 3] = -z; B[:, 2, 3] = y
    B[:, 0, 4] = z;  B[:, 2, 4] = -x
    B[:, 0, 5] = -y; B[:, 1, 5] = x
    return B


def _elasticity_problem(name, N, nu, E_elem, iters, start, seed_pert=1, meta=None):
    (rowptr, col, val), (nxn, nyn, nzn), coords = elasticity_q1(N, nu, E_elem)
    nnode = nxn * nyn * nzn
    xi = np.arange(nnode) % nxn
    yi = (np.arange(nnode) // nxn) % nyn
    zi = np.arange(nnode) // (nxn * nyn) + 1
    is_c_node = (xi % 2 == 0) & (yi % 2 == 0) & (zi % 2 == 0)
    ncn = int(is_c_node.sum())
    cid_node = np.full(nnode, -1, dtype=np.int64)
    cid_node[is_c_node] = np.arange(ncn)
    Bn = _rbm(coords)                       # [nnode, 3, 6]
    Bc_node = Bn[is_c_node]
    fine_nodes = np.flatnonzero(~is_c_node)
    wp, wc, used = _grow_pattern((nxn, nyn, nzn), 1, is_c_node, cid_node, fine_nodes,
                                 "chebyshev", Bc_node, 6, 3)
    n = 3 * nnode
    is_c = np.repeat(is_c_node, 3)
    # point-level pattern: F dof rows of node -> {3c+b}, C dof rows identity
    cntn = np.diff(wp)
    cnt = np.ones(n, dtype=np.int64)
    fpt = (3 * fine_nodes[:, None] + np.arange(3)[None, :]).reshape(-1)
    cnt[fpt] = np.repeat(3 * cntn, 3)
    P_rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=P_rowptr[1:])
    P_col = np.empty(int(P_rowptr[-1]), dtype=np.int32)
    cpt = np.flatnonzero(is_c)
    cid_pt = 3 * np.repeat(cid_node[is_c_node], 3) + np.tile(np.arange(3), ncn)
    P_col[P_rowptr[cpt]] = cid_pt
    node_cols3 = (3 * wc[:, None] + np.arange(3)[None, :]).reshape(-1)    # per node segment, 3|J|
    seg = np.repeat(np.arange(fine_nodes.size), 3 * cntn)
    # each of the 3 dof rows of a fine node gets the same expanded list
    for d in range(3):
        rows = 3 * fine_nodes + d
        dst = _segment_positions(P_rowptr, rows, 3 * cntn)
        P_col[dst] = node_cols3
    del seg
    B = Bn.reshape(n, 6)
    Bc = B[is_c].copy()
    P_val = _start_values(start, n, is_c, None, P_rowptr, seed_pert)
    m = dict(dims=(nxn, nyn, nzn), zlo=1, growth=used, n_cnode=ncn, n_fnode=int(fine_nodes.size),
             **(meta or {}))
    return Problem(name, n, 3 * ncn, rowptr, col, val, is_c.astype(np.uint8), P_rowptr, P_col,
                   P_val, 6, B, Bc, iters, 3, m)


CONFIGS = {
    # name: (builder, default size, iters) -- BASELINE.json configs[0..4]
    "1": "2D Poisson 5-pt 32^2, equal-weight start, 20 it",
    "1b": "config 1 with the perturbed start (SURVEY §8d)",
    "2": "3D 7-pt (1,1,1e-3) 64^3, least-norm start, 30 it",
    "2b": "config 2 with the perturbed start",
    "3": "FV lognormal 128^3, corr 8, least-norm start, 40 it",
    "4": "Q1 elasticity 48^3, E=1, nu=0.3, bottom clamped, 30 it",
    "5": "Q1 elasticity 160^3, 8 layers E in 10^U(-2,2), nu=0.25, 40 it",
}


def poisson1d_problem(n=33, dist=3, start="leastnorm"):
    """1D Dirichlet Laplacian (tridiag -1, 2, -1), n odd, C = even indices,
    B = 1, pattern = C points within graph distance ``dist`` (closed-form
    pin of SURVEY §8c: converged W = 1/2 on the two adjacent C columns)."""
    shape = (1, 1, n)
    one = np.ones(shape)
    csr = _scalar_7pt(shape, {(2, -1): one, (2, 1): one}, 2.0 * one)
    rowptr, col, val = csr
    is_c = (np.arange(n) % 2 == 0)
    cid = np.full(n, -1, dtype=np.int64)
    cid[is_c] = np.arange(int(is_c.sum()))
    nc = int(is_c.sum())
    fine = np.flatnonzero(~is_c)
    c, cl = _box_pattern((n, 1, 1), 0, is_c, cid, dist, "manhattan", sel=fine)
    wp = np.zeros(fine.size + 1, dtype=np.int64)
    np.cumsum(c, out=wp[1:])
    P_rowptr, P_col = _merge_pattern(n, is_c, cid, fine, wp, cl, 1)
    P_val = _start_values(start, n, is_c, fine, P_rowptr, 1)
    return Problem(f"1d@{n}", n, nc, rowptr, col, val, is_c.astype(np.uint8), P_rowptr, P_col,
                   P_val, 1, np.ones((n, 1)), np.ones((nc, 1)), 40, 1, dict(dims=(n, 1, 1)))


def make_config(name: str, size: Optional[int] = None, seed: int = 0,
                start: Optional[str] = None) -> Problem:
    """Build BASELINE config ``name`` ('1','1b','2','2b','3','4','5'), or a
    reduced instance of the same generator with ``size`` grid points
    (scalar) / elements (elasticity) per side."""
    if name == "1d":
        return poisson1d_problem(size or 33, start=start or "leastnorm")
    if name == "1v3":
        # test workload (not a BASELINE config): config 1's operator with the
        # linear near kernel {1, x, y}, perturbed start
        n = size or 16
        csr, dims = poisson2d(n)
        return _scalar_problem(f"1v3@{n}", csr, dims, 20, start or "perturbed", meta=dict(config="1v3"),
                               linear_modes=True)
    if name in ("1", "1b"):
        n = size or 32
        csr, dims = poisson2d(n)
        st = start or ("equal" if name == "1" else "perturbed")
        return _scalar_problem(f"{name}@{n}", csr, dims, 20, st, meta=dict(config=name))
    if name in ("2", "2b"):
        n = size or 64
        csr, dims = poisson3d(n)
        st = start or ("leastnorm" if name == "2" else "perturbed")
        return _scalar_problem(f"{name}@{n}", csr, dims, 30, st, meta=dict(config=name))
    if name == "3":
        n = size or 128
        csr, dims, _k = fv_diffusion(n, seed=seed)
        return _scalar_problem(f"3@{n}", csr, dims, 40, start or "leastnorm",
                               meta=dict(config="3", seed=seed))
    if name == "4":
        N = size or 48
        E = np.ones((N, N, N))
        return _elasticity_problem(f"4@{N}", N, 0.3, E, 30, start or "leastnorm",
                                   meta=dict(config="4"))
    if name == "5":
        N = size or 160
        rng = np.random.Generator(np.random.PCG64(seed))
        El = 10.0 ** rng.uniform(-2.0, 2.0, 8)
        layer = np.minimum((np.arange(N) * 8) // N, 7)        # z_elem // (N/8)
        E = np.broadcast_to(El[layer][:, None, None], (N, N, N)).copy()
        return _elasticity_problem(f"5@{N}", N, 0.25, E, 40, start or "leastnorm",
                                   meta=dict(config="5", seed=seed, E_layers=El.tolist()))
    raise KeyError(name)


def coarse_split(dims, zlo=0):
    """Geometric 2x coarsening of a lexicographic node grid (x fastest), the
    splitting every level of the configs uses (reading A26: PMIS is out of
    scope): node (x, y, zlo + z) is a C node iff x, y and zlo + z are even.
    Returns (is_c_node bool [nx*ny*nz], coarse dims, coarse zlo); coarse ids
    (ranks among the C nodes) are again lexicographic on the coarse grid."""
    nx, ny, nz = dims
    nodes = np.arange(nx * ny * nz)
    x, y, z = nodes % nx, (nodes // nx) % ny, zlo + nodes // (nx * ny)
    is_c = (x % 2 == 0) & (y % 2 == 0) & (z % 2 == 0)
    zc = np.arange(zlo, zlo + nz)
    zc = zc[zc % 2 == 0]
    cdims = ((nx + 1) // 2, (ny + 1) // 2, int(zc.size))
    czlo = int(zc[0] // 2) if zc.size else 0
    return is_c, cdims, czlo


def coarse_problem(prob: Problem, Ac_rowptr, Ac_col, Ac_val, iters: Optional[int] = None) -> Problem:
    """The next level of a hierarchy: operator A_c (=
    P^T A P, computed by the caller), C/F from ``coarse_split`` of the coarse
    grid, near kernel B_next = B_c of this level, B_c,next its injection;
    P's pattern is left to the caller (P_rowptr / P_col None: Alg. 1's growth
    on the graph of A_c), least-norm start (P_val None)."""
    dims, zlo = prob.meta["dims"], prob.meta.get("zlo", 0)
    bs = prob.block_size
    is_c_node, cdims, czlo = coarse_split(dims, zlo)
    if not np.array_equal(np.repeat(is_c_node, bs), prob.is_coarse.astype(bool)):
        raise ValueError("prob's C/F splitting is not the geometric one")
    # the next level's nodes are this level's C nodes (lexicographic on cdims)
    is_c2 = np.repeat(coarse_split(cdims, czlo)[0], bs)
    B2 = np.ascontiguousarray(prob.Bc)
    Bc2 = B2[is_c2].copy()
    lev = prob.meta.get("level", 1) + 1
    meta = dict(dims=cdims, zlo=czlo, level=lev, config=prob.meta.get("config"))
    return Problem(f"{prob.name}/L{lev}", prob.nc, int(is_c2.sum()), np.asarray(Ac_rowptr, np.int64),
                   np.asarray(Ac_col, np.int32), np.asarray(Ac_val, np.float64), is_c2.astype(np.uint8),
                   None, None, None, prob.nv, B2, Bc2, iters or prob.iters, bs, meta)


def sgs_key(prob: Problem, kind: str = "natural") -> Optional[np.ndarray]:
    """Ordering key (int64 per global row) for the SGS preconditioner's sweeps
    (reading A23: the unknowns of each K block are visited in ascending
    (key, row) order).  'natural': None (row order, the paper's enumeration).
    'color': a proper colouring of the grid graph -- red-black (x + y + z) % 2
    for the 5/7-point scalar stencils, the 8 parity classes (x%2, y%2, z%2) of
    the 27-point node graph for elasticity (all 3 dofs of a node share the
    node's colour) -- so that each sweep has few dependency levels."""
    if kind == "natural":
        return None
    if kind != "color":
        raise KeyError(kind)
    nx, ny, nz = prob.meta["dims"]
    nodes = np.arange(prob.n // prob.block_size)
    x, y, z = nodes % nx, (nodes // nx) % ny, nodes // (nx * ny)
    if prob.block_size == 1:
        col = (x + y + z) % 2
    else:
        col = (x % 2) + 2 * (y % 2) + 4 * (z % 2)
    return np.repeat(col, prob.block_size).astype(np.int64)
