// sgs.cu -- projected symmetric Gauss-Seidel preconditioner M_2 of Alg. 3
// (SURVEY §8f NEXT-1), selected with emin_opts.precond = 1.
//
//   z = Pi M_SGS^{-1} r,  M_SGS^{-1} = (L+D)^{-T} D (L+D)^{-1},  K = L + D + L^T
//
// K is block diagonal over the coarse columns j of W, block j = A(I_j, I_j)
// (Eq. 11blk), so one forward (L+D) solve updates every column at
// once, row by row:
//   u(i,j) = (r(i,j) - sum_{k before i} A(i,k) u(k,j)) / A(i,i)
// and the backward (L+D)^T solve, with v = D u,
//   z(i,j) = (v(i,j) - sum_{k after i} A(k,i) z(k,j)) / A(i,i),  A(k,i) = A(i,k),
// both matrix-free on the W layout exactly like the masked product (P:996-
// 1004: "the symmetric Gauss-Seidel step is then performed matrix-free,
// similar to the A P product").  "before" = ascending (sgs_key, row)
// (reading A23; key NULL = natural row order).
//
// GPU schedule: at setup the F rows get a dependency level (longest chain of
// predecessors in the A_FF graph, by in-place relaxation passes) and are
// bucketed by level; the forward sweep is one kernel per level ascending, the
// backward one per level descending, warp per row, lane per pattern position.
// A colouring key (red-black for 7-point operators, 8 parity classes of the
// 27-point node graph) gives 2-24 levels; the natural order gives O(grid
// diameter) levels.  The pending r update of the previous step is applied by
// the forward kernel (each row exactly once), Pi and the partial r.z by one
// row-parallel kernel.  Single GPU (the sweeps are sequential across ranks).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "emin_internal.cuh"
#include "dist.cuh"

struct SgsPlan {
  int64_t* key = nullptr;        // [nFh] ordering key of each F row (owned, then halo rows)
  int64_t* gid = nullptr;        // [nFh] global F id (the tie-break of the order)
  int32_t* lev = nullptr;        // [nF] dependency level
  int32_t* lvl_rows = nullptr;   // [nF] F rows bucketed by level
  int32_t* lvl_cnt = nullptr;    // [nlev + 1] scratch
  std::vector<int64_t> lvl_ptr;  // host [nlev + 1]
  int64_t nlev = 0;
  double* u = nullptr;           // [nnzW] u, then z in place
  // scalar-path fast sweeps (kernel_path 1): lane per W entry over windows
  // of <= 32 entries built from each level's row list
  const int4* rec = nullptr;     // the scalar path's A_FF records (not owned)
  uint8_t* dir = nullptr;        // [nnzAFF] per record: 0 diagonal, 1 predecessor, 2 successor
  int4* win = nullptr;           // [nwin] {j0 (into lvl_rows), head mask, nent, nrows}
  std::vector<int64_t> win_ptr;  // host [nlev + 1] window range of each level
  // nodal path (kernel_path 2, 3x3 blocks): levels and sweeps per F node
  int nodal = 0;
  const int2* nblk = nullptr;    // {wptr[3K], 3|J_K|} per block (not owned)
  const int64_t* bptr = nullptr;
  const uint8_t* pm8 = nullptr;
  const int64_t* pmoff = nullptr;
  int64_t nFn = 0;
  int32_t max_nb = 0;            // > 27: Galerkin level, sweeps stage the blocks in chunks
  uint8_t* bdir = nullptr;       // [nblk] 0 own node, 1 predecessor node, 2 successor node
  // direction-sorted copy (k_sgs_node_sort; max_nb <= 27): sweeps stage only what they couple
  double* sA = nullptr;          // [9 nblk]
  int2* sblk = nullptr;          // [nblk]
  uint8_t* spm = nullptr;        // byte map, same offsets as pm8
  int32_t* npred = nullptr;      // [nFn]
};

namespace {

constexpr int SGS_MAXC = EMIN_MAX_ROW / 32;   // pattern chunks of 32 lanes

// (key, global F id) order; key and gid cover the owned and the halo rows
// (local ids >= nF, multi-GPU), the global F id = the global row order
__device__ __forceinline__ bool sgs_before(const int64_t* __restrict__ key, const int64_t* __restrict__ gid,
                                           int32_t k, int32_t i) {
  const int64_t a = key[k], b = key[i];
  return a != b ? a < b : gid[k] < gid[i];
}

__global__ void k_sgs_key(int64_t nF, int64_t fbegin, const int64_t* __restrict__ frow,
                          const int64_t* __restrict__ key_own, int64_t* __restrict__ key, int64_t* __restrict__ gid) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nF; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = key_own ? key_own[frow[i]] : 0;
    gid[i] = fbegin + i;
  }
}

// per-unit values (rows, or nodes: stride 3) of the halo units from their
// owners, through the W-layout halo exchange: every W entry of an owned
// unit's first row carries the value's bits, the halo tail brings them back
// (every F row has >= 1 entry)
__global__ void k_sgs_units_to_w(const int64_t* __restrict__ wptr, int64_t nu, int stride,
                                 const int64_t* __restrict__ val64, const int32_t* __restrict__ val32,
                                 double* __restrict__ w) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = val64 ? val64[u] : (int64_t)val32[u];
    const double bits = __longlong_as_double(x);
    for (int64_t e = wptr[stride * u]; e < wptr[stride * u + 1]; ++e) w[e] = bits;
  }
}
__global__ void k_sgs_w_to_units(const int64_t* __restrict__ wptr, int64_t u0, int64_t u1, int stride,
                                 const double* __restrict__ w, int64_t* __restrict__ val64,
                                 int32_t* __restrict__ val32) {
  for (int64_t u = u0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < u1; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = __double_as_longlong(w[wptr[stride * u]]);
    if (val64) val64[u] = x; else val32[u] = (int32_t)x;
  }
}

// one relaxation pass of lev(i) = max over predecessors k of lev(k) + 1
// (in place: a pass propagates along every chain the grid happens to visit
// in order; repeated until no level changes)
__global__ void k_sgs_levels(DevView v, const int64_t* __restrict__ key, const int64_t* __restrict__ gid, int32_t* lev,
                             int32_t* changed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v.nF; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t m = 0;
    for (int64_t q = v.affptr[i]; q < v.affptr[i + 1]; ++q) {
      const int32_t k = v.affcol[q];
      if (k != (int32_t)i && sgs_before(key, gid, k, (int32_t)i)) m = max(m, ((volatile int32_t*)lev)[k] + 1);
    }
    if (m > lev[i]) {
      lev[i] = m;
      *changed = 1;
    }
  }
}

__global__ void k_sgs_maxlev(int64_t n, const int32_t* __restrict__ lev, int32_t* maxlev) {
  int32_t mx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, lev[i]);
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxlev, mx);
}

// level histogram / bucketing with warp-aggregated atomics (few levels =>
// every lane of a warp hits the same counter)
__global__ void k_sgs_count(int64_t nF, const int32_t* __restrict__ lev, int32_t* cnt, int32_t* maxlev) {
  int32_t mx = 0;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < nF; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const int32_t L = i < nF ? lev[i] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, L);
    if (L >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&cnt[L], __popc(grp));
    mx = max(mx, L);
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxlev, mx);
}

// per-level windows on the GPU: rows in level-bucket order j, entry offsets
// pst[j] (exclusive scan of the row lengths); a row whose offset from its
// level's start lies in [S w, S w + S) goes to window w of the level, S = 33 -
// the longest row (<= 8 on the scalar path): a window holds <= 32 entries.
// A window can be empty (rows of lengths 8, 8, 8, 6 with S = 25 all start in
// window 0 and leave window 1 zeroed {0, 0, 0, 0}); the sweeps skip those.
__global__ void k_sgs_wlen(int64_t nF, const int32_t* __restrict__ rows, const int64_t* __restrict__ wptr,
                           int64_t* __restrict__ len) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nF; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = rows[j];
    len[j] = wptr[i + 1] - wptr[i];
  }
}
__global__ void k_sgs_wgather(int64_t nlev, const int64_t* __restrict__ lptr, const int64_t* __restrict__ pst,
                              int64_t* __restrict__ out) {
  for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L <= nlev; L += (int64_t)gridDim.x * blockDim.x)
    out[L] = pst[lptr[L]];
}
__global__ void k_sgs_wfirst(int64_t nF, const int32_t* __restrict__ rows, const int32_t* __restrict__ lev,
                             const int64_t* __restrict__ lptr, const int64_t* __restrict__ base,
                             const int64_t* __restrict__ wbase, const int64_t* __restrict__ pst, int4* __restrict__ win,
                             int S) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nF; j += (int64_t)gridDim.x * blockDim.x) {
    const int L = lev[rows[j]];
    const int64_t wl = (pst[j] - base[L]) / S;
    const bool first = (j == lptr[L]) || ((pst[j - 1] - base[L]) / S != wl);
    if (first) win[wbase[L] + wl].x = (int)j;
  }
}
__global__ void k_sgs_wfill(int64_t nF, const int32_t* __restrict__ rows, const int32_t* __restrict__ lev,
                            const int64_t* __restrict__ base, const int64_t* __restrict__ wbase,
                            const int64_t* __restrict__ pst, const int64_t* __restrict__ len, int4* __restrict__ win,
                            int S) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nF; j += (int64_t)gridDim.x * blockDim.x) {
    const int L = lev[rows[j]];
    int4* w = &win[wbase[L] + (pst[j] - base[L]) / S];
    const int64_t o = pst[j] - pst[w->x];
    atomicOr(&w->y, (int)(1u << (unsigned)o));
    atomicAdd(&w->z, (int)len[j]);
    atomicAdd(&w->w, 1);
  }
}

__global__ void k_sgs_scatter(int64_t nF, const int32_t* __restrict__ lev, int32_t* cursor, int32_t* rows) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < nF; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const int32_t L = i < nF ? lev[i] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, L);
    const int leader = __ffs(grp) - 1;
    int32_t base = 0;
    if (L >= 0 && lane == leader) base = atomicAdd(&cursor[L], __popc(grp));
    base = __shfl_sync(grp, base, leader);
    if (L >= 0) rows[base + __popc(grp & ((1u << lane) - 1u))] = (int32_t)i;
  }
}

// Forward (L+D) solve on the rows of one level (FWD) or backward (L+D)^T
// solve (!FWD), warp per row, lane per pattern position t (chunks of 32).
//   FWD:  x = r [- alpha_pend yb, written back]; u = (x - sum_pred A u) / d
//   !FWD: z = (d u - sum_succ A z) / d, in place over u
// EDGE: the first forward level (rows without predecessors: lev 0 by
// definition) or the last backward level (rows without successors: a
// successor's level exceeds its predecessor's), so no coupling term exists
// and the record loop is skipped (u = x / d, z = v / d)
template <bool FWD, bool EDGE = false, bool TOP = false>
__global__ void __launch_bounds__(256)
k_sgs_sweep(DevView v, const int64_t* __restrict__ key, const int64_t* __restrict__ gid,
            const int32_t* __restrict__ rows, int32_t nrows, double* __restrict__ r, const double* __restrict__ yb,
            double* u) {
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = FWD ? st->pend : 0;
  const double ap = st->alpha_pend;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < nrows; w += nw) {
    const int32_t i = rows[w];
    const int64_t b = v.wptr[i];
    const int nj = (int)(v.wptr[i + 1] - b);
    const double di = v.d[i];
    double acc[SGS_MAXC];
    int32_t jt[SGS_MAXC];
#pragma unroll
    for (int c = 0; c < SGS_MAXC; ++c) {
      const int t = lane + 32 * c;
      jt[c] = t < nj ? v.wcol[b + t] : -1;
      double x = 0.0;
      if (t < nj) {
        if (FWD) {
          x = r[b + t];
          if (pend) { x = x - ap * yb[b + t]; r[b + t] = x; }
        } else {
          x = di * u[b + t];                    // v = D u
        }
      }
      acc[c] = x;
    }
    for (int64_t q = v.affptr[i]; !EDGE && q < v.affptr[i + 1]; ++q) {
      const int32_t k = v.affcol[q];
      if (k == i) continue;
      if (FWD != sgs_before(key, gid, k, i)) continue;   // FWD: predecessors, else successors
      const double a = v.affval[q];
      const int64_t kb = v.wptr[k];
      const int nk = (int)(v.wptr[k + 1] - kb);
#pragma unroll
      for (int c = 0; c < SGS_MAXC; ++c) {
        if (jt[c] >= 0) {
          const int p = lower_bound_i32(v.wcol + kb, nk, jt[c]);
          if (p < nk && v.wcol[kb + p] == jt[c]) acc[c] -= a * u[kb + p];
        }
      }
    }
#pragma unroll
    for (int c = 0; c < SGS_MAXC; ++c) {
      const int t = lane + 32 * c;
      if (t < nj) {
        double ue = acc[c] / di;
        if (TOP) ue = __ddiv_rn(__dmul_rn(di, ue), di);   // no successors: z = (D u) / d
        u[b + t] = ue;
      }
    }
  }
}

// record directions for the windowed sweeps: the scalar path stores row i's
// records diagonal first, then A's column order (k_plan_entries)
__global__ void k_sgs_dir(DevView v, const int64_t* __restrict__ key, const int64_t* __restrict__ gid,
                          uint8_t* __restrict__ dir) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v.nF; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qb = v.affptr[i], qe = v.affptr[i + 1];
    int64_t qd = qb;
    for (int64_t q = qb; q < qe; ++q)
      if (v.affcol[q] == (int32_t)i) { qd = q; break; }
    for (int64_t q = qb; q < qe; ++q) {
      const int64_t dst = (q == qd) ? qb : (q < qd ? q + 1 : q);
      const int32_t k = v.affcol[q];
      dir[dst] = (k == (int32_t)i) ? 0 : (sgs_before(key, gid, k, (int32_t)i) ? 1 : 2);
    }
  }
}

// The same sweep as k_sgs_sweep, lane per W entry (the scalar path's window
// decode of k_spgemm_win2): window {j0, head, nent, nrows} covers rows
// lvl_rows[j0 .. j0 + nrows) of one level, head bit p set where a row starts.
// Records are the scalar path's {a, wptr[k], pm} (pm nibble t = position of
// J_i[t] in J_k), filtered by dir.  Same order of operations as k_sgs_sweep.
// TOP (forward only): the level is the last one, its rows have no
// successors, so the backward solve of those rows, z = (D u) / d, is done
// right here (same operations as the backward kernel) and the backward sweep
// starts one level lower.
template <bool FWD, bool EDGE = false, bool TOP = false>
__global__ void __launch_bounds__(256)
k_sgs_sweep_win(DevView v, const int4* __restrict__ A4, const uint8_t* __restrict__ dir,
                const int4* __restrict__ win, int32_t nwin, const int32_t* __restrict__ rows,
                double* __restrict__ r, const double* __restrict__ yb, double* u) {
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = FWD ? st->pend : 0;
  const double ap = st->alpha_pend;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint8_t want = FWD ? 1 : 2;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int4 h = __ldg(win + w);
    const unsigned H = (unsigned)h.y;
    const int nent = h.z;
    if (nent == 0) continue;     // an empty window (warp-uniform): see k_sgs_wlen
    const bool act = lane < nent;
    const int l = act ? lane : nent - 1;
    const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
    const unsigned hu = H & upto;
    const int rloc = __popc(hu) - 1;
    const int rowbeg = 31 - __clz(hu);
    if (!act) continue;
    const int32_t i = rows[h.x + rloc];
    const int pos = lane - rowbeg;
    const int64_t e = v.wptr[i] + pos;
    const double di = v.d[i];
    double acc;
    if (FWD) {
      double x = r[e];
      if (pend) { x = x - ap * yb[e]; r[e] = x; }
      acc = x;
    } else {
      acc = di * u[e];                          // v = D u
    }
    const int qb = (int)v.affptr[i], qe = (int)v.affptr[i + 1];
    const unsigned sh4 = 4u * (unsigned)pos;
#pragma unroll 4
    for (int q = qb + 1; !EDGE && q < qe; ++q) {   // record qb is the diagonal
      if (__ldg(dir + q) != want) continue;
      const int4 en = __ldg(A4 + q);
      const unsigned sidx = ((unsigned)en.w >> sh4) & 0xFu;
      if (sidx != 0xFu) acc -= __hiloint2double(en.y, en.x) * u[en.z + (int)sidx];
    }
    double ue = acc / di;
    if (TOP) ue = __ddiv_rn(__dmul_rn(di, ue), di);   // z = (v - 0) / d, v = D u
    u[e] = ue;
  }
}

// ---- nodal path: the 3 dof rows of an F node share J and are visited
// consecutively (node-constant keys; reading A23 orders rows by (key, row),
// so node K precedes node I iff (key_K, K) < (key_I, I), and inside a node
// dof e precedes dof d iff e < d).
__global__ void k_sgs_node_key_ok(int64_t nFn, const int64_t* __restrict__ key, int32_t* bad) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < nFn; n += (int64_t)gridDim.x * blockDim.x)
    if (key[3 * n + 1] != key[3 * n] || key[3 * n + 2] != key[3 * n]) atomicExch(bad, 1);
}

__device__ __forceinline__ bool sgs_node_before(const int64_t* __restrict__ key, const int64_t* __restrict__ gid,
                                                int64_t K, int64_t I) {
  const int64_t a = key[3 * K], b = key[3 * I];
  return a != b ? a < b : gid[3 * K] < gid[3 * I];
}

__global__ void k_sgs_node_dir(DevView v, int64_t nFn, const int64_t* __restrict__ bptr,
                               const int64_t* __restrict__ key, const int64_t* __restrict__ gid,
                               uint8_t* __restrict__ bdir) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < nFn; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ab = v.affptr[3 * n];
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    for (int b = 0; b < nb; ++b) {
      const int64_t K = v.affcol[ab + 3 * b] / 3;
      bdir[bb + b] = (K == n) ? 0 : (sgs_node_before(key, gid, K, n) ? 1 : 2);
    }
  }
}

__global__ void k_sgs_node_levels(DevView v, int64_t nFn, const int64_t* __restrict__ bptr,
                                  const uint8_t* __restrict__ bdir, int32_t* lev, int32_t* changed) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < nFn; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ab = v.affptr[3 * n];
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    int32_t m = 0;
    for (int b = 0; b < nb; ++b)
      if (bdir[bb + b] == 1) m = max(m, ((volatile int32_t*)lev)[v.affcol[ab + 3 * b] / 3] + 1);
    if (m > lev[n]) {
      lev[n] = m;
      *changed = 1;
    }
  }
}

// direction-sorted copy of a node's blocks for k_sgs_sweep_nodal_ds: the
// own block first, then the predecessor nodes' blocks, then the successors'
// (each group in A's column order, so the sweeps add them in the same order
// as the unsorted kernel); A block-major (9 doubles), records and byte-map
// rows moved with them; npred per node.  Warp per node, lane per block.
__global__ void k_sgs_node_sort(DevView v, int64_t nFn, const int64_t* __restrict__ bptr,
                                const uint8_t* __restrict__ bdir, const int2* __restrict__ blk,
                                const uint8_t* __restrict__ pm8, const int64_t* __restrict__ pmoff,
                                double* __restrict__ sA, int2* __restrict__ sblk, uint8_t* __restrict__ spm,
                                int32_t* __restrict__ npred, int32_t* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = gw; n < nFn; n += nw) {
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    const int64_t ab = v.affptr[3 * n];
    const int rs = 3 * nb;
    const int nJ = (int)((v.wptr[3 * n + 1] - v.wptr[3 * n]) / 3);
    const uint8_t dl = lane < nb ? bdir[bb + lane] : 3;
    const unsigned below = (1u << lane) - 1u;
    const unsigned ownm = __ballot_sync(0xffffffffu, dl == 0);
    const unsigned prem = __ballot_sync(0xffffffffu, dl == 1);
    const unsigned sucm = __ballot_sync(0xffffffffu, dl == 2);
    const int np = __popc(prem);
    if (lane == 0) {
      npred[n] = np;
      if (__popc(ownm) != 1 || nb > 27) atomicExch(bad, 1);
    }
    if (lane < nb) {
      const int j = dl == 0 ? 0 : dl == 1 ? 1 + __popc(prem & below) : 1 + np + __popc(sucm & below);
      const int b = lane;
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = 0; e < 3; ++e) sA[9 * (bb + j) + 3 * d + e] = v.affval[ab + (int64_t)d * rs + 3 * b + e];
      sblk[bb + j] = blk[bb + b];
      const int64_t po = pmoff[n];
      for (int t = 0; t < nJ; ++t) spm[po + (int64_t)j * nJ + t] = pm8[po + (int64_t)b * nJ + t];
    }
  }
}

// Forward (FWD) / backward sweep over the F nodes of one level, warp per
// node, lane t owns pattern positions t and t + 32 of the node's 3 rows.
//   FWD:  acc_d = x_d - sum_{pred nodes K, e} A_IK[d][e] u_K[e](pos);
//         then the node's own 3x3 lower triangle, row by row:
//         u_d = (acc_d - sum_{e<d} A_II[d][e] u_e) / A_II[d][d]
//   !FWD: acc_d = A_II[d][d] u_d - sum_{succ nodes K, e} A_IK[d][e] z_K[e](pos);
//         z_d = (acc_d - sum_{e>d} A_II[d][e] z_e) / A_II[d][d], d = 2, 1, 0
// (the own-node terms come last, after the other blocks in A's column
// order; the oracle adds them at their column position -- a rounding-order
// difference only).
template <bool FWD, bool EDGE = false, bool TOP = false, bool WIDE = false>
__global__ void __launch_bounds__(256, 4)
k_sgs_sweep_nodal(DevView v, const int2* __restrict__ blk, const int64_t* __restrict__ bptr,
                  const uint8_t* __restrict__ pm8, const int64_t* __restrict__ pmoff,
                  const uint8_t* __restrict__ bdir, const int32_t* __restrict__ nodes, int32_t nnodes,
                  double* __restrict__ r, const double* __restrict__ yb, double* u) {
  // the node's A chunk (block-major, 10-double stride), block records,
  // position bytes and block directions are staged per warp in shared
  // memory with coalesced loads, as in the nodal SpGEMM (k_spgemm_nodal_v2)
  constexpr int MAXB = 27, MAXJ = 32, AST = 10;   // the nodal plan's limits (k_nodal_check)
  __shared__ __align__(16) double s_a[8][MAXB * AST];
  __shared__ int2 s_b[8][MAXB];
  __shared__ __align__(16) uint8_t s_pm[8][MAXB * MAXJ];
  __shared__ uint8_t s_dir[8][MAXB];
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = FWD ? st->pend : 0;
  const double ap = st->alpha_pend;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int t0 = lane, t1 = lane + 32;
  const int s0 = t0 / 3, b0 = t0 - 3 * s0, s1 = t1 / 3, b1 = t1 - 3 * s1;
  const uint8_t want = FWD ? 1 : 2;
  for (int64_t w = gw; w < nnodes; w += nw) {
    const int64_t n = nodes[w];
    const int64_t r3 = 3 * n;
    const int64_t wb = v.wptr[r3];
    const int n3 = (int)(v.wptr[r3 + 1] - wb);
    const int nJ = n3 / 3;
    const bool act0 = t0 < n3, act1 = t1 < n3;
    const bool any1 = n3 > 32;                         // warp-uniform
    const int64_t ab = v.affptr[r3];
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    const int rs = 3 * nb;
    const uint8_t* pm = pm8 + pmoff[n];
    double acc0[3], acc1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t ro = wb + (int64_t)d * n3;
      double x0 = 0.0, x1 = 0.0;
      if (FWD) {
        if (act0) { x0 = r[ro + t0]; if (pend) { x0 = x0 - ap * yb[ro + t0]; r[ro + t0] = x0; } }
        if (act1) { x1 = r[ro + t1]; if (pend) { x1 = x1 - ap * yb[ro + t1]; r[ro + t1] = x1; } }
      } else {
        const double dd = v.d[r3 + d];
        if (act0) x0 = dd * u[ro + t0];                    // v = D u
        if (act1) x1 = dd * u[ro + t1];
      }
      acc0[d] = x0;
      acc1[d] = x1;
    }
    double own[9];
    // nodes with more than MAXB blocks (Galerkin levels, NEXT-4; template
    // WIDE) are staged MAXB blocks at a time, in the same block order
    for (int cl = 0; cl < nb; cl += WIDE ? MAXB : nb) {
    const int c0 = WIDE ? cl : 0;
    const int cb = WIDE ? min(MAXB, nb - c0) : nb, cs = 3 * cb;
    __syncwarp();
    for (int k = lane; k < 9 * cb; k += 32) {
      const int d = k / cs, rem = k - d * cs, bk = rem / 3, e = rem - 3 * bk;
      const int64_t src = WIDE ? ab + (int64_t)d * rs + 3 * c0 + rem : ab + k;
      s_a[wib][bk * AST + d * 3 + e] = __ldg(v.affval + src);
    }
    for (int k = lane; k < cb; k += 32) { s_b[wib][k] = __ldg(blk + bb + c0 + k); s_dir[wib][k] = bdir[bb + c0 + k]; }
    if (!WIDE) {   // the node's byte map is 16-byte aligned and padded (k_nodal_check)
      const uint4* src4 = reinterpret_cast<const uint4*>(pm);
      uint4* dst4 = reinterpret_cast<uint4*>(&s_pm[wib][0]);
      for (int k = lane; k < ((nb * nJ + 15) >> 4); k += 32) dst4[k] = src4[k];
    } else {
      for (int k = lane; k < cb * nJ; k += 32) s_pm[wib][k] = pm[(int64_t)c0 * nJ + k];
    }
    __syncwarp();
    // the node's own block, and the coupled blocks (predecessor nodes in
    // the forward sweep, successors in the backward one) as a bit mask in
    // ascending block order (cb <= 27 < 32 lanes)
    const uint8_t dl = lane < cb ? s_dir[wib][lane] : 3;
    const unsigned ownm = __ballot_sync(0xffffffffu, dl == 0);
    unsigned cm = EDGE ? 0u : __ballot_sync(0xffffffffu, dl == want);
    if (ownm) {
      const int bo = __ffs(ownm) - 1;
      const double2* a2 = reinterpret_cast<const double2*>(&s_a[wib][bo * AST]);
      const double2 a01 = a2[0], a23 = a2[1], a45 = a2[2], a67 = a2[3], a8 = a2[4];
      own[0] = a01.x; own[1] = a01.y; own[2] = a23.x; own[3] = a23.y; own[4] = a45.x;
      own[5] = a45.y; own[6] = a67.x; own[7] = a67.y; own[8] = a8.x;
    }
    // two coupled blocks per round: all their gathers are issued before the
    // FMAs, which run in ascending block order (the order of the plain loop)
    while (cm) {
      const int bA = __ffs(cm) - 1;
      cm &= cm - 1u;
      const int bB = cm ? __ffs(cm) - 1 : -1;
      if (cm) cm &= cm - 1u;
      double yA0[3], yA1[3], yB0[3], yB1[3];
      bool mA0, mA1, mB0 = false, mB1 = false;
      {
        const int2 k = s_b[wib][bA];
        const int p0 = act0 ? s_pm[wib][bA * nJ + s0] : 0xFF;
        const int p1 = (any1 && act1) ? s_pm[wib][bA * nJ + s1] : 0xFF;
        mA0 = p0 != 0xFF;
        mA1 = p1 != 0xFF;
        const int64_t i0 = (int64_t)k.x + 3 * (mA0 ? p0 : 0) + b0, i1 = (int64_t)k.x + 3 * (mA1 ? p1 : 0) + b1;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          yA0[e] = mA0 ? u[i0 + e * k.y] : 0.0;
          yA1[e] = mA1 ? u[i1 + e * k.y] : 0.0;
        }
      }
      if (bB >= 0) {
        const int2 k = s_b[wib][bB];
        const int p0 = act0 ? s_pm[wib][bB * nJ + s0] : 0xFF;
        const int p1 = (any1 && act1) ? s_pm[wib][bB * nJ + s1] : 0xFF;
        mB0 = p0 != 0xFF;
        mB1 = p1 != 0xFF;
        const int64_t i0 = (int64_t)k.x + 3 * (mB0 ? p0 : 0) + b0, i1 = (int64_t)k.x + 3 * (mB1 ? p1 : 0) + b1;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          yB0[e] = mB0 ? u[i0 + e * k.y] : 0.0;
          yB1[e] = mB1 ? u[i1 + e * k.y] : 0.0;
        }
      }
      {
        const double2* a2 = reinterpret_cast<const double2*>(&s_a[wib][bA * AST]);
        const double2 a01 = a2[0], a23 = a2[1], a45 = a2[2], a67 = a2[3], a8 = a2[4];
        const double a[9] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y, a8.x};
        if (mA0) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc0[d] -= a[d * 3 + 0] * yA0[0];
            acc0[d] -= a[d * 3 + 1] * yA0[1];
            acc0[d] -= a[d * 3 + 2] * yA0[2];
          }
        }
        if (mA1) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc1[d] -= a[d * 3 + 0] * yA1[0];
            acc1[d] -= a[d * 3 + 1] * yA1[1];
            acc1[d] -= a[d * 3 + 2] * yA1[2];
          }
        }
      }
      if (bB >= 0) {
        const double2* a2 = reinterpret_cast<const double2*>(&s_a[wib][bB * AST]);
        const double2 a01 = a2[0], a23 = a2[1], a45 = a2[2], a67 = a2[3], a8 = a2[4];
        const double a[9] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y, a8.x};
        if (mB0) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc0[d] -= a[d * 3 + 0] * yB0[0];
            acc0[d] -= a[d * 3 + 1] * yB0[1];
            acc0[d] -= a[d * 3 + 2] * yB0[2];
          }
        }
        if (mB1) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc1[d] -= a[d * 3 + 0] * yB1[0];
            acc1[d] -= a[d * 3 + 1] * yB1[1];
            acc1[d] -= a[d * 3 + 2] * yB1[2];
          }
        }
      }
    }
    }  // chunks
    double o0[3], o1[3];
    if (FWD) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double a0 = acc0[d], a1 = acc1[d];
#pragma unroll
        for (int e = 0; e < 3; ++e)
          if (e < d) { a0 -= own[d * 3 + e] * o0[e]; a1 -= own[d * 3 + e] * o1[e]; }
        o0[d] = a0 / own[d * 3 + d];
        o1[d] = a1 / own[d * 3 + d];
      }
      if (TOP) {                                   // no successor nodes: the node's backward solve
        double u0[3], u1[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) { u0[d] = o0[d]; u1[d] = o1[d]; }
#pragma unroll
        for (int d = 2; d >= 0; --d) {
          const double dd = own[d * 3 + d];
          double a0 = __dmul_rn(dd, u0[d]), a1 = __dmul_rn(dd, u1[d]);
#pragma unroll
          for (int e = 0; e < 3; ++e)
            if (e > d) { a0 -= own[d * 3 + e] * o0[e]; a1 -= own[d * 3 + e] * o1[e]; }
          o0[d] = a0 / dd;
          o1[d] = a1 / dd;
        }
      }
    } else {
#pragma unroll
      for (int d = 2; d >= 0; --d) {
        double a0 = acc0[d], a1 = acc1[d];
#pragma unroll
        for (int e = 0; e < 3; ++e)
          if (e > d) { a0 -= own[d * 3 + e] * o0[e]; a1 -= own[d * 3 + e] * o1[e]; }
        o0[d] = a0 / own[d * 3 + d];
        o1[d] = a1 / own[d * 3 + d];
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t ro = wb + (int64_t)d * n3;
      if (act0) u[ro + t0] = o0[d];
      if (act1) u[ro + t1] = o1[d];
    }
  }
}

template <bool FWD, bool EDGE = false, bool TOP = false>
__global__ void __launch_bounds__(256, 4)
k_sgs_sweep_nodal_ds(DevView v, const int2* __restrict__ blk, const int64_t* __restrict__ bptr,
                     const uint8_t* __restrict__ pm8, const int64_t* __restrict__ pmoff,
                     const int32_t* __restrict__ npred, const double* __restrict__ sA,
                     const int32_t* __restrict__ nodes, int32_t nnodes,
                     double* __restrict__ r, const double* __restrict__ yb, double* u) {
  // the node's own block and the blocks this sweep couples (predecessor
  // nodes forward, successors backward) -- contiguous in the direction-
  // sorted copy of A, records and byte map built at setup (k_sgs_node_sort)
  // -- are staged per warp in shared memory: about half of what the
  // unsorted sweep (k_sgs_sweep_nodal) stages and filters
  constexpr int MAXB = 27, MAXJ = 32, AST = 10;   // the nodal plan's limits (k_nodal_check)
  __shared__ __align__(16) double s_a[8][MAXB * AST];
  __shared__ int2 s_b[8][MAXB];
  __shared__ __align__(16) uint8_t s_pm[8][MAXB * MAXJ];
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = FWD ? st->pend : 0;
  const double ap = st->alpha_pend;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int t0 = lane, t1 = lane + 32;
  const int s0 = t0 / 3, b0 = t0 - 3 * s0, s1 = t1 / 3, b1 = t1 - 3 * s1;
  for (int64_t w = gw; w < nnodes; w += nw) {
    const int64_t n = nodes[w];
    const int64_t r3 = 3 * n;
    const int64_t wb = v.wptr[r3];
    const int n3 = (int)(v.wptr[r3 + 1] - wb);
    const int nJ = n3 / 3;
    const bool act0 = t0 < n3, act1 = t1 < n3;
    const bool any1 = n3 > 32;                         // warp-uniform
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    const int np = npred[n];
    // the node's blocks are stored [own, predecessors, successors] (each
    // group in A's column order): this sweep stages the own block and its
    // coupled group only, cnt blocks, coupled ones from sorted index lo
    const int lo = FWD ? 1 : 1 + np;
    const int cnt = FWD ? 1 + np : nb - np;
    const uint8_t* pm = pm8 + pmoff[n];
    double acc0[3], acc1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t ro = wb + (int64_t)d * n3;
      double x0 = 0.0, x1 = 0.0;
      if (FWD) {
        if (act0) { x0 = r[ro + t0]; if (pend) { x0 = x0 - ap * yb[ro + t0]; r[ro + t0] = x0; } }
        if (act1) { x1 = r[ro + t1]; if (pend) { x1 = x1 - ap * yb[ro + t1]; r[ro + t1] = x1; } }
      } else {
        const double dd = v.d[r3 + d];
        if (act0) x0 = dd * u[ro + t0];                    // v = D u
        if (act1) x1 = dd * u[ro + t1];
      }
      acc0[d] = x0;
      acc1[d] = x1;
    }
    double own[9];
    {
    __syncwarp();
    const double* a0 = sA + 9 * bb;                       // own block
    const double* a1 = sA + 9 * (bb + lo - 1);            // (k >= 9: coupled blocks)
    for (int k = lane; k < 9 * cnt; k += 32) {
      const int j = k / 9, t = k - 9 * j;
      s_a[wib][j * AST + t] = __ldg((k < 9 ? a0 : a1) + k);
    }
    for (int j = lane; j < cnt; j += 32) s_b[wib][j] = __ldg(blk + bb + (j == 0 ? 0 : lo + j - 1));
    for (int k = lane; k < nJ; k += 32) s_pm[wib][k] = pm[k];
    for (int k = lane; k < (cnt - 1) * nJ; k += 32) s_pm[wib][nJ + k] = pm[lo * nJ + k];
    __syncwarp();
    {
      const double2* a2 = reinterpret_cast<const double2*>(&s_a[wib][0]);
      const double2 a01 = a2[0], a23 = a2[1], a45 = a2[2], a67 = a2[3], a8 = a2[4];
      own[0] = a01.x; own[1] = a01.y; own[2] = a23.x; own[3] = a23.y; own[4] = a45.x;
      own[5] = a45.y; own[6] = a67.x; own[7] = a67.y; own[8] = a8.x;
    }
    // coupled blocks 1 .. cnt-1 in ascending order (cnt <= 27)
    unsigned cm = EDGE ? 0u : (((cnt >= 32) ? 0xffffffffu : ((1u << cnt) - 1u)) & ~1u);
    // two coupled blocks per round: all their gathers are issued before the
    // FMAs, which run in ascending block order (the order of the plain loop)
    while (cm) {
      const int bA = __ffs(cm) - 1;
      cm &= cm - 1u;
      const int bB = cm ? __ffs(cm) - 1 : -1;
      if (cm) cm &= cm - 1u;
      double yA0[3], yA1[3], yB0[3], yB1[3];
      bool mA0, mA1, mB0 = false, mB1 = false;
      {
        const int2 k = s_b[wib][bA];
        const int p0 = act0 ? s_pm[wib][bA * nJ + s0] : 0xFF;
        const int p1 = (any1 && act1) ? s_pm[wib][bA * nJ + s1] : 0xFF;
        mA0 = p0 != 0xFF;
        mA1 = p1 != 0xFF;
        const int64_t i0 = (int64_t)k.x + 3 * (mA0 ? p0 : 0) + b0, i1 = (int64_t)k.x + 3 * (mA1 ? p1 : 0) + b1;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          yA0[e] = mA0 ? u[i0 + e * k.y] : 0.0;
          yA1[e] = mA1 ? u[i1 + e * k.y] : 0.0;
        }
      }
      if (bB >= 0) {
        const int2 k = s_b[wib][bB];
        const int p0 = act0 ? s_pm[wib][bB * nJ + s0] : 0xFF;
        const int p1 = (any1 && act1) ? s_pm[wib][bB * nJ + s1] : 0xFF;
        mB0 = p0 != 0xFF;
        mB1 = p1 != 0xFF;
        const int64_t i0 = (int64_t)k.x + 3 * (mB0 ? p0 : 0) + b0, i1 = (int64_t)k.x + 3 * (mB1 ? p1 : 0) + b1;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          yB0[e] = mB0 ? u[i0 + e * k.y] : 0.0;
          yB1[e] = mB1 ? u[i1 + e * k.y] : 0.0;
        }
      }
      {
        const double2* a2 = reinterpret_cast<const double2*>(&s_a[wib][bA * AST]);
        const double2 a01 = a2[0], a23 = a2[1], a45 = a2[2], a67 = a2[3], a8 = a2[4];
        const double a[9] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y, a8.x};
        if (mA0) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc0[d] -= a[d * 3 + 0] * yA0[0];
            acc0[d] -= a[d * 3 + 1] * yA0[1];
            acc0[d] -= a[d * 3 + 2] * yA0[2];
          }
        }
        if (mA1) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc1[d] -= a[d * 3 + 0] * yA1[0];
            acc1[d] -= a[d * 3 + 1] * yA1[1];
            acc1[d] -= a[d * 3 + 2] * yA1[2];
          }
        }
      }
      if (bB >= 0) {
        const double2* a2 = reinterpret_cast<const double2*>(&s_a[wib][bB * AST]);
        const double2 a01 = a2[0], a23 = a2[1], a45 = a2[2], a67 = a2[3], a8 = a2[4];
        const double a[9] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y, a8.x};
        if (mB0) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc0[d] -= a[d * 3 + 0] * yB0[0];
            acc0[d] -= a[d * 3 + 1] * yB0[1];
            acc0[d] -= a[d * 3 + 2] * yB0[2];
          }
        }
        if (mB1) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            acc1[d] -= a[d * 3 + 0] * yB1[0];
            acc1[d] -= a[d * 3 + 1] * yB1[1];
            acc1[d] -= a[d * 3 + 2] * yB1[2];
          }
        }
      }
    }
    }
    double o0[3], o1[3];
    if (FWD) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double a0 = acc0[d], a1 = acc1[d];
#pragma unroll
        for (int e = 0; e < 3; ++e)
          if (e < d) { a0 -= own[d * 3 + e] * o0[e]; a1 -= own[d * 3 + e] * o1[e]; }
        o0[d] = a0 / own[d * 3 + d];
        o1[d] = a1 / own[d * 3 + d];
      }
      if (TOP) {                                   // no successor nodes: the node's backward solve
        double u0[3], u1[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) { u0[d] = o0[d]; u1[d] = o1[d]; }
#pragma unroll
        for (int d = 2; d >= 0; --d) {
          const double dd = own[d * 3 + d];
          double a0 = __dmul_rn(dd, u0[d]), a1 = __dmul_rn(dd, u1[d]);
#pragma unroll
          for (int e = 0; e < 3; ++e)
            if (e > d) { a0 -= own[d * 3 + e] * o0[e]; a1 -= own[d * 3 + e] * o1[e]; }
          o0[d] = a0 / dd;
          o1[d] = a1 / dd;
        }
      }
    } else {
#pragma unroll
      for (int d = 2; d >= 0; --d) {
        double a0 = acc0[d], a1 = acc1[d];
#pragma unroll
        for (int e = 0; e < 3; ++e)
          if (e > d) { a0 -= own[d * 3 + e] * o0[e]; a1 -= own[d * 3 + e] * o1[e]; }
        o0[d] = a0 / own[d * 3 + d];
        o1[d] = a1 / own[d * 3 + d];
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t ro = wb + (int64_t)d * n3;
      if (act0) u[ro + t0] = o0[d];
      if (act1) u[ro + t1] = o1[d];
    }
  }
}

// z <- Pi z and the partial r . z on the nodal path (Q of row 3n shared by
// the node's 3 rows), warp per node
template <int NV>
__global__ void __launch_bounds__(256)
k_sgs_project_nodal(DevView v, int64_t nFn, const double* __restrict__ r, double* __restrict__ z,
                    double* __restrict__ partials) {
  __shared__ double sh[32];
  if (v.st->stopped) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int t0 = lane, t1 = lane + 32;
  double part = 0.0;
  for (int64_t n = gw; n < nFn; n += nw) {
    const int64_t wb = v.wptr[3 * n];
    const int n3 = (int)(v.wptr[3 * n + 1] - wb);
    const bool act0 = t0 < n3, act1 = t1 < n3;
    double q0[NV], q1[NV];
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      q0[m] = act0 ? v.Q[(wb + t0) * NV + m] : 0.0;
      q1[m] = act1 ? v.Q[(wb + t1) * NV + m] : 0.0;
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t ro = wb + (int64_t)d * n3;
      const double z0 = act0 ? z[ro + t0] : 0.0, z1 = act1 ? z[ro + t1] : 0.0;
      double s0v = 0.0, s1v = 0.0;
#pragma unroll
      for (int m = 0; m < NV; ++m) {
        const double dm = warp_sum(fma(q0[m], z0, q1[m] * z1));
        s0v = fma(q0[m], dm, s0v);
        s1v = fma(q1[m], dm, s1v);
      }
      if (act0) { const double zz = z0 - s0v; z[ro + t0] = zz; part = fma(r[ro + t0], zz, part); }
      if (act1) { const double zz = z1 - s1v; z[ro + t1] = zz; part = fma(r[ro + t1], zz, part); }
    }
  }
  const double tot = block_sum(part, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// z <- Pi z (per row, Q_i), partial r . z  (Alg. 3 lines P:840-841)
__global__ void __launch_bounds__(256)
k_sgs_project(DevView v, const double* __restrict__ r, double* __restrict__ z, double* __restrict__ partials) {
  __shared__ double sh[32];
  if (v.st->stopped) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = v.nv;
  double part = 0.0;
  for (int64_t i = gw; i < v.nF; i += nw) {
    const int64_t b = v.wptr[i];
    const int nj = (int)(v.wptr[i + 1] - b);
    double dots[EMIN_NV_MAX];
#pragma unroll
    for (int m = 0; m < EMIN_NV_MAX; ++m) dots[m] = 0.0;
    for (int t = lane; t < nj; t += 32) {
      const double zt = z[b + t];
#pragma unroll
      for (int m = 0; m < EMIN_NV_MAX; ++m)
        if (m < nv) dots[m] = fma(v.Q[(b + t) * nv + m], zt, dots[m]);
    }
#pragma unroll
    for (int m = 0; m < EMIN_NV_MAX; ++m)
      if (m < nv) dots[m] = warp_sum(dots[m]);
    for (int t = lane; t < nj; t += 32) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < EMIN_NV_MAX; ++m)
        if (m < nv) s = fma(v.Q[(b + t) * nv + m], dots[m], s);
      const double zt = z[b + t] - s;
      z[b + t] = zt;
      part = fma(r[b + t], zt, part);
    }
  }
  const double tot = block_sum(part, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// z <- Pi z, partial r . z on the scalar path (nv = 1): lane per W entry on
// the scalar window plan, row sums of q z through shared memory in a fixed
// order (the projection of k_spgemm_win2)
__global__ void __launch_bounds__(256)
k_sgs_project_win(DevView v, const int32_t* __restrict__ rowstart, int64_t nwin, const double* __restrict__ r,
                  double* __restrict__ z, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qz[8][32];
  if (v.st->stopped) return;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part = 0.0;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int r0 = rowstart[w];
    const int nrows = rowstart[w + 1] - r0;
    if (nrows == 0) continue;                          // warp-uniform
    const int myptr = (lane <= nrows) ? (int)v.wptr[r0 + lane] : 0;
    const int base = __shfl_sync(0xffffffffu, myptr, 0);
    const int nent = __shfl_sync(0xffffffffu, myptr, nrows) - base;
    const unsigned H = __reduce_or_sync(0xffffffffu, (lane < nrows) ? (1u << (unsigned)(myptr - base)) : 0u);
    const bool act = lane < nent;
    const int l = act ? lane : nent - 1;
    const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
    const unsigned hu = H & upto;
    const int rowbeg = 31 - __clz(hu);
    const unsigned after = H & ~upto;
    const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
    const int e = base + lane;
    const double qv = act ? v.Q[e] : 0.0;
    const double zv = act ? z[e] : 0.0;
    s_qz[wib][lane] = qv * zv;
    __syncwarp();
    double dot = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p)                       // |J_i| <= 8 on the scalar path
      if (p < rowlen) dot += s_qz[wib][rowbeg + p];
    __syncwarp();
    if (act) {
      const double zt = zv - qv * dot;
      z[e] = zt;
      part = fma(r[e], zt, part);
    }
  }
  const double tot = block_sum(part, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// stage II with a stored z: dw += alpha_pend y_old ; y = z + beta y_old
__global__ void __launch_bounds__(256)
k_sgs_stage2(DevView v, const double* __restrict__ z, double* __restrict__ y, double* __restrict__ dw) {
  const DevState* st = v.st;
  const int stopped = st->stopped;
  const int pendw = st->pendw;
  if (stopped && !pendw) return;
  const double ap = st->alpha_pend;
  const double beta = st->beta;
  const bool first = (st->k_total == 0);
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < v.nnzW; p += (int64_t)gridDim.x * blockDim.x) {
    const double yo = y[p];
    if (pendw) dw[p] = dw[p] + ap * yo;
    if (!stopped) y[p] = first ? z[p] : z[p] + beta * yo;
  }
}

}  // namespace

// ---------------------------------------------------------------- host side
// per-unit values of the halo units (multi-GPU): see k_sgs_units_to_w
static emin_status sgs_halo_units(emin_ctx c, int stride, int64_t* v64, int32_t* v32, double* tmpw, cudaStream_t s) {
  const int SM = emin_num_sms();
  const int64_t nu = c->nF / stride, nuh = c->nFh / stride;
  k_sgs_units_to_w<<<SM * 4, 256, 0, s>>>(c->wptr, nu, stride, v64, v32, tmpw);
  c->launches += 1;
  emin_status st = emin_dist_halo_values(c, tmpw, s);
  if (st != EMIN_OK) return st;
  if (nuh > nu) {
    k_sgs_w_to_units<<<SM * 4, 256, 0, s>>>(c->wptr, nu, nuh, stride, tmpw, v64, v32);
    c->launches += 1;
  }
  return EMIN_OK;
}

emin_status emin_sgs_plan(emin_ctx c, const int64_t* key_own, const int64_t* frow, cudaStream_t s) {
  SgsPlan* p = new SgsPlan();
  c->sgs = p;
  const int64_t nF = c->nF, nFh = c->nFh;
  const int SM = emin_num_sms();
  const int64_t* dkey = key_own;
  int64_t* tmp = nullptr;
  double* tmpw = nullptr;                            // W-layout scratch of the halo exchanges
  if (key_own && !c->opts.inputs_on_device) {
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&tmp, sizeof(int64_t) * std::max<int64_t>(c->m_owned, 1), s));
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(tmp, key_own, sizeof(int64_t) * c->m_owned, cudaMemcpyHostToDevice, s));
    dkey = tmp;
  }
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->key, sizeof(int64_t) * std::max<int64_t>(nFh, 1), s));
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->gid, sizeof(int64_t) * std::max<int64_t>(nFh, 1), s));
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->lev, sizeof(int32_t) * std::max<int64_t>(nFh, 1), s));
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->lvl_rows, sizeof(int32_t) * std::max<int64_t>(nF, 1), s));
  // u carries the halo tail: the sweeps read the halo rows' u / z
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->u, sizeof(double) * std::max<int64_t>(c->nnzWh, 1) + 64, s));
  EMIN_CUDA_TRY(c, cudaMemsetAsync(p->u, 0, sizeof(double) * std::max<int64_t>(c->nnzWh, 1), s));
  int32_t* flag;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&flag, sizeof(int32_t) * 2, s));
  const int64_t fbegin = c->dist ? c->dist->fbeg[c->rank] : 0;
  k_sgs_key<<<SM * 4, 256, 0, s>>>(nF, fbegin, frow, dkey, p->key, p->gid);
  EMIN_CUDA_TRY(c, cudaMemsetAsync(p->lev, 0, sizeof(int32_t) * std::max<int64_t>(nFh, 1), s));
  c->launches += 1;
  if (c->dist) {
    // the halo rows' keys and global ids from their owners (the sweeps
    // order the coupled rows across the partition exactly as on one GPU)
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&tmpw, sizeof(double) * std::max<int64_t>(c->nnzWh, 1), s));
    emin_status st = sgs_halo_units(c, 1, p->key, nullptr, tmpw, s);
    if (st == EMIN_OK) st = sgs_halo_units(c, 1, p->gid, nullptr, tmpw, s);
    if (st != EMIN_OK) return st;
  }
  // nodal path with node-constant keys: levels, buckets and sweeps per F node
  int64_t nunits = nF;                               // rows, or nodes on the nodal path
  if (!(c->opts.debug_flags & EMIN_DBG_SGS_GENERIC) &&
      emin_nodal_plan(c, &p->nblk, &p->bptr, &p->pm8, &p->pmoff, &p->nFn, &p->max_nb)) {
    int32_t hb = 0;
    EMIN_CUDA_TRY(c, cudaMemsetAsync(flag, 0, sizeof(int32_t), s));
    k_sgs_node_key_ok<<<SM * 4, 256, 0, s>>>(p->nFn, p->key, flag);
    c->launches += 1;
    if (c->dist) {                                   // every rank takes the same path
      emin_status st = emin_dist_allreduce_max_i32(c, flag, s);
      if (st != EMIN_OK) return st;
    }
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(&hb, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
    if (!hb) {
      p->nodal = 1;
      nunits = p->nFn;
      EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->bdir, std::max<int64_t>(c->nnzAFF / 9, 1), s));
      k_sgs_node_dir<<<SM * 8, 256, 0, s>>>(c->view(), p->nFn, p->bptr, p->key, p->gid, p->bdir);
      c->launches += 1;
      if (p->max_nb <= 27 && !(c->opts.debug_flags & EMIN_DBG_AB1)) {
        const int64_t nblk = c->nnzAFF / 9;
        int64_t npm = 0;
        EMIN_CUDA_TRY(c, cudaMemcpyAsync(&npm, p->pmoff + p->nFn, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
        EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->sA, sizeof(double) * 9 * std::max<int64_t>(nblk, 1), s));
        EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->sblk, sizeof(int2) * std::max<int64_t>(nblk, 1), s));
        EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->spm, std::max<int64_t>(npm, 16), s));
        EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->npred, sizeof(int32_t) * std::max<int64_t>(p->nFn, 1), s));
        int32_t hbad = 0;
        EMIN_CUDA_TRY(c, cudaMemsetAsync(flag, 0, sizeof(int32_t), s));
        k_sgs_node_sort<<<SM * 8, 256, 0, s>>>(c->view(), p->nFn, p->bptr, p->bdir, p->nblk, p->pm8, p->pmoff, p->sA,
                                               p->sblk, p->spm, p->npred, flag);
        c->launches += 1;
        EMIN_CUDA_TRY(c, cudaMemcpyAsync(&hbad, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
        if (hbad) {                                   // (no own block: keep the unsorted sweeps)
          void* q[] = {p->sA, p->sblk, p->spm, p->npred};
          for (void* x : q) cudaFreeAsync(x, s);
          p->sA = nullptr; p->sblk = nullptr; p->spm = nullptr; p->npred = nullptr;
        }
      }
    }
  }
  // relaxation passes until no level changes (<= longest chain + 1); on
  // several GPUs the halo units' levels are refreshed from their owners
  // after every pass and the pass repeats until no rank changed a level
  for (int64_t pass = 0; pass <= (c->dist ? c->n_global : nunits); ++pass) {
    int32_t h = 0;
    EMIN_CUDA_TRY(c, cudaMemsetAsync(flag, 0, sizeof(int32_t), s));
    if (p->nodal)
      k_sgs_node_levels<<<SM * 8, 256, 0, s>>>(c->view(), p->nFn, p->bptr, p->bdir, p->lev, flag);
    else
      k_sgs_levels<<<SM * 8, 256, 0, s>>>(c->view(), p->key, p->gid, p->lev, flag);
    c->launches += 1;
    if (c->dist) {
      emin_status st = sgs_halo_units(c, p->nodal ? 3 : 1, nullptr, p->lev, tmpw, s);
      if (st == EMIN_OK) st = emin_dist_allreduce_max_i32(c, flag, s);
      if (st != EMIN_OK) return st;
    }
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(&h, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
    if (!h) break;
  }
  if (tmpw) cudaFreeAsync(tmpw, s);
  // bucket the rows by level
  int32_t hmax = 0;
  EMIN_CUDA_TRY(c, cudaMemsetAsync(flag + 1, 0, sizeof(int32_t), s));
  // the highest level (over all ranks: every rank sweeps all global levels)
  k_sgs_maxlev<<<SM * 4, 256, 0, s>>>(nunits, p->lev, flag + 1);
  c->launches += 1;
  if (c->dist) {
    emin_status st = emin_dist_allreduce_max_i32(c, flag + 1, s);
    if (st != EMIN_OK) return st;
  }
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(&hmax, flag + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  p->nlev = (nunits > 0 || c->dist) ? (int64_t)hmax + 1 : 0;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->lvl_cnt, sizeof(int32_t) * (p->nlev + 2), s));
  EMIN_CUDA_TRY(c, cudaMemsetAsync(p->lvl_cnt, 0, sizeof(int32_t) * (p->nlev + 2), s));
  k_sgs_count<<<SM * 4, 256, 0, s>>>(nunits, p->lev, p->lvl_cnt, flag + 1);
  std::vector<int32_t> hc((size_t)p->nlev + 1, 0);
  if (p->nlev)
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(hc.data(), p->lvl_cnt, sizeof(int32_t) * p->nlev, cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  p->lvl_ptr.assign((size_t)p->nlev + 1, 0);
  for (int64_t L = 0; L < p->nlev; ++L) p->lvl_ptr[L + 1] = p->lvl_ptr[L] + hc[L];
  std::vector<int32_t> cur(p->lvl_ptr.begin(), p->lvl_ptr.end() - (p->nlev ? 1 : 0));
  if (p->nlev) {
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(p->lvl_cnt, cur.data(), sizeof(int32_t) * p->nlev, cudaMemcpyHostToDevice, s));
    k_sgs_scatter<<<SM * 4, 256, 0, s>>>(nunits, p->lev, p->lvl_cnt, p->lvl_rows);
  }
  c->launches += 2;
  // scalar path: per-level windows of <= 32 entries (rows never straddle)
  p->rec = p->nodal ? nullptr : emin_scalar_records(c);
  if (p->rec && p->nlev && !(c->opts.debug_flags & EMIN_DBG_SGS_GENERIC)) {
    // windows built on the GPU (k_sgs_w*): only nlev + 1 offsets visit the host
    int64_t *len, *pst, *lptr, *base, *wbase, *tot2, *scr;
    const int64_t nl = p->nlev;
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&len, sizeof(int64_t) * (nF + 1), s));
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&pst, sizeof(int64_t) * (nF + 1), s));
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&lptr, sizeof(int64_t) * (nl + 1), s));
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&base, sizeof(int64_t) * (nl + 1), s));
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&wbase, sizeof(int64_t) * (nl + 1), s));
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&tot2, sizeof(int64_t), s));
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&scr, sizeof(int64_t) * emin_scan_scratch_elems(nF + 1), s));
    k_sgs_wlen<<<SM * 8, 256, 0, s>>>(nF, p->lvl_rows, c->wptr, len);
    EMIN_CUDA_TRY(c, emin_scan_i64(len, pst, nF, tot2, scr, s));
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(pst + nF, tot2, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(lptr, p->lvl_ptr.data(), sizeof(int64_t) * (nl + 1), cudaMemcpyHostToDevice, s));
    k_sgs_wgather<<<1, 256, 0, s>>>(nl, lptr, pst, base);
    std::vector<int64_t> hb((size_t)nl + 1);
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(hb.data(), base, sizeof(int64_t) * (nl + 1), cudaMemcpyDeviceToHost, s));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
    p->win_ptr.assign((size_t)nl + 1, 0);
    const int S = 33 - std::max(1, c->max_row);   // (max_row <= 8 on the scalar path)
    for (int64_t L = 0; L < nl; ++L) p->win_ptr[L + 1] = p->win_ptr[L] + (hb[L + 1] - hb[L] + S - 1) / S;
    const int64_t nw = p->win_ptr[nl];
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(wbase, p->win_ptr.data(), sizeof(int64_t) * (nl + 1), cudaMemcpyHostToDevice, s));
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->win, sizeof(int4) * std::max<int64_t>(nw, 1), s));
    EMIN_CUDA_TRY(c, cudaMemsetAsync(p->win, 0, sizeof(int4) * std::max<int64_t>(nw, 1), s));
    k_sgs_wfirst<<<SM * 8, 256, 0, s>>>(nF, p->lvl_rows, p->lev, lptr, base, wbase, pst, p->win, S);
    k_sgs_wfill<<<SM * 8, 256, 0, s>>>(nF, p->lvl_rows, p->lev, base, wbase, pst, len, p->win, S);
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&p->dir, std::max<int64_t>(c->nnzAFF, 1), s));
    k_sgs_dir<<<SM * 8, 256, 0, s>>>(c->view(), p->key, p->gid, p->dir);
    c->launches += 6;
    void* fr[] = {len, pst, lptr, base, wbase, tot2, scr};
    for (void* q : fr) cudaFreeAsync(q, s);
  } else {
    p->rec = nullptr;
  }
  cudaFreeAsync(flag, s);
  if (tmp) cudaFreeAsync(tmp, s);
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  EMIN_CUDA_TRY(c, cudaGetLastError());
  return EMIN_OK;
}

int64_t emin_sgs_levels(emin_ctx c) { return c->sgs ? c->sgs->nlev : 0; }

// z = Pi M_SGS^{-1} r and the partial sums of r.z (in c->partials); *grid =
// the grid of the projection kernel (= number of partials).  On several
// GPUs the halo rows' u (forward) / z (backward) are refreshed from their
// owners after every level (the sweep is matrix-free like the
// masked product, so it exchanges only values, never the pattern); every
// rank runs all global levels, so the exchanges pair up.
emin_status emin_sgs_enqueue(emin_ctx c, cudaStream_t s, int* grid) {
  SgsPlan* p = c->sgs;
  auto halo = [&]() -> emin_status { return c->dist ? emin_dist_halo_values(c, p->u, s) : EMIN_OK; };
  const DevView v = c->view();
  const int SM = emin_num_sms();
  auto grid_for = [&](int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)SM * 8));
  };
  // the sweeps (no partial sums): 8 CTAs per SM
  const int64_t sweep_per_sm = 8;
  auto sweep_grid = [&](int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)SM * sweep_per_sm));
  };
  if (p->nodal) {
    for (int64_t L = 0; L < p->nlev; ++L) {
      const int64_t n = p->lvl_ptr[L + 1] - p->lvl_ptr[L];
      const int32_t* rows = p->lvl_rows + p->lvl_ptr[L];
      const bool first = L == 0, top = L == p->nlev - 1;
#define NDF(E, T, W) k_sgs_sweep_nodal<true, E, T, W><<<sweep_grid(n), 256, 0, s>>>(v, p->nblk, p->bptr, p->pm8, \
                                                                     p->pmoff, p->bdir, rows, (int32_t)n, c->r, c->yb, p->u)
#define NDS(E, T) k_sgs_sweep_nodal_ds<true, E, T><<<sweep_grid(n), 256, 0, s>>>(v, p->sblk, p->bptr, p->spm, \
                                                     p->pmoff, p->npred, p->sA, rows, (int32_t)n, c->r, c->yb, p->u)
      if (p->max_nb > 27) {
        if (first && top) NDF(true, true, true); else if (first) NDF(true, false, true);
        else if (top) NDF(false, true, true); else NDF(false, false, true);
      } else if (p->sA) {
        if (first && top) NDS(true, true); else if (first) NDS(true, false);
        else if (top) NDS(false, true); else NDS(false, false);
      } else {
        if (first && top) NDF(true, true, false); else if (first) NDF(true, false, false);
        else if (top) NDF(false, true, false); else NDF(false, false, false);
      }
#undef NDF
#undef NDS
      const emin_status hs = halo();
      if (hs != EMIN_OK) return hs;
    }
    for (int64_t L = p->nlev - 2; L >= 0; --L) {     // the top level was solved by the forward launch
      const int64_t n = p->lvl_ptr[L + 1] - p->lvl_ptr[L];
      if (p->sA)
        k_sgs_sweep_nodal_ds<false><<<sweep_grid(n), 256, 0, s>>>(v, p->sblk, p->bptr, p->spm, p->pmoff, p->npred,
                                                                p->sA, p->lvl_rows + p->lvl_ptr[L], (int32_t)n,
                                                                c->r, c->yb, p->u);
      else if (p->max_nb > 27)
        k_sgs_sweep_nodal<false, false, false, true><<<sweep_grid(n), 256, 0, s>>>(
            v, p->nblk, p->bptr, p->pm8, p->pmoff, p->bdir, p->lvl_rows + p->lvl_ptr[L], (int32_t)n, c->r, c->yb, p->u);
      else
        k_sgs_sweep_nodal<false><<<sweep_grid(n), 256, 0, s>>>(v, p->nblk, p->bptr, p->pm8, p->pmoff, p->bdir,
                                                            p->lvl_rows + p->lvl_ptr[L], (int32_t)n, c->r, c->yb, p->u);
      if (L > 0) {
        const emin_status hs = halo();
        if (hs != EMIN_OK) return hs;
      }
    }
    const int g = grid_for(p->nFn);
    switch (c->nv) {
#define PN(N) case N: k_sgs_project_nodal<N><<<g, 256, 0, s>>>(v, p->nFn, c->r, p->u, c->partials); break;
      PN(1) PN(2) PN(3) PN(4) PN(5) PN(6) PN(7) PN(8)
#undef PN
    }
    *grid = g;
    return EMIN_OK;
  }
  if (p->rec) {
    for (int64_t L = 0; L < p->nlev; ++L) {
      const int64_t n = p->win_ptr[L + 1] - p->win_ptr[L];
      const bool first = L == 0, top = L == p->nlev - 1;
#define WF(E, T) k_sgs_sweep_win<true, E, T><<<grid_for(n), 256, 0, s>>>(v, p->rec, p->dir, p->win + p->win_ptr[L], \
                                                                        (int32_t)n, p->lvl_rows, c->r, c->yb, p->u)
      if (first && top) WF(true, true); else if (first) WF(true, false); else if (top) WF(false, true);
      else WF(false, false);
#undef WF
      const emin_status hs = halo();
      if (hs != EMIN_OK) return hs;
    }
    for (int64_t L = p->nlev - 2; L >= 0; --L) {     // the top level was solved by the forward launch
      const int64_t n = p->win_ptr[L + 1] - p->win_ptr[L];
      k_sgs_sweep_win<false><<<grid_for(n), 256, 0, s>>>(v, p->rec, p->dir, p->win + p->win_ptr[L], (int32_t)n,
                                                        p->lvl_rows, c->r, c->yb, p->u);
      if (L > 0) {
        const emin_status hs = halo();
        if (hs != EMIN_OK) return hs;
      }
    }
  } else {
    for (int64_t L = 0; L < p->nlev; ++L) {
      const int64_t n = p->lvl_ptr[L + 1] - p->lvl_ptr[L];
      const int32_t* rows = p->lvl_rows + p->lvl_ptr[L];
      const bool first = L == 0, top = L == p->nlev - 1;
#define GF(E, T) k_sgs_sweep<true, E, T><<<grid_for(n), 256, 0, s>>>(v, p->key, p->gid, rows, (int32_t)n, c->r, \
                                                                   c->yb, p->u)
      if (first && top) GF(true, true); else if (first) GF(true, false); else if (top) GF(false, true);
      else GF(false, false);
#undef GF
      const emin_status hs = halo();
      if (hs != EMIN_OK) return hs;
    }
    for (int64_t L = p->nlev - 2; L >= 0; --L) {     // the top level was solved by the forward launch
      const int64_t n = p->lvl_ptr[L + 1] - p->lvl_ptr[L];
      k_sgs_sweep<false><<<grid_for(n), 256, 0, s>>>(v, p->key, p->gid, p->lvl_rows + p->lvl_ptr[L], (int32_t)n,
                                                    c->r, c->yb, p->u);
      if (L > 0) {
        const emin_status hs = halo();
        if (hs != EMIN_OK) return hs;
      }
    }
  }
  int64_t nwin = 0;
  const int32_t* rowstart = emin_scalar_windows(c, &nwin);
  if (rowstart && p->rec) {
    const int g = grid_for(nwin);
    k_sgs_project_win<<<g, 256, 0, s>>>(v, rowstart, nwin, c->r, p->u, c->partials);
    *grid = g;
    return EMIN_OK;
  }
  const int g = grid_for(c->nF);
  k_sgs_project<<<g, 256, 0, s>>>(v, c->r, p->u, c->partials);
  *grid = g;
  return EMIN_OK;
}

void emin_sgs_stage2(emin_ctx c, cudaStream_t s) {
  const int SM = emin_num_sms();
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((c->nnzW + 255) / 256, (int64_t)SM * 8));
  k_sgs_stage2<<<g, 256, 0, s>>>(c->view(), c->sgs->u, c->y, c->dw);
}

void emin_sgs_free(emin_ctx c) {
  SgsPlan* p = c->sgs;
  if (!p) return;
  void* ptrs[] = {p->key, p->gid, p->lev, p->lvl_rows, p->lvl_cnt, p->u, p->dir, p->win, p->bdir,
                  p->sA, p->sblk, p->spm, p->npred};
  for (void* q : ptrs)
    if (q) cudaFreeAsync(q, c->stream);
  delete p;
  c->sgs = nullptr;
}
