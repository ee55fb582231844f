// setup.cu -- emin_setup: validation, F-row index preparation, Alg. 2
// (EMIN_SetUp) per F row, r0 and E0 (start of Alg. 3).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "emin_internal.cuh"
#include "dist.cuh"
#include "masked.cuh"

namespace {

thread_local std::string g_setup_error;

// ------------------------------------------------------------ index prep
__global__ void k_coarse_flags(const uint8_t* __restrict__ isc, int64_t n, int64_t* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    out[r] = isc[r] ? 1 : 0;
}

struct RowsArgs {
  int64_t m, row_begin, row_end, n_global, nc_global;
  int64_t fbegin;                 // global F id of the first owned F row
  const int64_t* Arp; const int32_t* Acol; const double* Aval;
  const uint8_t* isc; const int64_t* cidx;   // exclusive scan of is_coarse (global)
  const int64_t* Prp; const int32_t* Pcol; const double* Pval;
  int64_t* cnt_ff; int64_t* cnt_fc; int64_t* cnt_w;  // per owned F row
  double* d; double* dcc;          // F-row diagonal; C-row diagonal (per owned row, 0 for F)
  int32_t* err; int64_t* err_row; int32_t* max_row;
};

__device__ __forceinline__ void raise_err(const RowsArgs& a, int32_t bit, int64_t row) {
  atomicOr(a.err, bit);
  atomicMin((unsigned long long*)a.err_row, (unsigned long long)row);
}

// Validation + per-row counts (one thread per owned row; setup only).
__global__ void k_rows(RowsArgs a) {
  int32_t wmax = 0;                           // longest pattern row seen by this thread
  for (int64_t rl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rl < a.m;
       rl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = a.row_begin + rl;
    const bool coarse = a.isc[r] != 0;
    const int64_t fl = (r - a.cidx[r]) - a.fbegin;   // local F id (valid if !coarse)
    // ---- A row (no early exit: the loads of a row are independent, the
    // error bits and the first bad row are the same)
    const int64_t qb = a.Arp[rl] - a.Arp[0], qe = a.Arp[rl + 1] - a.Arp[0];
    if (qe < qb) { raise_err(a, EF_CSR, r); continue; }
    int64_t nff = 0, nfc = 0;
    double diag = 0.0;
    bool has_diag = false, bad = false, nonfin = false;
    int32_t prev = -1;
#pragma unroll 4
    for (int64_t q = qb; q < qe; ++q) {
      const int32_t c = a.Acol[q];
      const double v = a.Aval[q];
      const bool ok = c >= 0 && c < a.n_global && c > prev;
      bad |= !ok;
      prev = c;
      nonfin |= !isfinite(v);
      if (c == r) { diag = v; has_diag = true; }
      if (ok) { if (a.isc[c]) ++nfc; else ++nff; }
    }
    if (bad) { raise_err(a, EF_CSR, r); continue; }
    if (nonfin) raise_err(a, EF_NONFINITE, r);
    if (coarse) {
      a.dcc[rl] = diag;
    } else {
      a.dcc[rl] = 0.0;
      if (!has_diag || !(diag > 0.0)) raise_err(a, EF_DIAG, r);
      a.d[fl] = diag;
      a.cnt_ff[fl] = nff;
      a.cnt_fc[fl] = nfc;
    }
    // ---- P row
    const int64_t pb = a.Prp[rl] - a.Prp[0], pe = a.Prp[rl + 1] - a.Prp[0];
    const int64_t len = pe - pb;
    if (len < 0) { raise_err(a, EF_PATTERN, r); continue; }
    if (coarse) {
      if (len != 1 || a.Pcol[pb] != (int32_t)a.cidx[r] || (a.Pval && a.Pval[pb] != 1.0))
        raise_err(a, EF_PATTERN, r);
    } else {
      if (len == 0) raise_err(a, EF_PATTERN, r);
      if (len > EMIN_MAX_ROW) raise_err(a, EF_ROWLEN, r);
      int32_t pp = -1;
      bool pbad = false, pnf = false;
#pragma unroll 4
      for (int64_t q = pb; q < pe; ++q) {
        const int32_t c = a.Pcol[q];
        pbad |= !(c >= 0 && c < a.nc_global && c > pp);
        pp = c;
        if (a.Pval) pnf |= !isfinite(a.Pval[q]);
      }
      if (pbad) raise_err(a, EF_PATTERN, r);
      if (pnf) raise_err(a, EF_NONFINITE, r);
      a.cnt_w[fl] = len;
      wmax = max(wmax, (int32_t)(len < INT_MAX ? len : INT_MAX));
    }
  }
  // one atomic per warp for the longest row (not one per F row)
  wmax = __reduce_max_sync(0xffffffffu, wmax);
  if ((threadIdx.x & 31) == 0 && wmax > 0) atomicMax(a.max_row, wmax);
}

__global__ void k_check_B(int64_t m, int64_t row_begin, int32_t nv, const uint8_t* __restrict__ isc,
                          const int64_t* __restrict__ cidx, const double* __restrict__ B,
                          const double* __restrict__ Bc, int64_t nc, int32_t* err, int64_t* err_row) {
  const int64_t tot = m * nv;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rl = e / nv;
    const int mm = (int)(e % nv);
    const int64_t r = row_begin + rl;
    const double b = B[e];
    if (!isfinite(b)) { atomicOr(err, EF_NONFINITE); atomicMin((unsigned long long*)err_row, (unsigned long long)r); }
    if (isc[r] && Bc[cidx[r] * nv + mm] != b) {
      atomicOr(err, EF_BC);
      atomicMin((unsigned long long*)err_row, (unsigned long long)r);
    }
  }
  const int64_t tc = nc * nv;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tc; e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(Bc[e])) atomicOr(err, EF_NONFINITE);
}

struct FillArgs {
  int64_t m, row_begin, row_end, fbegin, nF;
  const int64_t* Arp; const int32_t* Acol; const double* Aval;
  const uint8_t* isc; const int64_t* cidx;
  const int64_t* Prp; const int32_t* Pcol; const double* Pval;
  const int64_t* wptr; const int64_t* affptr; const int64_t* afcptr;
  int32_t* wcol; double* what; int64_t* pofs;
  int32_t* affcol; double* affval; int32_t* afccol; double* afcval;
  int64_t* frow;   // local F id -> local row
  const int64_t* hpos;   // multi-GPU: halo slot of a global F id (null on one GPU)
  int32_t* adiag;  // position of A(i,i) in A_FF row i (the record plan puts it first)
};

// F rows: copy the pattern into the W layout, split A into A_FF (local F
// ids) and A_FC (coarse ids).  One warp per owned row (coalesced copies).
// Groups of FILL_G lanes per row; loops have warp-uniform trip counts because
// of the warp-wide ballots.
constexpr int FILL_G = 8;
__global__ void k_fill(FillArgs a) {
  const int lane = threadIdx.x & 31;
  const int lg = lane & (FILL_G - 1);
  const int gshift = lane & ~(FILL_G - 1);
  const unsigned gmask = ((1u << FILL_G) - 1u) << gshift;
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / FILL_G;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / FILL_G;
  for (int64_t rl = gid; __any_sync(0xffffffffu, rl < a.m); rl += ng) {
    bool act = rl < a.m;
    const int64_t r = a.row_begin + (act ? rl : 0);
    if (act && a.isc[r]) act = false;
    const int64_t fl = act ? (r - a.cidx[r]) - a.fbegin : 0;
    int64_t qb = 0, qe = 0, off_ff = 0, off_fc = 0;
    if (act) {
      if (lg == 0) { a.frow[fl] = rl; a.pofs[fl] = a.Prp[rl] - a.Prp[0]; }
      const int64_t pb = a.Prp[rl] - a.Prp[0];
      const int64_t wb = a.wptr[fl];
      const int len = (int)(a.wptr[fl + 1] - wb);
      for (int t = lg; t < len; t += FILL_G) {
        a.wcol[wb + t] = a.Pcol[pb + t];
        a.what[wb + t] = a.Pval ? a.Pval[pb + t] : 0.0;
      }
      qb = a.Arp[rl] - a.Arp[0];
      qe = a.Arp[rl + 1] - a.Arp[0];
      off_ff = a.affptr[fl];
      off_fc = a.afcptr[fl];
    }
    for (int64_t q0 = qb; __any_sync(0xffffffffu, q0 < qe); q0 += FILL_G) {
      const int64_t q = q0 + lg;
      const bool valid = q < qe;
      const int32_t c = valid ? a.Acol[q] : 0;
      const double v = valid ? a.Aval[q] : 0.0;
      const bool coarse = valid && a.isc[c];
      const bool fine = valid && !coarse;
      const unsigned mf = __ballot_sync(0xffffffffu, fine) & gmask;
      const unsigned mc = __ballot_sync(0xffffffffu, coarse) & gmask;
      const unsigned lt = (1u << lane) - 1u;
      if (fine) {
        const int64_t gF = (int64_t)c - a.cidx[c];
        int64_t loc = gF - a.fbegin;                          // owned row
        if (loc < 0 || loc >= a.nF) loc = a.nF + a.hpos[gF];  // halo row (multi-GPU)
        const int64_t pos = off_ff + __popc(mf & lt);
        a.affcol[pos] = (int32_t)loc;
        a.affval[pos] = v;
        if (loc == fl) a.adiag[fl] = (int32_t)(pos - a.affptr[fl]);
      }
      if (coarse) {
        const int64_t pos = off_fc + __popc(mc & lt);
        a.afccol[pos] = (int32_t)a.cidx[c];
        a.afcval[pos] = v;
      }
      off_ff += __popc(mf);
      off_fc += __popc(mc);
    }
  }
}

// ------------------------------------------------------------ Alg. 2
// One warp per owned F row i (P:626-659 with readings A5, A6):
//   M = B_c(J_i,:) (nj x nv), r = b_i - M^T w^_i,
//   QR branch (nj >= nv, rank(R) = nv): M = Q R by twice-iterated
//     classical Gram-Schmidt (an economy QR; Pi depends only on range(M)),
//     delta = Q R^{-T} r (least-norm solution of M^T delta = r);
//   SVD branch otherwise: one-sided Jacobi SVD of M, k = #{s > tol s_max},
//     Q = U(:,1:k), delta = U_k S_k^{-1} V_k^T r.
//   w0 = w^ + delta ; Q stored row-major per entry, zero padded to nv.
template <int MAXC>
__global__ void __launch_bounds__(128)
k_alg2(DevView v, const double* __restrict__ Bc, const double* __restrict__ B,
       const int64_t* __restrict__ frow, const double* __restrict__ what, double tol,
       double* __restrict__ Qout, double* __restrict__ w0, unsigned long long* counters,
       const uint8_t* __restrict__ only = nullptr) {
  __shared__ double Rs[4][EMIN_NV_MAX][EMIN_NV_MAX];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = v.nv;
  double (*R)[EMIN_NV_MAX] = Rs[wib];
  for (int64_t i = gw; i < v.nF; i += nw) {
    if (only && !only[i / 3]) continue;          // (node-level fallback: flagged nodes only)
    const int64_t b = v.wptr[i];
    const int nj = (int)(v.wptr[i + 1] - b);
    const int64_t rl = frow[i];
    int32_t jj[MAXC];
    double wh[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int t = lane + 32 * c;
      jj[c] = (t < nj) ? v.wcol[b + t] : 0;
      wh[c] = (t < nj) ? what[b + t] : 0.0;
    }
    auto Mval = [&](int c, int m) -> double {
      return (lane + 32 * c < nj) ? __ldg(Bc + (int64_t)jj[c] * nv + m) : 0.0;
    };
    double rv[EMIN_NV_MAX];
#pragma unroll
    for (int m = 0; m < EMIN_NV_MAX; ++m) {
      rv[m] = 0.0;
      if (m < nv) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) s = fma(Mval(c, m), wh[c], s);
        rv[m] = B[rl * nv + m] - warp_sum(s);
      }
    }
    double q[MAXC][EMIN_NV_MAX];
    double delta[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) delta[c] = 0.0;
    bool qr_ok = false;
    int krank = 0;
    if (nj >= nv) {
      // ---- CGS2 QR
#pragma unroll
      for (int j = 0; j < EMIN_NV_MAX; ++j) {
        if (j >= nv) break;
        double vc[MAXC];
#pragma unroll
        for (int c = 0; c < MAXC; ++c) vc[c] = Mval(c, j);
        double rcol[EMIN_NV_MAX];
#pragma unroll
        for (int l = 0; l < EMIN_NV_MAX; ++l) rcol[l] = 0.0;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
          for (int l = 0; l < EMIN_NV_MAX; ++l) {
            if (l < j) {
              double s = 0.0;
#pragma unroll
              for (int c = 0; c < MAXC; ++c) s = fma(q[c][l], vc[c], s);
              const double h = warp_sum(s);
              rcol[l] += h;
#pragma unroll
              for (int c = 0; c < MAXC; ++c) vc[c] = fma(-h, q[c][l], vc[c]);
            }
          }
        }
        double s2 = 0.0;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) s2 = fma(vc[c], vc[c], s2);
        const double nrm = sqrt(warp_sum(s2));
        rcol[j] = nrm;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) q[c][j] = (nrm > 0.0) ? vc[c] / nrm : 0.0;
        if (lane == 0) {
#pragma unroll
          for (int l = 0; l < EMIN_NV_MAX; ++l) if (l <= j) R[l][j] = rcol[l];
        }
      }
      __syncwarp();
      double rmax = 0.0, rmin = INFINITY;
      for (int j = 0; j < nv; ++j) {
        const double a = fabs(R[j][j]);
        rmax = fmax(rmax, a);
        rmin = fmin(rmin, a);
      }
      qr_ok = (rmax > 0.0) && (rmin > tol * rmax);
      if (qr_ok) {
        // R^T u = r (forward substitution), delta = Q u
        double u[EMIN_NV_MAX];
#pragma unroll
        for (int j = 0; j < EMIN_NV_MAX; ++j) {
          u[j] = 0.0;
          if (j < nv) {
            double s = rv[j];
#pragma unroll
            for (int l = 0; l < EMIN_NV_MAX; ++l) if (l < j) s -= R[l][j] * u[l];
            u[j] = s / R[j][j];
          }
        }
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < EMIN_NV_MAX; ++j) if (j < nv) s = fma(q[c][j], u[j], s);
          delta[c] = s;
        }
        krank = nv;
      }
      __syncwarp();
    }
    if (!qr_ok) {
      // ---- one-sided Jacobi SVD; V lives in shared memory (R slot reused)
      double (*V)[EMIN_NV_MAX] = R;
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
#pragma unroll
        for (int j = 0; j < EMIN_NV_MAX; ++j) q[c][j] = (j < nv) ? Mval(c, j) : 0.0;
      if (lane < EMIN_NV_MAX)
        for (int j = 0; j < EMIN_NV_MAX; ++j) V[lane][j] = (lane == j) ? 1.0 : 0.0;
      __syncwarp();
      for (int sweep = 0; sweep < 100; ++sweep) {
        bool rotated = false;
#pragma unroll
        for (int p = 0; p < EMIN_NV_MAX - 1; ++p) {
#pragma unroll
          for (int qq = p + 1; qq < EMIN_NV_MAX; ++qq) {
            if (qq < nv) {
              double sa = 0.0, sb = 0.0, sc = 0.0;
#pragma unroll
              for (int c = 0; c < MAXC; ++c) {
                sa = fma(q[c][p], q[c][p], sa);
                sb = fma(q[c][qq], q[c][qq], sb);
                sc = fma(q[c][p], q[c][qq], sc);
              }
              const double a = warp_sum(sa), bb = warp_sum(sb), cc = warp_sum(sc);
              if (cc != 0.0 && fabs(cc) > 1e-15 * sqrt(a * bb)) {
                rotated = true;
                const double zeta = (bb - a) / (2.0 * cc);
                const double tt = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
#pragma unroll
                for (int c = 0; c < MAXC; ++c) {
                  const double up = q[c][p], uq = q[c][qq];
                  q[c][p] = cs * up - sn * uq;
                  q[c][qq] = sn * up + cs * uq;
                }
                if (lane < nv) {
                  const double vp = V[lane][p], vq = V[lane][qq];
                  V[lane][p] = cs * vp - sn * vq;
                  V[lane][qq] = sn * vp + cs * vq;
                }
                __syncwarp();
              }
            }
          }
        }
        if (!rotated) break;
      }
      double sig[EMIN_NV_MAX];
      double smax = 0.0;
#pragma unroll
      for (int j = 0; j < EMIN_NV_MAX; ++j) {
        sig[j] = 0.0;
        if (j < nv) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < MAXC; ++c) s = fma(q[c][j], q[c][j], s);
          sig[j] = sqrt(warp_sum(s));
          smax = fmax(smax, sig[j]);
        }
      }
      int ord[EMIN_NV_MAX];
      for (int j = 0; j < nv; ++j) ord[j] = j;
      for (int a = 1; a < nv; ++a)
        for (int bq = a; bq > 0 && sig[ord[bq]] > sig[ord[bq - 1]]; --bq) {
          const int tmp = ord[bq]; ord[bq] = ord[bq - 1]; ord[bq - 1] = tmp;
        }
      double qn[MAXC][EMIN_NV_MAX];
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
#pragma unroll
        for (int j = 0; j < EMIN_NV_MAX; ++j) qn[c][j] = 0.0;
      for (int a = 0; a < nv; ++a) {
        const int ja = ord[a];
        double sj = 0.0;
        double ucol[MAXC];
#pragma unroll
        for (int j = 0; j < EMIN_NV_MAX; ++j)
          if (j == ja) {
            sj = sig[j];
#pragma unroll
            for (int c = 0; c < MAXC; ++c) ucol[c] = q[c][j];
          }
        if (!(smax > 0.0 && sj > tol * smax)) continue;
        double vr = 0.0;
        for (int l = 0; l < nv; ++l) vr += V[l][ja] * rv[l];
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          const double u = ucol[c] / sj;
#pragma unroll
          for (int j = 0; j < EMIN_NV_MAX; ++j) if (j == krank) qn[c][j] = u;
          delta[c] = fma(u, vr / sj, delta[c]);
        }
        ++krank;
      }
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
#pragma unroll
        for (int j = 0; j < EMIN_NV_MAX; ++j) q[c][j] = qn[c][j];
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int t = lane + 32 * c;
      if (t < nj) {
#pragma unroll
        for (int j = 0; j < EMIN_NV_MAX; ++j) if (j < nv) Qout[(b + t) * nv + j] = q[c][j];
        w0[b + t] = wh[c] + delta[c];
      }
    }
    if (lane == 0) {
      if (!qr_ok) atomicAdd(counters + 0, 1ull);
      if (nj == krank) atomicAdd(counters + 1, 1ull);
    }
    __syncwarp();
  }
}

// Alg. 2 on the nodal path: the 3 rows of an F node share J, hence M = B_c(J,:)
// and its QR; one warp per node factors M once (the same CGS2 operations as
// k_alg2, so Q and R are bitwise the per-row ones) and solves the 3 right-hand
// sides.  Nodes whose QR is rank deficient are flagged and redone row by row
// by k_alg2 (SVD branch).
template <int MAXC>
__global__ void __launch_bounds__(128)
k_alg2_nodal(DevView v, const double* __restrict__ Bc, const double* __restrict__ B,
             const int64_t* __restrict__ frow, const double* __restrict__ what, double tol,
             double* __restrict__ Qout, double* __restrict__ w0, unsigned long long* counters,
             uint8_t* __restrict__ flag) {
  __shared__ double Rs[4][EMIN_NV_MAX][EMIN_NV_MAX];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = v.nv;
  double (*R)[EMIN_NV_MAX] = Rs[wib];
  unsigned long long frozen = 0, nflag = 0;
  for (int64_t nd = gw; nd < v.nF / 3; nd += nw) {
    const int64_t i0 = 3 * nd;
    const int64_t b0 = v.wptr[i0];
    const int nj = (int)(v.wptr[i0 + 1] - b0);
    int32_t jj[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int t = lane + 32 * c;
      jj[c] = (t < nj) ? v.wcol[b0 + t] : 0;
    }
    auto Mval = [&](int c, int m) -> double {
      return (lane + 32 * c < nj) ? __ldg(Bc + (int64_t)jj[c] * nv + m) : 0.0;
    };
    double q[MAXC][EMIN_NV_MAX];
    bool qr_ok = false;
    if (nj >= nv) {
#pragma unroll
      for (int j = 0; j < EMIN_NV_MAX; ++j) {
        if (j >= nv) break;
        double vc[MAXC];
#pragma unroll
        for (int c = 0; c < MAXC; ++c) vc[c] = Mval(c, j);
        double rcol[EMIN_NV_MAX];
#pragma unroll
        for (int l = 0; l < EMIN_NV_MAX; ++l) rcol[l] = 0.0;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
          for (int l = 0; l < EMIN_NV_MAX; ++l) {
            if (l < j) {
              double s = 0.0;
#pragma unroll
              for (int c = 0; c < MAXC; ++c) s = fma(q[c][l], vc[c], s);
              const double h = warp_sum(s);
              rcol[l] += h;
#pragma unroll
              for (int c = 0; c < MAXC; ++c) vc[c] = fma(-h, q[c][l], vc[c]);
            }
          }
        }
        double s2 = 0.0;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) s2 = fma(vc[c], vc[c], s2);
        const double nrm = sqrt(warp_sum(s2));
        rcol[j] = nrm;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) q[c][j] = (nrm > 0.0) ? vc[c] / nrm : 0.0;
        if (lane == 0) {
#pragma unroll
          for (int l = 0; l < EMIN_NV_MAX; ++l) if (l <= j) R[l][j] = rcol[l];
        }
      }
      __syncwarp();
      double rmax = 0.0, rmin = INFINITY;
      for (int j = 0; j < nv; ++j) {
        const double a = fabs(R[j][j]);
        rmax = fmax(rmax, a);
        rmin = fmin(rmin, a);
      }
      qr_ok = (rmax > 0.0) && (rmin > tol * rmax);
    }
    if (!qr_ok) {                                 // SVD branch: row by row (k_alg2)
      if (lane == 0) { flag[nd] = 1; ++nflag; }
      __syncwarp();
      continue;
    }
    for (int d = 0; d < 3; ++d) {
      const int64_t i = i0 + d;
      const int64_t b = v.wptr[i];
      const int64_t rl = frow[i];
      double wh[MAXC];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
        wh[c] = (t < nj) ? what[b + t] : 0.0;
      }
      double rv[EMIN_NV_MAX];
#pragma unroll
      for (int m = 0; m < EMIN_NV_MAX; ++m) {
        rv[m] = 0.0;
        if (m < nv) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < MAXC; ++c) s = fma(Mval(c, m), wh[c], s);
          rv[m] = B[rl * nv + m] - warp_sum(s);
        }
      }
      double u[EMIN_NV_MAX];
#pragma unroll
      for (int j = 0; j < EMIN_NV_MAX; ++j) {
        u[j] = 0.0;
        if (j < nv) {
          double s = rv[j];
#pragma unroll
          for (int l = 0; l < EMIN_NV_MAX; ++l) if (l < j) s -= R[l][j] * u[l];
          u[j] = s / R[j][j];
        }
      }
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
        if (t < nj) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < EMIN_NV_MAX; ++j) if (j < nv) s = fma(q[c][j], u[j], s);
#pragma unroll
          for (int j = 0; j < EMIN_NV_MAX; ++j) if (j < nv) Qout[(b + t) * nv + j] = q[c][j];
          w0[b + t] = wh[c] + s;
        }
      }
    }
    if (lane == 0 && nj == nv) frozen += 3;
    __syncwarp();
  }
  if (lane == 0) {
    if (frozen) atomicAdd(counters + 1, frozen);
    if (nflag) atomicAdd(counters + 3, nflag);
  }
}

__global__ void k_reduce_partials(const double* __restrict__ p, int np, double* out, double add) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int k = threadIdx.x; k < np; k += blockDim.x) s += p[k];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) *out = t + add;
}

// first pass of a deterministic two-pass sum: one partial per block
__global__ void k_block_sums(const double* __restrict__ x, int64_t n, double* __restrict__ partials) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    s += x[k];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// every context array carries 64 bytes of tail padding: the TMA-staged
// window kernel (win9) copies 16-byte-aligned spans that may end up to one
// element past an array's last entry (read, never used)
template <typename T>
cudaError_t dalloc(T** p, int64_t n, cudaStream_t s) {
  return emin_mallocAsync((void**)p, sizeof(T) * (size_t)(n > 0 ? n : 1) + 64, s);
}

}  // namespace

// ============================================================ host helpers
int emin_launch_masked(emin_ctx ctx, int mode, const double* X, const double* X2, double* out,
                       cudaStream_t s);
emin_status emin_finish_r0(emin_ctx ctx);
emin_status emin_plan(emin_ctx ctx);
bool emin_alg2_fast(emin_ctx c, const double* Bc, const double* B, const int64_t* frow, const double* what,
                    unsigned long long* counters, cudaStream_t s);
void emin_free_all(emin_ctx ctx);

extern "C" void emin_default_opts(emin_opts* o, int64_t n_global) {
  std::memset(o, 0, sizeof(*o));
  o->block_size = 1;
  o->rank_tol = 1e-10;
  o->tau = 0.0;
  o->project_after_jacobi = 0;
  o->stagnation_rel = 1e-30;
  o->stream = nullptr;
  o->nccl_comm = nullptr;
  o->row_begin = 0;
  o->row_end = n_global;
  o->inputs_on_device = 0;
  o->precond = EMIN_PREC_JACOBI;
  o->sgs_key = nullptr;
  o->start = EMIN_START_GIVEN;
}

static emin_status fail(emin_ctx ctx, emin_status st, const std::string& msg) {
  g_setup_error = msg;
  emin_dist_abort(ctx, msg);   // a loopback group must not wait for this rank
  if (ctx) emin_destroy(ctx);
  return st;
}

// debug_flags & EMIN_DBG_TRACE: synchronise and print the elapsed host time of
// each setup phase
struct SetupTrace {
  bool on = false;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(cudaStream_t s, const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[emin setup] %8.3f ms  %s\n", ms, what);
  }
};

#define SETUP_TRY(call)                                                                \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? EMIN_ERR_OOM : EMIN_ERR_CUDA, \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

extern "C" const char* emin_setup_error_internal() { return g_setup_error.c_str(); }

extern "C" emin_status emin_setup(emin_ctx* out, int64_t n_global, int64_t nc_global,
                                  const int64_t* A_rowptr, const int32_t* A_col, const double* A_val,
                                  const uint8_t* is_coarse, const int64_t* P_rowptr,
                                  const int32_t* P_col, const double* P_val, int32_t nv,
                                  const double* B, const double* Bc, const emin_opts* opts) {
  emin_ctx ctx = nullptr;
  if (!out) return fail(ctx, EMIN_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!opts || !A_rowptr || !A_col || !A_val || !is_coarse || !P_rowptr || !P_col || !B || !Bc)
    return fail(ctx, EMIN_ERR_ARG, "NULL argument");
  if (n_global <= 0 || nc_global < 0 || nc_global > n_global || nv < 1 || nv > EMIN_NV_MAX)
    return fail(ctx, EMIN_ERR_ARG, "bad n_global / nc_global / nv");
  if (opts->row_begin < 0 || opts->row_end > n_global || opts->row_end <= opts->row_begin)
    return fail(ctx, EMIN_ERR_ARG, "bad row range");
  if (n_global > INT32_MAX || nc_global > INT32_MAX)
    return fail(ctx, EMIN_ERR_ARG, "n_global exceeds the int32 column range");
  if (opts->precond != EMIN_PREC_JACOBI && opts->precond != EMIN_PREC_SGS)
    return fail(ctx, EMIN_ERR_ARG, "precond must be EMIN_PREC_JACOBI or EMIN_PREC_SGS");
  if (opts->start != EMIN_START_GIVEN && opts->start != EMIN_START_MAXVOL)
    return fail(ctx, EMIN_ERR_ARG, "start must be EMIN_START_GIVEN or EMIN_START_MAXVOL");
  if (opts->nccl_comm && opts->loopback)
    return fail(ctx, EMIN_ERR_ARG, "nccl_comm and loopback are mutually exclusive");

  SetupTrace trace;
  trace.on = (opts->debug_flags & EMIN_DBG_TRACE) != 0;
  ctx = new emin_ctx_s();
  ctx->opts = *opts;
  ctx->stream = (cudaStream_t)opts->stream;
  ctx->n_global = n_global;
  ctx->nc_global = nc_global;
  ctx->m_owned = opts->row_end - opts->row_begin;
  ctx->nv = nv;
  cudaStream_t s = ctx->stream;
  const int64_t m = ctx->m_owned;
  const int SM = emin_num_sms();
  if (opts->nccl_comm || opts->loopback) {
    emin_status st = emin_dist_attach(ctx, opts->nccl_comm, opts->loopback, opts->loopback_rank);
    if (st != EMIN_OK) return fail(ctx, st, ctx->last_error);
  }

  // ---- stage the inputs on the device (host pointers are copied)
  int64_t nnzA = 0, nnzP = 0, a0 = 0, p0 = 0;
  const int64_t *dArp = A_rowptr, *dPrp = P_rowptr;
  const int32_t *dAcol = A_col, *dPcol = P_col;
  const double *dAval = A_val, *dPval = P_val, *dB = B, *dBc = Bc;
  const uint8_t* dIsc = is_coarse;
  std::vector<void*> temps;
  auto tmp_free = [&]() { for (void* p : temps) cudaFreeAsync(p, s); temps.clear(); };
  if (!opts->inputs_on_device) {
    a0 = A_rowptr[0]; nnzA = A_rowptr[m] - a0;
    p0 = P_rowptr[0]; nnzP = P_rowptr[m] - p0;
    int64_t *t1; int32_t *t2; double *t3; uint8_t *t4;
    SETUP_TRY(dalloc(&t1, m + 1, s)); temps.push_back(t1);
    SETUP_TRY(cudaMemcpyAsync(t1, A_rowptr, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, s)); dArp = t1;
    SETUP_TRY(dalloc(&t2, nnzA, s)); temps.push_back(t2);
    SETUP_TRY(cudaMemcpyAsync(t2, A_col + a0, sizeof(int32_t) * nnzA, cudaMemcpyHostToDevice, s)); dAcol = t2;
    SETUP_TRY(dalloc(&t3, nnzA, s)); temps.push_back(t3);
    SETUP_TRY(cudaMemcpyAsync(t3, A_val + a0, sizeof(double) * nnzA, cudaMemcpyHostToDevice, s)); dAval = t3;
    SETUP_TRY(dalloc(&t4, n_global, s)); temps.push_back(t4);
    SETUP_TRY(cudaMemcpyAsync(t4, is_coarse, n_global, cudaMemcpyHostToDevice, s)); dIsc = t4;
    SETUP_TRY(dalloc(&t1, m + 1, s)); temps.push_back(t1);
    SETUP_TRY(cudaMemcpyAsync(t1, P_rowptr, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, s)); dPrp = t1;
    SETUP_TRY(dalloc(&t2, nnzP, s)); temps.push_back(t2);
    SETUP_TRY(cudaMemcpyAsync(t2, P_col + p0, sizeof(int32_t) * nnzP, cudaMemcpyHostToDevice, s)); dPcol = t2;
    if (P_val) {
      SETUP_TRY(dalloc(&t3, nnzP, s)); temps.push_back(t3);
      SETUP_TRY(cudaMemcpyAsync(t3, P_val + p0, sizeof(double) * nnzP, cudaMemcpyHostToDevice, s)); dPval = t3;
    }
    SETUP_TRY(dalloc(&t3, m * nv, s)); temps.push_back(t3);
    SETUP_TRY(cudaMemcpyAsync(t3, B, sizeof(double) * m * nv, cudaMemcpyHostToDevice, s)); dB = t3;
    SETUP_TRY(dalloc(&t3, nc_global * nv, s)); temps.push_back(t3);
    SETUP_TRY(cudaMemcpyAsync(t3, Bc, sizeof(double) * nc_global * nv, cudaMemcpyHostToDevice, s)); dBc = t3;
    // the copies start at the first owned entry; kernels index relative to rowptr[0]
  } else {
    int64_t hb[2];
    SETUP_TRY(cudaMemcpyAsync(hb, A_rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SETUP_TRY(cudaMemcpyAsync(hb + 1, A_rowptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    int64_t pb[2];
    SETUP_TRY(cudaMemcpyAsync(pb, P_rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SETUP_TRY(cudaMemcpyAsync(pb + 1, P_rowptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SETUP_TRY(cudaStreamSynchronize(s));
    a0 = hb[0]; nnzA = hb[1] - hb[0];
    p0 = pb[0]; nnzP = pb[1] - pb[0];
    dAcol = A_col + a0; dAval = A_val + a0; dPcol = P_col + p0;
    if (P_val) dPval = P_val + p0;
  }
  ctx->nnzP = nnzP;

  trace.mark(s, "inputs staged");
  // ---- coarse numbering: cidx = exclusive scan of is_coarse (global)
  int64_t *cidx, *scratch, *totals;
  SETUP_TRY(dalloc(&cidx, n_global + 1, s)); temps.push_back(cidx);
  SETUP_TRY(dalloc(&scratch, emin_scan_scratch_elems(n_global + m + 8), s)); temps.push_back(scratch);
  SETUP_TRY(dalloc(&totals, 8, s)); temps.push_back(totals);
  k_coarse_flags<<<SM * 8, 256, 0, s>>>(dIsc, n_global, cidx);
  SETUP_TRY(emin_scan_i64(cidx, cidx, n_global, totals + 0, scratch, s));
  int64_t h_nc = 0, h_cb = 0;
  SETUP_TRY(cudaMemcpyAsync(&h_nc, totals + 0, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SETUP_TRY(cudaMemcpyAsync(&h_cb, cidx + opts->row_begin, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  int64_t h_ce = 0;
  if (opts->row_end < n_global)
    SETUP_TRY(cudaMemcpyAsync(&h_ce, cidx + opts->row_end, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SETUP_TRY(cudaStreamSynchronize(s));
  if (opts->row_end == n_global) h_ce = h_nc;
  if (h_nc != nc_global) { tmp_free(); return fail(ctx, EMIN_ERR_ARG, "sum(is_coarse) != nc_global"); }
  const int64_t fbegin = opts->row_begin - h_cb;
  const int64_t nF = (opts->row_end - opts->row_begin) - (h_ce - h_cb);
  ctx->nF = nF;
  ctx->nFh = nF;
  ctx->n_crows = h_ce - h_cb;

  trace.mark(s, "coarse numbering");
  // ---- validation + counts
  int64_t *cnt_ff, *cnt_fc, *cnt_w;
  double* dcc;
  int32_t* err;
  int64_t* err_row;
  int32_t* max_row;
  SETUP_TRY(dalloc(&cnt_ff, nF + 1, s)); temps.push_back(cnt_ff);
  SETUP_TRY(dalloc(&cnt_fc, nF + 1, s)); temps.push_back(cnt_fc);
  SETUP_TRY(dalloc(&cnt_w, nF + 1, s)); temps.push_back(cnt_w);
  SETUP_TRY(dalloc(&dcc, m, s)); temps.push_back(dcc);
  SETUP_TRY(dalloc(&err, 4, s)); temps.push_back(err);
  SETUP_TRY(dalloc(&err_row, 1, s)); temps.push_back(err_row);
  max_row = err + 1;
  SETUP_TRY(dalloc(&ctx->d, nF, s));
  SETUP_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t) * 4, s));
  SETUP_TRY(cudaMemsetAsync(err_row, 0x7f, sizeof(int64_t), s));
  RowsArgs ra;
  ra.m = m; ra.row_begin = opts->row_begin; ra.row_end = opts->row_end; ra.n_global = n_global;
  ra.nc_global = nc_global; ra.fbegin = fbegin;
  ra.Arp = dArp; ra.Acol = dAcol; ra.Aval = dAval; ra.isc = dIsc; ra.cidx = cidx;
  ra.Prp = dPrp; ra.Pcol = dPcol; ra.Pval = dPval;
  ra.cnt_ff = cnt_ff; ra.cnt_fc = cnt_fc; ra.cnt_w = cnt_w; ra.d = ctx->d; ra.dcc = dcc;
  ra.err = err; ra.err_row = err_row; ra.max_row = max_row;
  // short in-order CTAs (config 5 validation 10.2 -> 8.5 ms, fill 13.7 -> 11.7 ms; CTAs per SM)
  const int grows = 32;
  k_rows<<<SM * grows, 256, 0, s>>>(ra);
  k_check_B<<<SM * 8, 256, 0, s>>>(m, opts->row_begin, nv, dIsc, cidx, dB, dBc, nc_global, err, err_row);
  SETUP_TRY(cudaGetLastError());
  if (ctx->dist) {
    // every rank fails together; the longest pattern row is global
    emin_status st1 = emin_dist_allreduce_max_i32(ctx, err, s);
    emin_status st2 = emin_dist_allreduce_max_i32(ctx, max_row, s);
    if (st1 != EMIN_OK || st2 != EMIN_OK) { tmp_free(); return fail(ctx, st1 != EMIN_OK ? st1 : st2, ctx->last_error); }
  }
  int32_t h_err[2];
  int64_t h_err_row;
  SETUP_TRY(cudaMemcpyAsync(h_err, err, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost, s));
  SETUP_TRY(cudaMemcpyAsync(&h_err_row, err_row, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SETUP_TRY(cudaStreamSynchronize(s));
  if (h_err[0]) {
    tmp_free();
    char buf[160];
    std::snprintf(buf, sizeof buf, "input validation failed (flags 0x%x) at global row %lld", h_err[0],
                  (long long)h_err_row);
    const int32_t f = h_err[0];
    emin_status st = (f & EF_CSR) ? EMIN_ERR_CSR : (f & EF_NONFINITE) ? EMIN_ERR_NONFINITE
                   : (f & (EF_PATTERN | EF_ROWLEN)) ? EMIN_ERR_PATTERN : (f & EF_BC) ? EMIN_ERR_BC
                   : EMIN_ERR_DIAG;
    return fail(ctx, st, buf);
  }
  ctx->max_row = h_err[1];
  trace.mark(s, "validation");

  // ---- multi-GPU: halo rows (F rows of other ranks referenced by A_FF)
  if (ctx->dist) {
    emin_status st = emin_dist_find_halo(ctx, fbegin, nF, n_global - nc_global, m, dArp, dAcol, dIsc, cidx,
                                         scratch);
    if (st != EMIN_OK) { tmp_free(); return fail(ctx, st, ctx->last_error); }
    ctx->nFh = nF + ctx->dist->nH;
  }

  // ---- row pointers of the W layout, A_FF and A_FC
  // (+2 elements: the TMA slices are read from 16-byte aligned bounds)
  SETUP_TRY(dalloc(&ctx->wptr, ctx->nFh + 1 + 2, s));
  SETUP_TRY(dalloc(&ctx->affptr, nF + 1 + 2, s));
  SETUP_TRY(dalloc(&ctx->afcptr, nF + 1, s));
  SETUP_TRY(emin_scan_i64(cnt_w, ctx->wptr, nF, totals + 1, scratch, s));
  SETUP_TRY(emin_scan_i64(cnt_ff, ctx->affptr, nF, totals + 2, scratch, s));
  SETUP_TRY(emin_scan_i64(cnt_fc, ctx->afcptr, nF, totals + 3, scratch, s));
  SETUP_TRY(cudaMemcpyAsync(ctx->wptr + nF, totals + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  SETUP_TRY(cudaMemcpyAsync(ctx->affptr + nF, totals + 2, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  SETUP_TRY(cudaMemcpyAsync(ctx->afcptr + nF, totals + 3, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  int64_t h_tot[3];
  SETUP_TRY(cudaMemcpyAsync(h_tot, totals + 1, sizeof(int64_t) * 3, cudaMemcpyDeviceToHost, s));
  SETUP_TRY(cudaStreamSynchronize(s));
  ctx->nnzW = ctx->nnzWh = h_tot[0];
  ctx->nnzAFF = h_tot[1];
  ctx->nnzAFC = h_tot[2];
  const int64_t W = ctx->nnzW;
  if (ctx->dist) {
    // halo row lengths -> wptr tail; send lists (once)
    emin_status st = emin_dist_halo_pattern_sizes(ctx, scratch);
    if (st != EMIN_OK) { tmp_free(); return fail(ctx, st, ctx->last_error); }
    ctx->nnzWh = W + ctx->dist->nHW;
  }
  const int64_t Wh = ctx->nnzWh;

  trace.mark(s, "row pointers");
  // ---- fill
  double* what;
  SETUP_TRY(dalloc(&ctx->wcol, Wh, s));
  SETUP_TRY(dalloc(&what, W, s)); temps.push_back(what);
  SETUP_TRY(dalloc(&ctx->pofs, nF, s));
  SETUP_TRY(dalloc(&ctx->cofs, m + 1, s));
  SETUP_TRY(cudaMemcpyAsync(ctx->cofs, dPrp, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToDevice, s));
  SETUP_TRY(dalloc(&ctx->isc_own, m, s));
  SETUP_TRY(cudaMemcpyAsync(ctx->isc_own, dIsc + opts->row_begin, m, cudaMemcpyDeviceToDevice, s));
  SETUP_TRY(dalloc(&ctx->affcol, ctx->nnzAFF, s));
  SETUP_TRY(dalloc(&ctx->affval, ctx->nnzAFF, s));
  SETUP_TRY(dalloc(&ctx->afccol, ctx->nnzAFC, s));
  SETUP_TRY(dalloc(&ctx->afcval, ctx->nnzAFC, s));
  int64_t* frow;
  SETUP_TRY(dalloc(&frow, nF, s)); temps.push_back(frow);
  FillArgs fa;
  fa.m = m; fa.row_begin = opts->row_begin; fa.row_end = opts->row_end; fa.fbegin = fbegin; fa.nF = nF;
  fa.Arp = dArp; fa.Acol = dAcol; fa.Aval = dAval; fa.isc = dIsc; fa.cidx = cidx;
  fa.Prp = dPrp; fa.Pcol = dPcol; fa.Pval = dPval;
  fa.wptr = ctx->wptr; fa.affptr = ctx->affptr; fa.afcptr = ctx->afcptr;
  fa.wcol = ctx->wcol; fa.what = what; fa.pofs = ctx->pofs;
  fa.affcol = ctx->affcol; fa.affval = ctx->affval; fa.afccol = ctx->afccol; fa.afcval = ctx->afcval;
  fa.frow = frow;
  fa.hpos = ctx->dist ? ctx->dist->hpos : nullptr;
  SETUP_TRY(dalloc(&ctx->adiag, std::max<int64_t>(nF, 1), s));
  fa.adiag = ctx->adiag;
  const int gfill = 64;
  k_fill<<<SM * gfill, 256, 0, s>>>(fa);
  SETUP_TRY(cudaGetLastError());
  if (ctx->dist) {
    emin_status st = emin_dist_halo_wcol(ctx);
    if (st != EMIN_OK) { tmp_free(); return fail(ctx, st, ctx->last_error); }
  }

  trace.mark(s, "fill");
  // ---- sum of the C-row diagonal (energy constant, Eq. trInc tr(A_cc))
  SETUP_TRY(dalloc(&ctx->partials, SM * 32, s));
  ctx->n_partials = SM * 32;
  double* dsum;
  SETUP_TRY(dalloc(&dsum, 4, s)); temps.push_back(dsum);
  k_block_sums<<<SM * 4, 256, 0, s>>>(dcc, m, ctx->partials);
  k_reduce_partials<<<1, 1024, 0, s>>>(ctx->partials, SM * 4, dsum, 0.0);

  // ---- kernel path (scalar window plan / generic) and launch geometry
  {
    emin_status pst = emin_plan(ctx);
    if (pst != EMIN_OK) { tmp_free(); return fail(ctx, pst, ctx->last_error); }
  }

  if (opts->precond == EMIN_PREC_SGS) {
    emin_status sst = emin_sgs_plan(ctx, opts->sgs_key, frow, s);
    if (sst != EMIN_OK) { tmp_free(); return fail(ctx, sst, ctx->last_error); }
  }
  trace.mark(s, "kernel plan");
  // ---- Alg. 2
  // w0, dw, y carry the halo tail (values of other ranks' rows)
  SETUP_TRY(dalloc(&ctx->Q, W * nv + 2, s));
  SETUP_TRY(dalloc(&ctx->w0, Wh + 2, s));
  SETUP_TRY(dalloc(&ctx->dw, Wh + 2, s));
  SETUP_TRY(dalloc(&ctx->r, W, s));
  SETUP_TRY(dalloc(&ctx->y, Wh + 2, s));
  SETUP_TRY(dalloc(&ctx->yb, W, s));
  SETUP_TRY(dalloc(&ctx->st, 1, s));
  unsigned long long* counters;
  SETUP_TRY(dalloc(&counters, 4, s)); temps.push_back(counters);
  SETUP_TRY(cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * 4, s));
  SETUP_TRY(cudaMemsetAsync(ctx->dw, 0, sizeof(double) * Wh, s));
  SETUP_TRY(cudaMemsetAsync(ctx->y, 0, sizeof(double) * Wh, s));
  SETUP_TRY(cudaMemsetAsync(ctx->yb, 0, sizeof(double) * W, s));
  const DevView v = ctx->view();
  const int agrid = (int)std::max<int64_t>(1, std::min<int64_t>((nF + 3) / 4, (int64_t)SM * 16));
  if (opts->start == EMIN_START_MAXVOL && nF > 0)      // Alg. 1 tentative start (NEXT-3, reading A24)
    emin_maxvol_start(ctx, dBc, dB, frow, what, counters + 2, s);
  bool alg2_done = emin_alg2_fast(ctx, dBc, dB, frow, what, counters, s);
  if (!alg2_done && ctx->kernel_path == 2 && ctx->max_row <= 128 && !(opts->debug_flags & EMIN_DBG_ALG2_ROWS)) {
    // nodal path: one QR per F node; rank-deficient nodes redone row by row
    uint8_t* nflag;
    SETUP_TRY(dalloc(&nflag, nF / 3 + 1, s)); temps.push_back(nflag);
    SETUP_TRY(cudaMemsetAsync(nflag, 0, nF / 3 + 1, s));
    const int64_t ngs = 16;   // short in-order CTAs (16 per SM)
    const int ng = (int)std::max<int64_t>(1, std::min<int64_t>((nF / 3 + 3) / 4, (int64_t)SM * ngs));
    if (ctx->max_row <= 32)
      k_alg2_nodal<1><<<ng, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters, nflag);
    else if (ctx->max_row <= 64)
      k_alg2_nodal<2><<<ng, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters, nflag);
    else
      k_alg2_nodal<4><<<ng, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters, nflag);
    unsigned long long h_nflag = 0;
    SETUP_TRY(cudaMemcpyAsync(&h_nflag, counters + 3, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SETUP_TRY(cudaStreamSynchronize(s));
    if (h_nflag) {
      if (ctx->max_row <= 32)
        k_alg2<1><<<agrid, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters, nflag);
      else if (ctx->max_row <= 64)
        k_alg2<2><<<agrid, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters, nflag);
      else
        k_alg2<4><<<agrid, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters, nflag);
    }
    alg2_done = true;
  }
  if (alg2_done)
    ;
  else if (ctx->max_row <= 32)
    k_alg2<1><<<agrid, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters);
  else if (ctx->max_row <= 64)
    k_alg2<2><<<agrid, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters);
  else
    k_alg2<4><<<agrid, 128, 0, s>>>(v, dBc, dB, frow, what, opts->rank_tol, ctx->Q, ctx->w0, counters);
  SETUP_TRY(cudaGetLastError());
  if (ctx->dist) {
    // W0 on the halo rows (needed by r0 and E0) and the global tr(A_CC)
    emin_status st1 = emin_dist_halo_values(ctx, ctx->w0, s);
    emin_status st2 = emin_dist_allreduce(ctx, dsum, dsum + 1, 1, s);
    if (st2 == EMIN_OK)
      SETUP_TRY(cudaMemcpyAsync(dsum, dsum + 1, sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (st1 != EMIN_OK || st2 != EMIN_OK) { tmp_free(); return fail(ctx, st1 != EMIN_OK ? st1 : st2, ctx->last_error); }
  }

  trace.mark(s, "Alg. 2");
  // ---- r0 = -Pi (A P0)|F and E0 = tr(P0^T A P0)
  // tr(A_CC) and the Alg. 2 counters stay on the device (emin_report reads
  // them; no host round trip here)
  SETUP_TRY(cudaMemcpyAsync(&ctx->st->sum_cc, dsum, sizeof(double), cudaMemcpyDeviceToDevice, s));
  SETUP_TRY(cudaMemcpyAsync(ctx->st->cnt, counters, sizeof(unsigned long long) * 3, cudaMemcpyDeviceToDevice, s));
  // kernels enqueued above: coarse flags, 4 scans x 3, rows, check_B, fill, 2 reduce, alg2
  ctx->launches += 1 + 3 + 2 + (nF > 0 ? 9 : 0) + 1 + 2 + 1;
  emin_status st = emin_finish_r0(ctx);
  tmp_free();
  if (st != EMIN_OK) return fail(ctx, st, ctx->last_error);
  // no final synchronisation: the caller's next call (the iteration graph's
  // build, typically) overlaps the tail of the setup kernels; a fault in them
  // surfaces at the next synchronising call
  SETUP_TRY(cudaGetLastError());
  trace.mark(s, "r0, E0 (done)");
  *out = ctx;
  return EMIN_OK;
}
