/*
 * emin_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * restricted PCG energy minimisation of an AMG prolongation
 * (arXiv 2208.02995, PAPER.md = /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2208_02995_b200/csrc); neither includes or links the other.
 *
 * What it computes, step by step in the paper's order and notation, with the
 * readings of SURVEY.md §8c / DESIGN.md §3 where the paper is garbled:
 *
 *   setup   Alg. 2 EMIN_SetUp per F row i, rows ascending:
 *           M_i = B_c(J_i,:) (|J_i| x nv, reading A5), r_i = b_i - M_i^T w^_i,
 *           economy Householder QR if |J_i| >= nv and rank(R) = nv
 *           (rank_tol relative, A6): delta_i = Q_i R_i^{-T} r_i ; otherwise
 *           one-sided Jacobi SVD, k_i = #{sigma > rank_tol sigma_max},
 *           Q_i = U(:,1:k_i), delta_i = U_k Sigma_k^{-1} V_k^T r_i.
 *           w0_i = w^_i + delta_i.
 *   r0      r = Pi_B (f - K w0) = -Pi_B (A P0)|_F-pattern  (Alg. 3 line 3,
 *           P:838, sign reading A1, projection reading A2).
 *   iterate Alg. 3 with readings A3 (k = 1), A4 (stop exits the
 *           loop without the update, P is still formed), A18 (guards):
 *             z = Pi_B M^{-1} r  (Jacobi, M = diag(K) = A(i,i) per row,
 *                                 Theorem 1; projected)
 *             gamma = r^T z ; gamma <= 0 -> converged stop
 *             y = z (k = 1) else y = z + (gamma/gamma_old) y
 *             gamma_old = gamma
 *             yb = Pi_B K y          (K y = A Y on the fixed pattern)
 *             den = y^T yb ; den < 0 -> breakdown ; den == 0 -> stop
 *             alpha = gamma/den ; dE_k = gamma alpha       (Eq. CG_dEa)
 *             tau > 0, k > 1, dE_k < tau dE_1 -> stop      (Eq. relRed)
 *             dE_k <= stag E0 -> stop                       (A18)
 *             dw += alpha y ; r -= alpha yb
 *   energy  tr(P^T A P) by its definition (Eq. trace), P = [W; I].
 *   pattern (NEXT-3) oracle_pattern: the pattern of P from the graph of A by
 *           Alg. 1's growth loop (reading A25); pinned bit-exactly against
 *           the independent box-arithmetic input generator.
 *   start   (optional) the tentative start W^ of Alg. 1
 *            on the prescribed pattern: per F row the max-vol
 *           selection of nv columns of V_c(J_i,:)^T (reading A24), the local
 *           system solved exactly on them, zero elsewhere; rows without a
 *           nonsingular selection keep W^ = 0.
 *   precond z = Pi M_2^{-1} r with the projected
 *           symmetric Gauss-Seidel preconditioner (Eq. SGS_prec
 *           simplified): M_SGS^{-1} = (L+D)^{-T} D (L+D)^{-1}, K = L + D + L^T
 *           (K block diagonal, block j = A(I_j, I_j) for coarse
 *           column j), the unknowns of each block visited in ascending
 *           (sgs_key, row) order (reading A23); applied matrix-free on the W
 *           layout as one forward and one backward sweep over the F rows, and
 *           always followed by Pi (only Jacobi may skip it).
 *   galerkin (reading A26) A_c = P^T A P, the next
 *           level's operator (the matrix whose trace is the energy,
 *           P:248-250; "sparse matrix-matrix product") by its
 *           two-product definition T = A P, A_c = P^T T; pinned against the
 *           1D textbook closed form, dense numpy products and
 *           A_c B_c = P^T A B whenever P B_c = B.
 *
 * Summation order: per-row sums ascending in A's column order; global sums
 * row-ascending with Neumaier compensation.
 *
 * Threads (OpenMP, -fopenmp): only loops whose iterations are independent
 * run in parallel -- the per-row loops of the projection, the masked
 * product, Alg. 2 and the Jacobi scaling, and the elementwise vector
 * updates.  Every global sum stays one serial Neumaier pass in the order
 * above (the energy's per-entry terms are formed in parallel into an array,
 * then summed serially), and the SGS sweeps stay serial, so the result does
 * not depend on the thread count (pinned: tests/test_oracle_pins.py compares
 * 1 thread with all of them bitwise).
 *
 * Parity pins (tests/test_oracle_*.py): dense KKT solve, null-space solve,
 * 1D closed form, config 1b/2b converge to the symmetric equal-weight P,
 * constraint at every iterate, monotone + telescoping energy, Theorem 1,
 * S:288 least-norm example, masked product == gather(dense A P),
 * energy == dense tr(P^T A P), QR/SVD vs numpy.linalg.
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_ARG 1
#define OR_ERR_CSR 2
#define OR_ERR_PATTERN 3
#define OR_ERR_BC 4
#define OR_ERR_DIAG 5
#define OR_ERR_NONFINITE 6
#define OR_ERR_BREAKDOWN 7

/* stop reasons */
#define OR_RUN 0
#define OR_STOP_GAMMA 1
#define OR_STOP_DEN 2
#define OR_STOP_TAU 3
#define OR_STOP_STAG 4

typedef struct {
    int64_t n, nc, nF, nnzW;
    int nv;
    double rank_tol, tau, stag;
    int project_z;                 /* 1: z = Pi M^-1 r (literal P:840) */
    int precond;                   /* 0 Jacobi M_1, 1 projected SGS M_2 */
    int64_t n_maxvol_fail;         /* F rows where max-vol found no nonsingular selection */
    int64_t *sgs_key;              /* F index -> SGS ordering key (0 if none given) */
    /* full operator, copied */
    int64_t *Arp; int32_t *Acol; double *Aval;
    uint8_t *isc;
    int64_t *coarse_of;            /* global -> coarse id or -1 */
    int64_t *fid;                  /* global -> F index or -1 */
    int64_t *frow;                 /* F index -> global row */
    /* full P pattern (all rows), copied */
    int64_t *Prp; int32_t *Pcol;
    /* W layout over F rows */
    int64_t *wptr; int32_t *wcol;
    double *Q;                     /* nnzW * nv, row-major per entry, zero-padded */
    int *krank;                    /* numerical rank k_i per F row */
    double *d;                     /* A(i,i) per F row */
    double *w0, *dw, *r, *y, *yb, *z;
    double sum_diag_cc;
    /* CG state */
    double gamma_old, dE1, E0;
    int64_t k_total;
    int stopped;
    /* report */
    int64_t n_svd, n_frozen;
} oracle_t;

/* ---------------- Neumaier-compensated accumulation -------------------- */
typedef struct { double s, c; } nsum_t;
static void nsum_add(nsum_t *a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
}
static double nsum_val(const nsum_t *a) { return a->s + a->c; }

/* ---------------- small dense helpers (column-major, local) ------------ */

/* Householder economy QR of M (n x m, n >= m, column-major, ld = n).
 * On return Q (n x m, column-major) and R (m x m, column-major, upper). */
static void householder_qr(int n, int m, const double *M, double *Q, double *R) {
    double *Wk = (double *)malloc(sizeof(double) * n * m);
    double *V = (double *)calloc((size_t)n * m, sizeof(double));  /* reflectors */
    double *vn = (double *)calloc(m, sizeof(double));              /* v^T v */
    memcpy(Wk, M, sizeof(double) * n * m);
    for (int j = 0; j < m; ++j) {
        double nrm2 = 0.0;
        for (int t = j; t < n; ++t) nrm2 += Wk[t + j * n] * Wk[t + j * n];
        double nrm = sqrt(nrm2);
        double x0 = Wk[j + j * n];
        double alpha = (x0 >= 0.0) ? -nrm : nrm;
        for (int t = j; t < n; ++t) V[t + j * n] = Wk[t + j * n];
        V[j + j * n] -= alpha;
        double vv = 0.0;
        for (int t = j; t < n; ++t) vv += V[t + j * n] * V[t + j * n];
        vn[j] = vv;
        if (vv > 0.0) {
            for (int c = j; c < m; ++c) {
                double s = 0.0;
                for (int t = j; t < n; ++t) s += V[t + j * n] * Wk[t + c * n];
                s = 2.0 * s / vv;
                for (int t = j; t < n; ++t) Wk[t + c * n] -= s * V[t + j * n];
            }
        }
    }
    for (int c = 0; c < m; ++c)
        for (int rr = 0; rr < m; ++rr) R[rr + c * m] = (rr <= c) ? Wk[rr + c * n] : 0.0;
    /* Q = H_0 ... H_{m-1} [I; 0] */
    for (int c = 0; c < m; ++c)
        for (int t = 0; t < n; ++t) Q[t + c * n] = (t == c) ? 1.0 : 0.0;
    for (int j = m - 1; j >= 0; --j) {
        if (vn[j] <= 0.0) continue;
        for (int c = 0; c < m; ++c) {
            double s = 0.0;
            for (int t = j; t < n; ++t) s += V[t + j * n] * Q[t + c * n];
            s = 2.0 * s / vn[j];
            for (int t = j; t < n; ++t) Q[t + c * n] -= s * V[t + j * n];
        }
    }
    free(Wk); free(V); free(vn);
}

/* One-sided (Hestenes) Jacobi SVD of M (n x m, column-major): on return
 * U holds the rotated columns (= U Sigma), V (m x m) the right vectors. */
static void jacobi_svd(int n, int m, const double *M, double *US, double *V) {
    memcpy(US, M, sizeof(double) * n * m);
    for (int c = 0; c < m; ++c)
        for (int rr = 0; rr < m; ++rr) V[rr + c * m] = (rr == c) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        int rotated = 0;
        for (int p = 0; p < m - 1; ++p) {
            for (int q = p + 1; q < m; ++q) {
                double a = 0.0, b = 0.0, c = 0.0;
                for (int t = 0; t < n; ++t) {
                    a += US[t + p * n] * US[t + p * n];
                    b += US[t + q * n] * US[t + q * n];
                    c += US[t + p * n] * US[t + q * n];
                }
                if (c == 0.0 || fabs(c) <= 1e-15 * sqrt(a * b)) continue;
                rotated = 1;
                double zeta = (b - a) / (2.0 * c);
                double tt = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
                for (int t = 0; t < n; ++t) {
                    double up = US[t + p * n], uq = US[t + q * n];
                    US[t + p * n] = cs * up - sn * uq;
                    US[t + q * n] = sn * up + cs * uq;
                }
                for (int t = 0; t < m; ++t) {
                    double vp = V[t + p * m], vq = V[t + q * m];
                    V[t + p * m] = cs * vp - sn * vq;
                    V[t + q * m] = sn * vp + cs * vq;
                }
            }
        }
        if (!rotated) break;
    }
}

/* Alg. 2 for one row.  M = B_c(J_i,:) (nj x nv, col-major), rvec = r_i (nv).
 * Writes Qrow (nj x nv, ROW-major per entry, zero-padded beyond k), delta (nj).
 * Returns k (numerical rank); *used_svd set if the SVD branch ran. */
static int emin_setup_row(int nj, int nv, const double *M, const double *rvec, double tol,
                          double *Qrow, double *delta, int *used_svd) {
    *used_svd = 0;
    for (int t = 0; t < nj * nv; ++t) Qrow[t] = 0.0;
    for (int t = 0; t < nj; ++t) delta[t] = 0.0;
    if (nj >= nv) {
        double *Q = (double *)malloc(sizeof(double) * nj * nv);
        double *R = (double *)malloc(sizeof(double) * nv * nv);
        householder_qr(nj, nv, M, Q, R);
        double rmax = 0.0, rmin = INFINITY;
        for (int j = 0; j < nv; ++j) {
            double a = fabs(R[j + j * nv]);
            if (a > rmax) rmax = a;
            if (a < rmin) rmin = a;
        }
        if (rmax > 0.0 && rmin > tol * rmax) {
            /* delta = Q R^{-T} r : solve R^T u = r (forward), delta = Q u */
            double *u = (double *)malloc(sizeof(double) * nv);
            for (int j = 0; j < nv; ++j) {
                double s = rvec[j];
                for (int l = 0; l < j; ++l) s -= R[l + j * nv] * u[l];
                u[j] = s / R[j + j * nv];
            }
            for (int t = 0; t < nj; ++t) {
                double s = 0.0;
                for (int j = 0; j < nv; ++j) s += Q[t + j * nj] * u[j];
                delta[t] = s;
                for (int j = 0; j < nv; ++j) Qrow[t * nv + j] = Q[t + j * nj];
            }
            free(u); free(Q); free(R);
            return nv;
        }
        free(Q); free(R);
    }
    /* SVD branch, P:648-653 (reading A5: delta = U_k Sigma_k^-1 V_k^T r) */
    *used_svd = 1;
    double *US = (double *)malloc(sizeof(double) * nj * nv);
    double *V = (double *)malloc(sizeof(double) * nv * nv);
    jacobi_svd(nj, nv, M, US, V);
    double smax = 0.0;
    double *sig = (double *)malloc(sizeof(double) * nv);
    for (int j = 0; j < nv; ++j) {
        double s = 0.0;
        for (int t = 0; t < nj; ++t) s += US[t + j * nj] * US[t + j * nj];
        sig[j] = sqrt(s);
        if (sig[j] > smax) smax = sig[j];
    }
    /* keep columns in descending sigma order (stable by index) */
    int k = 0;
    int *order = (int *)malloc(sizeof(int) * nv);
    for (int j = 0; j < nv; ++j) order[j] = j;
    for (int a = 1; a < nv; ++a)
        for (int b = a; b > 0 && sig[order[b]] > sig[order[b - 1]]; --b) {
            int tmp = order[b]; order[b] = order[b - 1]; order[b - 1] = tmp;
        }
    for (int a = 0; a < nv; ++a) {
        int j = order[a];
        if (!(smax > 0.0 && sig[j] > tol * smax)) continue;
        double vr = 0.0;
        for (int l = 0; l < nv; ++l) vr += V[l + j * nv] * rvec[l];
        for (int t = 0; t < nj; ++t) {
            double u = US[t + j * nj] / sig[j];
            Qrow[t * nv + k] = u;
            delta[t] += u * (vr / sig[j]);
        }
        ++k;
    }
    free(order); free(sig); free(US); free(V);
    return k;
}

/* ---------------- Alg. 1 tentative start: max-vol selection ------------- */
/* Reading A24 (the paper cites max vol [Knu85, Gor08] without details):
 *   M = V_c(J_i,:) (m x nv, column-major), the columns of V_c(J_i,:)^T are
 *   M's rows.
 *   initial selection: Gaussian elimination with partial pivoting on a copy
 *     of M, pivot of column c = the first unselected row t whose |entry| is
 *     within a factor (1 - 1e-12) of the column maximum; a zero maximum means
 *     no nonsingular selection (return 0);
 *   max-vol sweeps (<= 100): C = M B^{-1}, B = M(S,:); (t, c) = the first
 *     (row-major) entry with |C| within (1 - 1e-12) of max |C|; stop when
 *     max |C| <= 1 + 1e-8, else S[c] = t (the volume |det B| grows by |C|).
 *   w = 0 except w(S) = B^{-T} v (the local system B^T w = v solved exactly).
 * Returns 1 on success. */
static int maxvol_tol_first(const double *val, int n, double *vmax) {
    double mx = 0.0;
    for (int t = 0; t < n; ++t) if (val[t] > mx) mx = val[t];
    *vmax = mx;
    for (int t = 0; t < n; ++t) if (val[t] >= (1.0 - 1e-12) * mx && val[t] >= 0.0) return t;
    return -1;
}

/* inverse of the nv x nv matrix B (row-major) by Gauss-Jordan with partial
 * pivoting; returns 0 if singular */
static int gj_inverse(int nv, const double *Bm, double *inv) {
    double a[16 * 32];
    for (int r = 0; r < nv; ++r)
        for (int c = 0; c < 2 * nv; ++c) a[r * 2 * nv + c] = c < nv ? Bm[r * nv + c] : (c - nv == r ? 1.0 : 0.0);
    for (int c = 0; c < nv; ++c) {
        int p = c;
        for (int r = c + 1; r < nv; ++r) if (fabs(a[r * 2 * nv + c]) > fabs(a[p * 2 * nv + c])) p = r;
        if (a[p * 2 * nv + c] == 0.0) return 0;
        if (p != c)
            for (int k = 0; k < 2 * nv; ++k) { double t = a[c * 2 * nv + k]; a[c * 2 * nv + k] = a[p * 2 * nv + k]; a[p * 2 * nv + k] = t; }
        double piv = a[c * 2 * nv + c];
        for (int k = 0; k < 2 * nv; ++k) a[c * 2 * nv + k] /= piv;
        for (int r = 0; r < nv; ++r) {
            if (r == c) continue;
            double f = a[r * 2 * nv + c];
            if (f != 0.0) for (int k = 0; k < 2 * nv; ++k) a[r * 2 * nv + k] -= f * a[c * 2 * nv + k];
        }
    }
    for (int r = 0; r < nv; ++r)
        for (int c = 0; c < nv; ++c) inv[r * nv + c] = a[r * 2 * nv + nv + c];
    return 1;
}

int oracle_maxvol(int m, int nv, const double *M, int *S) {
    if (m < nv) return 0;
    double *W = (double *)malloc(sizeof(double) * m * nv);
    double *val = (double *)malloc(sizeof(double) * m);
    int *used = (int *)calloc(m, sizeof(int));
    memcpy(W, M, sizeof(double) * m * nv);
    int ok = 1;
    for (int c = 0; c < nv && ok; ++c) {
        double mx;
        for (int t = 0; t < m; ++t) val[t] = used[t] ? -1.0 : fabs(W[t + c * m]);
        int p = maxvol_tol_first(val, m, &mx);
        if (p < 0 || mx == 0.0) { ok = 0; break; }
        S[c] = p;
        used[p] = 1;
        for (int t = 0; t < m; ++t) {
            if (used[t]) continue;
            double f = W[t + c * m] / W[p + c * m];
            for (int k = c; k < nv; ++k) W[t + k * m] -= f * W[p + k * m];
        }
    }
    if (ok) {
        double Bm[256], inv[256];
        double *C = (double *)malloc(sizeof(double) * m * nv);
        for (int sweep = 0; sweep < 100 && ok; ++sweep) {
            for (int a = 0; a < nv; ++a)
                for (int b = 0; b < nv; ++b) Bm[a * nv + b] = M[S[a] + b * m];
            if (!gj_inverse(nv, Bm, inv)) { ok = 0; break; }
            double mx = 0.0;
            for (int t = 0; t < m; ++t)
                for (int c = 0; c < nv; ++c) {
                    double sum = 0.0;
                    for (int b = 0; b < nv; ++b) sum += M[t + b * m] * inv[b * nv + c];
                    C[t * nv + c] = fabs(sum);
                    if (C[t * nv + c] > mx) mx = C[t * nv + c];
                }
            if (mx <= 1.0 + 1e-8) break;
            int bt = -1, bc = -1;
            for (int t = 0; t < m && bt < 0; ++t)
                for (int c = 0; c < nv; ++c)
                    if (C[t * nv + c] >= (1.0 - 1e-12) * mx) { bt = t; bc = c; break; }
            S[bc] = bt;
        }
        free(C);
    }
    free(W); free(val); free(used);
    return ok;
}

/* w(S) = B^{-T} v, B = M(S,:); zero elsewhere.  Returns 0 if B is singular. */
static int maxvol_solve(int m, int nv, const double *M, const int *S, const double *v, double *w) {
    double Bm[256], inv[256];
    for (int a = 0; a < nv; ++a)
        for (int b = 0; b < nv; ++b) Bm[a * nv + b] = M[S[a] + b * m];
    if (!gj_inverse(nv, Bm, inv)) return 0;
    for (int t = 0; t < m; ++t) w[t] = 0.0;
    for (int a = 0; a < nv; ++a) {
        double sum = 0.0;
        for (int b = 0; b < nv; ++b) sum += inv[b * nv + a] * v[b];
        w[S[a]] = sum;
    }
    return 1;
}

/* ---------------- the pieces of the path -------------------------------- */

/* (Pi x)_i = x_i - Q_i (Q_i^T x_i)   (Pi_B = I - Q Q^T) */
void oracle_project(const oracle_t *o, const double *x, double *out) {
    int nv = o->nv;
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < o->nF; ++i) {
        int64_t b = o->wptr[i], e = o->wptr[i + 1];
        double c[16];
        for (int m = 0; m < nv; ++m) {
            double s = 0.0;
            for (int64_t p = b; p < e; ++p) s += o->Q[p * nv + m] * x[p];
            c[m] = s;
        }
        for (int64_t p = b; p < e; ++p) {
            double s = 0.0;
            for (int m = 0; m < nv; ++m) s += o->Q[p * nv + m] * c[m];
            out[p] = x[p] - s;
        }
    }
}

/* Masked product on the F pattern:
 *   out(i,j) = sum_{k in F} A(i,k) X(k,j)  [+ A(i,c_j) if with_fc]
 * for j in J_i, where X(k,j) = 0 if j not in J_k.  Summed in the order of
 * row i of A; J_i and J_k are merged as sorted lists. */
void oracle_masked_AX(const oracle_t *o, const double *X, int with_fc, double *out) {
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < o->nF; ++i) {
        int64_t g = o->frow[i];
        int64_t b = o->wptr[i], e = o->wptr[i + 1];
        for (int64_t p = b; p < e; ++p) out[p] = 0.0;
        for (int64_t q = o->Arp[g]; q < o->Arp[g + 1]; ++q) {
            int64_t c = o->Acol[q];
            double a = o->Aval[q];
            if (!o->isc[c]) {
                int64_t k = o->fid[c];
                int64_t pi = b, pk = o->wptr[k], ek = o->wptr[k + 1];
                while (pi < e && pk < ek) {
                    if (o->wcol[pi] == o->wcol[pk]) { out[pi] += a * X[pk]; ++pi; ++pk; }
                    else if (o->wcol[pi] < o->wcol[pk]) ++pi;
                    else ++pk;
                }
            } else if (with_fc) {
                int64_t j = o->coarse_of[c];
                for (int64_t p = b; p < e; ++p)
                    if (o->wcol[p] == j) out[p] += a;
            }
        }
    }
}

/* does F row k precede F row i in the SGS visiting order?  Ascending
 * (sgs_key, global row) -- reading A23 (the paper leaves the order of the
 * unknowns inside a K block open; natural order = all keys equal). */
static int sgs_before(const oracle_t *o, int64_t k, int64_t i) {
    if (o->sgs_key[k] != o->sgs_key[i]) return o->sgs_key[k] < o->sgs_key[i];
    return o->frow[k] < o->frow[i];
}

/* z = M_SGS^{-1} x = (L+D)^{-T} D (L+D)^{-1} x, K = L + D + L^T.
 * K is block diagonal over the coarse columns j, block j = A(I_j, I_j)
 * (Eq. 11blk): the unknown (i, j) couples to (k, j) with weight
 * A(i,k) for every F row k whose pattern also holds j; D = A(i,i).
 *   (L+D) u = x   forward:  u(i,j) = (x(i,j) - sum_{k before i} A(i,k) u(k,j)) / A(i,i)
 *   v = D u
 *   (L+D)^T z = v backward: z(i,j) = (v(i,j) - sum_{k after i} A(k,i) z(k,j)) / A(i,i)
 * with A(k,i) = A(i,k) (A symmetric); the sums run over row i of A in
 * its column order.  Rows are visited in the SGS order (sgs_before); every
 * entry of row i is solved at once (the blocks j are independent). */
static void sgs_apply(const oracle_t *o, const double *x, double *z) {
    int64_t nF = o->nF;
    int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (nF ? nF : 1));
    double *u = (double *)malloc(sizeof(double) * (o->nnzW ? o->nnzW : 1));
    for (int64_t i = 0; i < nF; ++i) ord[i] = i;
    /* insertion of the visiting order (stable; plain O(nF log nF) merge sort) */
    {
        int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (nF ? nF : 1));
        for (int64_t w = 1; w < nF; w *= 2) {
            for (int64_t lo = 0; lo < nF; lo += 2 * w) {
                int64_t mid = lo + w < nF ? lo + w : nF, hi = lo + 2 * w < nF ? lo + 2 * w : nF;
                int64_t a = lo, b = mid, t = lo;
                while (a < mid && b < hi) tmp[t++] = sgs_before(o, ord[b], ord[a]) ? ord[b++] : ord[a++];
                while (a < mid) tmp[t++] = ord[a++];
                while (b < hi) tmp[t++] = ord[b++];
            }
            memcpy(ord, tmp, sizeof(int64_t) * nF);
        }
        free(tmp);
    }
    /* forward sweep: (L + D) u = x */
    for (int64_t oi = 0; oi < nF; ++oi) {
        int64_t i = ord[oi], g = o->frow[i];
        int64_t b = o->wptr[i], e = o->wptr[i + 1];
        for (int64_t p = b; p < e; ++p) u[p] = x[p];
        for (int64_t q = o->Arp[g]; q < o->Arp[g + 1]; ++q) {
            int64_t c = o->Acol[q];
            if (o->isc[c] || c == g) continue;
            int64_t k = o->fid[c];
            if (!sgs_before(o, k, i)) continue;
            double a = o->Aval[q];
            int64_t pi = b, pk = o->wptr[k], ek = o->wptr[k + 1];
            while (pi < e && pk < ek) {
                if (o->wcol[pi] == o->wcol[pk]) { u[pi] -= a * u[pk]; ++pi; ++pk; }
                else if (o->wcol[pi] < o->wcol[pk]) ++pi;
                else ++pk;
            }
        }
        for (int64_t p = b; p < e; ++p) u[p] = u[p] / o->d[i];
    }
    /* v = D u, then backward sweep: (L + D)^T z = v */
    for (int64_t oi = nF - 1; oi >= 0; --oi) {
        int64_t i = ord[oi], g = o->frow[i];
        int64_t b = o->wptr[i], e = o->wptr[i + 1];
        for (int64_t p = b; p < e; ++p) z[p] = o->d[i] * u[p];
        for (int64_t q = o->Arp[g]; q < o->Arp[g + 1]; ++q) {
            int64_t c = o->Acol[q];
            if (o->isc[c] || c == g) continue;
            int64_t k = o->fid[c];
            if (!sgs_before(o, i, k)) continue;
            double a = o->Aval[q];
            int64_t pi = b, pk = o->wptr[k], ek = o->wptr[k + 1];
            while (pi < e && pk < ek) {
                if (o->wcol[pi] == o->wcol[pk]) { z[pi] -= a * z[pk]; ++pi; ++pk; }
                else if (o->wcol[pi] < o->wcol[pk]) ++pi;
                else ++pk;
            }
        }
        for (int64_t p = b; p < e; ++p) z[p] = z[p] / o->d[i];
    }
    free(ord);
    free(u);
}

/* z = Pi_B M^{-1} x for the selected preconditioner (Alg. 3 line P:840). */
void oracle_apply_prec(const oracle_t *o, const double *x, double *z) {
    if (o->precond == 1) {
        sgs_apply(o, x, z);
        oracle_project(o, z, z);          /* mandatory for SGS */
    } else {
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < o->nF; ++i)
            for (int64_t p = o->wptr[i]; p < o->wptr[i + 1]; ++p) z[p] = x[p] / o->d[i];
        if (o->project_z) oracle_project(o, z, z);
    }
}

static double dot_w(const oracle_t *o, const double *a, const double *b) {
    nsum_t s = {0.0, 0.0};
    for (int64_t p = 0; p < o->nnzW; ++p) nsum_add(&s, a[p] * b[p]);
    return nsum_val(&s);
}

/* tr(P^T A P) by definition, P = [W; I] on the full row set (Eq. trace):
 * the terms P(r,j) (A P)(r,j) over the pattern of P in CSR order, summed
 * row-ascending (Neumaier). */
double oracle_energy_of(const oracle_t *o, const double *W) {
    int64_t nnzP = o->Prp[o->n];
    double *term = (double *)malloc(sizeof(double) * (nnzP ? nnzP : 1));
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < o->n; ++r) {
        /* P row r: pattern and values */
        int64_t rb, re;
        const int32_t *rc;
        const double *rv;
        double one = 1.0;
        int32_t cself;
        if (o->isc[r]) { cself = (int32_t)o->coarse_of[r]; rc = &cself; rv = &one; rb = 0; re = 1; }
        else { int64_t i = o->fid[r]; rb = o->wptr[i]; re = o->wptr[i + 1]; rc = o->wcol; rv = W; }
        for (int64_t p = rb; p < re; ++p) {
            int32_t j = rc[p];
            double prj = rv[p];
            /* (A P)(r, j) */
            double apj = 0.0;
            for (int64_t q = o->Arp[r]; q < o->Arp[r + 1]; ++q) {
                int64_t k = o->Acol[q];
                double pkj = 0.0;
                if (o->isc[k]) pkj = (o->coarse_of[k] == j) ? 1.0 : 0.0;
                else {
                    int64_t kk = o->fid[k];
                    for (int64_t s = o->wptr[kk]; s < o->wptr[kk + 1]; ++s)
                        if (o->wcol[s] == j) { pkj = W[s]; break; }
                }
                apj += o->Aval[q] * pkj;
            }
            term[o->Prp[r] + (p - rb)] = prj * apj;
        }
    }
    nsum_t tot = {0.0, 0.0};
    for (int64_t q = 0; q < nnzP; ++q) nsum_add(&tot, term[q]);
    free(term);
    return nsum_val(&tot);
}

/* ---------------- lifecycle --------------------------------------------- */

void oracle_destroy(oracle_t *o) {
    if (!o) return;
    free(o->Arp); free(o->Acol); free(o->Aval); free(o->isc); free(o->coarse_of);
    free(o->fid); free(o->frow); free(o->Prp); free(o->Pcol); free(o->wptr);
    free(o->wcol); free(o->Q); free(o->krank); free(o->d); free(o->w0); free(o->dw);
    free(o->r); free(o->y); free(o->yb); free(o->z); free(o->sgs_key);
    free(o);
}

/* Build the oracle state; returns status, *out = NULL on failure. */
int oracle_create(oracle_t **out, int64_t n, int64_t nc,
                  const int64_t *A_rowptr, const int32_t *A_col, const double *A_val,
                  const uint8_t *is_coarse,
                  const int64_t *P_rowptr, const int32_t *P_col, const double *P_val,
                  int nv, const double *B, const double *Bc,
                  double rank_tol, double tau, double stag, int project_z,
                  int precond, const int64_t *sgs_key, int start) {
    *out = NULL;
    if (n <= 0 || nc < 0 || nv <= 0 || nv > 16) return OR_ERR_ARG;
    oracle_t *o = (oracle_t *)calloc(1, sizeof(oracle_t));
    o->n = n; o->nc = nc; o->nv = nv;
    o->rank_tol = rank_tol; o->tau = tau; o->stag = stag; o->project_z = project_z;
    if (precond < 0 || precond > 1) { free(o); return OR_ERR_ARG; }
    o->precond = precond;
    int64_t nnzA = A_rowptr[n];
    o->Arp = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    o->Acol = (int32_t *)malloc(sizeof(int32_t) * (nnzA ? nnzA : 1));
    o->Aval = (double *)malloc(sizeof(double) * (nnzA ? nnzA : 1));
    memcpy(o->Arp, A_rowptr, sizeof(int64_t) * (n + 1));
    memcpy(o->Acol, A_col, sizeof(int32_t) * nnzA);
    memcpy(o->Aval, A_val, sizeof(double) * nnzA);
    o->isc = (uint8_t *)malloc(n);
    memcpy(o->isc, is_coarse, n);
    /* CSR validity: rowptr monotone, columns in range and strictly increasing */
    if (A_rowptr[0] != 0) { oracle_destroy(o); return OR_ERR_CSR; }
    for (int64_t r = 0; r < n; ++r) {
        if (A_rowptr[r + 1] < A_rowptr[r]) { oracle_destroy(o); return OR_ERR_CSR; }
        for (int64_t q = A_rowptr[r]; q < A_rowptr[r + 1]; ++q) {
            if (A_col[q] < 0 || A_col[q] >= n) { oracle_destroy(o); return OR_ERR_CSR; }
            if (q > A_rowptr[r] && A_col[q] <= A_col[q - 1]) { oracle_destroy(o); return OR_ERR_CSR; }
            if (!isfinite(A_val[q])) { oracle_destroy(o); return OR_ERR_NONFINITE; }
        }
    }
    /* C/F numbering: coarse ids and F ids ascending with the global index */
    o->coarse_of = (int64_t *)malloc(sizeof(int64_t) * n);
    o->fid = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t cc = 0, ff = 0;
    for (int64_t r = 0; r < n; ++r) {
        if (is_coarse[r]) { o->coarse_of[r] = cc++; o->fid[r] = -1; }
        else { o->coarse_of[r] = -1; o->fid[r] = ff++; }
    }
    if (cc != nc) { oracle_destroy(o); return OR_ERR_ARG; }
    o->nF = ff;
    o->frow = (int64_t *)malloc(sizeof(int64_t) * (ff ? ff : 1));
    for (int64_t r = 0; r < n; ++r) if (!is_coarse[r]) o->frow[o->fid[r]] = r;
    o->sgs_key = (int64_t *)calloc(ff ? ff : 1, sizeof(int64_t));
    if (sgs_key) for (int64_t i = 0; i < ff; ++i) o->sgs_key[i] = sgs_key[o->frow[i]];
    /* pattern: C row c must be exactly {coarse(c)}; F rows non-empty, sorted */
    int64_t nnzP = P_rowptr[n];
    o->Prp = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    o->Pcol = (int32_t *)malloc(sizeof(int32_t) * (nnzP ? nnzP : 1));
    memcpy(o->Prp, P_rowptr, sizeof(int64_t) * (n + 1));
    memcpy(o->Pcol, P_col, sizeof(int32_t) * nnzP);
    o->wptr = (int64_t *)malloc(sizeof(int64_t) * (ff + 1));
    o->wptr[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        int64_t len = P_rowptr[r + 1] - P_rowptr[r];
        if (len < 0) { oracle_destroy(o); return OR_ERR_PATTERN; }
        for (int64_t q = P_rowptr[r]; q < P_rowptr[r + 1]; ++q) {
            if (P_col[q] < 0 || P_col[q] >= nc) { oracle_destroy(o); return OR_ERR_PATTERN; }
            if (q > P_rowptr[r] && P_col[q] <= P_col[q - 1]) { oracle_destroy(o); return OR_ERR_PATTERN; }
        }
        if (is_coarse[r]) {
            if (len != 1 || P_col[P_rowptr[r]] != o->coarse_of[r]) { oracle_destroy(o); return OR_ERR_PATTERN; }
            if (P_val && P_val[P_rowptr[r]] != 1.0) { oracle_destroy(o); return OR_ERR_PATTERN; }
        } else {
            if (len == 0) { oracle_destroy(o); return OR_ERR_PATTERN; }
            int64_t i = o->fid[r];
            o->wptr[i + 1] = o->wptr[i] + len;
        }
    }
    o->nnzW = o->wptr[ff];
    int64_t W = o->nnzW ? o->nnzW : 1;
    o->wcol = (int32_t *)malloc(sizeof(int32_t) * W);
    for (int64_t i = 0; i < ff; ++i) {
        int64_t r = o->frow[i];
        memcpy(o->wcol + o->wptr[i], P_col + P_rowptr[r], sizeof(int32_t) * (o->wptr[i + 1] - o->wptr[i]));
    }
    /* B_c(coarse(c),:) must equal B(c,:) exactly (reading A21) */
    for (int64_t r = 0; r < n; ++r)
        if (is_coarse[r])
            for (int m = 0; m < nv; ++m)
                if (Bc[o->coarse_of[r] * nv + m] != B[r * nv + m]) { oracle_destroy(o); return OR_ERR_BC; }
    /* diagonal of the F rows and sum of the C diagonal */
    o->d = (double *)malloc(sizeof(double) * (ff ? ff : 1));
    nsum_t dcc = {0.0, 0.0};
    for (int64_t r = 0; r < n; ++r) {
        double dv = 0.0;
        for (int64_t q = A_rowptr[r]; q < A_rowptr[r + 1]; ++q) if (A_col[q] == r) dv = A_val[q];
        if (is_coarse[r]) nsum_add(&dcc, dv);
        else {
            if (!(dv > 0.0)) { oracle_destroy(o); return OR_ERR_DIAG; }
            o->d[o->fid[r]] = dv;
        }
    }
    o->sum_diag_cc = nsum_val(&dcc);
    /* Alg. 2 per F row */
    o->Q = (double *)calloc((size_t)W * nv, sizeof(double));
    o->krank = (int *)calloc(ff ? ff : 1, sizeof(int));
    o->w0 = (double *)calloc(W, sizeof(double));
    o->dw = (double *)calloc(W, sizeof(double));
    o->r = (double *)calloc(W, sizeof(double));
    o->y = (double *)calloc(W, sizeof(double));
    o->yb = (double *)calloc(W, sizeof(double));
    o->z = (double *)calloc(W, sizeof(double));
    int64_t n_svd = 0, n_frozen = 0, n_mvf = 0;
    #pragma omp parallel for schedule(dynamic, 256) reduction(+ : n_svd, n_frozen, n_mvf)
    for (int64_t i = 0; i < ff; ++i) {
        int64_t r = o->frow[i], b = o->wptr[i];
        int nj = (int)(o->wptr[i + 1] - b);
        double *M = (double *)malloc(sizeof(double) * nj * nv);
        double *wh = (double *)malloc(sizeof(double) * nj);
        double *delta = (double *)malloc(sizeof(double) * nj);
        double rv[16];
        for (int t = 0; t < nj; ++t) {
            int32_t j = o->wcol[b + t];
            for (int m = 0; m < nv; ++m) M[t + m * nj] = Bc[(int64_t)j * nv + m];
            wh[t] = P_val ? P_val[P_rowptr[r] + t] : 0.0;
        }
        if (start == 1) {                            /* Alg. 1 tentative start (reading A24) */
            int S[16];
            int ok = oracle_maxvol(nj, nv, M, S) && maxvol_solve(nj, nv, M, S, B + r * nv, wh);
            if (!ok) { for (int t = 0; t < nj; ++t) wh[t] = 0.0; n_mvf++; }
        }
        for (int m = 0; m < nv; ++m) {              /* r_i = v_i - M^T w^ */
            double s = B[r * nv + m];
            for (int t = 0; t < nj; ++t) s -= M[t + m * nj] * wh[t];
            rv[m] = s;
        }
        int used_svd = 0;
        int k = emin_setup_row(nj, nv, M, rv, rank_tol, o->Q + b * nv, delta, &used_svd);
        o->krank[i] = k;
        if (used_svd) n_svd++;
        if (nj == k) n_frozen++;
        for (int t = 0; t < nj; ++t) o->w0[b + t] = wh[t] + delta[t];
        free(M); free(wh); free(delta);
    }
    o->n_svd = n_svd; o->n_frozen = n_frozen; o->n_maxvol_fail = n_mvf;
    /* r0 = -Pi (A P0)|F   (readings A1, A2) */
    double *G = (double *)malloc(sizeof(double) * W);
    oracle_masked_AX(o, o->w0, 1, G);
    oracle_project(o, G, o->r);
    for (int64_t p = 0; p < o->nnzW; ++p) o->r[p] = -o->r[p];
    free(G);
    o->E0 = oracle_energy_of(o, o->w0);
    o->k_total = 0; o->stopped = OR_RUN; o->gamma_old = 0.0; o->dE1 = 0.0;
    *out = o;
    return OR_OK;
}

/* Alg. 3 main loop, continuing from the current state for up to kmax
 * iterations.  dE (nullable, length kmax) receives dE of applied steps.
 * Returns status; *k_done = number of applied updates in this call. */
int oracle_iterate(oracle_t *o, int kmax, int *k_done, double *dE) {
    *k_done = 0;
    int64_t W = o->nnzW;
    for (int it = 0; it < kmax; ++it) {
        if (o->stopped) break;
        int64_t k = o->k_total + 1;
        /* z = Pi M^-1 r: Jacobi M_1 = A(i,i) per row block
         * or the projected SGS M_2 */
        oracle_apply_prec(o, o->r, o->z);
        double gamma = dot_w(o, o->r, o->z);
        if (!(gamma > 0.0)) { o->stopped = OR_STOP_GAMMA; break; }
        if (k == 1) {
            #pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < W; ++p) o->y[p] = o->z[p];
        } else {
            double beta = gamma / o->gamma_old;
            #pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < W; ++p) o->y[p] = o->z[p] + beta * o->y[p];
        }
        o->gamma_old = gamma;
        oracle_masked_AX(o, o->y, 0, o->yb);
        oracle_project(o, o->yb, o->yb);
        double den = dot_w(o, o->y, o->yb);
        if (den < 0.0) { o->stopped = OR_STOP_DEN; return OR_ERR_BREAKDOWN; }
        if (den == 0.0) { o->stopped = OR_STOP_DEN; break; }
        double alpha = gamma / den;
        double dEk = gamma * alpha;
        if (k == 1) o->dE1 = dEk;
        if (o->tau > 0.0 && k > 1 && dEk < o->tau * o->dE1) { o->stopped = OR_STOP_TAU; break; }
        if (dEk <= o->stag * o->E0) { o->stopped = OR_STOP_STAG; break; }
        #pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < W; ++p) {
            o->dw[p] += alpha * o->y[p];
            o->r[p] -= alpha * o->yb[p];
        }
        if (dE) dE[*k_done] = dEk;
        o->k_total = k;
        (*k_done)++;
    }
    return OR_OK;
}

/* w = w0 + dw */
void oracle_get_W(const oracle_t *o, double *W) {
    for (int64_t p = 0; p < o->nnzW; ++p) W[p] = o->w0[p] + o->dw[p];
}
/* full P values in the input CSR order, C rows = 1 */
void oracle_get_P(const oracle_t *o, double *Pval) {
    for (int64_t r = 0; r < o->n; ++r) {
        if (o->isc[r]) { Pval[o->Prp[r]] = 1.0; continue; }
        int64_t i = o->fid[r];
        for (int64_t t = 0; t < o->wptr[i + 1] - o->wptr[i]; ++t)
            Pval[o->Prp[r] + t] = o->w0[o->wptr[i] + t] + o->dw[o->wptr[i] + t];
    }
}
double oracle_energy(const oracle_t *o) {
    double *W = (double *)malloc(sizeof(double) * (o->nnzW ? o->nnzW : 1));
    oracle_get_W(o, W);
    double e = oracle_energy_of(o, W);
    free(W);
    return e;
}
void oracle_reset(oracle_t *o) {
    memset(o->dw, 0, sizeof(double) * o->nnzW);
    double *G = (double *)malloc(sizeof(double) * (o->nnzW ? o->nnzW : 1));
    oracle_masked_AX(o, o->w0, 1, G);
    oracle_project(o, G, o->r);
    for (int64_t p = 0; p < o->nnzW; ++p) o->r[p] = -o->r[p];
    free(G);
    o->k_total = 0; o->stopped = OR_RUN; o->gamma_old = 0.0; o->dE1 = 0.0;
}

/* ---------------- accessors for the Python wrapper ----------------------- */
/* threads of the parallel loops (1 = the serial order everywhere) */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}
int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
int64_t oracle_nF(const oracle_t *o) { return o->nF; }
int64_t oracle_nnzW(const oracle_t *o) { return o->nnzW; }
double oracle_E0(const oracle_t *o) { return o->E0; }
double oracle_dE1(const oracle_t *o) { return o->dE1; }
int64_t oracle_k_total(const oracle_t *o) { return o->k_total; }
int oracle_stopped(const oracle_t *o) { return o->stopped; }
int64_t oracle_n_svd(const oracle_t *o) { return o->n_svd; }
int64_t oracle_n_frozen(const oracle_t *o) { return o->n_frozen; }
int64_t oracle_n_maxvol_fail(const oracle_t *o) { return o->n_maxvol_fail; }
double oracle_sum_diag_cc(const oracle_t *o) { return o->sum_diag_cc; }
void oracle_copy_layout(const oracle_t *o, int64_t *wptr, int32_t *wcol, int64_t *frow) {
    memcpy(wptr, o->wptr, sizeof(int64_t) * (o->nF + 1));
    memcpy(wcol, o->wcol, sizeof(int32_t) * o->nnzW);
    memcpy(frow, o->frow, sizeof(int64_t) * o->nF);
}
void oracle_copy_vec(const oracle_t *o, int which, double *out) {
    const double *src = which == 0 ? o->w0 : which == 1 ? o->dw : which == 2 ? o->r
                      : which == 3 ? o->y : which == 4 ? o->yb : o->d;
    int64_t len = which == 5 ? o->nF : o->nnzW;
    memcpy(out, src, sizeof(double) * len);
}
void oracle_copy_Q(const oracle_t *o, double *Q, int *krank) {
    memcpy(Q, o->Q, sizeof(double) * o->nnzW * o->nv);
    memcpy(krank, o->krank, sizeof(int) * o->nF);
}
/* Setup-row entry point for the QR/SVD pins: M col-major nj x nv. */
int oracle_setup_row(int nj, int nv, const double *M, const double *rvec, double tol,
                     double *Qrow, double *delta, int *used_svd) {
    return emin_setup_row(nj, nv, M, rvec, tol, Qrow, delta, used_svd);
}

/* ---------------- Alg. 1 pattern growth (NEXT-3, reading A25) ----------- */
/* The sparsity pattern of P from the graph of A (Eq. enlPatt, and
 * the growth loop of Alg. 1): the graph has an edge i ~ k for every
 * off-diagonal nonzero of A (reading A12, no strength threshold); with
 * block_size 3 it is the node graph (node I ~ K if the 3x3 block (I,K) has a
 * nonzero; rows 3I..3I+2 of a node) and the pattern is applied blockwise.
 * For every F node: N_l = the C nodes within graph distance l, for
 * l = l0, l0+1, ... until the Gram matrix G = M^T M of M = V_c(J,:) (J = the
 * dofs of N_l) has lambda_min > 1e-10 lambda_max (full rank; the same
 * criterion as the input generator), and unconditionally at l = lmax.
 * Columns ascending (coarse ids).  C rows: {coarse(c)}. */

/* eigenvalues of the symmetric n x n matrix a (row-major, destroyed) by
 * cyclic Jacobi rotations; returns min and max */
static void jacobi_eig_minmax(int n, double *a, double *lmin, double *lmax) {
    for (int sweep = 0; sweep < 50; ++sweep) {
        /* converged when the off-diagonal mass is below (1e-16 trace)^2: the
         * eigenvalues are then exact to ~1e-16 lambda_max, far inside the
         * 1e-10 rank threshold */
        double off = 0.0, tr = 0.0;
        for (int p = 0; p < n; ++p) {
            tr += fabs(a[p * n + p]);
            for (int q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
        }
        if (off <= 1e-32 * tr * tr) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                double apq = a[p * n + q];
                if (apq == 0.0) continue;
                double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) {          /* columns p, q */
                    double akp = a[k * n + p], akq = a[k * n + q];
                    a[k * n + p] = c * akp - s * akq;
                    a[k * n + q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {          /* rows p, q */
                    double apk = a[p * n + k], aqk = a[q * n + k];
                    a[p * n + k] = c * apk - s * aqk;
                    a[q * n + k] = s * apk + c * aqk;
                }
            }
    }
    double mn = a[0], mx = a[0];
    for (int k = 1; k < n; ++k) { if (a[k * n + k] < mn) mn = a[k * n + k]; if (a[k * n + k] > mx) mx = a[k * n + k]; }
    *lmin = mn; *lmax = mx;
}

int oracle_gram_full_rank(int nv, const double *G) {
    double a[256], mn, mx;
    memcpy(a, G, sizeof(double) * nv * nv);
    jacobi_eig_minmax(nv, a, &mn, &mx);
    if (mx < 0.0) mx = 0.0;
    return mn > 1e-10 * mx;
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Returns the number of nonzeros of the pattern (all rows); fills P_rowptr
 * [n+1] and, if P_col != NULL, P_col.  Also the histogram of the distance
 * used per F node (hist[l], l <= lmax) if hist != NULL. */
int64_t oracle_pattern(int64_t n, const int64_t *A_rowptr, const int32_t *A_col, const uint8_t *is_coarse,
                       int block_size, int nv, const double *Bc, int l0, int lmax,
                       int64_t *P_rowptr, int32_t *P_col, int64_t *hist) {
    int bs = block_size;
    int64_t nn = n / bs;                          /* nodes */
    int64_t *cid = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t nc = 0;
    for (int64_t u = 0; u < nn; ++u) cid[u] = is_coarse[u * bs] ? nc++ : -1;
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * nn);
    for (int64_t u = 0; u < nn; ++u) stamp[u] = -1;
    int64_t *front = (int64_t *)malloc(sizeof(int64_t) * nn), *next = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t *clist = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t nnz = 0;
    if (hist) for (int l = 0; l <= lmax; ++l) hist[l] = 0;
    P_rowptr[0] = 0;
    for (int64_t I = 0; I < nn; ++I) {
        int64_t cnt = 0;
        if (cid[I] >= 0) {
            cnt = 1;
        } else {
            int64_t nf = 1, ncl = 0;
            front[0] = I;
            stamp[I] = I;
            int lused = lmax;
            for (int l = 1; l <= lmax; ++l) {
                int64_t nx = 0;
                for (int64_t f = 0; f < nf; ++f) {
                    int64_t u = front[f], r = u * bs;
                    for (int64_t q = A_rowptr[r]; q < A_rowptr[r + 1]; ++q) {
                        int64_t w = A_col[q] / bs;
                        if (stamp[w] == I) continue;
                        stamp[w] = I;
                        next[nx++] = w;
                        if (cid[w] >= 0) clist[ncl++] = cid[w];
                    }
                }
                memcpy(front, next, sizeof(int64_t) * nx);
                nf = nx;
                if (l < l0) continue;
                if (l == lmax) break;
                if (ncl == 0) continue;
                double G[256];
                for (int k = 0; k < nv * nv; ++k) G[k] = 0.0;
                for (int64_t t = 0; t < ncl; ++t)
                    for (int b = 0; b < bs; ++b) {
                        const double *row = Bc + (bs * clist[t] + b) * nv;
                        for (int p = 0; p < nv; ++p)
                            for (int q = 0; q < nv; ++q) G[p * nv + q] += row[p] * row[q];
                    }
                if (oracle_gram_full_rank(nv, G)) { lused = l; break; }
            }
            if (hist) hist[lused]++;
            qsort(clist, ncl, sizeof(int64_t), cmp_i64);
            cnt = ncl * bs;
            if (P_col)
                for (int64_t t = 0; t < ncl; ++t)
                    for (int b = 0; b < bs; ++b) P_col[nnz + t * bs + b] = (int32_t)(bs * clist[t] + b);
        }
        const int64_t base = nnz;
        if (cid[I] >= 0) {                          /* C rows: each dof row its own column */
            if (P_col) for (int b = 0; b < bs; ++b) P_col[base + b] = (int32_t)(bs * cid[I] + b);
        } else if (P_col) {                         /* the bs rows of an F node share the list */
            for (int b = 1; b < bs; ++b) memcpy(P_col + base + b * cnt, P_col + base, sizeof(int32_t) * cnt);
        }
        for (int b = 0; b < bs; ++b) {
            nnz += cnt;
            P_rowptr[I * bs + b + 1] = nnz;
        }
    }
    free(cid); free(stamp); free(front); free(next); free(clist);
    return nnz;
}

/* ------------------------------------------------------------------------
 * galerkin (reading A26): the coarse operator of the next
 * level, A_c = P^T A P -- the matrix whose trace is the energy the method
 * minimises (Eq. trace), formed by the "sparse matrix-matrix
 * product" of the coarse grid construction.  Textbook
 * two-product definition, in this order:
 *   T = A P            row i of T: T(i,j) = sum_k A(i,k) P(k,j), k in A's
 *                      column order, one rounding per multiply and add;
 *   A_c = P^T T        row c of A_c: A_c(c,j) = sum_i P(i,c) T(i,j), i
 *                      ascending.
 * Structural pattern: (c, j) is stored if some product term exists (values
 * that cancel to 0 are kept); columns ascending.  Returns nnz(A_c); fills
 * Ac_rowptr [nc+1] and, when Ac_col != NULL, Ac_col / Ac_val.
 * ------------------------------------------------------------------------ */
int64_t oracle_galerkin(int64_t n, int64_t nc, const int64_t *A_rowptr, const int32_t *A_col,
                        const double *A_val, const int64_t *P_rowptr, const int32_t *P_col,
                        const double *P_val, int64_t *Ac_rowptr, int32_t *Ac_col, double *Ac_val) {
    /* T = A P, dense accumulator + marker per row (Gustavson) */
    double *acc = (double *)calloc(nc > 0 ? nc : 1, sizeof(double));
    int64_t *mark = (int64_t *)malloc(sizeof(int64_t) * (nc > 0 ? nc : 1));
    int64_t *list = (int64_t *)malloc(sizeof(int64_t) * (nc > 0 ? nc : 1));
    for (int64_t j = 0; j < nc; ++j) mark[j] = -1;
    int64_t *Trp = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    int64_t cap = 1024, nnzT = 0;
    int32_t *Tcol = (int32_t *)malloc(sizeof(int32_t) * cap);
    double *Tval = (double *)malloc(sizeof(double) * cap);
    Trp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t m = 0;
        for (int64_t q = A_rowptr[i]; q < A_rowptr[i + 1]; ++q) {
            int64_t k = A_col[q];
            for (int64_t s = P_rowptr[k]; s < P_rowptr[k + 1]; ++s) {
                int64_t j = P_col[s];
                if (mark[j] != i) { mark[j] = i; acc[j] = 0.0; list[m++] = j; }
                acc[j] = acc[j] + A_val[q] * P_val[s];
            }
        }
        if (nnzT + m > cap) {
            while (nnzT + m > cap) cap *= 2;
            Tcol = (int32_t *)realloc(Tcol, sizeof(int32_t) * cap);
            Tval = (double *)realloc(Tval, sizeof(double) * cap);
        }
        for (int64_t t = 0; t < m; ++t) { Tcol[nnzT] = (int32_t)list[t]; Tval[nnzT] = acc[list[t]]; ++nnzT; }
        Trp[i + 1] = nnzT;
    }
    /* P^T by counting (rows i ascending within each column c) */
    int64_t nnzP = P_rowptr[n];
    int64_t *Ptp = (int64_t *)calloc(nc + 1, sizeof(int64_t));
    for (int64_t s = 0; s < nnzP; ++s) Ptp[P_col[s] + 1]++;
    for (int64_t c = 0; c < nc; ++c) Ptp[c + 1] += Ptp[c];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (nc > 0 ? nc : 1));
    for (int64_t c = 0; c < nc; ++c) fill[c] = Ptp[c];
    int64_t *Ptrow = (int64_t *)malloc(sizeof(int64_t) * (nnzP > 0 ? nnzP : 1));
    double *Ptval = (double *)malloc(sizeof(double) * (nnzP > 0 ? nnzP : 1));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t s = P_rowptr[i]; s < P_rowptr[i + 1]; ++s) {
            int64_t c = P_col[s];
            Ptrow[fill[c]] = i; Ptval[fill[c]] = P_val[s]; fill[c]++;
        }
    /* A_c = P^T T */
    for (int64_t j = 0; j < nc; ++j) mark[j] = -1;
    int64_t nnz = 0;
    Ac_rowptr[0] = 0;
    for (int64_t c = 0; c < nc; ++c) {
        int64_t m = 0;
        for (int64_t s = Ptp[c]; s < Ptp[c + 1]; ++s) {
            int64_t i = Ptrow[s];
            for (int64_t t = Trp[i]; t < Trp[i + 1]; ++t) {
                int64_t j = Tcol[t];
                if (mark[j] != c) { mark[j] = c; acc[j] = 0.0; list[m++] = j; }
                acc[j] = acc[j] + Ptval[s] * Tval[t];
            }
        }
        qsort(list, m, sizeof(int64_t), cmp_i64);
        if (Ac_col)
            for (int64_t t = 0; t < m; ++t) { Ac_col[nnz + t] = (int32_t)list[t]; Ac_val[nnz + t] = acc[list[t]]; }
        nnz += m;
        Ac_rowptr[c + 1] = nnz;
    }
    free(acc); free(mark); free(list); free(Trp); free(Tcol); free(Tval);
    free(Ptp); free(fill); free(Ptrow); free(Ptval);
    return nnz;
}
