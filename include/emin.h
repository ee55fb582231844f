/*
 * emin.h -- C ABI of the B200-native restricted-PCG energy minimisation of an
 * AMG prolongation (arXiv 2208.02995).  PAPER.md = /root/reference/PAPER.md,
 * cited as P:<line> [section / equation / algorithm].
 *
 * Problem (Eq. inKern + trace, Eq. TSP/Constr):
 *     minimise tr(P^T A P)  over P = [W; I] (Eq. prol)
 *     subject to  W on a fixed sparsity pattern and P B_c = B.
 * Method: Alg. 2 EMIN_SetUp once, then Alg. 3 EMIN_PCG
 * with the Jacobi preconditioner M_1, K applied
 * matrix-free as the masked product A.P on the pattern, Pi_B
 * applied row by row from small orthonormal Q_i.  Readings of the
 * garbled passages are listed in DESIGN.md §3.
 *
 * Conventions for every call
 *  - All functions return emin_status; EMIN_OK (= 0) on success.
 *  - Layouts: CSR with int64 row pointers and int32 column indices, values
 *    fp64; dense blocks row-major.  Rows of A, P and B are the rows this
 *    process OWNS, [row_begin, row_end) of the global numbering (the whole
 *    matrix on one GPU); column indices are GLOBAL.
 *  - Pointers are host pointers unless opts->inputs_on_device = 1, in which
 *    case they are device pointers on the current CUDA device.  Inputs are
 *    read only during emin_setup (copied); the caller keeps ownership.
 *  - The context owns all device memory it allocates and releases it in
 *    emin_destroy.  Outputs go to caller-allocated buffers.
 *  - Work is enqueued on opts->stream (cudaStream_t, NULL = legacy default).
 *    emin_iterate is asynchronous unless k_done or dE is non-NULL.
 *  - Multi-GPU: emin_setup, emin_iterate, emin_energy, emin_get_P and
 *    emin_reset are collective over opts->nccl_comm (or the in-process
 *    opts->loopback group): every rank calls them in the same order;
 *    nccl_comm = loopback = NULL means one GPU owning all rows.
 *  - After a failing call other than emin_setup the context stays valid;
 *    emin_destroy is always safe (also on NULL).
 */
#ifndef EMIN_H_
#define EMIN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct emin_ctx_s* emin_ctx;

typedef enum {
  EMIN_OK = 0,
  EMIN_ERR_ARG = 1,        /* bad scalar argument, NULL pointer, nv out of [1,8] */
  EMIN_ERR_CSR = 2,        /* A rowptr not monotone, column out of range, unsorted or duplicate */
  EMIN_ERR_PATTERN = 3,    /* C row != {coarse(c)} (value 1 if P_val given), F row empty,
                              unsorted or out of [0, nc), or an F row longer than EMIN_MAX_ROW */
  EMIN_ERR_BC = 4,         /* B_c(coarse(c),:) != B(c,:) bitwise (reading A21) */
  EMIN_ERR_DIAG = 5,       /* A(i,i) missing or <= 0 on an F row (Jacobi) */
  EMIN_ERR_NONFINITE = 6,  /* NaN/Inf in A, B, B_c or P_val */
  EMIN_ERR_BREAKDOWN = 7,  /* y^T Pi K y < 0 (SPD A makes it >= 0) */
  EMIN_ERR_CUDA = 8,
  EMIN_ERR_NCCL = 9,
  EMIN_ERR_OOM = 10,
  EMIN_ERR_STATE = 11      /* call on a context in the wrong state */
} emin_status;

/* Longest F-row pattern the kernels accept (|J_i|). */
#define EMIN_MAX_ROW 128

typedef struct {
  int32_t block_size;           /* 1 = point rows; 3 = nodal hint: rows 3m..3m+2 share J
                                   (elasticity), enables the 3x3 block kernels when valid */
  double  rank_tol;             /* relative rank tolerance of Alg. 2's QR/SVD tests, 1e-10
                                   (reading A6) */
  double  tau;                  /* stop when dE_k < tau dE_1, k > 1 (Eq. relRed);
                                   0 = run exactly k steps.  Paper default 0.1 */
  int32_t project_after_jacobi; /* 1 = literal Alg. 3 line P:840 (z = Pi M^-1 r); 0 = skip the
                                   post-projection, exact for Jacobi (reading A7) */
  double  stagnation_rel;       /* stop (no update) when dE_k <= stagnation_rel * E_0
                                   (reading A18; 1e-30 default, 0 disables) */
  void*   stream;               /* cudaStream_t */
  void*   nccl_comm;            /* ncclComm_t or NULL (one GPU) */
  int64_t row_begin, row_end;   /* owned global rows; [0, n_global) on one GPU */
  int32_t inputs_on_device;     /* 1: the array arguments of emin_setup are device pointers */
  int32_t precond;              /* EMIN_PREC_JACOBI: M_1 = diag(K), row-wise scaling;
                                   EMIN_PREC_SGS: projected symmetric Gauss-Seidel
                                   M_2^-1 = Z^T (L+D)^-T D (L+D)^-1 Z, applied
                                   matrix-free as a forward and a backward sweep over the F rows
                                    and always followed by Pi_B.  On several ranks
                                   every rank sweeps all global dependency levels and the halo
                                   rows' values are exchanged after each level (the order is
                                   global: (sgs_key, global row)). */
  const int64_t* sgs_key;       /* nullable, [m] per owned row: SGS visits the unknowns of each
                                   K block (coarse column) in ascending (key, global
                                   row) order (reading A23); NULL = natural row order.  Host or
                                   device pointer as the other arrays.  A colouring key makes the
                                   sweeps short (few dependency levels). */
  int32_t start;                /* EMIN_START_GIVEN: W^ = P_val, or the least-norm start if
                                   P_val is NULL (reading A9);  EMIN_START_MAXVOL: the tentative
                                   start of Alg. 1 on the given pattern -- per F row
                                   the max-vol selection of nv columns of V_c(J_i,:)^T, the local
                                   system solved exactly on them, zero elsewhere (reading A24;
                                   P_val ignored).  Rows without a nonsingular selection keep
                                   W^ = 0 (counted in emin_report_t.n_maxvol_fail). */
  void*   loopback;             /* emin_loopback handle or NULL: the row-partitioned path with
                                   R ranks as R contexts on ONE device in one process (one
                                   thread per rank), exchanging through device-to-device
                                   copies ordered by events and host barriers instead of NCCL
                                   (see emin_loopback_create).  Mutually exclusive with
                                   nccl_comm.  Iterations are enqueued eagerly (no CUDA graph). */
  int32_t loopback_rank;        /* this context's rank in the loopback group */
  int32_t debug_flags;          /* 0 for production.  Bits (EMIN_DBG_*) select reference or
                                   alternative code paths for tests and A/B measurements; they
                                   never change the method, only which kernels compute it. */
} emin_opts;

/* emin_opts.debug_flags bits */
#define EMIN_DBG_FORCE_GENERIC 1   /* generic warp-per-row kernels instead of the scalar / nodal
                                      specialisations (the reference the fast paths are tested
                                      against) */
#define EMIN_DBG_UNSCALED 512      /* scalar Jacobi path: the CG vectors in the original variables
                                      (z = r / d by division, per-entry row gathers of d) instead of
                                      the symmetrically scaled ones (D^-1/2 A D^-1/2 records) */
#define EMIN_DBG_AB2 128           /* scalar path: the per-iteration masked product with one W
                                      entry per lane (k_spgemm_wd) instead of two (k_spgemm_wp) */
#define EMIN_DBG_NO_R0E 2          /* r0 and E0 by two masked passes instead of the fused one */
#define EMIN_DBG_SGS_GENERIC 4     /* generic warp-per-row SGS sweeps */
#define EMIN_DBG_TRACE 8           /* synchronise and print each setup phase's host time */
#define EMIN_DBG_FUSE_SCALARS 16   /* one GPU: CG scalar steps in the last block of the producing
                                      kernels instead of separate single-block kernels */
#define EMIN_DBG_ALG2_ROWS 32      /* nodal path: Alg. 2 row by row instead of once per node */
#define EMIN_DBG_AB1 64            /* A/B switch of the kernel under study;
                                      currently: the nodal SGS sweeps on the unsorted blocks
                                      (the reference the direction-sorted sweeps are tested
                                      against) */

#define EMIN_PREC_JACOBI 0
#define EMIN_PREC_SGS 1
#define EMIN_START_GIVEN 0
#define EMIN_START_MAXVOL 1

typedef struct {
  double  E0;          /* tr(P0^T A P0) after Alg. 2 */
  double  dE1;         /* first energy decrease (0 before the first step) */
  int64_t k_total;     /* accepted PCG steps since setup/reset */
  int32_t stop_reason; /* 0 running, 1 gamma <= 0, 2 y'Ky == 0, 3 tau, 4 stagnation,
                          5 breakdown */
  int64_t n_svd_rows;  /* F rows that took Alg. 2's SVD branch */
  int64_t n_frozen_rows;  /* F rows with |J_i| == rank (no free dof) */
  int64_t n_fine, nnz_W, nnz_AFF;  /* owned F rows, W entries, A_FF entries */
  int32_t kernel_path; /* 0 generic warp-per-row, 1 scalar lane-per-entry, 2 nodal 3x3 */
  int32_t nranks;
  int64_t launches;    /* kernels this context has enqueued so far (setup included) */
  int32_t precond;     /* EMIN_PREC_JACOBI or EMIN_PREC_SGS */
  int64_t sgs_levels;  /* dependency levels of one SGS sweep (0 for Jacobi) */
  int64_t n_maxvol_fail;  /* F rows where the max-vol start found no nonsingular selection */
  int32_t rank;        /* this context's rank (0 on one GPU) */
  int64_t n_halo_rows; /* F rows of other ranks whose pattern / values this rank receives */
  int64_t n_halo_entries;  /* their W entries (doubles received per halo exchange) */
  int64_t n_send_entries;  /* W entries this rank sends per halo exchange */
  int64_t n_interior_units;  /* units (windows / nodes / rows of the kernel path) of y^ = Pi K y
                                computed while the halo is exchanged (0: no overlap) */
} emin_report_t;

/* Fill opts with defaults (rank_tol 1e-10, tau 0, project_after_jacobi 0,
 * stagnation_rel 1e-30, block_size 1, one GPU over [0, n_global), Jacobi). */
void emin_default_opts(emin_opts* opts, int64_t n_global);

/* Alg. 2 + the start of Alg. 3:
 *   validates the inputs, builds the F-row structures, per F row i the
 *   orthonormal Q_i of M_i = B_c(J_i,:) and the correction delta_i, the
 *   start W0 = W^ + delta, r0 = Pi_B(f - K w0) = -Pi_B (A P0)|_F (reading A1)
 *   and E0.
 * n_global, nc_global : global row count and coarse count.
 * A_rowptr [m+1], A_col, A_val : owned rows of A (m = row_end - row_begin),
 *   global column ids, strictly increasing per row; A must be SPD.
 * is_coarse [n_global] : 1 for C points, 0 for F points (global).  Coarse
 *   id of a C point = its rank among C points in ascending global order.
 * P_rowptr [m+1], P_col : pattern of the owned rows of P, coarse ids,
 *   strictly increasing; C rows must be exactly {coarse(c)}.
 * P_val (nullable, same layout) : starting W^ (NULL: W^ = 0, least-norm
 *   start, reading A9); its C-row values must be 1.
 * nv in [1, 8]; B [m x nv] owned rows of the near kernel; Bc [nc_global x nv].
 * On failure *out = NULL and the status says why. */
emin_status emin_setup(emin_ctx* out, int64_t n_global, int64_t nc_global,
                       const int64_t* A_rowptr, const int32_t* A_col, const double* A_val,
                       const uint8_t* is_coarse,
                       const int64_t* P_rowptr, const int32_t* P_col, const double* P_val,
                       int32_t nv, const double* B, const double* Bc,
                       const emin_opts* opts);

/* Run up to k steps of Alg. 3 from the current state.
 * k_done (nullable): accepted steps in this call; dE (nullable, length k):
 * their energy decreases dE_j = gamma alpha (Eq. CG_dEa).  Passing
 * either forces a stream synchronisation.  emin_iterate(k1); emin_iterate(k2)
 * is bitwise equal to emin_iterate(k1 + k2).  EMIN_ERR_BREAKDOWN is reported
 * by the first call that observes it (synchronously only if k_done/dE given,
 * else by the next emin_report/emin_energy/emin_get_P). */
emin_status emin_iterate(emin_ctx ctx, int32_t k, int32_t* k_done, double* dE);

/* E = tr(P^T A P) of the current iterate (Eq. trace; by
 * Eq. trInc P:417-426 = sum_F W.(A_FF W + 2 A_FC) + tr(A_CC)).  Synchronous.
 * Collective. */
emin_status emin_energy(emin_ctx ctx, double* E);

/* Current P values of the owned rows in the input CSR order (C rows = 1),
 * W = W0 + dW.  P_val is a host pointer unless
 * opts.inputs_on_device, then a device pointer.  Synchronous. */
emin_status emin_get_P(emin_ctx ctx, double* P_val);

/* Back to W0, r0 (for benchmark repeats).  Collective. */
emin_status emin_reset(emin_ctx ctx);

/* Counters and scalars (synchronous). */
emin_status emin_report(emin_ctx ctx, emin_report_t* rep);

void emin_destroy(emin_ctx ctx);

const char* emin_status_str(emin_status s);

/* Device memory: every allocation of the library comes from a library-owned
 * stream-ordered pool per device (the device's default pool is left as it
 * is).  Freed blocks stay cached in that pool, so repeated emin_setup calls
 * reuse them; emin_release_memory() synchronises the device and returns all
 * cached blocks to the driver (emin_galerkin and emin_pattern release their
 * temporaries themselves). */
void emin_release_memory(void);
/* Last error message recorded on ctx (or of the last failed emin_setup when
 * ctx == NULL).  Never NULL. */
const char* emin_last_error(emin_ctx ctx);

/* Index structure the context built (for parity tests), host outputs:
 * wptr [n_fine+1] W-layout row pointers of the owned F rows (ascending
 * global order), wcol [nnz_W] coarse ids, pofs [n_fine] offset of each F
 * row in the caller's P CSR (relative to P_rowptr[0]).  Synchronous. */
emin_status emin_get_layout(emin_ctx ctx, int64_t* wptr, int32_t* wcol, int64_t* pofs);

/* Alg. 1's pattern growth (P:527-540 with Eq. enlPatt; SURVEY §8f
 * NEXT-3, reading A25) on one GPU: the sparsity pattern of P from the graph
 * of A.  Graph: an edge i ~ k per off-diagonal nonzero of A (no strength
 * threshold, reading A12); block_size 3 = the node graph of 3x3 blocks (row
 * 3I lists node I's neighbours), pattern applied blockwise.  For every F node
 * the C nodes within graph distance l, l = l0, l0+1, ... until
 * lambda_min(M^T M) > 1e-10 lambda_max(M^T M), M = Bc(J,:) (J = their
 * dofs), and unconditionally at l = lmax; columns ascending; C rows
 * {coarse(c)} (coarse id = rank among C points).
 *   n, A_rowptr [n+1], A_col : the whole matrix (global); is_coarse [n];
 *   Bc [nc x nv] row-major; P_rowptr [n+1] out; P_col [nnz] out or NULL
 *   (count only); P_col_cap its capacity (EMIN_ERR_ARG if < nnz, P_rowptr
 *   and *nnz_out still filled: call again); all pointers host, or device if
 *   inputs_on_device; stream = cudaStream_t.  Synchronous.
 * EMIN_ERR_PATTERN if a neighbourhood exceeds the kernel's shared-memory sets
 * (2048 visited nodes / 1024 frontier or C nodes per F node). */
emin_status emin_pattern(int64_t n, const int64_t* A_rowptr, const int32_t* A_col, const uint8_t* is_coarse,
                         int32_t block_size, int32_t nv, const double* Bc, int64_t nc, int32_t l0,
                         int32_t lmax, int64_t* P_rowptr, int32_t* P_col, int64_t P_col_cap,
                         int64_t* nnz_out, int32_t inputs_on_device, void* stream);
const char* emin_pattern_error(void);

/* The next level's operator A_c = P^T A P (reading A26):
 * the matrix whose trace is the energy (Eq. trace), formed by the
 * coarse grid construction's sparse matrix-matrix product before
 * the method is re-run on the next level.  T = A P, then A_c = P^T T; every
 * entry is the sum of its product terms in X order (A's column order, then
 * P's rows ascending), one rounding per multiply and add -- bitwise
 * reproducible; structural pattern (cancelled values are kept), columns
 * ascending.
 *   n, A_rowptr [n+1], A_col, A_val : A (n x n CSR);  P_rowptr [n+1], P_col
 *   (coarse ids < nc), P_val : P (n x nc CSR, e.g. from emin_get_P with the
 *   caller's pattern);  Ac_rowptr [nc+1] out;  Ac_col / Ac_val [Ac_cap] out,
 *   or Ac_col = NULL to count only (EMIN_ERR_ARG if Ac_cap < nnz, Ac_rowptr
 *   and *nnz_out still filled: call again);  all pointers host, or device if
 *   flags & EMIN_GALERKIN_DEVICE;  stream = cudaStream_t.  Synchronous; temporaries
 *   (T, P^T) are allocated on the stream and freed before returning.
 * EMIN_ERR_CSR on decreasing row pointers or column ids out of range;
 * EMIN_ERR_ARG if a row of T or A_c has more than 8192 distinct columns
 * (the 3x3-block product handles node rows of up to 1024 node columns and
 * hands wider ones to the point product). */
emin_status emin_galerkin(int64_t n, int64_t nc, const int64_t* A_rowptr, const int32_t* A_col,
                          const double* A_val, const int64_t* P_rowptr, const int32_t* P_col,
                          const double* P_val, int64_t* Ac_rowptr, int32_t* Ac_col, double* Ac_val,
                          int64_t Ac_cap, int64_t* nnz_out, int32_t flags, void* stream);
const char* emin_galerkin_error(void);
/* emin_galerkin flags: bit 0 (EMIN_GALERKIN_DEVICE) = all pointers are device
 * pointers; bit 1 (EMIN_GALERKIN_POINT) = always the point product (test of
 * the 3x3-block path, which must equal it bitwise). */
#define EMIN_GALERKIN_DEVICE 1
#define EMIN_GALERKIN_POINT 2
/* Which product the last emin_galerkin call of this thread used: 1 = the 3x3
 * block path (A in full 3x3 node blocks, P blockwise on F nodes and the
 * identity on C nodes -- the elasticity structure; same sums, bitwise), 0 =
 * the point path. */
int32_t emin_galerkin_path(void);

/* Multi-GPU helpers (one process per GPU, NCCL over NVLink/NVSwitch).
 * emin_nccl_unique_id fills id[128] on one rank; the caller broadcasts it
 * (e.g. with torch.distributed) and every rank calls emin_nccl_comm_init;
 * the resulting ncclComm_t goes into emin_opts.nccl_comm.  Row ranges must
 * be contiguous, ascending with the rank and cover [0, n_global).  Halo
 * rows (F rows of other ranks that the owned A_FF rows reference) are
 * found and their pattern exchanged once in emin_setup; per
 * iteration only y on those rows and two scalars are exchanged.
 * EMIN_ERR_NCCL if the library was built without NCCL. */
emin_status emin_nccl_unique_id(uint8_t* id128);
emin_status emin_nccl_comm_init(void** comm, int32_t nranks, const uint8_t* id128, int32_t rank);
emin_status emin_nccl_comm_destroy(void* comm);

/* In-process loopback transport (tests and single-GPU emulation of the
 * row-partitioned path).  R contexts, each set up by its
 * own host thread with opts.loopback = the handle and opts.loopback_rank = r,
 * share one device.  Every collective of the NCCL path has a loopback
 * counterpart with the same data movement: the halo exchange
 * becomes one cudaMemcpyAsync per (sender, receiver) pair from the sender's
 * packed buffer into the receiver's halo tail, ordered by CUDA events; the
 * scalar sums (allreduce) are one small kernel per rank adding the R rank-local
 * sums in rank order; setup-time gathers go through host memory.  Host threads
 * rendezvous at a barrier inside each collective, so all R ranks must call the
 * collective calls (emin_setup, emin_iterate, emin_energy, emin_reset,
 * emin_get_P) in the same order, each from its own thread.  No kernel waits on
 * another rank's kernel (stream-ordered copies only).
 * emin_loopback_create: nranks in [1, 64]; *out = handle.  destroy after every
 * context of the group is destroyed. */
emin_status emin_loopback_create(void** out, int32_t nranks);
void emin_loopback_destroy(void* lb);

/* Device time of the most recent emin_iterate's kernels, per kernel class,
 * accumulated with CUDA events on the launching stream when profiling is
 * enabled (emin_set_profiling(ctx, 1)); ms[0] stage I, ms[1] stage II,
 * ms[2] masked SpGEMM, ms[3] scalar/reduction kernels; launches[4] counts. */
emin_status emin_set_profiling(emin_ctx ctx, int32_t on);
emin_status emin_kernel_times(emin_ctx ctx, double* ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* EMIN_H_ */
