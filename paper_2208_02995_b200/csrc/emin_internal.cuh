// emin_internal.cuh -- internal types and device helpers of libemin (sm_100a).
// Not part of the ABI; see include/emin.h.  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/emin.h"

#define EMIN_NV_MAX 8
#define EMIN_WARP 32

// Device-resident CG scalars (Alg. 3 state).  One instance per
// context; updated only by the single-block scalar kernels, read by all.
struct DevState {
  double gamma;       // r^T z of the current step
  double gamma_old;
  double beta;        // gamma / gamma_old
  double alpha_pend;  // alpha of the accepted step whose updates are pending
  double den;         // y^T Pi K y
  double dE1;         // dE of the first step (Eq. relRed)
  double E0;          // tr(P0^T A P0)
  double tau, stag;
  int64_t k_total;    // accepted steps since setup / reset
  int32_t stopped;    // 0 running, 1 gamma<=0, 2 den==0, 3 tau, 4 stagnation, 5 breakdown
  int32_t pend;       // r -= alpha_pend yb pending (applied by stage I); 1: with dw += alpha_pend y, 2: without
  int32_t pendw;      // dw += alpha_pend y pending (applied by stage II)
  int32_t k_call;     // accepted steps in the current emin_iterate call
  double red[4];      // multi-GPU: rank-local sums [0] gamma, [1] y.yb, [2] energy
  double redg[4];     // ... and their sums over the ranks (allreduce red -> redg)
  uint32_t ctr[2];    // fused scalar steps: blocks done in stage I [0] / SpGEMM [1]
  double sum_cc;      // sum of A(c,c) over the C rows (all ranks; Eq. trInc), set at setup
  unsigned long long cnt[3];   // setup counters: SVD-branch rows, frozen rows, max-vol failures
};

struct DistPlan;
struct SgsPlan;

// Error flag bits raised by the validation kernels.
enum : int32_t {
  EF_CSR = 1, EF_PATTERN = 2, EF_BC = 4, EF_DIAG = 8, EF_NONFINITE = 16, EF_ROWLEN = 32
};

// Plain-pointer view of the device data used by the kernels.
struct DevView {
  int64_t nF;       // owned F rows
  int64_t nFh;      // owned + halo F rows (halo rows are appended)
  int64_t nnzW;     // owned W entries
  int32_t nv;
  const int64_t* wptr;   // [nFh+1]
  const int32_t* wcol;   // [wptr[nFh]]
  const int64_t* affptr; // [nF+1] A_FF in local F ids
  const int32_t* affcol;
  const double* affval;
  const int64_t* afcptr; // [nF+1] A_FC with coarse ids (setup / energy only)
  const int32_t* afccol;
  const double* afcval;
  const double* d;       // A(i,i) per owned F row
  const double* Q;       // [nnzW * nv] row-major per entry, zero padded
  DevState* st;
  int32_t pingpong;      // L2 ping-pong traversal order (see iterate.cu)
  int32_t fuse;          // 1: the last block of stage I / SpGEMM applies the scalar step;
                         // 2: it writes the rank-local sum to st->red[] (allreduce follows)
  double* dE_hist;       // per-step energy decrements (scalar step of the SpGEMM)
  // the y^ = Pi K y launch (MM_ITER) may be split into an interior and a
  // boundary launch (multi-GPU overlap, iterate.cu): units [ubeg, uend)
  // (windows / nodes / rows of the kernel path; uend < 0 = all) and the
  // launch's first slot in the partial-sum array
  int64_t ubeg, uend;
  int64_t ugap0, ugap1;  // ... minus the units [ugap0, ugap1) (the boundary launch skips the interior)
  int32_t poff;
};

// unit range of a (possibly split) y^ launch: idx in [0, unit_count) -> unit
__device__ __forceinline__ int64_t unit_count(const DevView& v, int64_t n) {
  return (v.uend < 0 ? n : v.uend) - v.ubeg - (v.ugap1 - v.ugap0);
}
__device__ __forceinline__ int64_t unit_of(const DevView& v, int64_t idx) {
  const int64_t w = v.ubeg + idx;
  return w >= v.ugap0 ? w + (v.ugap1 - v.ugap0) : w;
}

struct emin_ctx_s {
  emin_opts opts;
  cudaStream_t stream = nullptr;
  void* comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t n_global = 0, nc_global = 0, m_owned = 0;
  int64_t nF = 0, nFh = 0, nnzW = 0, nnzWh = 0, nnzAFF = 0, nnzAFC = 0, nnzP = 0;
  int32_t nv = 1;
  int32_t max_row = 0;
  int32_t group = 1;           // lanes per row in the streaming stages
  int32_t kernel_path = 0;
  int32_t pingpong = 0;        // alternate traversal directions (L2 ping-pong, iterate.cu)
  int32_t fuse = 0;            // scalar steps fused into the producing kernels (EMIN_DBG_FUSE_SCALARS)
  int32_t iter_kernels = 5;    // our kernel launches per CG iteration (set at graph capture)
  // y^ launch split (multi-GPU): the view of the launch being enqueued
  int64_t mm_ubeg = 0, mm_uend = -1, mm_ugap0 = 0, mm_ugap1 = 0;
  int32_t mm_poff = 0;
  // interior units [split_u0, split_u1) of the y^ launch: no halo row among
  // their A_FF neighbours (computed by emin_dist_split; split_on = 0: none)
  int32_t split_on = 0;
  int64_t split_u0 = 0, split_u1 = 0, split_n = 0;
  cudaStream_t comm_stream = nullptr;       // halo exchange overlapped with the interior launch
  cudaEvent_t ev_y = nullptr, ev_halo = nullptr;
  // device arrays (owned by ctx)
  int64_t *wptr = nullptr, *affptr = nullptr, *afcptr = nullptr, *pofs = nullptr, *cofs = nullptr;
  uint8_t* isc_own = nullptr;  // is_coarse of the owned rows
  cudaStream_t cap_stream = nullptr;  // capture stream for the CUDA graphs
  int64_t k_launched = 0;      // upper bound of k_total (host side)
  int64_t launches = 0;        // kernels enqueued by this context
  void* fast = nullptr;        // specialised-path plan (kernels_fast.cuh)
  void* nodal = nullptr;       // nodal 3x3 path plan (kernels_nodal.cuh)
  int32_t* erow = nullptr;     // F-row id of every W entry (streaming stages)
  int32_t* adiag = nullptr;    // position of A(i,i) in A_FF row i (setup: the record plan)
  double* dinv = nullptr;      // 1 / A(i,i) per owned F row
  // symmetric Jacobi scaling (scalar path, one GPU, Jacobi without the
  // post-projection): the CG runs on r~ = S r, y~ = S^-1 y, dW~ = S^-1 dW with
  // S = D^-1/2 and the records D^-1/2 A_FF D^-1/2, so z~ = r~
  int32_t sym = 0;
  double* srow = nullptr;      // S = 1 / sqrt(A(i,i)) per owned (+ halo) F row (sym)
  double* affvalS = nullptr;   // S A_FF S in A_FF's layout (sym on the nodal path)
  double* wtmp = nullptr;      // W = W0 + dW scratch of the energy pass (with the halo tail)
  DistPlan* dist = nullptr;    // multi-GPU halo plan (dist.cu), null on one GPU
  SgsPlan* sgs = nullptr;      // SGS preconditioner plan (sgs.cu), null for Jacobi
  int breakdown_reported = 0;
  int32_t *wcol = nullptr, *affcol = nullptr, *afccol = nullptr;
  double *affval = nullptr, *afcval = nullptr, *d = nullptr, *Q = nullptr;
  double *w0 = nullptr, *dw = nullptr, *r = nullptr, *r0 = nullptr, *y = nullptr, *yb = nullptr;
  double *partials = nullptr;  // per-block reduction partials
  int32_t n_partials = 0;
  double *dE_hist = nullptr;
  int64_t dE_cap = 0;
  DevState* st = nullptr;
  int64_t n_crows = 0;         // (tr(A_CC) and the Alg. 2 counters live in DevState)
  // launch geometry
  int grid_rows = 0, grid_spgemm = 0, grid_red = 0;
  // graphs: one per k (cached)
  cudaGraphExec_t graph = nullptr;
  int graph_k = -1;
  int graph_prof = 0;
  // profiling
  cudaGraphExec_t graph_prof_exec = nullptr;   // iteration graph with 6 event-record nodes
  cudaGraph_t graph_prof_src = nullptr;        // its source graph (owns the node handles)
  cudaGraphNode_t prof_node[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t prof_pending = 0;                    // iterations recorded, not yet folded
  int profiling = 0;
  std::vector<cudaEvent_t> ev;
  double prof_ms[4] = {0, 0, 0, 0};
  int64_t prof_launches[4] = {0, 0, 0, 0};
  std::string last_error;
  DevView view() const {
    DevView v;
    v.nF = nF; v.nFh = nFh; v.nnzW = nnzW; v.nv = nv;
    v.wptr = wptr; v.wcol = wcol; v.affptr = affptr; v.affcol = affcol; v.affval = affval;
    v.afcptr = afcptr; v.afccol = afccol; v.afcval = afcval; v.d = d; v.Q = Q; v.st = st;
    v.pingpong = pingpong;
    v.fuse = fuse;
    v.dE_hist = dE_hist;
    v.ubeg = mm_ubeg;
    v.uend = mm_uend;
    v.ugap0 = mm_ugap0;
    v.ugap1 = mm_ugap1;
    v.poff = mm_poff;
    return v;
  }
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum over aligned groups of G lanes (butterfly; identical result in every
// lane of the group; fixed order => deterministic).
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of one double (fixed tree); result valid in
// thread 0.  blockDim.x must be a multiple of 32 and <= 1024.
__device__ __forceinline__ double block_sum(double v, double* sh /* >= 32 */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double t = 0.0;
  if (w == 0) {
    t = (l < nw) ? sh[l] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// ---- the CG scalar steps (Alg. 3), applied by one thread
// gamma = r.z; stop if gamma <= 0; beta = gamma / gamma_old
__device__ __forceinline__ void scalar_gamma_apply(DevState* st, double g) {
  st->pendw = st->pend == 1;           // pend 2: a flush already applied dw += alpha y
  st->pend = 0;
  if (!(g > 0.0)) { st->stopped = 1; return; }
  st->beta = (st->k_total == 0) ? 0.0 : g / st->gamma_old;
  st->gamma = g;
  st->gamma_old = g;
}
// alpha = gamma / y.yb; dE = gamma alpha; stop tests (A4, A18)
__device__ __forceinline__ void scalar_alpha_apply(DevState* st, double den, double* dE_hist) {
  st->den = den;
  if (den < 0.0) { st->stopped = 5; return; }
  if (den == 0.0) { st->stopped = 2; return; }
  const double alpha = st->gamma / den;
  const double dE = st->gamma * alpha;
  const int64_t k = st->k_total + 1;
  if (k == 1) st->dE1 = dE;
  if (st->tau > 0.0 && k > 1 && dE < st->tau * st->dE1) { st->stopped = 3; return; }
  if (dE <= st->stag * st->E0) { st->stopped = 4; return; }
  st->alpha_pend = alpha;
  st->pend = 1;
  dE_hist[st->k_total] = dE;
  st->k_total = k;
  st->k_call += 1;
}

// Epilogue of a kernel producing per-block partial sums.  which = 0 (stage
// I: gamma) or 1 (SpGEMM: y.yb) with v.fuse set: the last block to finish
// (threadfence + counter, as in the CUDA threadFenceReduction sample) sums
// all partials in a fixed order and applies the scalar step, replacing the
// separate single-block scalar kernel.  All other blocks have already read
// the DevState fields the step writes (they read them at kernel start).
// which < 0 or !v.fuse: plain partial write (consumer kernel reduces).
__device__ __forceinline__ void block_partial_out(const DevView& v, double* partials, double tot, double* sh,
                                                  int which) {
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    partials[v.poff + blockIdx.x] = tot;
    int last = 0;
    if (which >= 0 && v.fuse) {
      __threadfence();
      last = atomicAdd(&v.st->ctr[which], 1u) == gridDim.x - 1;
    }
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // (a split launch: the earlier launches' partials [0, poff) precede in
  // stream order and are complete)
  double sum = 0.0;
  for (int k = threadIdx.x; k < v.poff + (int)gridDim.x; k += blockDim.x) sum += __ldcg(partials + k);
  sum = block_sum(sum, sh);
  if (threadIdx.x == 0) {
    if (v.fuse == 2) v.st->red[which] = sum;       // rank-local sum (multi-GPU: allreduce, scalar kernel)
    else if (which == 0) scalar_gamma_apply(v.st, sum);
    else {
      v.st->pendw = 0;
      if (!v.st->stopped) scalar_alpha_apply(v.st, sum, v.dE_hist);
    }
    v.st->ctr[which] = 0;
  }
}
// a fused SpGEMM that returns early on a stopped state still retires the
// pending dw update flag (what the separate alpha kernel did)
__device__ __forceinline__ void iter_stopped(const DevView& v) {
  if (v.fuse == 1 && blockIdx.x == 0 && threadIdx.x == 0) v.st->pendw = 0;
}

// lower_bound of key in sorted a[0..n)
__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ a, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// -------------------------------------------------------------- host side
#define EMIN_CUDA_TRY(ctx, call)                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      if (ctx) (ctx)->last_error = std::string(#call) + ": " + cudaGetErrorString(e_); \
      return (e_ == cudaErrorMemoryAllocation) ? EMIN_ERR_OOM : EMIN_ERR_CUDA;     \
    }                                                                              \
  } while (0)

// exclusive scan of int64 counts (in may alias out); returns total via *total_dev
// (device pointer, may be null).  Implemented in util.cu.
cudaError_t emin_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total_dev,
                          int64_t* scratch, cudaStream_t s);
int64_t emin_scan_scratch_elems(int64_t n);

int emin_num_sms();

// stream-ordered allocation from the library's own pool (util.cu); freed with
// cudaFreeAsync
cudaError_t emin_mallocAsync(void** p, size_t bytes, cudaStream_t s);
template <typename T>
inline cudaError_t emin_mallocAsync(T** p, size_t bytes, cudaStream_t s) {
  return emin_mallocAsync(reinterpret_cast<void**>(p), bytes, s);
}
void emin_pool_trim(cudaStream_t s);   // synchronises s, returns the pool's free blocks

// Alg. 1 tentative start (maxvol.cu)
void emin_maxvol_start(emin_ctx c, const double* Bc, const double* B, const int64_t* frow, double* what,
                       unsigned long long* fails, cudaStream_t s);

// projected SGS preconditioner (sgs.cu)
emin_status emin_sgs_plan(emin_ctx c, const int64_t* key_own, const int64_t* frow, cudaStream_t s);
emin_status emin_sgs_enqueue(emin_ctx c, cudaStream_t s, int* grid);
void emin_sgs_stage2(emin_ctx c, cudaStream_t s);
void emin_sgs_free(emin_ctx c);
int64_t emin_sgs_levels(emin_ctx c);
const int4* emin_scalar_records(emin_ctx c);   // iterate.cu
const int32_t* emin_scalar_windows(emin_ctx c, int64_t* nwin);
bool emin_nodal_plan(emin_ctx c, const int2** blk, const int64_t** bptr, const uint8_t** pm8,
                     const int64_t** pmoff, int64_t* nFn, int32_t* max_nb);
