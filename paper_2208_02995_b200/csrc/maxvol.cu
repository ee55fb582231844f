// maxvol.cu -- the tentative start of Alg. 1 (PTent_SetUp, P:487-544;
// SURVEY §8f NEXT-3) on the prescribed pattern, emin_opts.start =
// EMIN_START_MAXVOL: per F row i, with M = V_c(J_i,:) (|J_i| x nv),
//   select nv rows of M (= columns of V_c(J_i,:)^T) by max vol [Gor08],
//   solve the local system B^T w = v exactly on them (B = M(S,:)), zero
//   elsewhere ("Select the best columns ... using max vol ...
//   least-squares solution ... ||v - B w|| = 0").
// The pattern growth of Alg. 1 (distance l = 1, 2, ...) is the caller's
// (the pattern is an input of emin_setup); rows where no nonsingular
// selection exists keep W^ = 0 and are counted (reading A24).
//
// Reading A24 fixes the procedure (max vol is cited without details):
// partial-pivoting elimination for the first selection, then swap sweeps
// on C = M B^{-1} until max|C| <= 1 + 1e-8 (<= 100 sweeps); ties = the first
// candidate within a factor (1 - 1e-12) of the maximum.  The selection is a
// discrete decision, so the arithmetic that feeds it is done in the same
// order and without FMA contraction as the plain description (__dmul_rn,
// __dadd_rn, __ddiv_rn), and B^{-1} by the same Gauss-Jordan sweep.
//
// One warp per F row, lane t owns rows t, t + 32, ... of M (|J_i| <= 128).
#include <algorithm>

#include "emin_internal.cuh"

namespace {


// Gauss-Jordan inverse with partial pivoting of the N x N row-major B (one
// thread, fully unrolled: registers); false if singular
template <int N>
__device__ bool mv_gj_inverse_t(const double* __restrict__ Bm, double* __restrict__ inv) {
  double a[N][2 * N];
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < 2 * N; ++c) a[r][c] = c < N ? Bm[r * N + c] : (c - N == r ? 1.0 : 0.0);
#pragma unroll
  for (int c = 0; c < N; ++c) {
    int p = c;
#pragma unroll
    for (int r = c + 1; r < N; ++r)
      if (fabs(a[r][c]) > fabs(a[p][c])) p = r;
    // row swap c <-> p by selects (p is data dependent)
    double pivrow[2 * N];
#pragma unroll
    for (int k = 0; k < 2 * N; ++k) {
      double v = a[c][k];
#pragma unroll
      for (int r = c + 1; r < N; ++r) if (r == p) v = a[r][k];
      pivrow[k] = v;
    }
#pragma unroll
    for (int r = c + 1; r < N; ++r)
      if (r == p)
#pragma unroll
        for (int k = 0; k < 2 * N; ++k) a[r][k] = a[c][k];
#pragma unroll
    for (int k = 0; k < 2 * N; ++k) a[c][k] = pivrow[k];
    if (a[c][c] == 0.0) return false;
    const double piv = a[c][c];
#pragma unroll
    for (int k = 0; k < 2 * N; ++k) a[c][k] = __ddiv_rn(a[c][k], piv);
#pragma unroll
    for (int r = 0; r < N; ++r) {
      if (r == c) continue;
      const double f = a[r][c];
      if (f != 0.0)
#pragma unroll
        for (int k = 0; k < 2 * N; ++k) a[r][k] = __dsub_rn(a[r][k], __dmul_rn(f, a[c][k]));
    }
  }
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) inv[r * N + c] = a[r][N + c];
  return true;
}

__device__ bool mv_gj_inverse(int nv, const double* __restrict__ Bm, double* __restrict__ inv) {
  switch (nv) {
    case 1: return mv_gj_inverse_t<1>(Bm, inv);
    case 2: return mv_gj_inverse_t<2>(Bm, inv);
    case 3: return mv_gj_inverse_t<3>(Bm, inv);
    case 4: return mv_gj_inverse_t<4>(Bm, inv);
    case 5: return mv_gj_inverse_t<5>(Bm, inv);
    case 6: return mv_gj_inverse_t<6>(Bm, inv);
    case 7: return mv_gj_inverse_t<7>(Bm, inv);
    default: return mv_gj_inverse_t<8>(Bm, inv);
  }
}

__device__ __forceinline__ double mv_warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ int mv_warp_min(int x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

template <int MAXC>
__global__ void __launch_bounds__(128)
k_maxvol_start(DevView v, int rstep, const double* __restrict__ Bc, const double* __restrict__ B,
               const int64_t* __restrict__ frow, double* __restrict__ what, unsigned long long* fails) {
  __shared__ double s_B[4][EMIN_NV_MAX * EMIN_NV_MAX];
  __shared__ double s_inv[4][EMIN_NV_MAX * EMIN_NV_MAX];
  __shared__ int s_ok[4];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = v.nv;
  // rows i, i + 1, .., i + rstep - 1 share J (nodal path: the 3 dof rows of
  // an F node), hence M and the selection; each solves with its own v
  for (int64_t i = gw * rstep; i < v.nF; i += nw * rstep) {
    const int64_t b = v.wptr[i];
    const int m = (int)(v.wptr[i + 1] - b);
    double M[MAXC][EMIN_NV_MAX], W[MAXC][EMIN_NV_MAX];
    bool used[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int t = lane + 32 * c;
      used[c] = false;
#pragma unroll
      for (int k = 0; k < EMIN_NV_MAX; ++k) {
        M[c][k] = (t < m && k < nv) ? Bc[(int64_t)v.wcol[b + t] * nv + k] : 0.0;
        W[c][k] = M[c][k];
      }
    }
    int S[EMIN_NV_MAX];
    bool ok = m >= nv;
    // ---- first selection: elimination with partial pivoting
    for (int j = 0; j < nv && ok; ++j) {
      double vmax = -1.0;
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
        double val = -1.0;
#pragma unroll
        for (int k = 0; k < EMIN_NV_MAX; ++k)
          if (k == j) val = (t < m && !used[c]) ? fabs(W[c][k]) : -1.0;
        vmax = fmax(vmax, val);
      }
      const double mx = mv_warp_max(vmax);
      if (!(mx > 0.0)) { ok = false; break; }
      int cand = 1 << 30;
#pragma unroll
      for (int c = MAXC - 1; c >= 0; --c) {
        const int t = lane + 32 * c;
        double val = -1.0;
#pragma unroll
        for (int k = 0; k < EMIN_NV_MAX; ++k)
          if (k == j) val = (t < m && !used[c]) ? fabs(W[c][k]) : -1.0;
        if (val >= 0.0 && val >= (1.0 - 1e-12) * mx) cand = t;
      }
      const int p = mv_warp_min(cand);
      S[j] = p;
      // the pivot row (columns j .. nv-1)
      double prow[EMIN_NV_MAX];
#pragma unroll
      for (int k = 0; k < EMIN_NV_MAX; ++k) {
        double mine = 0.0;
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
          if (c == p / 32) mine = W[c][k];
        prow[k] = __shfl_sync(0xffffffffu, mine, p & 31);
      }
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
        if (t == p) used[c] = true;
        if (t < m && !used[c]) {
          double wj = 0.0, pj = 0.0;
#pragma unroll
          for (int k = 0; k < EMIN_NV_MAX; ++k)
            if (k == j) { wj = W[c][k]; pj = prow[k]; }
          const double f = __ddiv_rn(wj, pj);
#pragma unroll
          for (int k = 0; k < EMIN_NV_MAX; ++k)
            if (k >= j && k < nv) W[c][k] = __dsub_rn(W[c][k], __dmul_rn(f, prow[k]));
        }
      }
    }
    // ---- max-vol swap sweeps on C = M B^{-1}
    auto load_inverse = [&]() -> bool {
      // the owners of the selected rows write B = M(S,:) to shared memory
      __syncwarp();
      for (int a = 0; a < nv; ++a) {
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
          if (lane + 32 * c == S[a])
#pragma unroll
            for (int k = 0; k < EMIN_NV_MAX; ++k)
              if (k < nv) s_B[wib][a * nv + k] = M[c][k];
      }
      __syncwarp();
      if (lane == 0) s_ok[wib] = mv_gj_inverse(nv, s_B[wib], s_inv[wib]) ? 1 : 0;
      __syncwarp();
      return s_ok[wib] != 0;
    };
    for (int sweep = 0; sweep < 100 && ok; ++sweep) {
      if (!load_inverse()) { ok = false; break; }
      double cabs[MAXC][EMIN_NV_MAX];
      double lmax = 0.0;
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
#pragma unroll
        for (int cc = 0; cc < EMIN_NV_MAX; ++cc) {
          double sum = 0.0;
          if (t < m && cc < nv)
            for (int bb = 0; bb < nv; ++bb) {
              double mb = 0.0;
#pragma unroll
              for (int k = 0; k < EMIN_NV_MAX; ++k)
                if (k == bb) mb = M[c][k];
              sum = __dadd_rn(sum, __dmul_rn(mb, s_inv[wib][bb * nv + cc]));
            }
          cabs[c][cc] = (t < m && cc < nv) ? fabs(sum) : -1.0;
          lmax = fmax(lmax, cabs[c][cc]);
        }
      }
      const double mx = mv_warp_max(lmax);
      if (mx <= 1.0 + 1e-8) break;
      // first (row-major) entry within the tie band
      int ct = 1 << 30, cc_sel = 0;
#pragma unroll
      for (int c = MAXC - 1; c >= 0; --c) {
        const int t = lane + 32 * c;
        int first = -1;
#pragma unroll
        for (int cc = EMIN_NV_MAX - 1; cc >= 0; --cc)
          if (cabs[c][cc] >= 0.0 && cabs[c][cc] >= (1.0 - 1e-12) * mx) first = cc;
        if (first >= 0) { ct = t; cc_sel = first; }
      }
      const int tsel = mv_warp_min(ct);
      const int csel = __shfl_sync(0xffffffffu, cc_sel, tsel & 31);
      for (int a = 0; a < nv; ++a)
        if (a == csel) S[a] = tsel;
    }
    // ---- w(S) = B^{-T} v, zero elsewhere
    if (ok && !load_inverse()) ok = false;
    for (int d = 0; d < rstep; ++d) {
      const double* vrow = B + frow[i + d] * nv;
      const int64_t bd = v.wptr[i + d];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
        if (t >= m) continue;
        double w = 0.0;
        if (ok)
          for (int a = 0; a < nv; ++a)
            if (S[a] == t) {
              double sum = 0.0;
              for (int bb = 0; bb < nv; ++bb) sum = __dadd_rn(sum, __dmul_rn(s_inv[wib][bb * nv + a], vrow[bb]));
              w = sum;
            }
        what[bd + t] = w;
      }
    }
    if (!ok && lane == 0) atomicAdd(fails, (unsigned long long)rstep);
    __syncwarp();
  }
}

}  // namespace

// overwrite the start W^ (W layout) with the max-vol tentative start
void emin_maxvol_start(emin_ctx c, const double* Bc, const double* B, const int64_t* frow, double* what,
                       unsigned long long* fails, cudaStream_t s) {
  const int SM = emin_num_sms();
  const int rstep = c->kernel_path == 2 ? 3 : 1;   // nodal path: one selection per F node
  const int64_t units = c->nF / rstep;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((units + 3) / 4, (int64_t)SM * 16));
  const DevView v = c->view();
  if (c->max_row <= 32) k_maxvol_start<1><<<g, 128, 0, s>>>(v, rstep, Bc, B, frow, what, fails);
  else if (c->max_row <= 64) k_maxvol_start<2><<<g, 128, 0, s>>>(v, rstep, Bc, B, frow, what, fails);
  else k_maxvol_start<4><<<g, 128, 0, s>>>(v, rstep, Bc, B, frow, what, fails);
  c->launches += 1;
}
