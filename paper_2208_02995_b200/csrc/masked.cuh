// masked.cuh -- the masked product K y = (A Y) restricted to the fixed
// pattern of P ("the product K p as a SpMM ... with a fixed,
// prescribed pattern on P"), fused with the row projection Pi_B
// and the reduction the next CG scalar needs.
//
// Generic path: one warp per F row i; lane t owns pattern positions
// t, t+32, ... of J_i (MAXC chunks, |J_i| <= 32*MAXC).  For every A_FF
// entry (i,k) the lane binary-searches its column j in J_k and accumulates
// A(i,k) Y(k,j).  Works for any pattern; the specialised scalar and nodal
// kernels (kernels_fast.cuh) replace it on the hot path when they apply.
#pragma once
#include <climits>
#include "emin_internal.cuh"

enum MaskedMode : int {
  MM_ITER = 0,    // out = Pi (A_FF Y)|pattern ; partial += X . out
  MM_R0 = 1,      // out = -Pi (A P)|pattern  incl. the C-identity term (reading A1)
  MM_ENERGY = 2,  // partial += W . (A_FF W + 2 A_FC)|pattern           (Eq. trInc)
  MM_R0E = 3      // MM_R0 and MM_ENERGY of W = X in one pass (setup: r0 and E0 share A P0)
};

// X (and X2 when SUMX: X + X2, used for W = W0 + dW) is read on the owned
// and halo rows; out is written on the owned rows.
template <int MODE, int MAXC, bool SUMX>
__global__ void __launch_bounds__(256)
k_masked_generic(DevView v, const double* __restrict__ X, const double* __restrict__ X2,
                 double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  if (MODE == MM_ITER && v.st->stopped) { iter_stopped(v); return; }   // uniform over the grid
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = v.nv;
  double part = 0.0;
  const int64_t icnt = unit_count(v, v.nF);
  for (int64_t i1 = gw; i1 < icnt; i1 += nw) {
    const int64_t i = unit_of(v, i1);
    const int64_t b = v.wptr[i];
    const int nj = (int)(v.wptr[i + 1] - b);
    int32_t jj[MAXC];
    double acc[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int t = lane + 32 * c;
      jj[c] = (t < nj) ? v.wcol[b + t] : INT_MAX;
      acc[c] = 0.0;
    }
    const int64_t qb = v.affptr[i], qe = v.affptr[i + 1];
    for (int64_t q = qb; q < qe; ++q) {
      const int32_t k = __ldg(v.affcol + q);
      const double a = __ldg(v.affval + q);
      const int64_t kb = __ldg(v.wptr + k);
      const int kn = (int)(__ldg(v.wptr + k + 1) - kb);
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        if (lane + 32 * c < nj) {
          const int s = lower_bound_i32(v.wcol + kb, kn, jj[c]);
          if (s < kn && __ldg(v.wcol + kb + s) == jj[c]) {
            const double xv = SUMX ? (X[kb + s] + X2[kb + s]) : X[kb + s];
            acc[c] = fma(a, xv, acc[c]);
          }
        }
      }
    }
    double fc[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) fc[c] = 0.0;
    if (MODE != MM_ITER) {
      const int64_t fb = v.afcptr[i];
      const int fn = (int)(v.afcptr[i + 1] - fb);
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        if (lane + 32 * c < nj) {
          const int s = lower_bound_i32(v.afccol + fb, fn, jj[c]);
          if (s < fn && __ldg(v.afccol + fb + s) == jj[c]) fc[c] = __ldg(v.afcval + fb + s);
        }
      }
    }
    if (MODE == MM_ENERGY || MODE == MM_R0E) {
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
        if (t < nj) {
          const double w = SUMX ? (X[b + t] + X2[b + t]) : X[b + t];
          part += w * (acc[c] + 2.0 * fc[c]);
        }
      }
      if (MODE == MM_ENERGY) continue;
    }
    double g[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) g[c] = (MODE == MM_R0 || MODE == MM_R0E) ? acc[c] + fc[c] : acc[c];
    // Pi_B on row i: g <- g - Q_i (Q_i^T g)   (all dots first, then subtract).
    // r0 is projected twice (Pi^2 = Pi): when the start is already optimal
    // (configs 1, 2) Pi G is pure round-off, and the second pass puts that
    // round-off in ker(B^T) to its own precision, so that skipping the
    // post-Jacobi projection (reading A7) stays exact for it too.
#pragma unroll
    for (int pass = 0; pass < ((MODE == MM_R0 || MODE == MM_R0E) ? 2 : 1); ++pass) {
      double dots[EMIN_NV_MAX];
#pragma unroll
      for (int m = 0; m < EMIN_NV_MAX; ++m) {
        dots[m] = 0.0;
        if (m < nv) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < MAXC; ++c) {
            const int t = lane + 32 * c;
            if (t < nj) s = fma(__ldg(v.Q + (b + t) * nv + m), g[c], s);
          }
          dots[m] = warp_sum(s);
        }
      }
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int t = lane + 32 * c;
        if (t < nj) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < EMIN_NV_MAX; ++m)
            if (m < nv) s = fma(__ldg(v.Q + (b + t) * nv + m), dots[m], s);
          g[c] = g[c] - s;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int t = lane + 32 * c;
      if (t < nj) {
        if (MODE == MM_ITER) {
          out[b + t] = g[c];
          part = fma(X[b + t], g[c], part);
        } else {
          out[b + t] = -g[c];
        }
      }
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, MODE == MM_ITER ? 1 : -1);
}
