// iterate.cu -- Alg. 3 EMIN_PCG on the device: the two streaming
// stages, the masked SpGEMM step, the single-block scalar kernels, CUDA-graph
// capture of k iterations, and the remaining ABI calls.
//
// Per iteration (all scalars stay in device memory, no host sync):
//   stage I   r -= alpha_{k-1} yb (deferred update of step k-1);
//             z = D^-1 r [Pi]; partial gamma = r.z
//   scalar    gamma; stop if gamma <= 0; beta = gamma/gamma_old
//   stage II  dw += alpha_{k-1} y_{k-1} (deferred);
//             y = z + beta y (y = z at k = 1)
//   SpGEMM    yb = Pi K y = Pi (A Y)|pattern; partial y.yb
//   scalar    alpha = gamma / y.yb ; dE = gamma alpha ; stop tests   (A4, A18)
// The deferral moves no arithmetic: each element sees exactly the update
// Alg. 3 applies, one kernel later; a stopped step leaves nothing pending.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "emin_internal.cuh"
#include "masked.cuh"
#include "kernels_fast.cuh"
#include "dist.cuh"
#include "kernels_nodal.cuh"
#include <utility>

namespace {

// ------------------------------------------------------------ stage I
template <int G, bool PROJ>
__global__ void __launch_bounds__(256)
k_stage1(DevView v, double* __restrict__ r, const double* __restrict__ yb, double* __restrict__ partials) {
  __shared__ double sh[32];
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = st->pend;
  const double ap = st->alpha_pend;
  const int lg = threadIdx.x & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  const int nv = v.nv;
  double part = 0.0;
  // warp-uniform trip count: the PROJ path shuffles inside the loop
  for (int64_t i = gid; __any_sync(0xffffffffu, i < v.nF); i += ng) {
    const bool act = i < v.nF;
    const int64_t b = act ? v.wptr[i] : 0, e = act ? v.wptr[i + 1] : 0;
    const double di = act ? v.d[i] : 1.0;
    if (!PROJ) {
      for (int64_t p = b + lg; p < e; p += G) {
        double rv = r[p];
        if (pend) { rv = rv - ap * yb[p]; r[p] = rv; }
        const double z = rv / di;
        part = fma(rv, z, part);
      }
    } else {
      double dots[EMIN_NV_MAX];
#pragma unroll
      for (int m = 0; m < EMIN_NV_MAX; ++m) dots[m] = 0.0;
      for (int64_t p = b + lg; p < e; p += G) {
        double rv = r[p];
        if (pend) { rv = rv - ap * yb[p]; r[p] = rv; }
        const double z = rv / di;
#pragma unroll
        for (int m = 0; m < EMIN_NV_MAX; ++m) if (m < nv) dots[m] = fma(v.Q[p * nv + m], z, dots[m]);
      }
#pragma unroll
      for (int m = 0; m < EMIN_NV_MAX; ++m) if (m < nv) dots[m] = group_sum<G>(dots[m]);
      for (int64_t p = b + lg; p < e; p += G) {
        const double rv = r[p];
        double z = rv / di, s = 0.0;
#pragma unroll
        for (int m = 0; m < EMIN_NV_MAX; ++m) if (m < nv) s = fma(v.Q[p * nv + m], dots[m], s);
        z -= s;
        part = fma(rv, z, part);
      }
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 0);
}

// ------------------------------------------------------------ stage II
template <int G, bool PROJ>
__global__ void __launch_bounds__(256)
k_stage2(DevView v, const double* __restrict__ r, double* __restrict__ y, double* __restrict__ dw) {
  const DevState* st = v.st;
  const int stopped = st->stopped;
  const int pendw = st->pendw;
  if (stopped && !pendw) return;
  const double ap = st->alpha_pend;
  const double beta = st->beta;
  const bool first = (st->k_total == 0);
  const int lg = threadIdx.x & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  const int nv = v.nv;
  // warp-uniform trip count: the PROJ path shuffles inside the loop
  for (int64_t i = gid; __any_sync(0xffffffffu, i < v.nF); i += ng) {
    const bool act = i < v.nF;
    const int64_t b = act ? v.wptr[i] : 0, e = act ? v.wptr[i + 1] : 0;
    const double di = act ? v.d[i] : 1.0;
    double dots[EMIN_NV_MAX];
#pragma unroll
    for (int m = 0; m < EMIN_NV_MAX; ++m) dots[m] = 0.0;
    if (PROJ && !stopped) {
      for (int64_t p = b + lg; p < e; p += G) {
        const double z = r[p] / di;
#pragma unroll
        for (int m = 0; m < EMIN_NV_MAX; ++m) if (m < nv) dots[m] = fma(v.Q[p * nv + m], z, dots[m]);
      }
#pragma unroll
      for (int m = 0; m < EMIN_NV_MAX; ++m) if (m < nv) dots[m] = group_sum<G>(dots[m]);
    }
    for (int64_t p = b + lg; p < e; p += G) {
      const double yo = y[p];
      if (pendw) dw[p] = dw[p] + ap * yo;
      if (!stopped) {
        double z = r[p] / di;
        if (PROJ) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < EMIN_NV_MAX; ++m) if (m < nv) s = fma(v.Q[p * nv + m], dots[m], s);
          z -= s;
        }
        y[p] = first ? z : z + beta * yo;
      }
    }
  }
}

// ------------------------------------------------------------ entry-parallel stages
// (no post-Jacobi projection): one thread per pair of W entries, row from erow[].

// z = r / d (Jacobi) from a precomputed 1/d: q0 = r (1/d) and one
// FMA residual correction, which reproduces the IEEE quotient (Markstein)
// without the register-heavy DDIV sequence.
__device__ __forceinline__ double jacobi_div(double r, double d, double dinv) {
  const double q0 = r * dinv;
  const double res = fma(-q0, d, r);
  return fma(res, dinv, q0);
}

// Each thread moves pairs of entries with 16-byte loads and stores (double2 /
// int2); the odd tail entry is handled by thread 0.
__global__ void __launch_bounds__(256, 4)
k_stage1_v(DevView v, const int32_t* __restrict__ erow, const double* __restrict__ dinv, double* __restrict__ r,
           const double* __restrict__ yb, double* __restrict__ partials) {
  __shared__ double sh[32];
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = st->pend;
  const double ap = st->alpha_pend;
  const int64_t np = v.nnzW >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double2* r2 = reinterpret_cast<const double2*>(r);
  const double2* yb2 = reinterpret_cast<const double2*>(yb);
  const int2* er2 = reinterpret_cast<const int2*>(erow);
  double part = 0.0;
  // L2 ping-pong: odd steps sweep backwards, so the first pairs read are
  // the last ones the previous kernel wrote (still in the 126 MB L2)
  const bool rev = v.pingpong && (st->k_total & 1);
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < np; p0 += 2 * stride) {
    double2 rv[2];
    double dv[4], iv[4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t p = p0 + u * stride;
      if (p < np) {
        const int64_t pp = rev ? np - 1 - p : p;
        rv[u] = r2[pp];
        if (pend) {
          const double2 b = yb2[pp];
          rv[u].x = rv[u].x - ap * b.x;
          rv[u].y = rv[u].y - ap * b.y;
        }
        const int2 i = er2[pp];
        dv[2 * u] = v.d[i.x]; iv[2 * u] = dinv[i.x];
        dv[2 * u + 1] = v.d[i.y]; iv[2 * u + 1] = dinv[i.y];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t p = p0 + u * stride;
      if (p < np) {
        if (pend) reinterpret_cast<double2*>(r)[rev ? np - 1 - p : p] = rv[u];
        part = fma(rv[u].x, jacobi_div(rv[u].x, dv[2 * u], iv[2 * u]), part);
        part = fma(rv[u].y, jacobi_div(rv[u].y, dv[2 * u + 1], iv[2 * u + 1]), part);
      }
    }
  }
  if ((v.nnzW & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t e = v.nnzW - 1;
    double x = r[e];
    if (pend) { x = x - ap * yb[e]; r[e] = x; }
    part = fma(x, jacobi_div(x, v.d[erow[e]], dinv[erow[e]]), part);
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 0);
}

__global__ void __launch_bounds__(256, 4)
k_stage2_v(DevView v, const int32_t* __restrict__ erow, const double* __restrict__ dinv,
           const double* __restrict__ r, double* __restrict__ y, double* __restrict__ dw) {
  const DevState* st = v.st;
  const int stopped = st->stopped;
  const int pendw = st->pendw;
  if (stopped && !pendw) return;
  const double ap = st->alpha_pend;
  const double beta = st->beta;
  const bool first = (st->k_total == 0);
  const int64_t np = v.nnzW >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double2* y2 = reinterpret_cast<double2*>(y);
  double2* dw2 = reinterpret_cast<double2*>(dw);
  const double2* r2 = reinterpret_cast<const double2*>(r);
  const int2* er2 = reinterpret_cast<const int2*>(erow);
  const bool rev = v.pingpong && !(st->k_total & 1);   // opposite to stage I (L2 ping-pong)
  for (int64_t p1 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p1 < np; p1 += stride) {
    const int64_t p = rev ? np - 1 - p1 : p1;
    const double2 yo = y2[p];
    if (pendw) {
      double2 d = dw2[p];
      d.x = d.x + ap * yo.x;
      d.y = d.y + ap * yo.y;
      dw2[p] = d;
    }
    if (!stopped) {
      const double2 rv = r2[p];
      const int2 i = er2[p];
      const double z0 = jacobi_div(rv.x, v.d[i.x], dinv[i.x]);
      const double z1 = jacobi_div(rv.y, v.d[i.y], dinv[i.y]);
      double2 yn;
      yn.x = first ? z0 : z0 + beta * yo.x;
      yn.y = first ? z1 : z1 + beta * yo.y;
      y2[p] = yn;
    }
  }
  if ((v.nnzW & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t e = v.nnzW - 1;
    const double yo = y[e];
    if (pendw) dw[e] = dw[e] + ap * yo;
    if (!stopped) {
      const double z = jacobi_div(r[e], v.d[erow[e]], dinv[erow[e]]);
      y[e] = first ? z : z + beta * yo;
    }
  }
}

// ---- the same two stages under the symmetric Jacobi scaling (ctx sym):
// z~ = S D^-1 r = S r = r~, so gamma = r~.r~ and y~ = r~ + beta y~ are plain
// streams with no row ids and no division (24 and 40 bytes per W entry).
__global__ void __launch_bounds__(256, 4)
k_stage1_s(DevView v, double* __restrict__ r, const double* __restrict__ yb, double* __restrict__ partials) {
  __shared__ double sh[32];
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = st->pend;
  const double ap = st->alpha_pend;
  const int64_t np = v.nnzW >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* yb2 = reinterpret_cast<const double2*>(yb);
  double part = 0.0;
  const bool rev = v.pingpong && (st->k_total & 1);   // L2 ping-pong (see k_stage1_v)
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < np; p0 += 2 * stride) {
    double2 rv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t p = p0 + u * stride;
      if (p < np) {
        const int64_t pp = rev ? np - 1 - p : p;
        rv[u] = r2[pp];
        if (pend) {
          const double2 b = yb2[pp];
          rv[u].x = rv[u].x - ap * b.x;
          rv[u].y = rv[u].y - ap * b.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t p = p0 + u * stride;
      if (p < np) {
        if (pend) r2[rev ? np - 1 - p : p] = rv[u];
        part = fma(rv[u].x, rv[u].x, part);
        part = fma(rv[u].y, rv[u].y, part);
      }
    }
  }
  if ((v.nnzW & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t e = v.nnzW - 1;
    double x = r[e];
    if (pend) { x = x - ap * yb[e]; r[e] = x; }
    part = fma(x, x, part);
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 0);
}

__global__ void __launch_bounds__(256, 4)
k_stage2_s(DevView v, const double* __restrict__ r, double* __restrict__ y, double* __restrict__ dw) {
  const DevState* st = v.st;
  const int stopped = st->stopped;
  const int pendw = st->pendw;
  if (stopped && !pendw) return;
  const double ap = st->alpha_pend;
  const double beta = st->beta;
  const bool first = (st->k_total == 0);
  const int64_t np = v.nnzW >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double2* y2 = reinterpret_cast<double2*>(y);
  double2* dw2 = reinterpret_cast<double2*>(dw);
  const double2* r2 = reinterpret_cast<const double2*>(r);
  const bool rev = v.pingpong && !(st->k_total & 1);   // opposite to stage I (L2 ping-pong)
  for (int64_t p1 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p1 < np; p1 += stride) {
    const int64_t p = rev ? np - 1 - p1 : p1;
    const double2 yo = y2[p];
    if (pendw) {
      double2 d = dw2[p];
      d.x = d.x + ap * yo.x;
      d.y = d.y + ap * yo.y;
      dw2[p] = d;
    }
    if (!stopped) {
      const double2 rv = r2[p];
      double2 yn;
      yn.x = first ? rv.x : rv.x + beta * yo.x;
      yn.y = first ? rv.y : rv.y + beta * yo.y;
      y2[p] = yn;
    }
  }
  if ((v.nnzW & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t e = v.nnzW - 1;
    const double yo = y[e];
    if (pendw) dw[e] = dw[e] + ap * yo;
    if (!stopped) y[e] = first ? r[e] : r[e] + beta * yo;
  }
}

// x_e *= s(row(e)) (r~ = S r0 at setup / reset)
__global__ void k_scale_rows(double* __restrict__ x, const int32_t* __restrict__ erow,
                             const double* __restrict__ srow, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    x[e] = x[e] * srow[erow[e]];
}
// out = w0 + S dW~ (W under the symmetric scaling, for the energy pass)
__global__ void k_wsum_s(const double* __restrict__ w0, const double* __restrict__ dw, const int32_t* __restrict__ erow,
                         const double* __restrict__ srow, int64_t n, double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = w0[e] + srow[erow[e]] * dw[e];
}

__global__ void k_recip(const double* __restrict__ d, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = 1.0 / d[i];
}

__global__ void k_build_erow(const int64_t* __restrict__ wptr, int64_t nF, int32_t* __restrict__ erow) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nF; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = wptr[i]; p < wptr[i + 1]; ++p) erow[p] = (int32_t)i;
}

// ------------------------------------------------------------ scalars
__device__ double reduce_partials(const double* __restrict__ p, int np, double* sh) {
  if (np < 0) return p[0];   // already reduced over the ranks (DevState::red)
  // four independent accumulators (loads in flight), combined in a fixed order
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const int st = blockDim.x;
  int k = threadIdx.x;
  for (; k + 3 * st < np; k += 4 * st) {
    s0 += p[k];
    s1 += p[k + st];
    s2 += p[k + 2 * st];
    s3 += p[k + 3 * st];
  }
  for (; k < np; k += st) s0 += p[k];
  return block_sum((s0 + s1) + (s2 + s3), sh);
}

// The single-block scalar steps.  Thread 0 prefetches the CG state's lines
// into L1 while the block loads the partial sums, and the stopped test comes
// after the reduction: one global round trip instead of three (stopped flag,
// partials, state fields); the arithmetic and the summation order are
// unchanged.
__device__ __forceinline__ void prefetch_state(const DevState* st) {
  if (threadIdx.x == 0) {
    const char* p = reinterpret_cast<const char*>(st);
    for (int o = 0; o < (int)sizeof(DevState); o += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + o));
  }
}

__global__ void __launch_bounds__(1024) k_scalar_gamma(DevState* st, const double* __restrict__ partials, int np) {
  __shared__ double sh[32];
  prefetch_state(st);
  const double g = reduce_partials(partials, np, sh);
  if (threadIdx.x == 0 && !st->stopped) scalar_gamma_apply(st, g);
}

__global__ void __launch_bounds__(1024) k_scalar_alpha(DevState* st, const double* __restrict__ partials, int np,
                                                       double* __restrict__ dE_hist) {
  __shared__ double sh[32];
  prefetch_state(st);
  const double den = reduce_partials(partials, np, sh);
  if (threadIdx.x == 0) {
    st->pendw = 0;
    if (!st->stopped) scalar_alpha_apply(st, den, dE_hist);
  }
}

// apply a pending update (before reading W or r from outside the loop)
__global__ void k_wsum(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                       double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

// W = W0 + dW is read outside the loop (energy, P): apply a pending
// dw += alpha y; the pending r -= alpha y^ stays with stage I (pend 1 -> 2),
// so the flush moves 24 instead of 48 bytes per entry and a later
// emin_iterate takes the same values in the same order
__global__ void k_flush(DevView v, double* __restrict__ dw, const double* __restrict__ y) {
  const DevState* st = v.st;
  if (st->pend != 1) return;
  const double ap = st->alpha_pend;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < v.nnzW;
       p += (int64_t)gridDim.x * blockDim.x)
    dw[p] = dw[p] + ap * y[p];
}
__global__ void k_flush_done(DevState* st) { if (st->pend == 1) st->pend = 2; }

__global__ void k_reset_state(DevState* st, const double* __restrict__ Epart, int np, double tau, double stag) {
  __shared__ double sh[32];
  const double e = reduce_partials(Epart, np, sh);
  if (threadIdx.x == 0) {
    st->gamma = st->gamma_old = st->beta = st->alpha_pend = st->den = st->dE1 = 0.0;
    st->E0 = e + st->sum_cc;
    st->tau = tau;
    st->stag = stag;
    st->k_total = 0;
    st->stopped = 0;
    st->pend = st->pendw = 0;
    st->k_call = 0;
    st->ctr[0] = st->ctr[1] = 0;
  }
}

// (add: a device scalar added to the sum, or null)
__global__ void k_energy_out(const double* __restrict__ partials, int np, const double* add, double* out) {
  __shared__ double sh[32];
  const double e = reduce_partials(partials, np, sh);
  if (threadIdx.x == 0) *out = add ? e + *add : e;
}

__global__ void k_get_P(DevView v, const double* __restrict__ w0, const double* __restrict__ dw,
                        const int64_t* __restrict__ pofs, double* __restrict__ out, const double* __restrict__ srow) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < v.nF; i += nw) {
    const int64_t b = v.wptr[i];
    const int nj = (int)(v.wptr[i + 1] - b);
    const int64_t o = pofs[i];
    const double si = srow ? srow[i] : 1.0;          // dW = S dW~ under the symmetric scaling
    for (int t = lane; t < nj; t += 32) out[o + t] = w0[b + t] + (srow ? si * dw[b + t] : dw[b + t]);
  }
}
// S A_FF S in A_FF's layout, warp per owned F row, lanes over its entries
// (nodal path, sym)
__global__ void k_scale_aff(const int64_t* __restrict__ affptr, const int32_t* __restrict__ affcol,
                            const double* __restrict__ affval, const double* __restrict__ srow, int64_t nF,
                            double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < nF; i += nw) {
    const double si = srow[i];
    for (int64_t q = affptr[i] + lane; q < affptr[i + 1]; q += 32) out[q] = (affval[q] * si) * srow[affcol[q]];
  }
}
__global__ void k_get_P_crows(int64_t m, const uint8_t* __restrict__ isc, const int64_t* __restrict__ prp,
                              double* __restrict__ out) {
  for (int64_t rl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rl < m; rl += (int64_t)gridDim.x * blockDim.x)
    if (isc[rl]) out[prp[rl] - prp[0]] = 1.0;
}

// ------------------------------------------------------------ interior / boundary split (multi-GPU)
// a row is a boundary row if one of its A_FF neighbours is a halo row (local
// id >= nF); lohi[0] = 1 + the last boundary row of the lower half, lohi[1] =
// the first boundary row of the upper half (z-slab partitions: the halo
// planes sit at both ends of the owned rows)
__global__ void k_boundary_bounds(const int64_t* __restrict__ affptr, const int32_t* __restrict__ affcol, int64_t nF,
                                  unsigned long long* lohi) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nF; i += (int64_t)gridDim.x * blockDim.x) {
    bool bnd = false;
    for (int64_t q = affptr[i]; q < affptr[i + 1]; ++q) bnd |= affcol[q] >= nF;
    if (bnd) {
      if (i < nF / 2) atomicMax(&lohi[0], (unsigned long long)(i + 1));
      else atomicMin(&lohi[1], (unsigned long long)i);
    }
  }
}
__global__ void k_boundary_count(const int64_t* __restrict__ affptr, const int32_t* __restrict__ affcol, int64_t nF,
                                 const unsigned long long* __restrict__ lohi, unsigned long long* cnt) {
  const int64_t ib = (int64_t)lohi[0], ie = (int64_t)lohi[1];
  for (int64_t i = ib + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ie; i += (int64_t)gridDim.x * blockDim.x) {
    bool bnd = false;
    for (int64_t q = affptr[i]; q < affptr[i + 1]; ++q) bnd |= affcol[q] >= nF;
    if (bnd) atomicAdd(cnt, 1ull);
  }
}
// scalar path: the windows whose rows all lie in [ib, ie)
__global__ void k_window_range(const int32_t* __restrict__ rowstart, int64_t nwin, const unsigned long long* lohi,
                               unsigned long long* out) {
  const int64_t ib = (int64_t)lohi[0], ie = (int64_t)lohi[1];
  int64_t lo = 0, hi = nwin;                 // first w with rowstart[w] >= ib
  while (lo < hi) { const int64_t m = (lo + hi) / 2; if (rowstart[m] < ib) lo = m + 1; else hi = m; }
  const int64_t w0 = lo;
  lo = 0; hi = nwin;                         // windows w with rowstart[w + 1] <= ie
  while (lo < hi) { const int64_t m = (lo + hi) / 2; if (rowstart[m + 1] <= ie) lo = m + 1; else hi = m; }
  out[0] = (unsigned long long)w0;
  out[1] = (unsigned long long)lo;
}

int pick_group(double avg) {
  int best = 1;
  double best_eff = 0.0;
  for (int G = 1; G <= 32; G <<= 1) {
    const double eff = avg / (std::ceil(avg / G) * G);
    if (eff >= best_eff - 1e-12) { best = G; best_eff = eff; }
  }
  return best;
}

template <int G>
void launch_stage1_g(emin_ctx c, cudaStream_t s) {
  const DevView v = c->view();
  if (c->opts.project_after_jacobi)
    k_stage1<G, true><<<c->grid_rows, 256, 0, s>>>(v, c->r, c->yb, c->partials);
  else
    k_stage1<G, false><<<c->grid_rows, 256, 0, s>>>(v, c->r, c->yb, c->partials);
}
template <int G>
void launch_stage2_g(emin_ctx c, cudaStream_t s) {
  const DevView v = c->view();
  if (c->opts.project_after_jacobi)
    k_stage2<G, true><<<c->grid_rows, 256, 0, s>>>(v, c->r, c->y, c->dw);
  else
    k_stage2<G, false><<<c->grid_rows, 256, 0, s>>>(v, c->r, c->y, c->dw);
}
void launch_stage(emin_ctx c, int which, cudaStream_t s) {
  if (c->sym) {
    if (which == 1)
      k_stage1_s<<<c->grid_rows, 256, 0, s>>>(c->view(), c->r, c->yb, c->partials);
    else
      k_stage2_s<<<c->grid_rows, 256, 0, s>>>(c->view(), c->r, c->y, c->dw);
    return;
  }
  if (!c->opts.project_after_jacobi) {
    if (which == 1)
      k_stage1_v<<<c->grid_rows, 256, 0, s>>>(c->view(), c->erow, c->dinv, c->r, c->yb, c->partials);
    else
      k_stage2_v<<<c->grid_rows, 256, 0, s>>>(c->view(), c->erow, c->dinv, c->r, c->y, c->dw);
    return;
  }
  switch (c->group) {
#define CASE_G(GG) case GG: which == 1 ? launch_stage1_g<GG>(c, s) : launch_stage2_g<GG>(c, s); break;
    CASE_G(1) CASE_G(2) CASE_G(4) CASE_G(8) CASE_G(16) CASE_G(32)
#undef CASE_G
  }
}

}  // namespace

// ============================================================ internal API
// mode: MM_ITER (X = y), MM_R0 (X = w0), MM_ENERGY (X = w0, X2 = dw)
int emin_launch_masked(emin_ctx c, int mode, const double* X, const double* X2, double* out,
                       cudaStream_t s) {
  // returns the grid (= number of partial sums), or -1 if the kernel path
  // has no MM_R0E (fused r0 + E0) kernel -- the caller then runs MM_R0 and
  // MM_ENERGY separately
  const DevView v = c->view();
  const int grid = c->grid_spgemm;
  if (c->kernel_path == 1) {
    if (!launch_scalar_masked(c, mode, X, X2, out, s)) return -1;
    return mode == MM_ITER ? scalar_iter_launch_grid(c) : grid;
  }
  if (c->kernel_path == 2) {
    const NodalPlan* np = static_cast<const NodalPlan*>(c->nodal);
    if (!launch_nodal(c, np, mode, X, X2, out, s)) return -1;
    return nodal_grid(c, np);
  }
  const int mc = c->max_row <= 32 ? 1 : c->max_row <= 64 ? 2 : 4;
#define LAUNCH_M(MODE, MC, SUMX) \
  k_masked_generic<MODE, MC, SUMX><<<grid, 256, 0, s>>>(v, X, X2, out, c->partials)
  if (mode == MM_ITER) {
    if (mc == 1) LAUNCH_M(MM_ITER, 1, false); else if (mc == 2) LAUNCH_M(MM_ITER, 2, false); else LAUNCH_M(MM_ITER, 4, false);
  } else if (mode == MM_R0) {
    if (mc == 1) LAUNCH_M(MM_R0, 1, false); else if (mc == 2) LAUNCH_M(MM_R0, 2, false); else LAUNCH_M(MM_R0, 4, false);
  } else if (mode == MM_R0E) {
    if (mc == 1) LAUNCH_M(MM_R0E, 1, false); else if (mc == 2) LAUNCH_M(MM_R0E, 2, false); else LAUNCH_M(MM_R0E, 4, false);
  } else {
    if (mc == 1) LAUNCH_M(MM_ENERGY, 1, true); else if (mc == 2) LAUNCH_M(MM_ENERGY, 2, true); else LAUNCH_M(MM_ENERGY, 4, true);
  }
#undef LAUNCH_M
  return grid;
}

// Interior units of the y^ launch (multi-GPU): rows / windows / nodes whose
// A_FF neighbours are all owned, so their part of the masked product can run
// while the halo of y is exchanged (only the halo rows need the
// peers' values).  Stays off (split_on = 0) without an interior range.
static emin_status emin_split_plan(emin_ctx c) {
  c->split_on = 0;
  if (!c->dist || c->nF < 64) return EMIN_OK;
  cudaStream_t s = c->stream;
  const int SM = emin_num_sms();
  unsigned long long* d;
  EMIN_CUDA_TRY(c, emin_mallocAsync(&d, sizeof(unsigned long long) * 5, s));
  const unsigned long long init[5] = {0ull, (unsigned long long)c->nF, 0ull, 0ull, 0ull};
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_boundary_bounds<<<SM * 4, 256, 0, s>>>(c->affptr, c->affcol, c->nF, d);
  k_boundary_count<<<SM * 4, 256, 0, s>>>(c->affptr, c->affcol, c->nF, d, d + 2);
  c->launches += 2;
  int64_t nunits = c->nF;
  if (c->kernel_path == 1) {
    int64_t nwin = 0;
    const int32_t* rs = scalar_iter_windows(c, &nwin);
    k_window_range<<<1, 1, 0, s>>>(rs, nwin, d, d + 3);
    c->launches += 1;
    nunits = nwin;
  }
  unsigned long long h[5];
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  cudaFreeAsync(d, s);
  const int64_t ib = (int64_t)h[0], ie = (int64_t)h[1];
  if (h[2] != 0 || ie <= ib) return EMIN_OK;          // boundary rows inside: no split
  int64_t u0 = ib, u1 = ie;
  if (c->kernel_path == 1) { u0 = (int64_t)h[3]; u1 = (int64_t)h[4]; }
  if (c->kernel_path == 2) { u0 = (ib + 2) / 3; u1 = ie / 3; nunits = c->nF / 3; }
  if (u1 <= u0) return EMIN_OK;
  c->split_u0 = u0;
  c->split_u1 = u1;
  c->split_n = nunits;
  EMIN_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  EMIN_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_y, cudaEventDisableTiming));
  EMIN_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  c->split_on = 1;
  return EMIN_OK;
}

// kernel path + launch geometry (end of the index preparation in setup)
emin_status emin_plan(emin_ctx c) {
  const int SM = emin_num_sms();
  c->group = pick_group(c->nF ? (double)c->nnzW / (double)c->nF : 1.0);
  c->grid_rows = (int)std::max<int64_t>(1, std::min<int64_t>((c->nF * c->group + 255) / 256, (int64_t)SM * 8));
  c->grid_spgemm = (int)std::max<int64_t>(1, std::min<int64_t>((c->nF + 7) / 8, (int64_t)SM * 8));
  c->kernel_path = select_fast_path(c);
  if (c->kernel_path != 1 && c->sym) {        // the scaled records exist on the scalar path only
    c->sym = 0;
    if (c->srow) { cudaFreeAsync(c->srow, c->stream); c->srow = nullptr; }
  }
  if (c->kernel_path == 0 && (c->opts.row_begin % 3) == 0) {
    NodalPlan* np = nullptr;
    if (select_nodal_path(c, np)) {
      c->nodal = np;
      c->kernel_path = 2;
    }
  }
  if (c->kernel_path == 1) c->grid_spgemm = scalar_spgemm_grid(c);
  if (c->kernel_path == 2 && c->opts.precond == EMIN_PREC_JACOBI && !c->opts.project_after_jacobi &&
      !(c->opts.debug_flags & EMIN_DBG_UNSCALED)) {
    // symmetric Jacobi scaling on the nodal path: the per-iteration product
    // reads S A_FF S (a scaled copy of A_FF's values); the stages, r0, P and
    // the energy as on the scalar path
    c->sym = 1;
    emin_status sst = emin_build_srow(c);
    if (sst != EMIN_OK) return sst;
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&c->affvalS, sizeof(double) * std::max<int64_t>(c->nnzAFF, 1),
                                      c->stream));
    k_scale_aff<<<SM * 16, 256, 0, c->stream>>>(c->affptr, c->affcol, c->affval, c->srow, c->nF, c->affvalS);
    c->launches += 1;
  }
  if (!c->opts.project_after_jacobi) {
    // entry-parallel streaming stages: row id per W entry
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&c->erow, sizeof(int32_t) * std::max<int64_t>(c->nnzW, 1), c->stream));
    k_build_erow<<<SM * 8, 256, 0, c->stream>>>(c->wptr, c->nF, c->erow);
    c->launches += 1;
    if (!c->sym) {            // the unscaled stages' exact quotient r / d
      EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&c->dinv, sizeof(double) * std::max<int64_t>(c->nF, 1), c->stream));
      k_recip<<<SM * 4, 256, 0, c->stream>>>(c->d, c->nF, c->dinv);
      c->launches += 1;
    }
    // one wave (4 CTAs of 256 per SM, the launch bound): config 3 stage I/II
    // 39.3 / 51.0 -> 38.3 / 48.6 us, config 4 60.4 / 84.5 -> 59.5 / 82.3 us,
    // config 5 neutral
    c->grid_rows = (int)std::max<int64_t>(1, std::min<int64_t>((c->nnzW + 255) / 256, (int64_t)SM * 4));
    c->pingpong = 1;
  }
  c->grid_red = std::max(c->grid_rows, c->grid_spgemm);
  if (c->kernel_path == 1) c->grid_red = std::max(c->grid_red, scalar_iter_launch_grid(c));
  if (c->kernel_path == 2) c->grid_red = std::max(c->grid_red, nodal_grid(c, static_cast<NodalPlan*>(c->nodal)));
  if (c->dist) {
    // the y^ launch may run as an interior and a boundary launch (both
    // write partial sums): room for two grids
    c->grid_red *= 2;
    emin_status sst = emin_split_plan(c);
    if (sst != EMIN_OK) return sst;
  }
  if (c->grid_red > c->n_partials) {
    cudaFreeAsync(c->partials, c->stream);
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&c->partials, sizeof(double) * c->grid_red, c->stream));
    c->n_partials = c->grid_red;
  }
  EMIN_CUDA_TRY(c, cudaGetLastError());
  return EMIN_OK;
}

// the scalar path's per-A_FF-entry records {a, wptr[k], pm} (diagonal first
// per row, then A's column order), or null off the scalar path (sgs.cu)
const int4* emin_scalar_records(emin_ctx c) {
  return c->kernel_path == 1 ? reinterpret_cast<const int4*>(fast_of(c)->sc.ent) : nullptr;
}
// the nodal path's plan (sgs.cu): per F node n its blocks [bptr[n], bptr[n+1])
// with records {wptr[3K], 3|J_K|} and the byte map pm8 + pmoff[n] (position of
// J_I[s] in J_K per block, 0xFF absent); false off the nodal path
bool emin_nodal_plan(emin_ctx c, const int2** blk, const int64_t** bptr, const uint8_t** pm8,
                     const int64_t** pmoff, int64_t* nFn, int32_t* max_nb) {
  if (c->kernel_path != 2 || !c->nodal) return false;
  const NodalPlan* np = static_cast<const NodalPlan*>(c->nodal);
  *max_nb = np->max_nb;
  *blk = reinterpret_cast<const int2*>(np->blk);
  *bptr = np->bptr;
  *pm8 = np->pm8;
  *pmoff = np->pmoff;
  *nFn = np->nFn;
  return true;
}

// the scalar path's window plan: rows [rowstart[w], rowstart[w+1]) of window
// w hold <= 32 entries (sgs.cu)
const int32_t* emin_scalar_windows(emin_ctx c, int64_t* nwin) {
  if (c->kernel_path != 1) { *nwin = 0; return nullptr; }
  *nwin = fast_of(c)->sc.nwin;
  return fast_of(c)->sc.rowstart;
}

// Alg. 2 on a specialised path (false: use the generic warp kernel)
bool emin_alg2_fast(emin_ctx c, const double* Bc, const double* B, const int64_t* frow, const double* what,
                    unsigned long long* counters, cudaStream_t s) {
  if (c->kernel_path != 1) return false;
  launch_scalar_alg2(c, Bc, B, frow, what, counters, s);
  return true;
}

// Sum of the per-block partials; on several GPUs: rank-local sum into
// st->red[slot], allreduce into st->redg[slot], and the consumer reads that
// (np = -1).  *res = the (pointer, np) pair the consumer kernel takes.
static emin_status global_sum(emin_ctx c, int np, int slot, cudaStream_t s, std::pair<const double*, int>* res,
                              bool local_done = false) {
  if (!c->dist) { *res = {c->partials, np}; return EMIN_OK; }
  if (!local_done) {     // (fused: the producing kernel's last block wrote st->red[slot])
    k_energy_out<<<1, 1024, 0, s>>>(c->partials, np, nullptr, &c->st->red[slot]);
    c->launches += 1;
  }
  *res = {&c->st->redg[slot], -1};
  return emin_dist_allreduce(c, &c->st->red[slot], &c->st->redg[slot], 1, s);
}

// r0 = -Pi (A P0)|F, E0, fresh CG state (end of setup and emin_reset)

emin_status emin_finish_r0(emin_ctx c) {
  cudaStream_t s = c->stream;
  EMIN_CUDA_TRY(c, cudaMemsetAsync(c->dw, 0, sizeof(double) * std::max<int64_t>(c->nnzWh, 1), s));
  // r0 and the energy of P0 (dw = 0) share the masked product A P0: one
  // MM_R0E pass where the kernel path has it, else MM_R0 then MM_ENERGY
  int g = (c->opts.debug_flags & EMIN_DBG_NO_R0E) ? -1 : emin_launch_masked(c, MM_R0E, c->w0, nullptr, c->r, s);
  if (g < 0) {
    emin_launch_masked(c, MM_R0, c->w0, nullptr, c->r, s);
    g = emin_launch_masked(c, MM_ENERGY, c->w0, c->dw, nullptr, s);
  }
  if (c->sym) {                                   // r~ = S r0 (symmetric Jacobi scaling)
    k_scale_rows<<<emin_num_sms() * 8, 256, 0, s>>>(c->r, c->erow, c->srow, c->nnzW);
    c->launches += 1;
  }
  std::pair<const double*, int> red;
  {
    emin_status st = global_sum(c, g, 2, s, &red);
    if (st != EMIN_OK) return st;
  }
  k_reset_state<<<1, 1024, 0, s>>>(c->st, red.first, red.second, c->opts.tau,
                                   c->opts.stagnation_rel);
  c->launches += 3;
  EMIN_CUDA_TRY(c, cudaGetLastError());
  c->k_launched = 0;
  c->breakdown_reported = 0;
  return EMIN_OK;
}

static emin_status enqueue_iteration(emin_ctx c, cudaStream_t s, cudaEvent_t* ev, int external) {
  auto rec = [&](int t) {
    if (ev) cudaEventRecordWithFlags(ev[t], s, external ? cudaEventRecordExternal : cudaEventRecordDefault);
  };
  // fused mode (one GPU, EMIN_DBG_FUSE_SCALARS): the scalar steps run in the
  // last block of stage I and of the SpGEMM (block_partial_out); measured
  // 3.4 us per iteration SLOWER on config 3 than the single-block kernels
  // (the last block's serial tail -- counter atomic, partial reduction,
  // dependent DevState loads -- costs what the separate launch did;
  // profiles/r01b/spgemm_ab_c3.txt), so it is not the default
  c->fuse = (!c->dist && (c->opts.debug_flags & EMIN_DBG_FUSE_SCALARS)) ? 1 : 0;
  // several GPUs: the rank-local sums are folded into the producing kernels'
  // last block (st->red[]), so each CG scalar costs one allreduce and the
  // scalar kernel, no separate reduction kernel
  if (c->dist) c->fuse = 2;
  if (c->sgs) c->fuse = 0;
  const bool fused_local = c->fuse == 2;
  std::pair<const double*, int> red;
  emin_status st = EMIN_OK;
  rec(0);
  int g1 = c->grid_rows;
  if (c->sgs) {                              // z = Pi M_2^-1 r, partial r.z
    st = emin_sgs_enqueue(c, s, &g1);
    if (st != EMIN_OK) return st;
  } else {
    launch_stage(c, 1, s);
  }
  rec(1);
  if (c->fuse != 1) {
    st = global_sum(c, g1, 0, s, &red, fused_local);
    if (st != EMIN_OK) return st;
    k_scalar_gamma<<<1, 1024, 0, s>>>(c->st, red.first, red.second);
  }
  rec(2);
  if (c->sgs) emin_sgs_stage2(c, s);
  else launch_stage(c, 2, s);
  int g = 0;
  if (c->dist && c->split_on) {
    // the halo of y on the comm stream, overlapped with the
    // interior part of y^; the boundary part waits for it
    cudaEventRecord(c->ev_y, s);
    cudaStreamWaitEvent(c->comm_stream, c->ev_y, 0);
    st = emin_dist_halo_values(c, c->y, c->comm_stream);
    if (st != EMIN_OK) return st;
    cudaEventRecord(c->ev_halo, c->comm_stream);
    rec(3);
    const int32_t fz = c->fuse;
    c->fuse = 0;                                       // the interior launch only writes partials
    c->mm_ubeg = c->split_u0; c->mm_uend = c->split_u1; c->mm_ugap0 = c->mm_ugap1 = 0; c->mm_poff = 0;
    const int gi = emin_launch_masked(c, MM_ITER, c->y, nullptr, c->yb, s);
    c->fuse = fz;
    cudaStreamWaitEvent(s, c->ev_halo, 0);
    c->mm_ubeg = 0; c->mm_uend = c->split_n; c->mm_ugap0 = c->split_u0; c->mm_ugap1 = c->split_u1; c->mm_poff = gi;
    const int gb = emin_launch_masked(c, MM_ITER, c->y, nullptr, c->yb, s);
    c->mm_ubeg = 0; c->mm_uend = -1; c->mm_ugap0 = c->mm_ugap1 = 0; c->mm_poff = 0;
    g = gi + gb;
  } else {
    if (c->dist) {
      st = emin_dist_halo_values(c, c->y, s);     // y on the halo rows
      if (st != EMIN_OK) return st;
    }
    rec(3);
    g = emin_launch_masked(c, MM_ITER, c->y, nullptr, c->yb, s);
  }
  rec(4);
  if (c->fuse != 1) {
    st = global_sum(c, g, 1, s, &red, fused_local);
    if (st != EMIN_OK) return st;
    k_scalar_alpha<<<1, 1024, 0, s>>>(c->st, red.first, red.second, c->dE_hist);
  }
  rec(5);
  // kernels of ours per iteration: stage I, stage II, y^ (+ the two scalar
  // kernels; + on several GPUs the halo pack and, with the interior /
  // boundary split, a second y^ launch; + with the loopback transport its
  // two rank-sum kernels)
  const bool lb = c->dist && !emin_dist_capturable(c);
  c->iter_kernels = 3 + (c->fuse == 1 ? 0 : 2) + (c->dist ? (c->dist->nSE ? 1 : 0) + (c->split_on ? 1 : 0) : 0) +
                    (lb ? 2 : 0) + (c->sgs ? (int32_t)(2 * emin_sgs_levels(c) - 1) : 0);
  return cudaGetLastError() == cudaSuccess ? EMIN_OK : EMIN_ERR_CUDA;
}

// timing events of this context's profiling mode (created on its device,
// destroyed by emin_destroy)
static std::vector<cudaEvent_t>& event_pool(emin_ctx c) { return c->ev; }

// One iteration captured as a CUDA graph (5 kernel nodes, cheap to
// instantiate per context); emin_iterate(k) launches it k times.  The
// profiling variant adds 6 event-record nodes around the kernels; before each
// launch their events are re-pointed (cudaGraphExecEventRecordNodeSetEvent)
// to fresh events of the pool, so k launches leave 6k timestamps and no
// synchronisation is needed until emin_kernel_times reads them.
static emin_status build_graph(emin_ctx c, int prof) {
  cudaGraphExec_t& ge = prof ? c->graph_prof_exec : c->graph;
  if (ge) { cudaGraphExecDestroy(ge); ge = nullptr; }
  // capture on the calling thread's own capture stream (one per thread and
  // device, kept for the thread's lifetime: the capture mode is
  // thread-local, and creating and destroying a stream per context cost
  // ~0.1 ms per bench step)
  static thread_local cudaStream_t cap[64] = {};
  {
    int dev = 0;
    EMIN_CUDA_TRY(c, cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return EMIN_ERR_CUDA;
    if (!cap[dev]) EMIN_CUDA_TRY(c, cudaStreamCreateWithFlags(&cap[dev], cudaStreamNonBlocking));
    c->cap_stream = cap[dev];
  }
  std::vector<cudaEvent_t>& ev = event_pool(c);
  while (prof && ev.size() < 6) {
    cudaEvent_t e;
    EMIN_CUDA_TRY(c, cudaEventCreate(&e));
    ev.push_back(e);
  }
  cudaStream_t s = c->cap_stream;
  EMIN_CUDA_TRY(c, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  const emin_status est = enqueue_iteration(c, s, prof ? ev.data() : nullptr, prof ? 1 : 0);
  cudaGraph_t g;
  EMIN_CUDA_TRY(c, cudaStreamEndCapture(s, &g));
  if (est != EMIN_OK) {    // a collective failed while the graph was built
    cudaGraphDestroy(g);
    if (c->last_error.empty()) c->last_error = "enqueue of the iteration failed";
    return est;
  }
  if (prof) {
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    for (int t = 0; t < 6; ++t) c->prof_node[t] = nullptr;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      cudaGraphNodeGetType(nd, &ty);
      if (ty != cudaGraphNodeTypeEventRecord) continue;
      cudaEvent_t e;
      cudaGraphEventRecordNodeGetEvent(nd, &e);
      for (int t = 0; t < 6; ++t)
        if (e == ev[t]) c->prof_node[t] = nd;
    }
  }
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  if (prof) {
    // the event-record node handles stay valid only while their graph lives
    if (c->graph_prof_src) cudaGraphDestroy(c->graph_prof_src);
    c->graph_prof_src = g;
  } else {
    cudaGraphDestroy(g);
  }
  EMIN_CUDA_TRY(c, e);
  return EMIN_OK;
}

// fold the recorded iterations into the per-class totals (synchronises)
static emin_status fold_profile(emin_ctx c) {
  if (!c->prof_pending) return EMIN_OK;
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  std::vector<cudaEvent_t>& ev = event_pool(c);
  for (int64_t it = 0; it < c->prof_pending; ++it) {
    cudaEvent_t* e = &ev[6 * (it + 1)];
    float t[5];
    for (int j = 0; j < 5; ++j) cudaEventElapsedTime(&t[j], e[j], e[j + 1]);
    c->prof_ms[0] += t[0];
    c->prof_ms[1] += t[2];
    c->prof_ms[2] += t[3];
    c->prof_ms[3] += t[1] + t[4];
    c->prof_launches[0] += 1; c->prof_launches[1] += 1; c->prof_launches[2] += 1;
    c->prof_launches[3] += 2;
  }
  c->prof_pending = 0;
  return EMIN_OK;
}

static emin_status ensure_hist(emin_ctx c, int64_t need) {
  if (need <= c->dE_cap) return EMIN_OK;
  int64_t cap = std::max<int64_t>(need, std::max<int64_t>(1024, 2 * c->dE_cap));
  double* nh;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&nh, sizeof(double) * cap, c->stream));
  if (c->dE_hist) {
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(nh, c->dE_hist, sizeof(double) * c->dE_cap, cudaMemcpyDeviceToDevice, c->stream));
    cudaFreeAsync(c->dE_hist, c->stream);
  }
  c->dE_hist = nh;
  c->dE_cap = cap;
  if (c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }   // they captured the old pointer
  if (c->graph_prof_exec) { cudaGraphExecDestroy(c->graph_prof_exec); c->graph_prof_exec = nullptr; }
  return EMIN_OK;
}

extern "C" emin_status emin_iterate(emin_ctx c, int32_t k, int32_t* k_done, double* dE) {
  if (!c) return EMIN_ERR_ARG;
  if (k < 0) { c->last_error = "k < 0"; return EMIN_ERR_ARG; }
  if (k_done) *k_done = 0;
  if (k == 0) return EMIN_OK;
  emin_status st = ensure_hist(c, c->k_launched + k);
  if (st != EMIN_OK) return st;
  EMIN_CUDA_TRY(c, cudaMemsetAsync(&c->st->k_call, 0, sizeof(int32_t), c->stream));
  if (!emin_dist_capturable(c)) {
    // loopback transport: its collectives rendezvous on the host, so the
    // iterations are enqueued eagerly (same kernels, same order)
    for (int it = 0; it < k; ++it) {
      st = enqueue_iteration(c, c->stream, nullptr, 0);
      if (st != EMIN_OK) {
        emin_dist_abort(c, c->last_error);
        return st;
      }
    }
  } else if (c->profiling) {
    if (!c->graph_prof_exec) {
      st = build_graph(c, 1);
      if (st != EMIN_OK) return st;
    }
    std::vector<cudaEvent_t>& ev = event_pool(c);
    const size_t need = (size_t)6 * (c->prof_pending + k + 1);
    while (ev.size() < need) {
      cudaEvent_t e;
      EMIN_CUDA_TRY(c, cudaEventCreate(&e));
      ev.push_back(e);
    }
    for (int it = 0; it < k; ++it) {
      cudaEvent_t* e = &ev[6 * (c->prof_pending + 1)];
      for (int t = 0; t < 6; ++t)
        if (c->prof_node[t]) EMIN_CUDA_TRY(c, cudaGraphExecEventRecordNodeSetEvent(c->graph_prof_exec, c->prof_node[t], e[t]));
      EMIN_CUDA_TRY(c, cudaGraphLaunch(c->graph_prof_exec, c->stream));
      c->prof_pending += 1;
    }
  } else {
    if (!c->graph) {
      st = build_graph(c, 0);
      if (st != EMIN_OK) return st;
    }
    for (int it = 0; it < k; ++it) EMIN_CUDA_TRY(c, cudaGraphLaunch(c->graph, c->stream));
  }
  c->launches += c->iter_kernels * (int64_t)k;
  c->k_launched += k;
  if (k_done || dE) {
    DevState h;
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(&h, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (k_done) *k_done = h.k_call;
    if (dE && h.k_call > 0)
      EMIN_CUDA_TRY(c, cudaMemcpy(dE, c->dE_hist + (h.k_total - h.k_call), sizeof(double) * h.k_call,
                                  cudaMemcpyDeviceToHost));
    if (h.stopped == 5 && !c->breakdown_reported) {
      c->breakdown_reported = 1;
      c->last_error = "y^T Pi K y < 0 (breakdown)";
      return EMIN_ERR_BREAKDOWN;
    }
  }
  EMIN_CUDA_TRY(c, cudaGetLastError());
  return EMIN_OK;
}

static void flush(emin_ctx c) {
  const int SM = emin_num_sms();
  k_flush<<<SM * 8, 256, 0, c->stream>>>(c->view(), c->dw, c->y);
  k_flush_done<<<1, 1, 0, c->stream>>>(c->st);
}

extern "C" emin_status emin_energy(emin_ctx c, double* E) {
  if (!c || !E) return EMIN_ERR_ARG;
  flush(c);
  if (c->dist && !c->sym) {
    emin_status st = emin_dist_halo_values(c, c->dw, c->stream);   // W = W0 + dW on the halo rows
    if (st != EMIN_OK) return st;
  }
  int g;
  // W = W0 + dW is summed once into a scratch vector (not y^: the flush
  // leaves the pending r -= alpha y^ to the next stage I)
  if ((c->sym || (c->kernel_path == 2 && !c->dist)) && !c->wtmp)
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&c->wtmp, sizeof(double) * std::max<int64_t>(c->nnzWh, 1), c->stream));
  if (c->sym) {
    // W = W0 + S dW~; on several GPUs its halo rows from their owners
    k_wsum_s<<<emin_num_sms() * 8, 256, 0, c->stream>>>(c->w0, c->dw, c->erow, c->srow, c->nnzW, c->wtmp);
    c->launches += 1;
    if (c->dist) {
      emin_status st = emin_dist_halo_values(c, c->wtmp, c->stream);
      if (st != EMIN_OK) return st;
    }
    g = emin_launch_masked(c, MM_ENERGY, c->wtmp, nullptr, nullptr, c->stream);
  } else if (c->kernel_path == 2 && !c->dist) {
    // nodal path: W = W0 + dW once, so the energy pass gathers one vector
    // instead of two (same sums; on the scalar path the extra pass costs
    // what it saves: 10.13 vs 10.15 ms/step)
    k_wsum<<<emin_num_sms() * 8, 256, 0, c->stream>>>(c->w0, c->dw, c->nnzW, c->wtmp);
    c->launches += 1;
    g = emin_launch_masked(c, MM_ENERGY, c->wtmp, nullptr, nullptr, c->stream);
  } else {
    g = emin_launch_masked(c, MM_ENERGY, c->w0, c->dw, nullptr, c->stream);
  }
  double* dev;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&dev, sizeof(double), c->stream));
  std::pair<const double*, int> red;
  {
    emin_status st = global_sum(c, g, 2, c->stream, &red);
    if (st != EMIN_OK) { cudaFreeAsync(dev, c->stream); return st; }
  }
  k_energy_out<<<1, 1024, 0, c->stream>>>(red.first, red.second, &c->st->sum_cc, dev);
  c->launches += 4;
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(E, dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  cudaFreeAsync(dev, c->stream);
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EMIN_OK;
}

extern "C" emin_status emin_get_P(emin_ctx c, double* P_val) {
  if (!c || !P_val) return EMIN_ERR_ARG;
  flush(c);
  const int SM = emin_num_sms();
  double* out = P_val;
  if (!c->opts.inputs_on_device)
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&out, sizeof(double) * std::max<int64_t>(c->nnzP, 1), c->stream));
  if (c->kernel_path == 1)
    launch_scalar_get_P(c, out, c->stream);
  else
    k_get_P<<<SM * 8, 256, 0, c->stream>>>(c->view(), c->w0, c->dw, c->pofs, out, c->sym ? c->srow : nullptr);
  k_get_P_crows<<<SM * 8, 256, 0, c->stream>>>(c->m_owned, c->isc_own, c->cofs, out);
  c->launches += 4;
  EMIN_CUDA_TRY(c, cudaGetLastError());
  if (!c->opts.inputs_on_device) {
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(P_val, out, sizeof(double) * c->nnzP, cudaMemcpyDeviceToHost, c->stream));
    cudaFreeAsync(out, c->stream);
  }
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EMIN_OK;
}

extern "C" emin_status emin_reset(emin_ctx c) {
  if (!c) return EMIN_ERR_ARG;
  return emin_finish_r0(c);
}

extern "C" emin_status emin_report(emin_ctx c, emin_report_t* rep) {
  if (!c || !rep) return EMIN_ERR_ARG;
  DevState h;
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(&h, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  std::memset(rep, 0, sizeof(*rep));
  rep->E0 = h.E0;
  rep->dE1 = h.dE1;
  rep->k_total = h.k_total;
  rep->stop_reason = h.stopped;
  rep->n_svd_rows = (int64_t)h.cnt[0];       // (Alg. 2 counters, kept on the device at setup)
  rep->n_frozen_rows = (int64_t)h.cnt[1];
  rep->n_fine = c->nF;
  rep->nnz_W = c->nnzW;
  rep->nnz_AFF = c->nnzAFF;
  rep->kernel_path = c->kernel_path;
  rep->nranks = c->nranks;
  rep->launches = c->launches;
  rep->precond = c->opts.precond;
  rep->sgs_levels = emin_sgs_levels(c);
  rep->n_maxvol_fail = (int64_t)h.cnt[2];
  rep->rank = c->rank;
  if (c->dist) {
    rep->n_halo_rows = c->dist->nH;
    rep->n_halo_entries = c->dist->nHW;
    rep->n_send_entries = c->dist->nSE;
    rep->n_interior_units = c->split_on ? c->split_u1 - c->split_u0 : 0;
  }
  if (h.stopped == 5 && !c->breakdown_reported) {
    c->breakdown_reported = 1;
    return EMIN_ERR_BREAKDOWN;
  }
  return EMIN_OK;
}

extern "C" emin_status emin_get_layout(emin_ctx c, int64_t* wptr, int32_t* wcol, int64_t* pofs) {
  if (!c) return EMIN_ERR_ARG;
  if (wptr) EMIN_CUDA_TRY(c, cudaMemcpyAsync(wptr, c->wptr, sizeof(int64_t) * (c->nF + 1), cudaMemcpyDeviceToHost, c->stream));
  if (wcol && c->nnzW)
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(wcol, c->wcol, sizeof(int32_t) * c->nnzW, cudaMemcpyDeviceToHost, c->stream));
  if (pofs && c->nF) EMIN_CUDA_TRY(c, cudaMemcpyAsync(pofs, c->pofs, sizeof(int64_t) * c->nF, cudaMemcpyDeviceToHost, c->stream));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EMIN_OK;
}

extern "C" emin_status emin_set_profiling(emin_ctx c, int32_t on) {
  if (!c) return EMIN_ERR_ARG;
  fold_profile(c);
  c->profiling = on ? 1 : 0;
  for (int j = 0; j < 4; ++j) { c->prof_ms[j] = 0.0; c->prof_launches[j] = 0; }
  return EMIN_OK;
}

extern "C" emin_status emin_kernel_times(emin_ctx c, double* ms, int64_t* launches) {
  if (!c) return EMIN_ERR_ARG;
  {
    emin_status st = fold_profile(c);
    if (st != EMIN_OK) return st;
  }
  for (int j = 0; j < 4; ++j) {
    if (ms) ms[j] = c->prof_ms[j];
    if (launches) launches[j] = c->prof_launches[j];
  }
  return EMIN_OK;
}

void emin_free_all(emin_ctx c) {
  cudaStream_t s = c->stream;
  void* ptrs[] = {c->wptr, c->affptr, c->afcptr, c->pofs, c->cofs, c->isc_own, c->wcol, c->affcol,
                  c->afccol, c->affval, c->afcval, c->d, c->Q, c->w0, c->dw, c->r, c->r0, c->y,
                  c->yb, c->partials, c->dE_hist, c->st, c->erow, c->dinv, c->adiag, c->srow, c->affvalS, c->wtmp};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, s);
  free_fast_path(c);
  {
    NodalPlan* np = static_cast<NodalPlan*>(c->nodal);
    free_nodal_path(c, np);
    c->nodal = nullptr;
  }
  emin_dist_free(c);
  emin_sgs_free(c);
  cudaStreamSynchronize(s);
}

extern "C" void emin_destroy(emin_ctx c) {
  if (!c) return;
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->graph_prof_exec) cudaGraphExecDestroy(c->graph_prof_exec);
  if (c->graph_prof_src) cudaGraphDestroy(c->graph_prof_src);
  emin_free_all(c);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  if (c->ev_y) cudaEventDestroy(c->ev_y);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  delete c;                                   // (the capture stream is kept per thread and device)
}

extern "C" const char* emin_setup_error_internal();
extern "C" const char* emin_last_error(emin_ctx c) {
  if (!c) return emin_setup_error_internal();
  return c->last_error.c_str();
}
