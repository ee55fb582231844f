// Round-1 A/B variants of the nodal masked SpGEMM (NOT compiled into libemin;
// kept for the record -- see README.md in this directory).
// y^ = Pi K y on the nodal path (+ partial y . y^)
template <int NV>
__global__ void __launch_bounds__(256)
k_spgemm_nodal(DevView v, const NodalBlk* __restrict__ blk, const int64_t* __restrict__ bptr,
               const uint8_t* __restrict__ pm8, const int64_t* __restrict__ pmoff, int64_t nFn,
               const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part = 0.0;
  for (int64_t n = gw; n < nFn; n += nw) {
    const int64_t r = 3 * n;
    const int64_t wb = v.wptr[r];
    const int n3 = (int)(v.wptr[r + 1] - wb);
    const int nJ = n3 / 3;
    const int t0 = lane, t1 = lane + 32;
    const bool act0 = t0 < n3, act1 = t1 < n3;
    const int s0 = t0 / 3, b0 = t0 - 3 * s0, s1 = t1 / 3, b1 = t1 - 3 * s1;
    const int64_t ab = v.affptr[r];
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    const int64_t rs = 3 * (int64_t)nb;          // row stride of the node's A chunk
    const int64_t po = pmoff[n];
    double acc0[3] = {0.0, 0.0, 0.0}, acc1[3] = {0.0, 0.0, 0.0};
    for (int b = 0; b < nb; ++b) {
      const NodalBlk k = blk[bb + b];
      double a[3][3];
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = 0; e < 3; ++e) a[d][e] = __ldg(v.affval + ab + d * rs + 3 * b + e);
      const int p0 = act0 ? pm8[po + (int64_t)b * nJ + s0] : 0xFF;
      const int p1 = act1 ? pm8[po + (int64_t)b * nJ + s1] : 0xFF;
      if (p0 != 0xFF) {
        double y[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) y[e] = X[(int64_t)k.ybase + e * k.nK3 + 3 * p0 + b0];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e = 0; e < 3; ++e) acc0[d] = fma(a[d][e], y[e], acc0[d]);
      }
      if (p1 != 0xFF) {
        double y[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) y[e] = X[(int64_t)k.ybase + e * k.nK3 + 3 * p1 + b1];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e = 0; e < 3; ++e) acc1[d] = fma(a[d][e], y[e], acc1[d]);
      }
    }
    // Pi_B per output row (Q of the node, row 3n, shared by its 3 rows)
    double q0[NV], q1[NV];
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      q0[m] = act0 ? v.Q[(wb + t0) * NV + m] : 0.0;
      q1[m] = act1 ? v.Q[(wb + t1) * NV + m] : 0.0;
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double dots[NV];
#pragma unroll
      for (int m = 0; m < NV; ++m) dots[m] = warp_sum(fma(q0[m], acc0[d], q1[m] * acc1[d]));
      double s0v = 0.0, s1v = 0.0;
#pragma unroll
      for (int m = 0; m < NV; ++m) {
        s0v = fma(q0[m], dots[m], s0v);
        s1v = fma(q1[m], dots[m], s1v);
      }
      const int64_t ro = wb + (int64_t)d * n3;
      if (act0) {
        const double g = acc0[d] - s0v;
        out[ro + t0] = g;
        part = fma(X[ro + t0], g, part);
      }
      if (act1) {
        const double g = acc1[d] - s1v;
        out[ro + t1] = g;
        part = fma(X[ro + t1], g, part);
      }
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

// Staged variant: the warp first copies its node's A chunk (9 nb doubles),
// block records and byte map into shared memory with coalesced loads (all
// independent), then the block loop only gathers y (two blocks per round so
// that six gathers per lane are in flight).
constexpr int ND_WARPS = 8;
constexpr int ND_MAXB = 27;      // blocks per node (27-point node stencil)
constexpr int ND_MAXJ = 32;      // C nodes per pattern row (3|J| <= 96 entries -> 2 chunks of 32 needs |J| <= 21)

template <int NV, int MODE>
__global__ void __launch_bounds__(ND_WARPS * 32, 4)
k_spgemm_nodal_s(DevView v, const NodalBlk* __restrict__ blk, const int64_t* __restrict__ bptr,
                 const uint8_t* __restrict__ pm8, const int64_t* __restrict__ pmoff, int64_t nFn,
                 const double* __restrict__ X, const double* __restrict__ X2, double* __restrict__ out,
                 double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_a[ND_WARPS][ND_MAXB * 9];
  __shared__ NodalBlk s_b[ND_WARPS][ND_MAXB];
  __shared__ uint8_t s_pm[ND_WARPS][ND_MAXB * ND_MAXJ];
  if (MODE == MM_ITER && v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool two = MODE == MM_ENERGY && X2 != nullptr;    // (X2 null: X already W0 + dW)
  auto xval = [&](int64_t idx) -> double { return two ? X[idx] + X2[idx] : X[idx]; };
  double part = 0.0;
  for (int64_t n = gw; n < nFn; n += nw) {
    const int64_t r = 3 * n;
    const int64_t wb = v.wptr[r];
    const int n3 = (int)(v.wptr[r + 1] - wb);
    const int nJ = n3 / 3;
    const int64_t ab = v.affptr[r];
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    const int64_t po = pmoff[n];
    // ---- stage the node's data (re-ordered A chunk: block-major 3x3)
    const int rs = 3 * nb;
    for (int k = lane; k < 9 * nb; k += 32) {
      const int d = k / rs, rem = k - d * rs, b = rem / 3, e = rem - 3 * b;
      s_a[wib][b * 9 + d * 3 + e] = __ldg(v.affval + ab + k);
    }
    for (int k = lane; k < nb; k += 32) s_b[wib][k] = blk[bb + k];
    for (int k = lane; k < nb * nJ; k += 32) s_pm[wib][k] = pm8[po + k];
    const int t0 = lane, t1 = lane + 32;
    const bool act0 = t0 < n3, act1 = t1 < n3;
    const int s0 = t0 / 3, b0 = t0 - 3 * s0, s1 = t1 / 3, b1 = t1 - 3 * s1;
    __syncwarp();
    double acc0[3] = {0.0, 0.0, 0.0}, acc1[3] = {0.0, 0.0, 0.0};
#pragma unroll 2
    for (int b = 0; b < nb; ++b) {
      const NodalBlk k = s_b[wib][b];
      const int p0 = act0 ? s_pm[wib][b * nJ + s0] : 0xFF;
      const int p1 = act1 ? s_pm[wib][b * nJ + s1] : 0xFF;
      double y0[3] = {0.0, 0.0, 0.0}, y1[3] = {0.0, 0.0, 0.0};
      if (p0 != 0xFF) {
#pragma unroll
        for (int e = 0; e < 3; ++e) y0[e] = xval((int64_t)k.ybase + e * k.nK3 + 3 * p0 + b0);
      }
      if (p1 != 0xFF) {
#pragma unroll
        for (int e = 0; e < 3; ++e) y1[e] = xval((int64_t)k.ybase + e * k.nK3 + 3 * p1 + b1);
      }
      const double* a = &s_a[wib][b * 9];
      if (p0 != 0xFF) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e = 0; e < 3; ++e) acc0[d] = fma(a[d * 3 + e], y0[e], acc0[d]);
      }
      if (p1 != 0xFF) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e = 0; e < 3; ++e) acc1[d] = fma(a[d * 3 + e], y1[e], acc1[d]);
      }
    }
    // Q of the node (row 3n) loaded after the block loop: keeps the loop's
    // register footprint small (occupancy)
    double q0[NV], q1[NV];
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      q0[m] = (MODE != MM_ENERGY && act0) ? v.Q[(wb + t0) * NV + m] : 0.0;
      q1[m] = (MODE != MM_ENERGY && act1) ? v.Q[(wb + t1) * NV + m] : 0.0;
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t ro = wb + (int64_t)d * n3;
      double g0 = acc0[d], g1 = acc1[d];
      if (MODE != MM_ITER) {          // C-identity term A(i, c_j) (setup / energy only)
        const int64_t fb = v.afcptr[r + d], fe = v.afcptr[r + d + 1];
        double f0 = 0.0, f1 = 0.0;
        if (act0) {
          const int32_t j = v.wcol[ro + t0];
          for (int64_t q = fb; q < fe; ++q) if (v.afccol[q] == j) { f0 = v.afcval[q]; break; }
        }
        if (act1) {
          const int32_t j = v.wcol[ro + t1];
          for (int64_t q = fb; q < fe; ++q) if (v.afccol[q] == j) { f1 = v.afcval[q]; break; }
        }
        if (MODE == MM_ENERGY) {
          if (act0) part = fma(xval(ro + t0), g0 + 2.0 * f0, part);
          if (act1) part = fma(xval(ro + t1), g1 + 2.0 * f1, part);
          continue;
        }
        g0 += f0;
        g1 += f1;
      }
      // Pi_B with the node's Q (twice for r0, see masked.cuh)
#pragma unroll
      for (int pass = 0; pass < (MODE == MM_R0 ? 2 : 1); ++pass) {
        double dots[NV];
#pragma unroll
        for (int m = 0; m < NV; ++m) dots[m] = warp_sum(fma(q0[m], g0, q1[m] * g1));
        double s0v = 0.0, s1v = 0.0;
#pragma unroll
        for (int m = 0; m < NV; ++m) {
          s0v = fma(q0[m], dots[m], s0v);
          s1v = fma(q1[m], dots[m], s1v);
        }
        g0 -= s0v;
        g1 -= s1v;
      }
      if (act0) {
        if (MODE == MM_ITER) { out[ro + t0] = g0; part = fma(X[ro + t0], g0, part); }
        else out[ro + t0] = -g0;
      }
      if (act1) {
        if (MODE == MM_ITER) { out[ro + t1] = g1; part = fma(X[ro + t1], g1, part); }
        else out[ro + t1] = -g1;
      }
    }
    __syncwarp();
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, MODE == MM_ITER ? 1 : -1);
}

