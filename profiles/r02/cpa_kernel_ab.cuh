// A/B record (round 2): cp.async gathers into shared memory (k_spgemm_cpa).
// Not part of the library; config 3: R=6 164.7 us, R=4 132.0 us vs k_spgemm_wd 116.6 us.
// y^ = Pi K y, window-descriptor kernel with the neighbour gathers issued as
// cp.async copies into shared memory (no registers held while they fly):
// every lane issues the gathers of all its row's records at once, waits
// once, then runs the FMAs in the same order as k_spgemm_wd (bitwise the
// same y^).  Records beyond the first R off-diagonal ones take the register
// loop.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <int R = 6>
__global__ void __launch_bounds__(256, 8)
k_spgemm_cpa(DevView v, const SpEnt* __restrict__ A, const int4* __restrict__ whdr, const uint32_t* __restrict__ wdesc,
             int32_t nwin, const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  __shared__ __align__(16) double s_y[8][R][32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  double part = 0.0;
  const bool rev = v.pingpong && (v.st->k_total & 1);
  const bool split = v.uend >= 0 || v.ubeg != 0 || v.ugap1 != v.ugap0;
  const int cnt = split ? (int)unit_count(v, nwin) : nwin;
  const int4* A4 = reinterpret_cast<const int4*>(A);
  const int2* A2 = reinterpret_cast<const int2*>(A);
  for (int w1 = gw; w1 < cnt; w1 += nw) {
    int w = rev ? cnt - 1 - w1 : w1;
    if (split) w = (int)unit_of(v, w);
    const int4 h = __ldg(whdr + w);
    const int nent = h.z;
    if (nent == 0) continue;
    const bool act = lane < nent;
    const int e = h.x + lane;
    const uint32_t dsc = act ? __ldg(wdesc + e) : 0u;
    const double qv = act ? v.Q[e] : 0.0;
    const double xo = act ? X[e] : 0.0;
    const int rowbeg = (int)(dsc & 31u);
    const int rowlen = (int)((dsc >> 5) & 7u) + 1;
    const int qb = h.y + (int)(dsc >> 16);
    const int qe = qb + (int)((dsc >> 8) & 255u);
    const int pos = lane - rowbeg;
    const unsigned sh4 = 4u * (unsigned)pos;
    const int nr = act ? min(qe - qb - 1, R) : 0;
    unsigned mk = 0u;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (j < nr) {
        const int2 zw = __ldg(A2 + 2 * (qb + 1 + j) + 1);     // {ybase, pm}
        const unsigned s = ((unsigned)zw.y >> sh4) & 0xFu;
        if (s != 0xFu) {
          cp_async8(&s_y[wib][j][lane], X + zw.x + (int)s);
          mk |= 1u << j;
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    double acc = act ? __hiloint2double(__ldg(&A4[qb]).y, __ldg(&A4[qb]).x) * xo : 0.0;
    double av[R];
#pragma unroll
    for (int j = 0; j < R; ++j) av[j] = ((mk >> j) & 1u) ? __ldg(&A[qb + 1 + j].a) : 0.0;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int j = 0; j < R; ++j)
      if ((mk >> j) & 1u) acc = fma(av[j], s_y[wib][j][lane], acc);
    if (act) {
      for (int q = qb + 1 + R; q < qe; ++q) {
        const int4 en = __ldg(&A4[q]);
        const unsigned s = ((unsigned)en.w >> sh4) & 0xFu;
        if (s != 0xFu) acc = fma(__hiloint2double(en.y, en.x), X[en.z + (int)s], acc);
      }
    }
    s_qa[wib][lane] = qv * acc;
    __syncwarp();
    double dot = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
      if (p < rowlen) dot += s_qa[wib][rowbeg + p];
    __syncwarp();
    if (act) {
      const double g = acc - qv * dot;
      out[e] = g;
      part = fma(xo, g, part);
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

