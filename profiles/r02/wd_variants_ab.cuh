// A/B record (round 2): k_spgemm_wd variants (GRP 1/2/3, PRED, CTA-contiguous order, 6 CTAs/SM).
// The library keeps GRP=1, 8 CTAs/SM, grid-stride order; timings in profiles/r02/spgemm_ab_c3.txt.
constexpr uint32_t WD_MAXREC = 255, WD_MAXREL = 65535;
template <int GRP = 2, int MINB = 8, bool PRED = false, bool CTAC = false>
__global__ void __launch_bounds__(256, MINB)
k_spgemm_wd(DevView v, const SpEnt* __restrict__ A, const int4* __restrict__ whdr, const uint32_t* __restrict__ wdesc,
            int32_t nwin, const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  double part = 0.0;
  const bool rev = v.pingpong && (v.st->k_total & 1);   // same direction as stage I (L2 ping-pong)
  const bool split = v.uend >= 0 || v.ubeg != 0 || v.ugap1 != v.ugap0;
  const int cnt = split ? (int)unit_count(v, nwin) : nwin;
  const int4* A4 = reinterpret_cast<const int4*>(A);
  // CTAC: each CTA sweeps a contiguous run of windows (its 8 warps on 8
  // consecutive windows at a time), so neighbour rows a few windows back
  // are still in this SM's L1
  const int per = CTAC ? (cnt + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int cb = CTAC ? (int)blockIdx.x * per : 0;
  const int ce = CTAC ? min(cnt, cb + per) : cnt;
  for (int w1 = CTAC ? cb + wib : gw; w1 < ce; w1 += CTAC ? 8 : nw) {
    int w = rev ? cnt - 1 - w1 : w1;
    if (split) w = (int)unit_of(v, w);
    const int4 h = __ldg(whdr + w);
    const int nent = h.z;
    if (nent == 0) continue;                           // warp-uniform
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
    double acc = 0.0;
    if (act) {
      // record qb is the diagonal A(i,i): its y value is the lane's own entry
      acc = __hiloint2double(__ldg(&A4[qb]).y, __ldg(&A4[qb]).x) * xo;
      const unsigned sh4 = 4u * (unsigned)pos;
      int q = qb + 1;
      if (GRP > 1) {
        for (; q + GRP <= qe; q += GRP) {
          int4 en[GRP];
          double y[GRP];
          bool m[GRP];
#pragma unroll
          for (int g = 0; g < GRP; ++g) en[g] = __ldg(&A4[q + g]);
#pragma unroll
          for (int g = 0; g < GRP; ++g) {
            const unsigned s = ((unsigned)en[g].w >> sh4) & 0xFu;
            m[g] = s != 0xFu;
            y[g] = m[g] ? X[en[g].z + (int)s] : 0.0;
          }
#pragma unroll
          for (int g = 0; g < GRP; ++g)
            if (PRED || m[g]) acc = fma(__hiloint2double(en[g].y, en[g].x), y[g], acc);
        }
      }
#pragma unroll 4
      for (; q < qe; ++q) {
        const int4 en = __ldg(&A4[q]);
        const unsigned s = ((unsigned)en.w >> sh4) & 0xFu;
        if (PRED) acc = fma(__hiloint2double(en.y, en.x), s != 0xFu ? X[en.z + (int)s] : 0.0, acc);
        else if (s != 0xFu) acc = fma(__hiloint2double(en.y, en.x), X[en.z + (int)s], acc);
      }
    }
    s_qa[wib][lane] = qv * acc;
    __syncwarp();
    double dot = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p)                       // |J_i| <= 8 on the scalar path
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

