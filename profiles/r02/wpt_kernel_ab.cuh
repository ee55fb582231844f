// A/B variant (not in the library): k_spgemm_wp on slot-major (window-transposed)
// records, with L1 prefetch of the window's record block (PF 1) and of its y / Q
// lines (PF 2).  profiles/r02/spgemm_ab_c3.txt has the numbers.

// k_spgemm_wp on window-transposed records: the same pair windows, lanes,
// terms and order (the same y^), but the records of a window's R rows are
// stored slot-major -- record q of row r at T_w + q R + r, rows shorter than
// the window's longest (M records) padded with pm = ~0 -- so a round's two
// record loads read R consecutive records (two L1 lines) instead of one line
// per row; the window's record block is prefetched into L1 when its header
// arrives.  (The pair kernel is bound by L1 data-pipe wavefronts: ncu 83 %
// of peak, ~5 wavefronts per load request.)
// thdr[w] = {first lane slot, T_w, lanes | R << 8 | M << 16, first W entry};
// tdesc[l] = {first entry, row's first lane | (|J_r| - 1) << 5 | row << 8}.
template <int NT = WP_NT, int MINB = WP_MINB, int UNR = WP_UNR, int PF = 1>
__global__ void __launch_bounds__(NT, MINB)
k_spgemm_wpt(DevView v, const SpEnt* __restrict__ AT, const int4* __restrict__ thdr, const int2* __restrict__ tdesc,
             int32_t nwin, const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[NT / 32][64];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  double part = 0.0;
  const bool rev = v.pingpong && (v.st->k_total & 1);   // same direction as stage I (L2 ping-pong)
  const bool split = v.uend >= 0 || v.ubeg != 0 || v.ugap1 != v.ugap0;
  const int cnt = split ? (int)unit_count(v, nwin) : nwin;
  const int2* I2 = reinterpret_cast<const int2*>(AT);
  const double* Ad = reinterpret_cast<const double*>(AT);
  for (int w1 = gw; w1 < cnt; w1 += nw) {
    int w = rev ? cnt - 1 - w1 : w1;
    if (split) w = (int)unit_of(v, w);
    const int4 h = __ldg(thdr + w);
    const int nl = h.z & 63;
    if (nl == 0) continue;                             // warp-uniform
    const int R = (h.z >> 8) & 63, M = h.z >> 16;
    if (PF && lane * 8 < R * M) pf_l1(AT + h.y + 8 * lane);   // the window's record block (<= 32 lines)
    if (PF >= 2) {
      // y and Q lines of the window's entries (<= 64 entries from the first)
      const int nent = min(64, 2 * (h.z & 63));
      if (lane < 8) { if (16 * lane < nent) pf_l1(X + h.w + 16 * lane); }
      else if (lane < 16) { if (16 * (lane - 8) < nent) pf_l1(v.Q + h.w + 16 * (lane - 8)); }
    }
    const bool act = lane < nl;
    const int2 d = act ? __ldg(tdesc + h.x + lane) : make_int2(0, 0);
    const int e0 = d.x;
    const uint32_t dsc = (uint32_t)d.y;
    const int rowbeg = (int)(dsc & 31u);
    const int rowlen = (int)((dsc >> 5) & 7u) + 1;
    const int p0 = 2 * (lane - rowbeg);                // the lane's first position in its row
    double acc0 = 0.0, acc1 = 0.0;
    if (act) {
      int slot = h.y + (int)(dsc >> 8);                // slot (0, row): the diagonal A(i,i)
      const int send = slot + M * R;
      const double ad = __ldg(Ad + 2 * slot);
      acc0 = ad * X[e0];
      if (p0 + 1 < rowlen) acc1 = ad * X[e0 + 1];
      const unsigned shp = 4u * (unsigned)p0;
      slot += R;
      // the record stream is padded by WPT_PAD slots: the look-ahead load
      // needs no bound check; an absent position adds a * 0
      int2 nxt = __ldg(I2 + 2 * slot + 1);
#pragma unroll UNR
      for (; slot < send; slot += R) {
        const int2 cur = nxt;
        nxt = __ldg(I2 + 2 * (slot + R) + 1);
        const unsigned pm = (unsigned)cur.y >> shp;    // positions past the row: 0xF
        const unsigned s0 = pm & 0xFu, s1 = (pm >> 4) & 0xFu;
        const double y0 = (s0 != 0xFu) ? X[cur.x + (int)s0] : 0.0;
        const double y1 = (s1 != 0xFu) ? X[cur.x + (int)s1] : 0.0;
        const double a = __ldg(Ad + 2 * slot);
        acc0 = fma(a, y0, acc0);
        acc1 = fma(a, y1, acc1);
      }
    }
    const double qv0 = act ? v.Q[e0] : 0.0;
    const double qv1 = (act && p0 + 1 < rowlen) ? v.Q[e0 + 1] : 0.0;
    s_qa[wib][2 * lane] = qv0 * acc0;
    s_qa[wib][2 * lane + 1] = qv1 * acc1;
    __syncwarp();
    double dot = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p)                       // |J_i| <= 8 on the scalar path
      if (p < rowlen) dot += s_qa[wib][2 * rowbeg + p];
    __syncwarp();
    if (act) {
      const double g0 = acc0 - qv0 * dot;
      out[e0] = g0;
      part = fma(X[e0], g0, part);
      if (p0 + 1 < rowlen) {
        const double g1 = acc1 - qv1 * dot;
        out[e0 + 1] = g1;
        part = fma(X[e0 + 1], g1, part);
      }
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

// k_spgemm_wpt's plan: padded slots R * M of each pair window
__global__ void k_plan_wt_count(const int64_t* __restrict__ affptr, const int32_t* __restrict__ rowstart,
                                int64_t nwin, int64_t* __restrict__ slots) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = rowstart[w], r1 = rowstart[w + 1];
    int64_t M = 0;
    for (int i = r0; i < r1; ++i) M = max(M, affptr[i + 1] - affptr[i]);
    slots[w] = (int64_t)(r1 - r0) * M;
  }
}
// warp per window, lane per row: slot-major records (pad pm = ~0), header
// and the rows' lane-slot descriptors
__global__ void k_plan_wt_fill(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr,
                               const int64_t* __restrict__ lptr, const int32_t* __restrict__ rowstart, int64_t nwin,
                               const int64_t* __restrict__ Tw, const SpEnt* __restrict__ ent, SpEnt* __restrict__ entT,
                               int4* __restrict__ thdr, int2* __restrict__ tdesc) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int r0 = rowstart[w], r1 = rowstart[w + 1];
    const int R = r1 - r0;
    const int64_t rb = (lane < R) ? affptr[r0 + lane] : 0;
    const int nr = (lane < R) ? (int)(affptr[r0 + lane + 1] - rb) : 0;
    const int M = __reduce_max_sync(0xffffffffu, nr);
    const int64_t T = Tw[w], lb = lptr[r0];
    if (lane == 0)
      thdr[w] = make_int4((int)lb, (int)T, (int)(lptr[r1] - lb) | (R << 8) | (M << 16), (int)wptr[r0]);
    if (lane < R) {
      const int i = r0 + lane;
      for (int q = 0; q < M; ++q) {
        SpEnt en;
        if (q < nr) en = ent[rb + q];
        else { en.a = 0.0; en.ybase = 0; en.pm = 0xFFFFFFFFu; }
        entT[T + (int64_t)q * R + lane] = en;
      }
      const int64_t l0 = lptr[i], l1 = lptr[i + 1];
      const int64_t len = wptr[i + 1] - wptr[i];
      const uint32_t d = (uint32_t)(l0 - lb) | ((uint32_t)(len - 1) << 5) | ((uint32_t)lane << 8);
      for (int64_t l = l0; l < l1; ++l) tdesc[l] = make_int2((int)(wptr[i] + 2 * (l - l0)), (int)d);
    }
  }
}

