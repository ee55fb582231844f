// y^ = Pi K y (nv = 1), "push" window kernel.  Same windows as win2 (a warp
// owns the rows whose first W entry lies in window w, <= 32 entries), but the
// loads are organised for memory-level parallelism instead of a per-lane
// dependent chain (win2: rowstart -> wptr -> affptr -> broadcast record ->
// gather, ~112 unique bytes per 512-byte register load):
//   1. one 16-byte header per window {r0, base, a0, head mask} (the next
//      window's header is prefetched), then in ONE round, all independent:
//      the window's A_FF records, coalesced (lane = record, 16 B each), the
//      rows' entry / record offsets (int32), the lane's own y and Q_i entry;
//   2. each record-lane finds its row (record head mask + ballot) and issues
//      all the gathers of its record at once -- y(k, s) for every position t
//      of its row where J_i[t] is in J_k (the nibble map) -- and writes the
//      products a_ik y(k, s) to shared memory slot [entry][rank of k in row i];
//   3. each entry-lane sums its row's products in record order (diagonal
//      first, then A's column order: deterministic), then Pi_B by the row dot
//      through shared memory as in win2.
// The products are rounded before the sum (win2 used one fma per record), so
// y^ agrees with win2 / the generic kernel to round-off (tested against the
// generic kernel).
template <int MAXR>
__global__ void __launch_bounds__(256)
k_spgemm_push(DevView v, const int4* __restrict__ A4, const int4* __restrict__ hdr, int64_t nwin,
              const int32_t* __restrict__ wptr32, const int32_t* __restrict__ aptr32,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  __shared__ double s_pr[8][32 * MAXR];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  double* pr = s_pr[wib];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part = 0.0;
  const bool rev = v.pingpong && (v.st->k_total & 1);   // same direction as stage I (L2 ping-pong)
  auto win_of = [&](int64_t w1) { return rev ? nwin - 1 - w1 : w1; };
  int4 h0 = {0, 0, 0, 0}, h1 = {0, 0, 0, 0};
  if (gw < nwin) { h0 = __ldg(hdr + win_of(gw)); h1 = __ldg(hdr + win_of(gw) + 1); }
  for (int64_t w1 = gw; w1 < nwin; w1 += nw) {
    const int r0 = h0.x, nrows = h1.x - h0.x;
    const int base = h0.y, nent = h1.y - h0.y;
    const int a0 = h0.z, nrec = h1.z - h0.z;
    const unsigned H = (unsigned)h0.w;
    // prefetch the next window's header
    if (w1 + nw < nwin) { h0 = __ldg(hdr + win_of(w1 + nw)); h1 = __ldg(hdr + win_of(w1 + nw) + 1); }
    if (nrows == 0) continue;                          // warp-uniform
    // ---- round 1: independent loads
    const bool act = lane < nent;
    const int e = base + lane;
    const int wofs = (lane <= nrows) ? __ldg(wptr32 + r0 + lane) - base : 0;   // row starts (entries)
    const int aofs = (lane <= nrows) ? __ldg(aptr32 + r0 + lane) - a0 : 0;     // row starts (records)
    const double qv = act ? __ldg(v.Q + e) : 0.0;
    const double xo = act ? X[e] : 0.0;
    int4 rc0 = {0, 0, 0, 0}, rc1 = {0, 0, 0, 0};
    if (lane < nrec) rc0 = __ldg(A4 + a0 + lane);
    if (32 + lane < nrec) rc1 = __ldg(A4 + a0 + 32 + lane);
    // ---- round 2: per record, its row and all its gathers
    for (int c = 0; 32 * c < nrec; ++c) {
      int4 rc = c == 0 ? rc0 : c == 1 ? rc1 : int4{0, 0, 0, 0};
      const int x = 32 * c + lane;
      if (c >= 2 && x < nrec) rc = __ldg(A4 + a0 + x);
      // rows starting before this chunk, and the row starts inside it
      const int nbefore = __popc(__ballot_sync(0xffffffffu, lane < nrows && aofs < 32 * c));
      const int rel = aofs - 32 * c;
      const unsigned Hr = __reduce_or_sync(0xffffffffu, (lane < nrows && rel >= 0 && rel < 32) ? (1u << rel) : 0u);
      const unsigned upto = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
      int row = nbefore + __popc(Hr & upto) - 1;
      row = row < 0 ? 0 : row;
      const int rank = x - __shfl_sync(0xffffffffu, aofs, row);
      const int rb = __shfl_sync(0xffffffffu, wofs, row);
      const int rlen = __shfl_sync(0xffffffffu, wofs, row + 1 <= nrows ? row + 1 : nrows) - rb;
      if (x < nrec) {
        const double a = __hiloint2double(rc.y, rc.x);
        const unsigned pm = (unsigned)rc.w;
        double yv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const unsigned sidx = (pm >> (4 * t)) & 0xFu;
          yv[t] = (t < rlen && sidx != 0xFu) ? X[rc.z + (int)sidx] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (t < rlen) pr[(rb + t) * MAXR + rank] = a * yv[t];
      }
    }
    __syncwarp();
    // ---- round 3: per entry, the sum over its row's records (record order)
    const int l = act ? lane : nent - 1;
    const unsigned uptoe = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
    const int rloc = __popc(H & uptoe) - 1;
    const int rowbeg = 31 - __clz(H & uptoe);
    const unsigned after = H & ~uptoe;
    const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
    const int ra = __shfl_sync(0xffffffffu, aofs, rloc);
    const int nr = __shfl_sync(0xffffffffu, aofs, rloc + 1) - ra;
    double acc = 0.0;
    if (act) {
      acc = pr[lane * MAXR];
      for (int r = 1; r < nr; ++r) acc += pr[lane * MAXR + r];
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

// window headers of the push kernel: hdr[w] = {r0, wptr[r0], affptr[r0],
// head mask (bit wptr[r] - wptr[r0] for the rows r of the window)}, w in
// [0, nwin] (hdr[nwin] = the end sentinel)
__global__ void k_plan_push_hdr(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr,
                                const int32_t* __restrict__ rowstart, int64_t nwin, int64_t nF,
                                int4* __restrict__ hdr) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w <= nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r0 = w < nwin ? rowstart[w] : (int32_t)nF;
    const int32_t r1 = w < nwin ? rowstart[w + 1] : (int32_t)nF;
    int4 h;
    h.x = r0;
    h.y = (int32_t)wptr[r0];
    h.z = (int32_t)affptr[r0];
    uint32_t head = 0;
    for (int32_t r = r0; r < r1; ++r) head |= 1u << (unsigned)(wptr[r] - wptr[r0]);
    h.w = (int32_t)head;
    hdr[w] = h;
  }
}

__global__ void k_narrow_ptr(const int64_t* __restrict__ p, int64_t n, int32_t* __restrict__ out,
