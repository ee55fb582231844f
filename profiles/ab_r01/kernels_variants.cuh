// kernels_variants.cuh -- alternative per-iteration masked-SpGEMM kernels of
// the scalar path, selectable with EMIN_SPGEMM for A/B runs
// (profiles/spgemm_variants.py) and parity-tested against the generic kernel
// (tests/test_gpu_parity.py::test_kernel_paths_agree).  All were measured
// slower than the default k_spgemm_win2 on config 3 (DESIGN.md §6 table,
// profiles/r01b/spgemm_ab_c3.txt); they stay as the record of what the
// latency / register / instruction trade-off of this kernel looks like.
// Included by kernels_fast.cuh after the shared helpers.
#pragma once

// per W entry: bit q set if record q of the entry's A_FF row matches the
// entry's column (setup; thread per row, rows with <= 16 A_FF entries)
__global__ void k_plan_emask(DevView v, const SpEnt* __restrict__ A, uint16_t* __restrict__ emask, int32_t* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v.nF; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = v.wptr[i];
    const int nj = (int)(v.wptr[i + 1] - b);
    const int64_t qb = v.affptr[i];
    const int nq = (int)(v.affptr[i + 1] - qb);
    if (nq > 16) atomicExch(bad, 1);
    for (int t = 0; t < nj; ++t) {
      uint32_t m = 0;
      for (int q = 0; q < nq && q < 16; ++q)
        if (((A[qb + q].pm >> (4 * t)) & 0xFu) != 0xFu) m |= 1u << q;
      emask[b + t] = (uint16_t)m;
    }
  }
}

// y^ = Pi K y (nv = 1): window headers (ALU decode), per-entry match masks
// (only the ~3.5 matching records of the row are visited, in A order, four
// loads in flight), row sums of q.g through shared memory (fixed order, no
// shuffles).
__global__ void __launch_bounds__(256, 8)
k_spgemm_mask(DevView v, const SpEnt* __restrict__ A, const WinHdr* __restrict__ hdr, int64_t nwin,
              const uint16_t* __restrict__ emask, const double* __restrict__ X, double* __restrict__ out,
              double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  const int4* H4 = reinterpret_cast<const int4*>(hdr);
  int4 hv = (w < nwin) ? H4[w] : make_int4(0, 0, 0, 0);
  while (w < nwin) {
    const int64_t wn = w + nw;
    const int4 hn = (wn < nwin) ? H4[wn] : make_int4(0, 0, 0, 0);
    if (hv.w > 0) {                                   // warp-uniform
      WinHdr h;
      h.r0 = hv.x; h.base = hv.y; h.head = (uint32_t)hv.z; h.nent = hv.w;
      const WinLane L = decode_hdr(h, lane);
      const int64_t i = (int64_t)h.r0 + L.rloc;
      const int64_t e = (int64_t)h.base + lane;
      const int64_t qb = v.affptr[i];
      uint32_t mask = L.act ? emask[e] : 0u;
      const double qv = L.act ? v.Q[e] : 0.0;
      const double xo = L.act ? X[e] : 0.0;
      const unsigned sh4 = 4u * (unsigned)(L.pos & 7);
      double acc = 0.0;
      while (mask) {
        int qa[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          qa[u] = mask ? __ffs(mask) - 1 : -1;
          mask &= mask - 1u;
        }
        SpEnt en[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (qa[u] >= 0) en[u] = A[qb + qa[u]];
        double yv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (qa[u] >= 0) yv[u] = X[(int64_t)en[u].ybase + ((en[u].pm >> sh4) & 0xFu)];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (qa[u] >= 0) acc = fma(en[u].a, yv[u], acc);
      }
      // Pi_B (nv = 1): row sum of q.g in a fixed order through shared memory
      s_qa[wib][lane] = qv * acc;
      __syncwarp();
      double dot = 0.0;
      for (int p = 0; p < L.rowlen; ++p) dot += s_qa[wib][L.rowbeg + p];
      __syncwarp();
      if (L.act) {
        const double g = acc - qv * dot;
        out[e] = g;
        part = fma(xo, g, part);
      }
    }
    hv = hn;
    w = wn;
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}


// win3: windows of up to 64 entries (two per lane: positions lane and
// lane + 32), so the per-window decode is amortised over twice the entries
// and every lane has two independent gather chains in flight.  Rows per
// window <= 63; head mask 64-bit.
__global__ void __launch_bounds__(256)
k_spgemm_win3(DevView v, const SpEnt* __restrict__ A, const int32_t* __restrict__ rowstart, int64_t nwin,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][64];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part = 0.0;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int r0 = rowstart[w];
    const int nrows = rowstart[w + 1] - r0;
    if (nrows == 0) continue;                          // warp-uniform
    const int p0 = (lane <= nrows) ? (int)v.wptr[r0 + lane] : 0;
    const int p1 = (lane + 32 <= nrows) ? (int)v.wptr[r0 + lane + 32] : 0;
    const int base = __shfl_sync(0xffffffffu, p0, 0);
    const int endp = (nrows < 32) ? __shfl_sync(0xffffffffu, p0, nrows) : __shfl_sync(0xffffffffu, p1, nrows - 32);
    const int nent = endp - base;
    const unsigned h0 = __reduce_or_sync(0xffffffffu, (lane < nrows && p0 - base < 32) ? (1u << (unsigned)(p0 - base)) : 0u) |
                        __reduce_or_sync(0xffffffffu, (lane + 32 < nrows && p1 - base < 32) ? (1u << (unsigned)(p1 - base)) : 0u);
    const unsigned h1 = __reduce_or_sync(0xffffffffu, (lane < nrows && p0 - base >= 32) ? (1u << (unsigned)(p0 - base - 32)) : 0u) |
                        __reduce_or_sync(0xffffffffu, (lane + 32 < nrows && p1 - base >= 32) ? (1u << (unsigned)(p1 - base - 32)) : 0u);
    const uint64_t H = ((uint64_t)h1 << 32) | h0;
    double acc[2], qv[2], xo[2];
    int rb[2], rl[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = lane + 32 * u;
      const bool act = t < nent;
      const int l = act ? t : nent - 1;
      const uint64_t upto = (l == 63) ? ~0ull : ((2ull << l) - 1ull);
      const uint64_t hu = H & upto;
      const int rloc = __popcll(hu) - 1;
      rb[u] = 63 - __clzll(hu);
      const uint64_t after = H & ~upto;
      rl[u] = (after ? (__ffsll(after) - 1) : nent) - rb[u];
      const int pos = t - rb[u];
      const int i = r0 + rloc;
      const int e = base + t;
      qv[u] = act ? v.Q[e] : 0.0;
      xo[u] = act ? X[e] : 0.0;
      acc[u] = 0.0;
      if (act) {
        const int qb = (int)v.affptr[i], qe = (int)v.affptr[i + 1];
        const unsigned sh4 = 4u * (unsigned)pos;
        double a = 0.0;
#pragma unroll 4
        for (int q = qb; q < qe; ++q) {
          const SpEnt en = A[q];
          const unsigned s = (en.pm >> sh4) & 0xFu;
          if (s != 0xFu) a = fma(en.a, X[en.ybase + (int)s], a);
        }
        acc[u] = a;
      }
      s_qa[wib][t] = qv[u] * acc[u];
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = lane + 32 * u;
      double dot = 0.0;
      for (int p = 0; p < rl[u]; ++p) dot += s_qa[wib][rb[u] + p];
      if (t < nent) {
        const double g = acc[u] - qv[u] * dot;
        out[base + t] = g;
        part = fma(xo[u], g, part);
      }
    }
    __syncwarp();
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

// ---------------------------------------------------------------------------
// win4 / win5: the window kernel without a dependent-load chain.
//
// win2 walks rowstart[w] -> wptr[r0..] -> affptr[i] -> A records -> y: four
// dependent DRAM round trips before the first gather, ~28 times per warp,
// which (not bandwidth) bounds it (profiles/r01: 52 % issue-active, DRAM at
// 44 % of peak).  Here a 32-byte header per window (built once at setup)
// holds everything the lane decode needs, so after the header every load
// of the window -- its A records (one coalesced 16-byte load per lane,
// staged in shared memory), the lanes' Q and y entries, the row pointers --
// is independent, and only the y gathers depend on the records.  PIPE
// additionally issues the next window's loads (and the header after it)
// before the current window's gathers.
// Arithmetic and summation order are those of win2 (bitwise equal).
// ---------------------------------------------------------------------------
struct Win4Hdr {
  int32_t r0, ebase, abase;
  uint32_t ehead;            // bit p: a row starts at window entry p
  int32_t nent, nrows, nrec, pad;
};
constexpr int W4_REC = 64;   // records staged per pass (2 per lane)

__global__ void k_plan_win4(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr,
                            const int32_t* __restrict__ rowstart, int64_t nwin, Win4Hdr* __restrict__ hdr) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r0 = rowstart[w], r1 = rowstart[w + 1];
    Win4Hdr h;
    h.r0 = r0;
    h.nrows = r1 - r0;
    h.ebase = (int32_t)(r1 > r0 ? wptr[r0] : 0);
    h.nent = (int32_t)(r1 > r0 ? wptr[r1] - wptr[r0] : 0);
    h.abase = (int32_t)(r1 > r0 ? affptr[r0] : 0);
    h.nrec = (int32_t)(r1 > r0 ? affptr[r1] - affptr[r0] : 0);
    uint32_t head = 0;
    for (int32_t r = r0; r < r1; ++r) head |= 1u << (unsigned)(wptr[r] - h.ebase);
    h.ehead = head;
    h.pad = 0;
    hdr[w] = h;
  }
}

struct Win4Loads {
  int4 ra, rb;     // records abase + lane, abase + 32 + lane (first pass)
  double qv, xo;   // Q and y of the lane's entry
  int ap;          // affptr[r0 + lane] - abase (lanes 0..nrows)
};

__device__ __forceinline__ Win4Loads win4_issue(const DevView& v, const int4* __restrict__ A4,
                                                const double* __restrict__ X, const Win4Hdr& h, int lane) {
  Win4Loads L;
  const int4 z4 = make_int4(0, 0, 0, 0);
  L.ra = lane < h.nrec ? __ldg(A4 + h.abase + lane) : z4;
  L.rb = lane + 32 < h.nrec ? __ldg(A4 + h.abase + 32 + lane) : z4;
  const bool act = lane < h.nent;
  L.qv = act ? __ldg(v.Q + h.ebase + lane) : 0.0;
  L.xo = act ? X[h.ebase + lane] : 0.0;
  L.ap = lane <= h.nrows ? (int)(__ldg(v.affptr + h.r0 + lane) - h.abase) : 0;
  return L;
}

template <bool PIPE>
__global__ void __launch_bounds__(256, PIPE ? 3 : 4)
k_spgemm_win4(DevView v, const int4* __restrict__ A4, const Win4Hdr* __restrict__ hdr, int64_t nwin,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  __shared__ int4 s_rec[8][W4_REC];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  // grid-stride over windows: all warps sweep one narrow front of rows, so
  // the y rows a window gathers were touched by its neighbours moments ago
  // (L2 hits); a contiguous run of windows per warp spreads the front over
  // the whole matrix and measured 1.6x slower.
  const Win4Hdr hz = {0, 0, 0, 0u, 0, 0, 0, 0};
  Win4Hdr h = w < nwin ? hdr[w] : hz;
  Win4Hdr hn = (PIPE && w + nw < nwin) ? hdr[w + nw] : hz;
  Win4Loads cur = win4_issue(v, A4, X, h, lane);
  while (w < nwin) {
    Win4Loads nxt;
    Win4Hdr hnn = hz;
    if (PIPE) {
      if (w + nw < nwin) nxt = win4_issue(v, A4, X, hn, lane);
      if (w + 2 * nw < nwin) hnn = hdr[w + 2 * nw];
    }
    const int nent = h.nent, nrows = h.nrows, nrec = h.nrec;
    if (nrows > 0) {                                   // warp-uniform
      const unsigned H = h.ehead;
      const bool act = lane < nent;
      const int l = act ? lane : nent - 1;
      const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
      const unsigned hu = H & upto;
      const int rloc = __popc(hu) - 1;
      const int rowbeg = 31 - __clz(hu);
      const unsigned after = H & ~upto;
      const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
      const unsigned sh4 = 4u * (unsigned)(lane - rowbeg);
      const int qb = __shfl_sync(0xffffffffu, cur.ap, rloc);
      const int qe = __shfl_sync(0xffffffffu, cur.ap, rloc + 1);
      double acc = 0.0;
      for (int p0 = 0; p0 < nrec; p0 += W4_REC) {      // warp-uniform; one pass unless nrec > 64
        if (p0 > 0) {
          __syncwarp();
          const int4 z4 = make_int4(0, 0, 0, 0);
          cur.ra = p0 + lane < nrec ? __ldg(A4 + h.abase + p0 + lane) : z4;
          cur.rb = p0 + 32 + lane < nrec ? __ldg(A4 + h.abase + p0 + 32 + lane) : z4;
        }
        s_rec[wib][lane] = cur.ra;
        s_rec[wib][lane + 32] = cur.rb;
        __syncwarp();
        if (act) {
          int lo = max(qb, p0);
          const int hi = min(qe, p0 + W4_REC);
          if (lo == qb && lo < hi) {
            // record qb is the diagonal A(i,i) (k_plan_entries): own y
            const int4 en = s_rec[wib][qb - p0];
            acc = __hiloint2double(en.y, en.x) * cur.xo;
            ++lo;
          }
#pragma unroll 4
          for (int q = lo; q < hi; ++q) {
            const int4 en = s_rec[wib][q - p0];         // {a (lo, hi), ybase, pm}
            const unsigned sidx = ((unsigned)en.w >> sh4) & 0xFu;
            if (sidx != 0xFu) acc = fma(__hiloint2double(en.y, en.x), X[en.z + (int)sidx], acc);
          }
        }
      }
      s_qa[wib][lane] = cur.qv * acc;
      __syncwarp();
      double dot = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p)                       // |J_i| <= 8 on the scalar path
        if (p < rowlen) dot += s_qa[wib][rowbeg + p];
      __syncwarp();
      if (act) {
        const double g = acc - cur.qv * dot;
        out[h.ebase + lane] = g;
        part = fma(cur.xo, g, part);
      }
    }
    w += nw;
    if (PIPE) {
      h = hn;
      hn = hnn;
      cur = nxt;
    } else if (w < nwin) {
      h = hdr[w];
      cur = win4_issue(v, A4, X, h, lane);
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

// ---------------------------------------------------------------------------
// win6: win2's lane map and arithmetic, with the next window's data pulled
// into L2 while the current window computes.
//
// win2 is latency bound (profiles/r01: 27 of 35 stall cycles per issued
// instruction are long-scoreboard waits at 99 % occupancy): per window it
// walks rowstart -> wptr -> affptr -> records -> y, four dependent DRAM
// misses and one L2 hit.  Here a 16-byte header per window {r0, abase,
// ebase, ehead} (nrows, nrec, nent are differences with the next header,
// so lanes 0 and 1 load both in one 32-byte access) replaces the first two
// steps, and the warp loads the header of its NEXT window one iteration
// ahead and issues prefetch.global.L2 for that window's row pointers,
// A records, Q and y entries before computing the current one.  The
// remaining chain -- affptr -> records -> y -- then runs on L2 hits.
// Registers stay at win2's level (no loads held across iterations).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pf_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// lanes [l0, l0 + nl) prefetch the 128-byte lines of [p, p + bytes), one each
__device__ __forceinline__ void pf_lines(const void* p, size_t bytes, int lane, int l0, int nl) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const int nlines = bytes ? (int)(((a + bytes - 1) >> 7) - (a >> 7)) + 1 : 0;
  const int j = lane - l0;
  if (j >= 0 && j < nl && j < nlines) pf_l2(reinterpret_cast<const void*>(((a >> 7) + j) << 7));
}

__global__ void k_plan_win6(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr,
                            const int32_t* __restrict__ rowstart, int64_t nwin, int4* __restrict__ hdr) {
  // hdr[w] for w in [0, nwin]; hdr[nwin] is the end sentinel
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w <= nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r0 = rowstart[w];
    const int32_t r1 = (w < nwin) ? rowstart[w + 1] : r0;
    uint32_t head = 0;
    for (int32_t r = r0; r < r1; ++r) head |= 1u << (unsigned)(wptr[r] - wptr[r0]);
    hdr[w] = make_int4(r0, (int32_t)affptr[r0], (int32_t)wptr[r0], (int32_t)head);
  }
}

__global__ void __launch_bounds__(256, 6)
k_spgemm_win6(DevView v, const int4* __restrict__ A4, const int4* __restrict__ hdr, int64_t nwin,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  // lanes 0 and 1 hold headers w and w + 1 of the current window
  int4 hc = (w < nwin && lane < 2) ? __ldg(hdr + w + lane) : make_int4(0, 0, 0, 0);
  while (w < nwin) {
    const int64_t wn = w + nw;
    // next window's header pair (consumed next iteration)
    const int4 hn = (wn < nwin && lane < 2) ? __ldg(hdr + wn + lane) : make_int4(0, 0, 0, 0);
    const int r0 = __shfl_sync(0xffffffffu, hc.x, 0);
    const int nrows = __shfl_sync(0xffffffffu, hc.x, 1) - r0;
    const int abase = __shfl_sync(0xffffffffu, hc.y, 0);
    const int base = __shfl_sync(0xffffffffu, hc.z, 0);
    const int nent = __shfl_sync(0xffffffffu, hc.z, 1) - base;
    const unsigned H = (unsigned)__shfl_sync(0xffffffffu, hc.w, 0);
    if (nrows > 0) {                                   // warp-uniform
      const bool act = lane < nent;
      const int l = act ? lane : nent - 1;
      const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
      const unsigned hu = H & upto;
      const int rloc = __popc(hu) - 1;
      const int rowbeg = 31 - __clz(hu);
      const unsigned after = H & ~upto;
      const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
      const int i = r0 + rloc;
      const int e = base + lane;
      const int qb = (int)v.affptr[i], qe = (int)v.affptr[i + 1];
      const double qv = act ? v.Q[e] : 0.0;
      const double xo = act ? X[e] : 0.0;
      (void)abase;
      double acc = 0.0;
      if (act) {
        acc = __hiloint2double(__ldg(&A4[qb]).y, __ldg(&A4[qb]).x) * xo;   // diagonal record first
        const unsigned sh4 = 4u * (unsigned)(lane - rowbeg);
#pragma unroll 4
        for (int q = qb + 1; q < qe; ++q) {
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
    // prefetch the next window into L2 (its header pair arrived meanwhile)
    if (wn < nwin) {
      const int nr0 = __shfl_sync(0xffffffffu, hn.x, 0);
      const int nr1 = __shfl_sync(0xffffffffu, hn.x, 1);
      const int nab = __shfl_sync(0xffffffffu, hn.y, 0);
      const int nae = __shfl_sync(0xffffffffu, hn.y, 1);
      const int neb = __shfl_sync(0xffffffffu, hn.z, 0);
      const int nee = __shfl_sync(0xffffffffu, hn.z, 1);
      if (nr1 > nr0) {
        // 128-byte lines of: records [nab, nae), Q and y [neb, nee), affptr [nr0, nr1]
        pf_lines(A4 + nab, (size_t)(nae - nab) * 16, lane, 0, 16);
        pf_lines(v.Q + neb, (size_t)(nee - neb) * 8, lane, 16, 4);
        pf_lines(X + neb, (size_t)(nee - neb) * 8, lane, 20, 4);
        pf_lines(v.affptr + nr0, (size_t)(nr1 - nr0 + 1) * 8, lane, 24, 4);
      }
    }
    hc = hn;
    w = wn;
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

// ---------------------------------------------------------------------------
// win7: ELL-padded A records.  Latency model of win2 (fits the measured
// 117 us on config 3 to 10 %): a warp spends ~8200 cycles per window, seven
// serialised memory round trips -- rowstart, wptr, affptr, two batches of
// records, two batches of y gathers.  Here
//  * row i's records sit at [W i, W i + W) (W = max A_FF row length <= 8,
//    padding records never match: pm = 0xFFFFFFFF, a = 0), so no affptr;
//  * a 16-byte window header {r0, ebase, ehead, nent}, loaded one window
//    ahead, replaces rowstart / wptr;
//  * all W records of the lane's row are loaded at once (full unroll), then
//    all its gathers,
// leaving two round trips per window (records, then y).  Same arithmetic and
// order as win2 (diagonal first, then A's column order).
// ---------------------------------------------------------------------------
__global__ void k_rowlen_max(const int64_t* __restrict__ ptr, int64_t n, int32_t* out) {
  int32_t m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int32_t)(ptr[i + 1] - ptr[i]));
  atomicMax(out, m);
}

__global__ void k_plan_ell(const int64_t* __restrict__ affptr, int64_t nF, int W, const int4* __restrict__ ent,
                           int4* __restrict__ ell) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nF * W; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / W;
    const int q = (int)(k - i * W);
    const int64_t qb = affptr[i], qe = affptr[i + 1];
    ell[k] = (qb + q < qe) ? ent[qb + q] : make_int4(0, 0, 0, (int)0xFFFFFFFFu);
  }
}

__global__ void k_plan_win7(const int64_t* __restrict__ wptr, const int32_t* __restrict__ rowstart, int64_t nwin,
                            int4* __restrict__ hdr) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r0 = rowstart[w], r1 = rowstart[w + 1];
    uint32_t head = 0;
    for (int32_t r = r0; r < r1; ++r) head |= 1u << (unsigned)(wptr[r] - wptr[r0]);
    hdr[w] = make_int4(r0, (int32_t)wptr[r0], (int32_t)head, (int32_t)(wptr[r1] - wptr[r0]));
  }
}

template <int W>
__global__ void __launch_bounds__(256, 4)
k_spgemm_win7(DevView v, const int4* __restrict__ ell, const int4* __restrict__ hdr, int64_t nwin,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  int4 h = w < nwin ? __ldg(hdr + w) : make_int4(0, 0, 0, 0);
  while (w < nwin) {
    const int64_t wn = w + nw;
    const int4 hn = wn < nwin ? __ldg(hdr + wn) : make_int4(0, 0, 0, 0);   // one window ahead
    const int nent = h.w;
    if (nent > 0) {                                     // warp-uniform
      const unsigned H = (unsigned)h.z;
      const bool act = lane < nent;
      const int l = act ? lane : nent - 1;
      const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
      const unsigned hu = H & upto;
      const int rloc = __popc(hu) - 1;
      const int rowbeg = 31 - __clz(hu);
      const unsigned after = H & ~upto;
      const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
      const int i = h.x + rloc;
      const int e = h.y + lane;
      const double qv = act ? v.Q[e] : 0.0;
      const double xo = act ? X[e] : 0.0;
      double acc = 0.0;
      if (act) {
        // three phases, so that no FMA waiting on a gather holds back the
        // next load (in-order issue): (1) the {ybase, pm} halves of the W
        // records, (2) all matching gathers, (3) the a halves (L1 hits: same
        // lines as phase 1) and the FMAs in A's order
        const int4* rec = ell + (int64_t)i * W;
        const unsigned sh4 = 4u * (unsigned)(lane - rowbeg);
        int yi[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) yi[q] = -1;
#pragma unroll
        for (int q = 1; q < W; ++q) {
          const int2 ip = __ldg(reinterpret_cast<const int2*>(rec + q) + 1);
          const unsigned s = ((unsigned)ip.y >> sh4) & 0xFu;
          yi[q] = (s != 0xFu) ? ip.x + (int)s : -1;
        }
        // scheduling fences (empty asm): every gather address waits for all
        // record loads, every FMA for all gathers -- ptxas otherwise places
        // each load just before its consumer, serialising the round trips
        asm volatile("" : "+r"(yi[1]), "+r"(yi[2]), "+r"(yi[3]), "+r"(yi[4]), "+r"(yi[5]), "+r"(yi[6]), "+r"(yi[7]));
        double yv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) yv[q] = 0.0;
#pragma unroll
        for (int q = 1; q < W; ++q) yv[q] = (yi[q] >= 0) ? __ldg(X + yi[q]) : 0.0;
        acc = __ldg(reinterpret_cast<const double*>(rec)) * xo;    // diagonal record first (own y)
        asm volatile("" : "+d"(acc) : "d"(yv[1]), "d"(yv[2]), "d"(yv[3]), "d"(yv[4]), "d"(yv[5]), "d"(yv[6]), "d"(yv[7]));
#pragma unroll
        for (int q = 1; q < W; ++q)
          if (yi[q] >= 0) acc = fma(__ldg(reinterpret_cast<const double*>(rec + q)), yv[q], acc);
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
    h = hn;
    w = wn;
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

// ---------------------------------------------------------------------------
// win8: per-warp double-buffered cp.async staging.
//
// Measured (profiles/r01b): win2 runs at 99 % occupancy but only ~1 KB of
// unique DRAM bytes in flight per SM-warp-window, because every lane holds
// its row's records in registers (a 32-lane broadcast load of 512 register
// bytes carries ~112 unique bytes); shortening the dependent chain in
// registers (win4/win7) cost the same factor in occupancy.  Here the window's
// A records, its lanes' Q and y entries and its row pointers are copied by
// cp.async straight into shared memory -- no registers wait on them -- for
// the NEXT window while the current one computes from the other buffer.
// Per window the only exposed latency left is the y gathers (L2).
// Header pairs as win6 ({r0, abase, ebase, ehead}; counts are differences
// with the next header).  Arithmetic and order are win2's.
// ---------------------------------------------------------------------------
constexpr int W8_REC = 96;      // records staged per window (more: read from global)
constexpr int W8_WARPS = 8;
struct W8Buf {
  int4 rec[W8_REC];
  double q[32];
  double x[32];
  int64_t ap[33];
  int64_t pad;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// header pair {r0, abase, ebase, ehead} of window w (lane 0) and w + 1 (lane 1)
struct W8Win {
  int r0, nrows, abase, nrec, ebase, nent;
  unsigned head;
};
__device__ __forceinline__ W8Win w8_decode(int4 hp) {
  W8Win d;
  d.r0 = __shfl_sync(0xffffffffu, hp.x, 0);
  d.nrows = __shfl_sync(0xffffffffu, hp.x, 1) - d.r0;
  d.abase = __shfl_sync(0xffffffffu, hp.y, 0);
  d.nrec = __shfl_sync(0xffffffffu, hp.y, 1) - d.abase;
  d.ebase = __shfl_sync(0xffffffffu, hp.z, 0);
  d.nent = __shfl_sync(0xffffffffu, hp.z, 1) - d.ebase;
  d.head = (unsigned)__shfl_sync(0xffffffffu, hp.w, 0);
  return d;
}
__device__ __forceinline__ void w8_issue(const W8Win& d, W8Buf* b, const DevView& v, const int4* __restrict__ A4,
                                         const double* __restrict__ X, int lane) {
  const int nr = min(d.nrec, W8_REC);
  for (int j = lane; j < nr; j += 32) cp_async16(&b->rec[j], A4 + d.abase + j);
  if (lane < d.nent) {
    cp_async8(&b->q[lane], v.Q + d.ebase + lane);
    cp_async8(&b->x[lane], X + d.ebase + lane);
  }
  if (lane <= d.nrows) cp_async8(&b->ap[lane], v.affptr + d.r0 + lane);
}

__global__ void __launch_bounds__(W8_WARPS * 32, 4)
k_spgemm_win8(DevView v, const int4* __restrict__ A4, const int4* __restrict__ hdr, int64_t nwin,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char w8_smem[];
  __shared__ double sh[32];
  __shared__ double s_qa[W8_WARPS][32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  W8Buf* bufs = reinterpret_cast<W8Buf*>(w8_smem) + 2 * wib;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  const int4 z4 = make_int4(0, 0, 0, 0);
  int4 hc = (w < nwin && lane < 2) ? __ldg(hdr + w + lane) : z4;
  int4 hn = (w + nw < nwin && lane < 2) ? __ldg(hdr + w + nw + lane) : z4;
  W8Win cur = w8_decode(hc);
  if (w < nwin) w8_issue(cur, &bufs[0], v, A4, X, lane);
  cp_async_commit();
  int bi = 0;
  while (w < nwin) {
    const int64_t wn = w + nw;
    const W8Win nxt = w8_decode(hn);
    if (wn < nwin) w8_issue(nxt, &bufs[bi ^ 1], v, A4, X, lane);
    cp_async_commit();
    const int4 hnn = (wn + nw < nwin && lane < 2) ? __ldg(hdr + wn + nw + lane) : z4;
    cp_async_wait<1>();                                // this window's group has landed
    __syncwarp();
    const W8Buf* b = &bufs[bi];
    if (cur.nrows > 0) {                               // warp-uniform
      const int nent = cur.nent;
      const unsigned H = cur.head;
      const bool act = lane < nent;
      const int l = act ? lane : nent - 1;
      const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
      const unsigned hu = H & upto;
      const int rloc = __popc(hu) - 1;
      const int rowbeg = 31 - __clz(hu);
      const unsigned after = H & ~upto;
      const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
      const double qv = act ? b->q[lane] : 0.0;
      const double xo = act ? b->x[lane] : 0.0;
      double acc = 0.0;
      if (act) {
        const int qb = (int)(b->ap[rloc] - cur.abase), qe = (int)(b->ap[rloc + 1] - cur.abase);
        const unsigned sh4 = 4u * (unsigned)(lane - rowbeg);
        if (qe <= W8_REC) {
          const int4 d0 = b->rec[qb];
          acc = __hiloint2double(d0.y, d0.x) * xo;     // diagonal record first (own y)
          // all gathers of a chunk are issued before the first FMA that
          // consumes one (in-order issue: an FMA waiting on its gather would
          // otherwise hold back the next gather -- one L2 round trip per
          // record, the measured bottleneck of win2/win8 v1)
          for (int q0 = qb + 1; q0 < qe; q0 += 8) {
            double yv[8];
            unsigned okm = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              // {ybase, pm} half of the record only (8-byte shared load)
              const int2 ip = reinterpret_cast<const int2*>(&b->rec[min(q0 + j, W8_REC - 1)])[1];
              const unsigned sidx = ((unsigned)ip.y >> sh4) & 0xFu;
              const bool ok = (q0 + j < qe) && sidx != 0xFu;
              okm |= ok ? (1u << j) : 0u;
              yv[j] = ok ? __ldg(X + ip.x + (int)sidx) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (okm & (1u << j))
                acc = fma(reinterpret_cast<const double*>(&b->rec[min(q0 + j, W8_REC - 1)])[0], yv[j], acc);
          }
        } else {                                        // records beyond the staged part
          const int4* g = A4 + cur.abase;
          const int4 d0 = __ldg(g + qb);
          acc = __hiloint2double(d0.y, d0.x) * xo;
          for (int q = qb + 1; q < qe; ++q) {
            const int4 en = __ldg(g + q);
            const unsigned s = ((unsigned)en.w >> sh4) & 0xFu;
            if (s != 0xFu) acc = fma(__hiloint2double(en.y, en.x), X[en.z + (int)s], acc);
          }
        }
      }
      s_qa[wib][lane] = qv * acc;
      __syncwarp();
      double dot = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < rowlen) dot += s_qa[wib][rowbeg + p];
      if (act) {
        const double g = acc - qv * dot;
        out[cur.ebase + lane] = g;
        part = fma(xo, g, part);
      }
    }
    __syncwarp();                                      // buffer bi is free for window w + 2 nw
    cur = nxt;
    hn = hnn;
    bi ^= 1;
    w = wn;
  }
  cp_async_wait<0>();
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}
static inline size_t w8_smem_bytes() { return sizeof(W8Buf) * 2 * W8_WARPS; }

// ---------------------------------------------------------------------------
// win9: win8 with the staging done by the bulk-copy (TMA) engine.  win8 cut
// the long-scoreboard stalls from 27 to 6.6 per issued instruction, but its
// per-lane cp.async code raised the instruction count 53 % (87 M vs 57 M on
// config 3).  Here one lane issues four cp.async.bulk copies per window
// (records; Q, y and affptr spans widened to 16-byte alignment -- every
// context array has 64 bytes of tail padding) on a per-warp mbarrier, and
// the gathers of a row are batched as in win8.
// ---------------------------------------------------------------------------
struct W9Buf {
  int4 rec[W8_REC];
  double q[34];
  double x[34];
  int64_t ap[34];
};

__global__ void __launch_bounds__(W8_WARPS * 32, 4)
k_spgemm_win9(DevView v, const int4* __restrict__ A4, const int4* __restrict__ hdr, int64_t nwin,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char w9_smem[];
  __shared__ double sh[32];
  __shared__ double s_qa[W8_WARPS][32];
  __shared__ __align__(8) uint64_t s_bar[W8_WARPS][2];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  W9Buf* bufs = reinterpret_cast<W9Buf*>(w9_smem) + 2 * wib;
  if (lane == 0) {
    mbar_init(&s_bar[wib][0], 1);
    mbar_init(&s_bar[wib][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  const int4 z4 = make_int4(0, 0, 0, 0);
  auto issue = [&](const W8Win& d, W9Buf* b, uint64_t* bar) {
    // lane 0 only
    const int nr = min(d.nrec, W8_REC);
    const int e0 = d.ebase & ~1, e1 = (d.ebase + d.nent + 1) & ~1;
    const int a0 = d.r0 & ~1, a1 = (d.r0 + d.nrows + 2) & ~1;
    const uint32_t bytes = (uint32_t)(nr * 16 + 2 * (e1 - e0) * 8 + (a1 - a0) * 8);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, bytes);
    if (nr) bulk_g2s(b->rec, A4 + d.abase, (uint32_t)(nr * 16), bar);
    bulk_g2s(b->q, v.Q + e0, (uint32_t)((e1 - e0) * 8), bar);
    bulk_g2s(b->x, X + e0, (uint32_t)((e1 - e0) * 8), bar);
    bulk_g2s(b->ap, v.affptr + a0, (uint32_t)((a1 - a0) * 8), bar);
  };
  int4 hc = (w < nwin && lane < 2) ? __ldg(hdr + w + lane) : z4;
  int4 hn = (w + nw < nwin && lane < 2) ? __ldg(hdr + w + nw + lane) : z4;
  W8Win cur = w8_decode(hc);
  if (w < nwin && lane == 0) issue(cur, &bufs[0], &s_bar[wib][0]);
  int it = 0;
  while (w < nwin) {
    const int bi = it & 1;
    const int64_t wn = w + nw;
    const W8Win nxt = w8_decode(hn);
    if (wn < nwin && lane == 0) issue(nxt, &bufs[bi ^ 1], &s_bar[wib][bi ^ 1]);
    const int4 hnn = (wn + nw < nwin && lane < 2) ? __ldg(hdr + wn + nw + lane) : z4;
    mbar_wait(&s_bar[wib][bi], (uint32_t)((it >> 1) & 1));
    const W9Buf* b = &bufs[bi];
    if (cur.nrows > 0) {                               // warp-uniform
      const int nent = cur.nent;
      const unsigned H = cur.head;
      const bool act = lane < nent;
      const int l = act ? lane : nent - 1;
      const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
      const unsigned hu = H & upto;
      const int rloc = __popc(hu) - 1;
      const int rowbeg = 31 - __clz(hu);
      const unsigned after = H & ~upto;
      const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
      const int es = cur.ebase & 1, as = cur.r0 & 1;
      const double qv = act ? b->q[es + lane] : 0.0;
      const double xo = act ? b->x[es + lane] : 0.0;
      double acc = 0.0;
      if (act) {
        const int qb = (int)(b->ap[as + rloc] - cur.abase), qe = (int)(b->ap[as + rloc + 1] - cur.abase);
        const unsigned sh4 = 4u * (unsigned)(lane - rowbeg);
        const int4* rec = (qe <= W8_REC) ? b->rec : A4 + cur.abase;   // beyond the staged part: global
        const int4 d0 = rec[qb];
        acc = __hiloint2double(d0.y, d0.x) * xo;       // diagonal record first (own y)
        for (int q0 = qb + 1; q0 < qe; q0 += 8) {
          double yv[8];
          unsigned okm = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int qq = min(q0 + j, qe - 1);
            const int2 ip = reinterpret_cast<const int2*>(&rec[qq])[1];
            const unsigned sidx = ((unsigned)ip.y >> sh4) & 0xFu;
            const bool ok = (q0 + j < qe) && sidx != 0xFu;
            okm |= ok ? (1u << j) : 0u;
            yv[j] = ok ? __ldg(X + ip.x + (int)sidx) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (okm & (1u << j)) acc = fma(reinterpret_cast<const double*>(&rec[q0 + j])[0], yv[j], acc);
        }
      }
      s_qa[wib][lane] = qv * acc;
      __syncwarp();
      double dot = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < rowlen) dot += s_qa[wib][rowbeg + p];
      if (act) {
        const double g = acc - qv * dot;
        out[cur.ebase + lane] = g;
        part = fma(xo, g, part);
      }
    }
    __syncwarp();                                      // buffer bi is free for window w + 2 nw
    cur = nxt;
    hn = hnn;
    ++it;
    w = wn;
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}
static inline size_t w9_smem_bytes() { return sizeof(W9Buf) * 2 * W8_WARPS; }

// ---------------------------------------------------------------------------
// win10: win2's lane map with the latency chain cut where it is cheap.
//  * a 32-byte window header (k_plan_win4) is loaded two windows ahead
//    (two warp-uniform 16-byte loads, no shuffles);
//  * lane 0 copies the NEXT window's A records and row pointers into a
//    per-warp shared buffer with cp.async.bulk on an mbarrier while the
//    current window computes (no registers wait on them);
//  * the lane's Q and y entries are plain coalesced loads;
//  * a row's gathers are issued together before its FMAs (fixed MAXR slots,
//    MAXR = longest A_FF row - 1), so they cost one L2 round trip, not one
//    per record.
// Order of the FMAs and of the row sums as win2 (diagonal first, then A's
// column order).
// ---------------------------------------------------------------------------
struct W10Buf {
  int4 rec[W8_REC];
  int64_t ap[36];
};

template <int MAXR>
__global__ void __launch_bounds__(W8_WARPS * 32)
k_spgemm_win10(DevView v, const int4* __restrict__ A4, const Win4Hdr* __restrict__ hdr, int64_t nwin,
               const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char w10_smem[];
  __shared__ double sh[32];
  __shared__ double s_qa[W8_WARPS][32];
  __shared__ __align__(8) uint64_t s_bar[W8_WARPS][2];
  if (v.st->stopped) return;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  W10Buf* bufs = reinterpret_cast<W10Buf*>(w10_smem) + 2 * wib;
  if (lane == 0) {
    mbar_init(&s_bar[wib][0], 1);
    mbar_init(&s_bar[wib][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  const int4* H4 = reinterpret_cast<const int4*>(hdr);
  const int4 z4 = make_int4(0, 0, 0, 0);
  auto issue = [&](int4 h0, int4 h1, W10Buf* b, uint64_t* bar) {   // lane 0 only
    // h0 = {r0, ebase, abase, ehead}, h1 = {nent, nrows, nrec, -}
    const int nr = min(h1.z, W8_REC);
    const int a0 = h0.x & ~1, a1 = (h0.x + h1.y + 2) & ~1;     // affptr[r0 .. r0 + nrows]
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)(nr * 16 + (a1 - a0) * 8));
    if (nr) bulk_g2s(b->rec, A4 + h0.z, (uint32_t)(nr * 16), bar);
    bulk_g2s(b->ap, v.affptr + a0, (uint32_t)((a1 - a0) * 8), bar);
  };
  int4 c0 = z4, c1 = z4, n0 = z4, n1 = z4;
  if (w < nwin) { c0 = __ldg(H4 + 2 * w); c1 = __ldg(H4 + 2 * w + 1); }
  if (w + nw < nwin) { n0 = __ldg(H4 + 2 * (w + nw)); n1 = __ldg(H4 + 2 * (w + nw) + 1); }
  if (w < nwin && lane == 0) issue(c0, c1, &bufs[0], &s_bar[wib][0]);
  int it = 0;
  while (w < nwin) {
    const int bi = it & 1;
    const int64_t wn = w + nw, wnn = w + 2 * nw;
    if (wn < nwin && lane == 0) issue(n0, n1, &bufs[bi ^ 1], &s_bar[wib][bi ^ 1]);
    int4 m0 = z4, m1 = z4;
    if (wnn < nwin) { m0 = __ldg(H4 + 2 * wnn); m1 = __ldg(H4 + 2 * wnn + 1); }
    const int nent = c1.x, nrows = c1.y;
    const bool act = lane < nent;
    const int e = c0.y + lane;
    const double qv = act ? __ldg(v.Q + e) : 0.0;
    const double xo = act ? X[e] : 0.0;
    mbar_wait(&s_bar[wib][bi], (uint32_t)((it >> 1) & 1));
    const W10Buf* b = &bufs[bi];
    if (nrows > 0) {                                   // warp-uniform
      const unsigned H = (unsigned)c0.w;
      const int l = act ? lane : nent - 1;
      const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
      const unsigned hu = H & upto;
      const int rloc = __popc(hu) - 1;
      const int rowbeg = 31 - __clz(hu);
      const unsigned after = H & ~upto;
      const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
      double acc = 0.0;
      if (act) {
        const int as = c0.x & 1;
        const int qb = (int)(b->ap[as + rloc] - c0.z), qe = (int)(b->ap[as + rloc + 1] - c0.z);
        const unsigned sh4 = 4u * (unsigned)(lane - rowbeg);
        const int4* rec = (qe <= W8_REC) ? b->rec : A4 + c0.z;   // beyond the staged part: global
        acc = reinterpret_cast<const double*>(rec + qb)[0] * xo;   // diagonal record first (own y)
        for (int q0 = qb + 1; q0 < qe; q0 += MAXR) {
          double yv[MAXR];
          unsigned okm = 0;
#pragma unroll
          for (int j = 0; j < MAXR; ++j) {
            const int qq = min(q0 + j, qe - 1);
            const int2 ip = reinterpret_cast<const int2*>(rec + qq)[1];
            const unsigned sidx = ((unsigned)ip.y >> sh4) & 0xFu;
            const bool ok = (q0 + j < qe) && sidx != 0xFu;
            okm |= ok ? (1u << j) : 0u;
            yv[j] = ok ? __ldg(X + ip.x + (int)sidx) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < MAXR; ++j)
            if (okm & (1u << j)) acc = fma(reinterpret_cast<const double*>(rec + q0 + j)[0], yv[j], acc);
        }
      }
      s_qa[wib][lane] = qv * acc;
      __syncwarp();
      double dot = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < rowlen) dot += s_qa[wib][rowbeg + p];
      if (act) {
        const double g = acc - qv * dot;
        out[e] = g;
        part = fma(xo, g, part);
      }
    }
    __syncwarp();                                      // buffer bi is free for window w + 2 nw
    c0 = n0; c1 = n1; n0 = m0; n1 = m1;
    ++it;
    w = wn;
  }
  const double tot = block_sum(part, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}
static inline size_t w10_smem_bytes() { return sizeof(W10Buf) * 2 * W8_WARPS; }

// y^ = Pi K y (nv = 1) on precomputed window headers, next header prefetched
__global__ void __launch_bounds__(256, 8)
k_spgemm_hdr(DevView v, const SpEnt* __restrict__ A, const WinHdr* __restrict__ hdr, int64_t nwin,
             const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double part = 0.0;
  // 32-bit indices throughout (the scalar path has nnz(W), nnz(A_FF) < 2^31)
  const int4* H4 = reinterpret_cast<const int4*>(hdr);
  int4 h = (w < nwin) ? H4[w] : make_int4(0, 0, 0, 0);
  while (w < nwin) {
    const int64_t wn = w + nw;
    const int4 hn = (wn < nwin) ? H4[wn] : make_int4(0, 0, 0, 0);
    if (h.w > 0) {                                    // warp-uniform
      WinHdr hh;
      hh.r0 = h.x; hh.base = h.y; hh.head = (uint32_t)h.z; hh.nent = h.w;
      const WinLane L = decode_hdr(hh, lane);
      const int i = h.x + L.rloc;
      const int e = h.y + lane;
      const int qb = (int)v.affptr[i], qe = (int)v.affptr[i + 1];
      const double qv = L.act ? v.Q[e] : 0.0;
      const double xo = L.act ? X[e] : 0.0;
      double acc = 0.0;
      if (L.act) {
        const unsigned sh4 = 4u * (unsigned)L.pos;
#pragma unroll 4
        for (int q = qb; q < qe; ++q) {
          const SpEnt en = A[q];
          const unsigned s = (en.pm >> sh4) & 0xFu;
          if (s != 0xFu) acc = fma(en.a, X[en.ybase + (int)s], acc);
        }
      }
      const double dot = row_sum(qv * acc, L);
      const double g = acc - qv * dot;
      if (L.act) {
        out[e] = g;
        part = fma(xo, g, part);
      }
    }
    h = hn;
    w = wn;
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}


