// kernels_variants_tile.cuh -- the persistent TMA-pipelined tile kernel
// (EMIN_SPGEMM=pipe), an A/B variant measured slower than k_spgemm_win2
// (DESIGN.md §6).  Included by kernels_fast.cuh after the tile kernel.
#pragma once

// ---------------------------------------------------------------------------
// Persistent, TMA-pipelined variant of the tile kernel (MM_ITER, the hot
// launch).  Each CTA walks tiles t = blockIdx.x, +gridDim.x, ...; thread 0
// streams the NEXT tile's contiguous slices (A_FF records, the Q and y
// slices of its W entries, the wptr / affptr slices) into the other smem
// stage with cp.async.bulk (1D TMA, completion on an mbarrier) while the CTA
// computes the current tile.  Only the y(k, s) gathers remain as loads.
// ---------------------------------------------------------------------------
struct PipeLayout {     // byte offsets of one stage, and of the shared tail
  uint32_t rec, q, x, wp, ap, stage_bytes;
  uint32_t erow, qa, dot, bars, total;
};

__host__ __device__ inline uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }

__host__ __device__ inline PipeLayout pipe_layout(int rec_cap, int rows_cap) {
  PipeLayout L;
  L.rec = 0;
  L.q = align16(L.rec + (uint32_t)rec_cap * 16u);
  L.x = align16(L.q + (TILE_E + 2) * 8u);
  L.wp = align16(L.x + (TILE_E + 2) * 8u);
  L.ap = align16(L.wp + ((uint32_t)rows_cap + 3) * 8u);
  L.stage_bytes = align16(L.ap + ((uint32_t)rows_cap + 3) * 8u);
  L.erow = 2 * L.stage_bytes;
  L.qa = align16(L.erow + TILE_E * 2u);
  L.dot = align16(L.qa + TILE_E * 8u);
  L.bars = align16(L.dot + ((uint32_t)rows_cap + 1) * 8u);
  L.total = L.bars + 16u;
  return L;
}

// issue the bulk copies of tile h into stage buffer sb (thread 0 only);
// 8-byte slices are copied from the 16-byte aligned element below their start
__device__ __forceinline__ void pipe_issue(const TileHdr& h, unsigned char* sb, const PipeLayout& L,
                                           const SpEnt* __restrict__ A, const double* __restrict__ Q,
                                           const double* __restrict__ X, const int64_t* __restrict__ wptr,
                                           const int64_t* __restrict__ affptr, uint64_t* bar) {
  const int64_t nrec = h.aend - h.abase;
  const int64_t e0 = h.base & ~1LL, e1 = (h.end + 1) & ~1LL;        // [e0, e1) even-aligned
  const int64_t r0 = h.r0 & ~1LL, r1 = (h.r1 + 2) & ~1LL;           // rows [r0, r1) cover r0..r1
  const uint32_t bytes = (uint32_t)(nrec * 16 + 2 * (e1 - e0) * 8 + 2 * (r1 - r0) * 8);
  mbar_expect_tx(bar, bytes);
  if (nrec) bulk_g2s(sb + L.rec, A + h.abase, (uint32_t)(nrec * 16), bar);
  bulk_g2s(sb + L.q, Q + e0, (uint32_t)((e1 - e0) * 8), bar);
  bulk_g2s(sb + L.x, X + e0, (uint32_t)((e1 - e0) * 8), bar);
  bulk_g2s(sb + L.wp, wptr + r0, (uint32_t)((r1 - r0) * 8), bar);
  bulk_g2s(sb + L.ap, affptr + r0, (uint32_t)((r1 - r0) * 8), bar);
}

__global__ void __launch_bounds__(TILE_T)
k_spgemm_pipe(DevView v, const SpEnt* __restrict__ A, const TileHdr* __restrict__ hdr, int64_t ntiles,
              int rec_cap, int rows_cap, const double* __restrict__ X, double* __restrict__ out,
              double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double sh[32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const PipeLayout L = pipe_layout(rec_cap, rows_cap);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bars);
  uint16_t* s_erow = reinterpret_cast<uint16_t*>(smem_raw + L.erow);
  double* s_qa = reinterpret_cast<double*>(smem_raw + L.qa);
  double* s_dot = reinterpret_cast<double*>(smem_raw + L.dot);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t t = blockIdx.x;
  if (tid == 0 && t < ntiles) pipe_issue(hdr[t], smem_raw, L, A, v.Q, X, v.wptr, v.affptr, &bars[0]);
  double part = 0.0;
  for (int it = 0; t < ntiles; ++it, t += gridDim.x) {
    const int st = it & 1;
    unsigned char* sb = smem_raw + st * L.stage_bytes;
    const TileHdr H = hdr[t];
    // prefetch the next tile into the other stage (its last readers passed
    // the __syncthreads that ended the previous iteration)
    if (tid == 0 && t + gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      pipe_issue(hdr[t + gridDim.x], smem_raw + (st ^ 1) * L.stage_bytes, L, A, v.Q, X, v.wptr, v.affptr,
                 &bars[st ^ 1]);
    }
    mbar_wait(&bars[st], (uint32_t)((it >> 1) & 1));
    const SpEnt* s_rec = reinterpret_cast<const SpEnt*>(sb + L.rec);
    const double* s_q = reinterpret_cast<const double*>(sb + L.q) + (H.base & 1);
    const double* s_x = reinterpret_cast<const double*>(sb + L.x) + (H.base & 1);
    const int64_t* s_wp = reinterpret_cast<const int64_t*>(sb + L.wp) + (H.r0 & 1);
    const int64_t* s_ap = reinterpret_cast<const int64_t*>(sb + L.ap) + (H.r0 & 1);
    const int nrows = H.r1 - H.r0;
    const int nent = (int)(H.end - H.base);
    for (int r = tid; r < nrows; r += TILE_T) {
      const int pb = (int)(s_wp[r] - H.base), pe = (int)(s_wp[r + 1] - H.base);
      for (int p = pb; p < pe; ++p) s_erow[p] = (uint16_t)r;
    }
    __syncthreads();
    double g[TILE_U], qv[TILE_U];
    int rl[TILE_U];
#pragma unroll
    for (int u = 0; u < TILE_U; ++u) {
      const int e = tid + u * TILE_T;
      g[u] = 0.0;
      qv[u] = 0.0;
      rl[u] = 0;
      if (e < nent) {
        const int r = s_erow[e];
        rl[u] = r;
        qv[u] = s_q[e];
        const unsigned sh4 = 4u * (unsigned)(e - (int)(s_wp[r] - H.base));
        const int q0 = (int)(s_ap[r] - H.abase), q1 = (int)(s_ap[r + 1] - H.abase);
        double acc = 0.0;
#pragma unroll 4
        for (int q = q0; q < q1; ++q) {
          const SpEnt en = s_rec[q];
          const unsigned s = (en.pm >> sh4) & 0xFu;
          if (s != 0xFu) acc = fma(en.a, X[(int64_t)en.ybase + s], acc);
        }
        g[u] = acc;
      }
    }
    // Pi_B (nv = 1): g - q (q . g) per row, fixed-order row sums
#pragma unroll
    for (int u = 0; u < TILE_U; ++u) {
      const int e = tid + u * TILE_T;
      if (e < nent) s_qa[e] = qv[u] * g[u];
    }
    __syncthreads();
    for (int r = tid; r < nrows; r += TILE_T) {
      const int pb = (int)(s_wp[r] - H.base), pe = (int)(s_wp[r + 1] - H.base);
      double s = 0.0;
      for (int p = pb; p < pe; ++p) s += s_qa[p];
      s_dot[r] = s;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < TILE_U; ++u) {
      const int e = tid + u * TILE_T;
      if (e < nent) {
        const double o = g[u] - qv[u] * s_dot[rl[u]];
        out[H.base + e] = o;
        part = fma(s_x[e], o, part);
      }
    }
    __syncthreads();   // stage st and the shared tail are free again
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

