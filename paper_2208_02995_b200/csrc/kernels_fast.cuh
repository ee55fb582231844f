// kernels_fast.cuh -- specialised hot-path kernels selected at setup.
//
// Scalar path (kernel_path 1): nv = 1 and |J_i| <= 8 (configs 1-3).
//   Lane-per-W-entry.  The W entries are cut into windows of S = 33 - max|J|
//   consecutive entries; warp w owns the rows whose first entry lies in
//   window w, so a warp never holds more than 32 entries and rows never
//   straddle warps.  Each lane finds its row from a head bitmask
//   (__reduce_or_sync + popc), so all loads of W-layout vectors are
//   coalesced and every lane does useful work (S/32 on average).
//   The masked product uses a per-A_FF-entry record built once at setup
//   (the pattern is fixed, "the sparsity pattern ... can be
//   communicated only once"):  {a = A(i,k), ybase = wptr[k], pm}, where
//   nibble t of pm is the position of J_i[t] in J_k (0xF: absent).  So the
//   inner loop is one 16-byte broadcast load, a nibble extract and one
//   gather of y(k, s) -- no search.
// Per-iteration kernel: k_spgemm_win2 (default); setup / energy modes: the
// tile kernel (k_spgemm_tile, fused MM_R0E at setup).  The A/B variants
// (EMIN_SPGEMM=win|win3..win10|hdr|mask|pipe) live in kernels_variants*.cuh.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "emin_internal.cuh"
#include "masked.cuh"

struct SpEnt {          // 16 bytes, one per A_FF entry
  double a;
  int32_t ybase;
  uint32_t pm;
};

struct TileHdr;
struct ScalarPlan {
  SpEnt* ent = nullptr;
  int32_t* rowstart = nullptr;   // [nwin + 1]
  int64_t nwin = 0;
  int32_t S = 0;
  TileHdr* hdr = nullptr;        // [ntiles] (staged tile kernel)
  int64_t ntiles = 0;
  size_t tile_smem = 0;
  int use_tiles = 0;
  int use_pipe = 0, pipe_grid = 0, rec_cap = 0, rows_cap = 0;   // TMA-pipelined persistent kernel
  uint32_t pipe_smem = 0;
  struct WinHdr* whdr = nullptr; // [nwin] window headers
  int variant = 0;               // per-iteration kernel: 0 hdr, 1 win, 2 tile, 3 pipe, 4 mask
  uint16_t* emask = nullptr;     // [nnzW] matching records per W entry (variant 4)
  int32_t* rowstart3 = nullptr;  // 64-entry windows (variant 6)
  int64_t nwin3 = 0;
  struct Win4Hdr* w4hdr = nullptr; // [nwin] 32-byte window headers (variants 7, 8)
  int4* w6hdr = nullptr;           // [nwin + 1] 16-byte window headers (variant 9)
  int4* ell = nullptr;             // [nF * ellW] ELL-padded records (variant 10)
  int4* w7hdr = nullptr;           // [nwin] {r0, ebase, ehead, nent} (variant 10)
  int ellW = 0;
  int w8grid = 0;                  // resident CTAs of win8 (variant 11)
};

// ---- shared-memory / mbarrier / bulk-copy helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}


// decode the window: rows [r0, r1), base entry, this lane's row and position
struct WinLane {
  int64_t base;   // first W entry of the window
  int nent;       // entries in the window (<= 32)
  int rloc;       // lane's row within the window
  int pos;        // lane's position in its row
  int rowbeg;     // lane index of its row's first entry
  int rowlen;
  bool act;
};

__device__ __forceinline__ WinLane decode_window(const int64_t* __restrict__ wptr, int64_t r0, int nrows,
                                                 int lane) {
  WinLane w;
  const int64_t myptr = (lane <= nrows) ? wptr[r0 + lane] : 0;
  w.base = __shfl_sync(0xffffffffu, myptr, 0);
  const int64_t end = __shfl_sync(0xffffffffu, myptr, nrows);
  w.nent = (int)(end - w.base);
  const unsigned bit = (lane < nrows) ? (1u << (unsigned)(myptr - w.base)) : 0u;
  const unsigned H = __reduce_or_sync(0xffffffffu, bit);
  const unsigned upto = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
  int rl = __popc(H & upto) - 1;
  if (rl < 0) rl = 0;
  if (rl >= nrows) rl = nrows - 1;
  w.rloc = rl;
  const int64_t rb = __shfl_sync(0xffffffffu, myptr, rl);
  const int64_t re = __shfl_sync(0xffffffffu, myptr, rl + 1 <= nrows ? rl + 1 : nrows);
  w.rowbeg = (int)(rb - w.base);
  w.rowlen = (int)(re - rb);
  w.pos = lane - w.rowbeg;
  w.act = lane < w.nent;
  return w;
}

// forward declaration (defined below)
struct WinHdr;

// sum of v over the lane's row (segmented inclusive scan, then the row's
// last lane broadcasts); identical in every lane of the row
__device__ __forceinline__ double row_sum(double v, const WinLane& L) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (L.pos >= o) v += t;
  }
  return __shfl_sync(0xffffffffu, v, L.rowbeg + L.rowlen - 1);
}

// Precomputed window header (one 16-byte load per warp; the lane decode is
// pure ALU): first row, first entry, head bitmask (bit p set if a row starts
// at window position p), entry count.
struct WinHdr {
  int32_t r0;
  int32_t base;
  uint32_t head;
  int32_t nent;
};

__device__ __forceinline__ WinLane decode_hdr(const WinHdr& h, int lane) {
  WinLane w;
  w.base = h.base;
  w.nent = h.nent;
  const int l = lane < h.nent ? lane : h.nent - 1;    // inactive lanes mirror the last entry
  const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
  const unsigned hu = h.head & upto;
  w.rloc = __popc(hu) - 1;
  w.rowbeg = 31 - __clz(hu);
  const unsigned after = h.head & ~upto;
  const int rowend = after ? (__ffs(after) - 1) : h.nent;
  w.rowlen = rowend - w.rowbeg;
  w.pos = lane - w.rowbeg;
  w.act = lane < h.nent;
  return w;
}

__global__ void k_plan_headers(const int64_t* __restrict__ wptr, const int32_t* __restrict__ rowstart,
                               int64_t nwin, WinHdr* __restrict__ hdr) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r0 = rowstart[w], r1 = rowstart[w + 1];
    WinHdr h;
    h.r0 = r0;
    h.base = (int32_t)(r1 > r0 ? wptr[r0] : 0);
    h.nent = (int32_t)(r1 > r0 ? wptr[r1] - wptr[r0] : 0);
    uint32_t head = 0;
    for (int32_t r = r0; r < r1; ++r) head |= 1u << (unsigned)(wptr[r] - h.base);
    h.head = head;
    hdr[w] = h;
  }
}

// y^ = Pi K y (nv = 1), window kernel with fewer warp collectives: the
// window decode derives row starts / lengths from the head bitmask by bit
// arithmetic (2 shuffles + 1 OR-reduction), the row projection sums q.g
// through shared memory in a fixed order (no shuffle scan).
template <int GRP = 1>
__global__ void __launch_bounds__(256)
k_spgemm_win2(DevView v, const SpEnt* __restrict__ A, const int32_t* __restrict__ rowstart, int64_t nwin,
              const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  if (v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part = 0.0;
  const bool rev = v.pingpong && (v.st->k_total & 1);   // same direction as stage I (L2 ping-pong)
  for (int64_t w1 = gw; w1 < nwin; w1 += nw) {
    const int64_t w = rev ? nwin - 1 - w1 : w1;
    const int r0 = rowstart[w];
    const int nrows = rowstart[w + 1] - r0;
    if (nrows == 0) continue;                          // warp-uniform
    const int myptr = (lane <= nrows) ? (int)v.wptr[r0 + lane] : 0;
    const int base = __shfl_sync(0xffffffffu, myptr, 0);
    const int nent = __shfl_sync(0xffffffffu, myptr, nrows) - base;
    const unsigned H = __reduce_or_sync(0xffffffffu, (lane < nrows) ? (1u << (unsigned)(myptr - base)) : 0u);
    const bool act = lane < nent;
    const int l = act ? lane : nent - 1;
    const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
    const unsigned hu = H & upto;
    const int rloc = __popc(hu) - 1;
    const int rowbeg = 31 - __clz(hu);
    const unsigned after = H & ~upto;
    const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
    const int pos = lane - rowbeg;
    const int i = r0 + rloc;
    const int e = base + lane;
    const int qb = (int)v.affptr[i], qe = (int)v.affptr[i + 1];
    const double qv = act ? v.Q[e] : 0.0;
    const double xo = act ? X[e] : 0.0;
    double acc = 0.0;
    if (act) {
      // record qb is the diagonal A(i,i) (k_plan_entries): its y value is the
      // lane's own entry, no gather
      const int4* A4 = reinterpret_cast<const int4*>(A);
      acc = __hiloint2double(__ldg(&A4[qb]).y, __ldg(&A4[qb]).x) * xo;
      const unsigned sh4 = 4u * (unsigned)pos;
      int q = qb + 1;
      if (GRP > 1) {
        // GRP records per round: their gathers are issued before the FMAs
        // (same ascending order of the sum)
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
            if (m[g]) acc = fma(__hiloint2double(en[g].y, en[g].x), y[g], acc);
        }
      }
#pragma unroll 4
      for (; q < qe; ++q) {
        const int4 en = __ldg(&A4[q]);              // one 16-byte load: {a, ybase, pm}
        const unsigned s = ((unsigned)en.w >> sh4) & 0xFu;
        if (s != 0xFu) acc = fma(__hiloint2double(en.y, en.x), X[en.z + (int)s], acc);
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

// win2's setup / energy modes (same window decode and record loop):
//   MM_R0      r0 = -Pi Pi (A P0)|F, the C-identity term A(i, c_j) added  (A1/A2)
//   MM_ENERGY  partial W . (A_FF W + 2 A_FC), W = X + X2                  (Eq. trInc)
template <int MODE>
__global__ void __launch_bounds__(256)
k_spgemm_win2m(DevView v, const SpEnt* __restrict__ A, const int32_t* __restrict__ rowstart, int64_t nwin,
               const double* __restrict__ X, const double* __restrict__ X2, double* __restrict__ out,
               double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[8][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // MM_ENERGY: W = X + X2, or X alone when the caller summed it (X2 null)
  const bool two = MODE == MM_ENERGY && X2 != nullptr;
  auto xval = [&](int idx) -> double { return two ? X[idx] + X2[idx] : X[idx]; };
  double part = 0.0;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int r0 = rowstart[w];
    const int nrows = rowstart[w + 1] - r0;
    if (nrows == 0) continue;                          // warp-uniform
    const int myptr = (lane <= nrows) ? (int)v.wptr[r0 + lane] : 0;
    const int base = __shfl_sync(0xffffffffu, myptr, 0);
    const int nent = __shfl_sync(0xffffffffu, myptr, nrows) - base;
    const unsigned H = __reduce_or_sync(0xffffffffu, (lane < nrows) ? (1u << (unsigned)(myptr - base)) : 0u);
    const bool act = lane < nent;
    const int l = act ? lane : nent - 1;
    const unsigned upto = (l == 31) ? 0xffffffffu : ((2u << l) - 1u);
    const unsigned hu = H & upto;
    const int rloc = __popc(hu) - 1;
    const int rowbeg = 31 - __clz(hu);
    const unsigned after = H & ~upto;
    const int rowlen = (after ? (__ffs(after) - 1) : nent) - rowbeg;
    const int pos = lane - rowbeg;
    const int i = r0 + rloc;
    const int e = base + lane;
    const double xo = act ? xval(e) : 0.0;
    double acc = 0.0, fc = 0.0;
    if (act) {
      const int qb = (int)v.affptr[i], qe = (int)v.affptr[i + 1];
      const int4* A4 = reinterpret_cast<const int4*>(A);
      acc = __hiloint2double(__ldg(&A4[qb]).y, __ldg(&A4[qb]).x) * xo;   // diagonal record first
      const unsigned sh4 = 4u * (unsigned)pos;
#pragma unroll 4
      for (int q = qb + 1; q < qe; ++q) {
        const int4 en = __ldg(&A4[q]);
        const unsigned sidx = ((unsigned)en.w >> sh4) & 0xFu;
        if (sidx != 0xFu) acc = fma(__hiloint2double(en.y, en.x), xval(en.z + (int)sidx), acc);
      }
      const int32_t j = v.wcol[e];                    // A(i, c_j): search the short A_FC row
      for (int64_t q = v.afcptr[i]; q < v.afcptr[i + 1]; ++q)
        if (v.afccol[q] == j) { fc = v.afcval[q]; break; }
    }
    if (MODE == MM_ENERGY) {
      if (act) part = fma(xo, acc + 2.0 * fc, part);
      continue;                                       // warp-uniform (MODE)
    }
    const double qv = act ? v.Q[e] : 0.0;
    double g = acc + fc;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {            // Pi applied twice (reading A2)
      s_qa[wib][lane] = qv * g;
      __syncwarp();
      double dot = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < rowlen) dot += s_qa[wib][rowbeg + p];
      __syncwarp();
      g = g - qv * dot;
    }
    if (act) out[e] = -g;
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, -1);
}

#include "kernels_variants.cuh"

// Masked product on the scalar path, modes as in masked.cuh:
//   MM_ITER    yb = Pi K y, partial y . yb
//   MM_R0      r0 = -Pi Pi (A P0)|F (C-identity term included)    (A1)
//   MM_ENERGY  partial W . (A_FF W + 2 A_FC), W = X + X2          (Eq. trInc)
template <int MODE>
__global__ void __launch_bounds__(256)
k_spgemm_scalar(DevView v, const SpEnt* __restrict__ A, const int32_t* __restrict__ rowstart, int64_t nwin,
                const double* __restrict__ X, const double* __restrict__ X2, double* __restrict__ out,
                double* __restrict__ partials) {
  __shared__ double sh[32];
  if (MODE == MM_ITER && v.st->stopped) { iter_stopped(v); return; }
  const bool two = MODE == MM_ENERGY && X2 != nullptr;      // (X2 null: X is already W)
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part = 0.0;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int64_t r0 = rowstart[w];
    const int nrows = (int)(rowstart[w + 1] - r0);
    if (nrows == 0) continue;                          // warp-uniform
    const WinLane L = decode_window(v.wptr, r0, nrows, lane);
    const int64_t i = r0 + L.rloc;
    const int64_t e = L.base + lane;
    double acc = 0.0, fc = 0.0;
    if (L.act) {
      const int64_t qb = v.affptr[i], qe = v.affptr[i + 1];
      const unsigned sh4 = 4u * (unsigned)L.pos;
      for (int64_t q = qb; q < qe; ++q) {
        const SpEnt en = A[q];
        const unsigned s = (en.pm >> sh4) & 0xFu;
        if (s != 0xFu) {
          const int64_t src = (int64_t)en.ybase + s;
          const double xv = two ? X[src] + X2[src] : X[src];
          acc = fma(en.a, xv, acc);
        }
      }
      if (MODE != MM_ITER) {            // A(i, c_j): search the short A_FC row
        const int32_t j = v.wcol[e];
        for (int64_t q = v.afcptr[i]; q < v.afcptr[i + 1]; ++q)
          if (v.afccol[q] == j) { fc = v.afcval[q]; break; }
      }
    }
    if (MODE == MM_ENERGY) {
      if (L.act) part += (two ? X[e] + X2[e] : X[e]) * (acc + 2.0 * fc);
      continue;
    }
    // Pi_B, nv = 1: g - q (q . g) over the row
    const double qv = L.act ? v.Q[e] : 0.0;
    double g = (MODE == MM_R0) ? acc + fc : acc;
#pragma unroll
    for (int pass = 0; pass < (MODE == MM_R0 ? 2 : 1); ++pass) {
      const double dot = row_sum(qv * g, L);
      g = g - qv * dot;
    }
    if (L.act) {
      if (MODE == MM_ITER) {
        out[e] = g;
        part = fma(X[e], g, part);
      } else {
        out[e] = -g;
      }
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, MODE == MM_ITER ? 1 : -1);
}

// Alg. 2 for nv = 1 on the window plan (the CGS2 QR of k_alg2 reduces to
// q = M / |M|, delta = q (r / |M|); |M| = 0 is the rank-0 SVD branch)
__global__ void __launch_bounds__(256)
k_alg2_nv1(DevView v, const int32_t* __restrict__ rowstart, int64_t nwin, const double* __restrict__ Bc,
           const double* __restrict__ B, const int64_t* __restrict__ frow, const double* __restrict__ what,
           double* __restrict__ Qout, double* __restrict__ w0, unsigned long long* counters) {
  __shared__ unsigned long long cnt[2];
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned n_svd = 0, n_frozen = 0;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int64_t r0 = rowstart[w];
    const int nrows = (int)(rowstart[w + 1] - r0);
    if (nrows == 0) continue;
    const WinLane L = decode_window(v.wptr, r0, nrows, lane);
    const int64_t e = L.base + lane;
    const int64_t i = r0 + L.rloc;
    const double m = L.act ? Bc[v.wcol[e]] : 0.0;
    const double wh = L.act ? what[e] : 0.0;
    const double smm = row_sum(m * m, L);
    const double smw = row_sum(m * wh, L);
    if (L.act) {
      const double rv = B[frow[i]] - smw;
      const double R = sqrt(smm);
      double q = 0.0, delta = 0.0;
      int k = 0;
      if (R > 0.0) {
        q = m / R;
        delta = q * (rv / R);
        k = 1;
      }
      Qout[e] = q;
      w0[e] = wh + delta;
      if (L.pos == 0) {
        n_svd += (k == 0);
        n_frozen += (L.rowlen == k);
      }
    }
  }
  atomicAdd(&cnt[0], (unsigned long long)n_svd);
  atomicAdd(&cnt[1], (unsigned long long)n_frozen);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (cnt[0]) atomicAdd(counters + 0, cnt[0]);
    if (cnt[1]) atomicAdd(counters + 1, cnt[1]);
  }
}

// P out on the window plan
__global__ void __launch_bounds__(256)
k_get_P_win(DevView v, const int32_t* __restrict__ rowstart, int64_t nwin, const double* __restrict__ w0,
            const double* __restrict__ dw, const int64_t* __restrict__ pofs, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int64_t r0 = rowstart[w];
    const int nrows = (int)(rowstart[w + 1] - r0);
    if (nrows == 0) continue;
    const WinLane L = decode_window(v.wptr, r0, nrows, lane);
    if (L.act) {
      const int64_t e = L.base + lane;
      out[pofs[r0 + L.rloc] + L.pos] = w0[e] + dw[e];
    }
  }
}

// stage I on the window plan: r -= alpha_pend yb ; partial r . (r / d)
__global__ void __launch_bounds__(256)
k_stage1_win(DevView v, const int32_t* __restrict__ rowstart, int64_t nwin, double* __restrict__ r,
             const double* __restrict__ yb, double* __restrict__ partials) {
  __shared__ double sh[32];
  const DevState* st = v.st;
  if (st->stopped) return;
  const int pend = st->pend;
  const double ap = st->alpha_pend;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double part = 0.0;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int64_t r0 = rowstart[w];
    const int nrows = (int)(rowstart[w + 1] - r0);
    if (nrows == 0) continue;
    const WinLane L = decode_window(v.wptr, r0, nrows, lane);
    if (L.act) {
      const int64_t e = L.base + lane;
      const double di = v.d[r0 + L.rloc];
      double rv = r[e];
      if (pend) { rv = rv - ap * yb[e]; r[e] = rv; }
      const double z = rv / di;
      part = fma(rv, z, part);
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 0);
}

// stage II on the window plan: dw += alpha_pend y_old ; y = z + beta y_old
__global__ void __launch_bounds__(256)
k_stage2_win(DevView v, const int32_t* __restrict__ rowstart, int64_t nwin, const double* __restrict__ r,
             double* __restrict__ y, double* __restrict__ dw) {
  const DevState* st = v.st;
  const int stopped = st->stopped;
  const int pendw = st->pendw;
  if (stopped && !pendw) return;
  const double ap = st->alpha_pend;
  const double beta = st->beta;
  const bool first = (st->k_total == 0);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < nwin; w += nw) {
    const int64_t r0 = rowstart[w];
    const int nrows = (int)(rowstart[w + 1] - r0);
    if (nrows == 0) continue;
    const WinLane L = decode_window(v.wptr, r0, nrows, lane);
    if (L.act) {
      const int64_t e = L.base + lane;
      const double yo = y[e];
      if (pendw) dw[e] = dw[e] + ap * yo;
      if (!stopped) {
        const double z = r[e] / v.d[r0 + L.rloc];
        y[e] = first ? z : z + beta * yo;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Tiled variant: one CTA per tile of consecutive rows whose first entry lies
// in [t S_T, (t+1) S_T) (S_T = TILE_E - max|J| + 1, so a tile holds at most
// TILE_E entries).  Phase A stages the tile's contiguous slices -- the A_FF
// records [abase, aend), the row pointers -- into shared memory with
// coalesced 16-byte loads, and loads each thread's own Q and y entries into
// registers, all independent of one another (one round trip after the tile
// header).  Phase B does the masked product from shared memory; only the
// y(k, s) gathers go to L2/HBM.  The row projection sums q.g per row in a
// fixed order through shared memory (deterministic).
// ---------------------------------------------------------------------------
constexpr int TILE_T = 256;                 // threads per CTA
constexpr int TILE_U = 2;                   // W entries per thread
constexpr int TILE_E = TILE_T * TILE_U;     // W entries per tile (max)

struct TileHdr {
  int32_t r0, r1;        // rows [r0, r1)
  int64_t base, end;     // W entries [base, end)
  int64_t abase, aend;   // A_FF records [abase, aend)
};

template <int MODE>
__global__ void __launch_bounds__(TILE_T)
k_spgemm_tile(DevView v, const SpEnt* __restrict__ A, const TileHdr* __restrict__ hdr,
              const double* __restrict__ X, const double* __restrict__ X2, double* __restrict__ out,
              double* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double sh[32];
  if (MODE == MM_ITER && v.st->stopped) { iter_stopped(v); return; }
  const bool two = MODE == MM_ENERGY && X2 != nullptr;      // (X2 null: X is already W)
  const int tid = threadIdx.x;
  const TileHdr H = hdr[blockIdx.x];
  const int nrows = H.r1 - H.r0;
  const int nent = (int)(H.end - H.base);
  const int nrec = (int)(H.aend - H.abase);
  SpEnt* s_rec = reinterpret_cast<SpEnt*>(smem_raw);                    // [nrec]
  int32_t* s_wptr = reinterpret_cast<int32_t*>(s_rec + nrec);          // [nrows+1]
  int32_t* s_aptr = s_wptr + (TILE_E + 1);                              // [nrows+1]
  uint16_t* s_erow = reinterpret_cast<uint16_t*>(s_aptr + (TILE_E + 1));// [nent]
  double* s_qa = reinterpret_cast<double*>(s_erow + TILE_E + 8 - (TILE_E % 8)); // [nent]
  double* s_dot = s_qa + TILE_E;                                        // [nrows]
  // ---- phase A: staged loads
  for (int k = tid; k < nrec; k += TILE_T) s_rec[k] = A[H.abase + k];
  for (int r = tid; r <= nrows; r += TILE_T) {
    s_wptr[r] = (int32_t)(v.wptr[H.r0 + r] - H.base);
    s_aptr[r] = (int32_t)(v.affptr[H.r0 + r] - H.abase);
  }
  double qv[TILE_U], xo[TILE_U];
#pragma unroll
  for (int u = 0; u < TILE_U; ++u) {
    const int e = tid + u * TILE_T;
    qv[u] = 0.0;
    xo[u] = 0.0;
    if (e < nent) {
      if (MODE != MM_ENERGY) qv[u] = v.Q[H.base + e];
      if (MODE == MM_ITER || MODE == MM_R0E) xo[u] = X[H.base + e];
      if (MODE == MM_ENERGY) xo[u] = two ? X[H.base + e] + X2[H.base + e] : X[H.base + e];
    }
  }
  __syncthreads();
  for (int r = tid; r < nrows; r += TILE_T)
    for (int p = s_wptr[r]; p < s_wptr[r + 1]; ++p) s_erow[p] = (uint16_t)r;
  __syncthreads();
  // ---- phase B: masked product from shared memory
  double part = 0.0;
  double g[TILE_U];
  int rl[TILE_U];
#pragma unroll
  for (int u = 0; u < TILE_U; ++u) {
    const int e = tid + u * TILE_T;
    g[u] = 0.0;
    rl[u] = 0;
    if (e < nent) {
      const int r = s_erow[e];
      rl[u] = r;
      const unsigned sh4 = 4u * (unsigned)(e - s_wptr[r]);
      double acc = 0.0;
      const int q1 = s_aptr[r + 1];
#pragma unroll 4
      for (int q = s_aptr[r]; q < q1; ++q) {
        const SpEnt en = s_rec[q];
        const unsigned s = (en.pm >> sh4) & 0xFu;
        if (s != 0xFu) {
          const int64_t src = (int64_t)en.ybase + s;
          const double xv = two ? X[src] + X2[src] : X[src];
          acc = fma(en.a, xv, acc);
        }
      }
      double fc = 0.0;
      if (MODE != MM_ITER) {
        const int64_t i = H.r0 + r;
        const int32_t j = v.wcol[H.base + e];
        for (int64_t q = v.afcptr[i]; q < v.afcptr[i + 1]; ++q)
          if (v.afccol[q] == j) { fc = v.afcval[q]; break; }
      }
      if (MODE == MM_ENERGY) g[u] = acc + 2.0 * fc;
      else if (MODE == MM_R0 || MODE == MM_R0E) g[u] = acc + fc;
      else g[u] = acc;
      if (MODE == MM_R0E) part = fma(xo[u], acc + 2.0 * fc, part);   // E0 term, as MM_ENERGY
    }
  }
  if (MODE == MM_ENERGY) {
#pragma unroll
    for (int u = 0; u < TILE_U; ++u)
      if (tid + u * TILE_T < nent) part = fma(xo[u], g[u], part);
  } else {
    // ---- Pi_B (nv = 1), twice for r0 (see masked.cuh)
#pragma unroll
    for (int pass = 0; pass < ((MODE == MM_R0 || MODE == MM_R0E) ? 2 : 1); ++pass) {
      __syncthreads();
#pragma unroll
      for (int u = 0; u < TILE_U; ++u) {
        const int e = tid + u * TILE_T;
        if (e < nent) s_qa[e] = qv[u] * g[u];
      }
      __syncthreads();
      for (int r = tid; r < nrows; r += TILE_T) {
        double s = 0.0;
        for (int p = s_wptr[r]; p < s_wptr[r + 1]; ++p) s += s_qa[p];
        s_dot[r] = s;
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < TILE_U; ++u)
        if (tid + u * TILE_T < nent) g[u] = g[u] - qv[u] * s_dot[rl[u]];
    }
#pragma unroll
    for (int u = 0; u < TILE_U; ++u) {
      const int e = tid + u * TILE_T;
      if (e < nent) {
        if (MODE == MM_ITER) {
          out[H.base + e] = g[u];
          part = fma(xo[u], g[u], part);
        } else {
          out[H.base + e] = -g[u];
        }
      }
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, MODE == MM_ITER ? 1 : -1);
}

#include "kernels_variants_tile.cuh"

__global__ void k_tile_headers(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr,
                               const int32_t* __restrict__ trow, int64_t ntiles, TileHdr* __restrict__ hdr,
                               int32_t* __restrict__ maxrec) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    TileHdr h;
    h.r0 = trow[t];
    h.r1 = trow[t + 1];
    h.base = wptr[h.r0];
    h.end = wptr[h.r1];
    h.abase = affptr[h.r0];
    h.aend = affptr[h.r1];
    hdr[t] = h;
    atomicMax(maxrec, (int32_t)(h.aend - h.abase));
    atomicMax(maxrec + 1, h.r1 - h.r0);
  }
}

static inline size_t tile_smem_bytes(int maxrec) {
  return (size_t)maxrec * sizeof(SpEnt) + 2 * sizeof(int32_t) * (TILE_E + 1) +
         sizeof(uint16_t) * (TILE_E + 8) + sizeof(double) * (2 * TILE_E) + 16;
}

// ---- setup of the scalar plan
__global__ void k_plan_rowstart(const int64_t* __restrict__ wptr, int64_t nF, int32_t S, int64_t nwin,
                                int32_t* __restrict__ rowstart) {
  // rowstart[w] = first row i with wptr[i] >= w S (lower bound), w in [0, nwin]
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nF; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t hi = (i < nF) ? wptr[i] : INT64_MAX / 2;
    const int64_t lo = (i > 0) ? wptr[i - 1] : -1;
    // windows w with lo < w S <= hi
    int64_t w0 = lo < 0 ? 0 : lo / S + 1;
    int64_t w1 = hi / S;
    if (w1 > nwin) w1 = nwin;
    for (int64_t w = w0; w <= w1; ++w) rowstart[w] = (int32_t)i;
  }
}

// one group of 8 lanes per F row, lane per A_FF entry (setup only)
__global__ void k_plan_entries(DevView v, SpEnt* __restrict__ ent) {
  const int lg = threadIdx.x & 7;
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 3;
  for (int64_t i = gid; i < v.nF; i += ng) {
    const int64_t b = v.wptr[i];
    const int nj = (int)(v.wptr[i + 1] - b);
    int32_t ji[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) ji[t] = (t < nj) ? v.wcol[b + t] : -1;
    // the diagonal record goes first (win2 takes its term from the lane's
    // own y value); the others keep A's column order
    const int64_t qb = v.affptr[i], qe = v.affptr[i + 1];
    int64_t qd = qb;
    for (int64_t q = qb; q < qe; ++q)
      if (v.affcol[q] == (int32_t)i) { qd = q; break; }
    for (int64_t q = qb + lg; q < qe; q += 8) {
      const int64_t dst = (q == qd) ? qb : (q < qd ? q + 1 : q);
      const int32_t k = v.affcol[q];
      const int64_t kb = v.wptr[k];
      const int nk = (int)(v.wptr[k + 1] - kb);
      int32_t jk[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) jk[s] = (s < nk) ? v.wcol[kb + s] : -2;
      uint32_t pm = 0xFFFFFFFFu;
#pragma unroll
      for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (ji[t] == jk[s]) pm = (pm & ~(0xFu << (4 * t))) | ((uint32_t)s << (4 * t));
      SpEnt e;
      e.a = v.affval[q];
      e.ybase = (int32_t)kb;
      e.pm = pm;
      ent[dst] = e;
    }
  }
}

// ---- host side ------------------------------------------------------------
struct FastPaths {
  ScalarPlan sc;
};
static FastPaths* fast_of(emin_ctx c) { return reinterpret_cast<FastPaths*>(c->fast); }

static inline int select_fast_path(emin_ctx c) {
  if (c->nv != 1 || c->max_row > 8 || c->nnzWh >= INT32_MAX || c->nF >= INT32_MAX || c->nnzAFF >= INT32_MAX ||
      c->nF == 0)
    return 0;
  if (getenv("EMIN_FORCE_GENERIC")) return 0;
  FastPaths* f = new FastPaths();
  c->fast = f;
  ScalarPlan& p = f->sc;
  p.S = std::min(31, 33 - c->max_row);   // <= 31 rows per window (lane nrows loads the end)
  p.nwin = (c->nnzW + p.S - 1) / p.S;
  cudaStream_t s = c->stream;
  if (cudaMallocAsync((void**)&p.rowstart, sizeof(int32_t) * (p.nwin + 1), s) != cudaSuccess) return 0;
  if (cudaMallocAsync((void**)&p.ent, sizeof(SpEnt) * (size_t)std::max<int64_t>(c->nnzAFF, 1), s) != cudaSuccess) return 0;
  const int SM = emin_num_sms();
  k_plan_rowstart<<<SM * 8, 256, 0, s>>>(c->wptr, c->nF, p.S, p.nwin, p.rowstart);
  // short in-order CTAs (kernel-plan phase 0.45 -> 0.37 ms on config 3; EMIN_PLAN_GRID: CTAs per SM)
  k_plan_entries<<<SM * (getenv("EMIN_PLAN_GRID") ? atoi(getenv("EMIN_PLAN_GRID")) : 32), 256, 0, s>>>(c->view(), p.ent);
  c->launches += 2;
  // per-iteration kernel variant (EMIN_SPGEMM, default win2); the tile plan
  // and the window headers are built only for the variants that use them
  const char* var = getenv("EMIN_SPGEMM");
  const bool need_tiles = !getenv("EMIN_SETUP_WIN2M") || (var && (!strcmp(var, "tile") || !strcmp(var, "pipe")));
  const bool need_whdr = var && (!strcmp(var, "hdr") || !strcmp(var, "mask"));
  int32_t hmax[2] = {0, 0};
  if (need_tiles) {
    // tile plan for the staged kernel
    const int ST = TILE_E - c->max_row + 1;
    p.ntiles = (c->nnzW + ST - 1) / ST;
    int32_t* trow = nullptr;
    int32_t* dmax = nullptr;
    if (cudaMallocAsync((void**)&trow, sizeof(int32_t) * (p.ntiles + 1), s) != cudaSuccess ||
        cudaMallocAsync((void**)&p.hdr, sizeof(TileHdr) * std::max<int64_t>(p.ntiles, 1), s) != cudaSuccess ||
        cudaMallocAsync((void**)&dmax, sizeof(int32_t) * 2, s) != cudaSuccess)
      return 1;
    cudaMemsetAsync(dmax, 0, sizeof(int32_t) * 2, s);
    k_plan_rowstart<<<SM * 8, 256, 0, s>>>(c->wptr, c->nF, ST, p.ntiles, trow);
    k_tile_headers<<<SM * 4, 256, 0, s>>>(c->wptr, c->affptr, trow, p.ntiles, p.hdr, dmax);
    c->launches += 2;
    cudaMemcpyAsync(hmax, dmax, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(trow, s);
    cudaFreeAsync(dmax, s);
    cudaStreamSynchronize(s);
    p.tile_smem = tile_smem_bytes(hmax[0]);
  }
  if (need_whdr) {
    // window headers (lane decode without the rowstart -> wptr round trips)
    if (cudaMallocAsync((void**)&p.whdr, sizeof(WinHdr) * std::max<int64_t>(p.nwin, 1), s) != cudaSuccess) return 1;
    k_plan_headers<<<SM * 4, 256, 0, s>>>(c->wptr, p.rowstart, p.nwin, p.whdr);
    c->launches += 1;
  }
  p.variant = 5;   // default: win2 (fastest measured, profiles/r01/spgemm_variants_c3.log)
  if (var && !strcmp(var, "hdr")) p.variant = 0;
  if (var && !strcmp(var, "win")) p.variant = 1;
  if (var && !strcmp(var, "tile")) p.variant = 2;
  if (var && !strcmp(var, "pipe")) p.variant = 3;
  if (var && !strcmp(var, "mask")) p.variant = 4;
  if (var && !strcmp(var, "win2")) p.variant = 5;
  if (var && !strcmp(var, "win3")) p.variant = 6;
  if (var && !strcmp(var, "win4")) p.variant = 7;
  if (var && !strcmp(var, "win5")) p.variant = 8;
  if (var && !strcmp(var, "win6")) p.variant = 9;
  if (var && !strcmp(var, "win7")) p.variant = 10;
  if (var && !strcmp(var, "win8")) p.variant = 11;
  if (var && !strcmp(var, "win9")) p.variant = 12;
  if (var && !strcmp(var, "win10")) p.variant = 13;
  if (var && !strcmp(var, "win2g1")) p.variant = 14;
  if (var && !strcmp(var, "win2g2")) p.variant = 5;
  if (var && !strcmp(var, "win2g3")) p.variant = 15;
  if (var && !strcmp(var, "win2g4")) p.variant = 16;
  if (p.variant == 13) {
    int32_t* dmx = nullptr;
    int32_t hw = 0;
    if (cudaMallocAsync((void**)&dmx, sizeof(int32_t), s) == cudaSuccess) {
      cudaMemsetAsync(dmx, 0, sizeof(int32_t), s);
      k_rowlen_max<<<SM * 4, 256, 0, s>>>(c->affptr, c->nF, dmx);
      cudaMemcpyAsync(&hw, dmx, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaFreeAsync(dmx, s);
      cudaStreamSynchronize(s);
      c->launches += 1;
    }
    p.ellW = std::max(2, hw) - 1;                    // MAXR = longest row - 1 (diagonal apart)
    int per_sm = 0;
    if (p.ellW <= 8) {
      auto kfun = p.ellW <= 4 ? k_spgemm_win10<4> : p.ellW <= 6 ? k_spgemm_win10<6> : k_spgemm_win10<8>;
      cudaFuncSetAttribute(kfun, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w10_smem_bytes());
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfun, W8_WARPS * 32, w10_smem_bytes());
    }
    if (per_sm < 1 || cudaMallocAsync((void**)&p.w4hdr, sizeof(Win4Hdr) * std::max<int64_t>(p.nwin, 1), s) != cudaSuccess) {
      p.variant = 5;
    } else {
      p.w8grid = (int)std::max<int64_t>(1, std::min<int64_t>((p.nwin + W8_WARPS - 1) / W8_WARPS, (int64_t)SM * per_sm));
      k_plan_win4<<<SM * 4, 256, 0, s>>>(c->wptr, c->affptr, p.rowstart, p.nwin, p.w4hdr);
      c->launches += 1;
    }
  }
  if (p.variant == 12) {
    int per_sm = 0;
    cudaFuncSetAttribute(k_spgemm_win9, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w9_smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spgemm_win9, W8_WARPS * 32, w9_smem_bytes());
    if (per_sm < 1 || cudaMallocAsync((void**)&p.w6hdr, sizeof(int4) * (p.nwin + 1), s) != cudaSuccess) {
      p.variant = 5;
    } else {
      p.w8grid = (int)std::max<int64_t>(1, std::min<int64_t>((p.nwin + W8_WARPS - 1) / W8_WARPS, (int64_t)SM * per_sm));
      k_plan_win6<<<SM * 4, 256, 0, s>>>(c->wptr, c->affptr, p.rowstart, p.nwin, p.w6hdr);
      c->launches += 1;
    }
  }
  if (p.variant == 11) {
    int per_sm = 0;
    cudaFuncSetAttribute(k_spgemm_win8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w8_smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spgemm_win8, W8_WARPS * 32, w8_smem_bytes());
    if (per_sm < 1 || cudaMallocAsync((void**)&p.w6hdr, sizeof(int4) * (p.nwin + 1), s) != cudaSuccess) {
      p.variant = 5;
    } else {
      p.w8grid = (int)std::max<int64_t>(1, std::min<int64_t>((p.nwin + W8_WARPS - 1) / W8_WARPS, (int64_t)SM * per_sm));
      k_plan_win6<<<SM * 4, 256, 0, s>>>(c->wptr, c->affptr, p.rowstart, p.nwin, p.w6hdr);
      c->launches += 1;
    }
  }
  if (p.variant == 10) {
    int32_t* dmx = nullptr;
    int32_t hw = 0;
    if (cudaMallocAsync((void**)&dmx, sizeof(int32_t), s) == cudaSuccess) {
      cudaMemsetAsync(dmx, 0, sizeof(int32_t), s);
      k_rowlen_max<<<SM * 4, 256, 0, s>>>(c->affptr, c->nF, dmx);
      cudaMemcpyAsync(&hw, dmx, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaFreeAsync(dmx, s);
      cudaStreamSynchronize(s);
      c->launches += 1;
    }
    p.ellW = std::max(4, hw);
    if (hw < 1 || hw > 8 ||
        cudaMallocAsync((void**)&p.ell, sizeof(int4) * (size_t)c->nF * p.ellW, s) != cudaSuccess ||
        cudaMallocAsync((void**)&p.w7hdr, sizeof(int4) * std::max<int64_t>(p.nwin, 1), s) != cudaSuccess) {
      p.variant = 5;
    } else {
      k_plan_ell<<<SM * 8, 256, 0, s>>>(c->affptr, c->nF, p.ellW, reinterpret_cast<const int4*>(p.ent), p.ell);
      k_plan_win7<<<SM * 4, 256, 0, s>>>(c->wptr, p.rowstart, p.nwin, p.w7hdr);
      c->launches += 2;
    }
  }
  if (p.variant == 9) {
    if (cudaMallocAsync((void**)&p.w6hdr, sizeof(int4) * (p.nwin + 1), s) != cudaSuccess) {
      p.variant = 5;
    } else {
      k_plan_win6<<<SM * 4, 256, 0, s>>>(c->wptr, c->affptr, p.rowstart, p.nwin, p.w6hdr);
      c->launches += 1;
    }
  }
  if (p.variant == 7 || p.variant == 8) {
    if (cudaMallocAsync((void**)&p.w4hdr, sizeof(Win4Hdr) * std::max<int64_t>(p.nwin, 1), s) != cudaSuccess) {
      p.variant = 5;
    } else {
      k_plan_win4<<<SM * 4, 256, 0, s>>>(c->wptr, c->affptr, p.rowstart, p.nwin, p.w4hdr);
      c->launches += 1;
    }
  }
  if (p.variant == 6) {
    const int S3 = std::min(63, 65 - c->max_row);
    p.nwin3 = (c->nnzW + S3 - 1) / S3;
    if (cudaMallocAsync((void**)&p.rowstart3, sizeof(int32_t) * (p.nwin3 + 1), s) != cudaSuccess) {
      p.variant = 5;
    } else {
      k_plan_rowstart<<<SM * 8, 256, 0, s>>>(c->wptr, c->nF, S3, p.nwin3, p.rowstart3);
      c->launches += 1;
    }
  }
  if (p.variant == 4) {
    int32_t* bad = nullptr;
    if (cudaMallocAsync((void**)&p.emask, sizeof(uint16_t) * std::max<int64_t>(c->nnzW, 1), s) != cudaSuccess ||
        cudaMallocAsync((void**)&bad, sizeof(int32_t), s) != cudaSuccess) {
      p.variant = 1;
    } else {
      cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
      k_plan_emask<<<SM * 8, 256, 0, s>>>(c->view(), p.ent, p.emask, bad);
      c->launches += 1;
      int32_t hb = 0;
      cudaMemcpyAsync(&hb, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaFreeAsync(bad, s);
      cudaStreamSynchronize(s);
      if (hb) p.variant = 1;
    }
  }
  if (need_tiles && p.tile_smem <= 160 * 1024) {
    p.use_tiles = 1;
    cudaFuncSetAttribute(k_spgemm_tile<MM_ITER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.tile_smem);
    cudaFuncSetAttribute(k_spgemm_tile<MM_R0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.tile_smem);
    cudaFuncSetAttribute(k_spgemm_tile<MM_ENERGY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.tile_smem);
    cudaFuncSetAttribute(k_spgemm_tile<MM_R0E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.tile_smem);
  } else if (p.variant == 2) {
    p.variant = 5;
  }
  if (p.variant == 3) {
    // persistent TMA-pipelined kernel
    p.rec_cap = (hmax[0] + 1) & ~1;
    p.rows_cap = hmax[1] + 1;
    p.pipe_smem = pipe_layout(p.rec_cap, p.rows_cap).total;
    int per_sm = 0;
    if (p.pipe_smem <= 200 * 1024) {
      cudaFuncSetAttribute(k_spgemm_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.pipe_smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spgemm_pipe, TILE_T, p.pipe_smem);
    }
    if (per_sm > 0) {
      p.use_pipe = 1;
      p.pipe_grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.ntiles, (int64_t)SM * per_sm));
    } else {
      p.variant = 5;
    }
  }
  return 1;
}

static inline int scalar_grid(emin_ctx c) {
  const int SM = emin_num_sms();
  const int64_t nwin = fast_of(c)->sc.nwin;
  const int64_t per_sm = getenv("EMIN_SCALAR_GRID") ? atoi(getenv("EMIN_SCALAR_GRID")) : 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>((nwin + 7) / 8, (int64_t)SM * per_sm));
}
// grid of the one-off window kernels (Alg. 2 for nv = 1, P out): short
// in-order CTAs (EMIN_WIN_GRID CTAs per SM, A/B)
static inline int setup_win_grid(emin_ctx c) {
  const int SM = emin_num_sms();
  const int64_t nwin = fast_of(c)->sc.nwin;
  const int64_t per_sm = getenv("EMIN_WIN_GRID") ? atoi(getenv("EMIN_WIN_GRID")) : 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>((nwin + 7) / 8, (int64_t)SM * per_sm));
}
// grid of the setup-time masked launches (MM_R0, MM_ENERGY)
static inline int scalar_spgemm_grid(emin_ctx c) {
  const ScalarPlan& p = fast_of(c)->sc;
  return p.use_tiles ? (int)std::max<int64_t>(1, p.ntiles) : scalar_grid(c);
}
// grid of the per-iteration masked launch (MM_ITER)
static inline int scalar_iter_grid(emin_ctx c) {
  const ScalarPlan& p = fast_of(c)->sc;
  switch (p.variant) {
    case 2: return (int)std::max<int64_t>(1, p.ntiles);
    case 3: return p.pipe_grid;
    case 11: case 12: case 13: return p.w8grid;
    default: return scalar_grid(c);
  }
}

static inline bool launch_scalar_masked(emin_ctx c, int mode, const double* X, const double* X2, double* out,
                                        cudaStream_t s) {
  const ScalarPlan& p = fast_of(c)->sc;
  const DevView v = c->view();
  if (mode == MM_ITER) {
    switch (p.variant) {
      case 0:
        k_spgemm_hdr<<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.whdr, p.nwin, X, out, c->partials);
        return true;
      case 4:
        k_spgemm_mask<<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.whdr, p.nwin, p.emask, X, out, c->partials);
        return true;
      case 5:     // default: two records per round (119.1 vs 120.8 us with one, config 3)
        k_spgemm_win2<2><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, out, c->partials);
        return true;
      case 14:
        k_spgemm_win2<1><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, out, c->partials);
        return true;
      case 15:
        k_spgemm_win2<3><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, out, c->partials);
        return true;
      case 16:
        k_spgemm_win2<4><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, out, c->partials);
        return true;
      case 7:
      case 8: {
        const int g = scalar_grid(c);
        if (p.variant == 7)
          k_spgemm_win4<false><<<g, 256, 0, s>>>(v, reinterpret_cast<const int4*>(p.ent),
                                                 p.w4hdr, p.nwin, X, out,
                                                 c->partials);
        else
          k_spgemm_win4<true><<<g, 256, 0, s>>>(v, reinterpret_cast<const int4*>(p.ent),
                                                p.w4hdr, p.nwin, X, out,
                                                c->partials);
        return true;
      }
      case 11:
        k_spgemm_win8<<<p.w8grid, W8_WARPS * 32, w8_smem_bytes(), s>>>(v, reinterpret_cast<const int4*>(p.ent),
                                                                      p.w6hdr, p.nwin, X, out, c->partials);
        return true;
      case 13: {
        const auto kfun = p.ellW <= 4 ? k_spgemm_win10<4> : p.ellW <= 6 ? k_spgemm_win10<6> : k_spgemm_win10<8>;
        kfun<<<p.w8grid, W8_WARPS * 32, w10_smem_bytes(), s>>>(v, reinterpret_cast<const int4*>(p.ent), p.w4hdr,
                                                               p.nwin, X, out, c->partials);
        return true;
      }
      case 12:
        k_spgemm_win9<<<p.w8grid, W8_WARPS * 32, w9_smem_bytes(), s>>>(v, reinterpret_cast<const int4*>(p.ent),
                                                                      p.w6hdr, p.nwin, X, out, c->partials);
        return true;
      case 10: {
        const int g = scalar_grid(c);
#define W7(WW) case WW: k_spgemm_win7<WW><<<g, 256, 0, s>>>(v, p.ell, p.w7hdr, p.nwin, X, out, c->partials); break;
        switch (p.ellW) { W7(4) W7(5) W7(6) W7(7) W7(8) }
#undef W7
        return true;
      }
      case 9:
        k_spgemm_win6<<<scalar_grid(c), 256, 0, s>>>(v, reinterpret_cast<const int4*>(p.ent), p.w6hdr, p.nwin, X,
                                                     out, c->partials);
        return true;
      case 6:
        k_spgemm_win3<<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart3, p.nwin3, X, out, c->partials);
        return true;
      case 1:
        k_spgemm_scalar<MM_ITER><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, X2, out,
                                                                c->partials);
        return true;
      case 2:
        k_spgemm_tile<MM_ITER><<<(int)std::max<int64_t>(1, p.ntiles), TILE_T, p.tile_smem, s>>>(
            v, p.ent, p.hdr, X, X2, out, c->partials);
        return true;
      default:
        k_spgemm_pipe<<<p.pipe_grid, TILE_T, p.pipe_smem, s>>>(v, p.ent, p.hdr, p.ntiles, p.rec_cap, p.rows_cap,
                                                              X, out, c->partials);
        return true;
    }
  }
  if (mode == MM_R0E) {                      // fused r0 + E0: the tile kernel only
    if (!p.use_tiles) return false;
    k_spgemm_tile<MM_R0E><<<(int)std::max<int64_t>(1, p.ntiles), TILE_T, p.tile_smem, s>>>(v, p.ent, p.hdr, X, X2,
                                                                                         out, c->partials);
    return true;
  }
  if (!p.use_tiles) {
    // setup / energy modes on win2's window kernel (EMIN_SETUP_WIN2M=1; measured
    // slower than the tile kernel on config 3: r0 + E0 0.47 ms either way,
    // emin_energy 0.34 vs 0.28 ms)
    if (mode == MM_R0)
      k_spgemm_win2m<MM_R0><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, X2, out, c->partials);
    else
      k_spgemm_win2m<MM_ENERGY><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, X2, out,
                                                              c->partials);
    return true;
  }
  const int g = (int)std::max<int64_t>(1, p.ntiles);
  if (mode == MM_R0)
    k_spgemm_tile<MM_R0><<<g, TILE_T, p.tile_smem, s>>>(v, p.ent, p.hdr, X, X2, out, c->partials);
  else
    k_spgemm_tile<MM_ENERGY><<<g, TILE_T, p.tile_smem, s>>>(v, p.ent, p.hdr, X, X2, out, c->partials);
  return true;
}
static inline void launch_scalar_alg2(emin_ctx c, const double* Bc, const double* B, const int64_t* frow,
                                      const double* what, unsigned long long* counters, cudaStream_t s) {
  const ScalarPlan& p = fast_of(c)->sc;
  k_alg2_nv1<<<setup_win_grid(c), 256, 0, s>>>(c->view(), p.rowstart, p.nwin, Bc, B, frow, what, c->Q, c->w0,
                                            counters);
}
static inline void launch_scalar_get_P(emin_ctx c, double* out, cudaStream_t s) {
  const ScalarPlan& p = fast_of(c)->sc;
  k_get_P_win<<<setup_win_grid(c), 256, 0, s>>>(c->view(), p.rowstart, p.nwin, c->w0, c->dw, c->pofs, out);
}
static inline void launch_scalar_stage(emin_ctx c, int which, cudaStream_t s) {
  const ScalarPlan& p = fast_of(c)->sc;
  if (which == 1)
    k_stage1_win<<<c->grid_rows, 256, 0, s>>>(c->view(), p.rowstart, p.nwin, c->r, c->yb, c->partials);
  else
    k_stage2_win<<<c->grid_rows, 256, 0, s>>>(c->view(), p.rowstart, p.nwin, c->r, c->y, c->dw);
}

static inline void free_fast_path(emin_ctx c) {
  FastPaths* f = fast_of(c);
  if (!f) return;
  if (f->sc.rowstart) cudaFreeAsync(f->sc.rowstart, c->stream);
  if (f->sc.ent) cudaFreeAsync(f->sc.ent, c->stream);
  if (f->sc.hdr) cudaFreeAsync(f->sc.hdr, c->stream);
  if (f->sc.whdr) cudaFreeAsync(f->sc.whdr, c->stream);
  if (f->sc.emask) cudaFreeAsync(f->sc.emask, c->stream);
  if (f->sc.rowstart3) cudaFreeAsync(f->sc.rowstart3, c->stream);
  if (f->sc.w4hdr) cudaFreeAsync(f->sc.w4hdr, c->stream);
  if (f->sc.w6hdr) cudaFreeAsync(f->sc.w6hdr, c->stream);
  if (f->sc.ell) cudaFreeAsync(f->sc.ell, c->stream);
  if (f->sc.w7hdr) cudaFreeAsync(f->sc.w7hdr, c->stream);
  delete f;
  c->fast = nullptr;
}
