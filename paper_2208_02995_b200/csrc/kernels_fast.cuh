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
// Per-iteration kernel: k_spgemm_wp (two W entries per lane on pair
// windows, one record load per two gathers; k_spgemm_wd -- one entry per
// lane, win2's windows with the decode precomputed at setup -- is its A/B
// reference, k_spgemm_win2 the fallback when the descriptors overflow);
// setup / energy modes: k_spgemm_wdm on wd's windows, else the tile kernel
// (k_spgemm_tile, fused MM_R0E at setup), or win2's modes (k_spgemm_win2m)
// when a tile's records do not fit in shared memory.  The round-1 A/B
// variants (profiles/ab_r01/) are not part of the library.
#pragma once
#include <algorithm>
#include "emin_internal.cuh"
#include "masked.cuh"
#include "bulk.cuh"
#include "dist.cuh"

struct SpEnt {          // 16 bytes, one per A_FF entry
  double a;
  int32_t ybase;
  uint32_t pm;
};

struct TileHdr;
struct ScalarPlan {
  SpEnt* ent = nullptr;
  SpEnt* entS = nullptr;         // the records of D^-1/2 A_FF D^-1/2 (ctx sym; per-iteration product)
  int32_t* rowstart = nullptr;   // [nwin + 1]
  int4* whdr = nullptr;          // [nwin] {first W entry, first record, entries, first row} (k_spgemm_wd)
  uint32_t* wdesc = nullptr;     // [nnzW] lane descriptor (k_spgemm_wd)
  // pair-lane plan of the per-iteration kernel (k_spgemm_wp)
  int64_t* lptr = nullptr;       // [nF + 1] first lane slot of each row
  int32_t* prowstart = nullptr;  // [npwin + 1] first row of each pair window
  int4* phdr = nullptr;          // [npwin] {first lane slot, first record, lanes, first row}
  int2* pdesc = nullptr;         // [lanes] {first entry, packed row / record fields}
  int64_t npwin = 0;
  int64_t nwin = 0;
  int32_t S = 0;
  TileHdr* hdr = nullptr;        // [ntiles] (staged tile kernel, setup / energy modes)
  int64_t ntiles = 0;
  size_t tile_smem = 0;
  int use_tiles = 0;
};

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
  const int64_t cnt = unit_count(v, nwin);
  for (int64_t w1 = gw; w1 < cnt; w1 += nw) {
    const int64_t w = unit_of(v, rev ? cnt - 1 - w1 : w1);
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

// y^ = Pi K y (nv = 1), window-descriptor kernel: the same windows, records
// and arithmetic as k_spgemm_win2 (bitwise the same y^ and partial sums), but
// the window decode is precomputed at setup -- a 16-byte header per window
// {first W entry, first record, entries} and a 32-bit descriptor per W entry
// {row's first lane, row length, row's record count and first record
// relative to the window's} -- so the per-window dependent-load chain
// rowstart -> wptr -> affptr -> record (4 latencies, 41 % of win2's stall
// samples, profiles/r02) becomes header -> descriptor -> record.  In the
// record loop the {ybase, pm} halves of the next LA records are loaded ahead
// (a record's gather no longer waits for its own record load) and a(q) is
// read at use from the line already in L1; LEAN re-reads Q and the own y
// entry after the loop so that LA = 2 fits 32 registers.
constexpr uint32_t WD_MAXREC = 255, WD_MAXREL = 65535;
constexpr int WD_NT = 1024;    // threads per CTA of the per-iteration launch
constexpr int WD_LA = 2;       // records whose {ybase, pm} are in flight ahead of the current one
template <int NT = 256, int LA = 0, bool LEAN = false>
__global__ void __launch_bounds__(NT, 2048 / NT)
k_spgemm_wd(DevView v, const SpEnt* __restrict__ A, const int4* __restrict__ whdr, const uint32_t* __restrict__ wdesc,
            int32_t nwin, const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[NT / 32][32];
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
  for (int w1 = gw; w1 < cnt; w1 += nw) {
    int w = rev ? cnt - 1 - w1 : w1;
    if (split) w = (int)unit_of(v, w);
    const int4 h = __ldg(whdr + w);
    const int nent = h.z;
    if (nent == 0) continue;                           // warp-uniform
    const bool act = lane < nent;
    const int e = h.x + lane;
    const uint32_t dsc = act ? __ldg(wdesc + e) : 0u;
    // LEAN: Q and the own y entry are (re)read after the record loop (fewer
    // live registers in it; the y line is still in L1)
    double qv = (!LEAN && act) ? v.Q[e] : 0.0;
    double xo = act ? X[e] : 0.0;
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
      if constexpr (LA > 0) {
        // the {ybase, pm} halves of the next LA records are in flight while
        // record q's gather runs; a(q) is read at use (same line: L1 hit)
        const int2* I2 = reinterpret_cast<const int2*>(A);
        const double* Ad = reinterpret_cast<const double*>(A);
        int2 la[LA > 0 ? LA : 1];
#pragma unroll
        for (int j = 0; j < LA; ++j) la[j] = (q + j < qe) ? __ldg(I2 + 2 * (q + j) + 1) : make_int2(0, -1);
#pragma unroll 2
        for (; q < qe; ++q) {
          const int2 cur = la[0];
#pragma unroll
          for (int j = 0; j + 1 < LA; ++j) la[j] = la[j + 1];
          la[LA - 1] = (q + LA < qe) ? __ldg(I2 + 2 * (q + LA) + 1) : make_int2(0, -1);
          const unsigned s = ((unsigned)cur.y >> sh4) & 0xFu;
          if (s != 0xFu) acc = fma(__ldg(Ad + 2 * q), X[cur.x + (int)s], acc);
        }
      } else {
#pragma unroll 4
      for (; q < qe; ++q) {
        const int4 en = __ldg(&A4[q]);
        const unsigned s = ((unsigned)en.w >> sh4) & 0xFu;
        if (s != 0xFu) acc = fma(__hiloint2double(en.y, en.x), X[en.z + (int)s], acc);
      }
      }
    }
    if (LEAN && act) { qv = v.Q[e]; xo = X[e]; }
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

// y^ = Pi K y (nv = 1), pair-lane kernel: a lane owns TWO consecutive W
// entries of its row (positions 2t and 2t+1), so one record load {a, ybase,
// pm} and its decode serve two gathers and two FMAs, and a window of 32
// lanes covers up to 64 entries (half as many windows, each with twice the
// gathers in flight per warp).  Lane slots: row r has ceil(|J_r| / 2) of
// them (lptr = their prefix sum); windows are cut on lane slots like wd's on
// entries.  Per window a 16-byte header {first lane slot, first record,
// lanes, first row}; per lane slot an int2 {first entry e0, row's first
// lane | (|J_r| - 1) << 5 | records << 8 | first record rel. << 16}.  Each
// entry's sum and the row projection take the same terms in the same order
// as wd (bitwise the same y^); only the y^T y partials are grouped per lane.
constexpr int WP_PAD = 4;      // records allocated past nnz(A_FF) (k_spgemm_wp's look-ahead)
// launch shape of k_spgemm_wp (config 3, us per launch, profiles/r02/spgemm_ab_c3.txt):
// 512-thread CTAs, 3 per SM (40 registers, 48 warps/SM), record loop unrolled
// twice: 95.2; 1024 x 2 (32 registers) 97.8-99.1; 768 x 2 96.3-98.5; four
// entries per lane 122-155
constexpr int WP_NT = 512, WP_MINB = 3, WP_UNR = 2;
// the unit-diagonal (scaled) instance: 512 x 4 per SM, 31 registers, loop not
// unrolled: 85.2-85.4 us vs 87.1-87.3 at 512 x 3 / unroll 2 (config 3;
// 1024 x 2 / unroll 1 the same 85.2-85.3, 256 x 6..8 and 768 x 2 85.6-88.6)
constexpr int WPS_NT = 512, WPS_MINB = 4, WPS_UNR = 1;
template <int NT = WD_NT, int MINB = 2048 / NT, int UNR = 1, int E = 2, bool SYM = false>
__global__ void __launch_bounds__(NT, MINB)
k_spgemm_wp(DevView v, const SpEnt* __restrict__ A, const int4* __restrict__ phdr, const int2* __restrict__ pdesc,
            int32_t nwin, const double* __restrict__ X, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[NT / 32][32 * E];
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
  const double* Ad = reinterpret_cast<const double*>(A);
  for (int w1 = gw; w1 < cnt; w1 += nw) {
    int w = rev ? cnt - 1 - w1 : w1;
    if (split) w = (int)unit_of(v, w);
    const int4 h = __ldg(phdr + w);
    const int nl = h.z;
    if (nl == 0) continue;                             // warp-uniform
    const bool act = lane < nl;
    const int2 d = act ? __ldg(pdesc + h.x + lane) : make_int2(0, 0);
    const int e0 = d.x;
    const uint32_t dsc = (uint32_t)d.y;
    const int rowbeg = (int)(dsc & 31u);
    const int rowlen = (int)((dsc >> 5) & 7u) + 1;
    const int p0 = E * (lane - rowbeg);                // the lane's first position in its row
    double acc[E];
#pragma unroll
    for (int j = 0; j < E; ++j) acc[j] = 0.0;
    if (act) {
      const int qb = h.y + (int)(dsc >> 16);
      const int qe = qb + (int)((dsc >> 8) & 255u);
      if (SYM) {
        // S A_FF S: unit diagonal, the records hold the off-diagonal terms
#pragma unroll
        for (int j = 0; j < E; ++j)
          if (p0 + j < rowlen) acc[j] = X[e0 + j];
      } else {
        const double ad = __ldg(Ad + 2 * qb);          // record qb: the diagonal A(i,i), own y entries
#pragma unroll
        for (int j = 0; j < E; ++j)
          if (p0 + j < rowlen) acc[j] = ad * X[e0 + j];
      }
      const unsigned shp = 4u * (unsigned)p0;
      // one 16-byte load per record {a, ybase, pm}, one record ahead (split
      // 8-byte loads of {ybase, pm} and a cost twice the L1 tag requests:
      // 95.2 vs 91.4 us on config 3); the record stream is padded by WP_PAD
      // records, so the look-ahead needs no bound check; an absent position
      // gathers nothing and adds a * 0 (the value of skipping the term, up
      // to the sign of a zero)
      const int q0 = SYM ? qb : qb + 1;
      int4 nxt = __ldg(A4 + q0);
#pragma unroll UNR
      for (int q = q0; q < qe; ++q) {
        const int4 cur = nxt;
        nxt = __ldg(A4 + q + 1);
        const unsigned pm = (unsigned)cur.w >> shp;    // positions past the row: 0xF
        double y[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const unsigned sj = (pm >> (4 * j)) & 0xFu;
          y[j] = (sj != 0xFu) ? X[cur.z + (int)sj] : 0.0;
        }
        const double a = __hiloint2double(cur.y, cur.x);
#pragma unroll
        for (int j = 0; j < E; ++j) acc[j] = fma(a, y[j], acc[j]);
      }
    }
    double qv[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      qv[j] = (act && p0 + j < rowlen) ? v.Q[e0 + j] : 0.0;
      s_qa[wib][E * lane + j] = qv[j] * acc[j];
    }
    __syncwarp();
    double dot = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p)                       // |J_i| <= 8 on the scalar path
      if (p < rowlen) dot += s_qa[wib][E * rowbeg + p];
    __syncwarp();
    if (act) {
#pragma unroll
      for (int j = 0; j < E; ++j)
        if (p0 + j < rowlen) {
          const double g = acc[j] - qv[j] * dot;
          out[e0 + j] = g;
          part = fma(X[e0 + j], g, part);
        }
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, 1);
}

// k_spgemm_wp's setup / energy modes on the pair windows (wdm's terms in
// wdm's order per entry -- the same r0 -- with the partial sums grouped per
// lane):
//   MM_R0      r0 = -Pi Pi (A P0)|F, the C-identity term A(i, c_j) added  (A1/A2)
//   MM_ENERGY  partial W . (A_FF W + 2 A_FC), W = X + X2 (or X)           (Eq. trInc)
//   MM_R0E     both (setup: they share A P0)
// The lane's row: the window's first row (header .w) + the row heads before it.
template <int MODE, int NT = WP_NT, int MINB = WP_MINB>
__global__ void __launch_bounds__(NT, MINB)
k_spgemm_wpm(DevView v, const SpEnt* __restrict__ A, const int4* __restrict__ phdr, const int2* __restrict__ pdesc,
             int32_t nwin, const double* __restrict__ X, const double* __restrict__ X2, double* __restrict__ out,
             double* __restrict__ partials, int32_t compact) {
  __shared__ double sh[32];
  __shared__ double s_qa[NT / 32][64];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const bool two = MODE == MM_ENERGY && X2 != nullptr;
  auto xval = [&](int idx) -> double { return two ? X[idx] + X2[idx] : X[idx]; };
  const int4* A4 = reinterpret_cast<const int4*>(A);
  const double* Ad = reinterpret_cast<const double*>(A);
  double part = 0.0;
  for (int w = gw; w < nwin; w += nw) {
    const int4 h = __ldg(phdr + w);
    const int nl = h.z;
    if (nl == 0) continue;                             // warp-uniform
    const bool act = lane < nl;
    const int2 d = act ? __ldg(pdesc + h.x + lane) : make_int2(0, 0);
    const int e0 = d.x;
    const uint32_t dsc = (uint32_t)d.y;
    const int rowbeg = (int)(dsc & 31u);
    const int rowlen = (int)((dsc >> 5) & 7u) + 1;
    const int p0 = 2 * (lane - rowbeg);
    const bool has1 = p0 + 1 < rowlen;
    const unsigned heads = __ballot_sync(0xffffffffu, act && p0 == 0);
    const int i = h.w + __popc(heads & ((2u << rowbeg) - 1u)) - 1;
    double acc0 = 0.0, acc1 = 0.0, fc0 = 0.0, fc1 = 0.0, xo0 = 0.0, xo1 = 0.0;
    if (act) {
      // compact descriptors (symmetric scaling) count the diagonal-free
      // records: row i's full run in A starts i records later, one longer
      const int qb = h.y + (int)(dsc >> 16) + (compact ? i : 0);
      const int qe = qb + (int)((dsc >> 8) & 255u) + (compact ? 1 : 0);
      const double ad = Ad[2 * qb];                    // diagonal record first
      xo0 = xval(e0);
      acc0 = ad * xo0;
      if (has1) { xo1 = xval(e0 + 1); acc1 = ad * xo1; }
      const unsigned shp = 4u * (unsigned)p0;
      for (int q = qb + 1; q < qe; ++q) {
        const int4 cur = __ldg(A4 + q);
        const unsigned pm = (unsigned)cur.w >> shp;
        const unsigned s0 = pm & 0xFu, s1 = (pm >> 4) & 0xFu;
        const double a = __hiloint2double(cur.y, cur.x);
        if (s0 != 0xFu) acc0 = fma(a, xval(cur.z + (int)s0), acc0);
        if (s1 != 0xFu) acc1 = fma(a, xval(cur.z + (int)s1), acc1);
      }
      // A(i, c_j): search the short A_FC row
      const int32_t j0 = v.wcol[e0], j1 = has1 ? v.wcol[e0 + 1] : -1;
      for (int64_t q = v.afcptr[i]; q < v.afcptr[i + 1]; ++q) {
        const int32_t cq = v.afccol[q];
        if (cq == j0) fc0 = v.afcval[q];
        if (cq == j1) fc1 = v.afcval[q];
      }
    }
    if (MODE == MM_ENERGY || MODE == MM_R0E)
      if (act) {
        part = fma(xo0, acc0 + 2.0 * fc0, part);
        if (has1) part = fma(xo1, acc1 + 2.0 * fc1, part);
      }
    if (MODE == MM_ENERGY) continue;                  // warp-uniform (MODE)
    const double qv0 = act ? v.Q[e0] : 0.0;
    const double qv1 = (act && has1) ? v.Q[e0 + 1] : 0.0;
    double g0 = acc0 + fc0, g1 = acc1 + fc1;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {            // Pi applied twice (reading A2)
      s_qa[wib][2 * lane] = qv0 * g0;
      s_qa[wib][2 * lane + 1] = qv1 * g1;
      __syncwarp();
      double dot = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < rowlen) dot += s_qa[wib][2 * rowbeg + p];
      __syncwarp();
      g0 = g0 - qv0 * dot;
      g1 = g1 - qv1 * dot;
    }
    if (act) {
      out[e0] = -g0;
      if (has1) out[e0 + 1] = -g1;
    }
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, -1);
}

// Alg. 2 for nv = 1 on the pair windows (q = M / |M|, delta = q (r / |M|);
// |M| = 0 is the rank-0 SVD branch): the row sums of m m and m w^ in
// ascending position order through shared memory
template <int NT = 256>
__global__ void __launch_bounds__(NT)
k_alg2_nv1_wp(DevView v, const int4* __restrict__ phdr, const int2* __restrict__ pdesc, int32_t nwin,
              const double* __restrict__ Bc, const double* __restrict__ B, const int64_t* __restrict__ frow,
              const double* __restrict__ what, double* __restrict__ Qout, double* __restrict__ w0,
              unsigned long long* counters) {
  __shared__ unsigned long long cnt[2];
  __shared__ double s_m[NT / 32][64];
  __shared__ double s_w[NT / 32][64];
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  unsigned n_svd = 0, n_frozen = 0;
  for (int w = gw; w < nwin; w += nw) {
    const int4 h = __ldg(phdr + w);
    if (h.z == 0) continue;                            // warp-uniform
    const bool act = lane < h.z;
    const int2 d = act ? __ldg(pdesc + h.x + lane) : make_int2(0, 0);
    const int e0 = d.x;
    const uint32_t dsc = (uint32_t)d.y;
    const int rowbeg = (int)(dsc & 31u);
    const int rowlen = (int)((dsc >> 5) & 7u) + 1;
    const int p0 = 2 * (lane - rowbeg);
    const bool has1 = p0 + 1 < rowlen;
    const unsigned heads = __ballot_sync(0xffffffffu, act && p0 == 0);
    const int i = h.w + __popc(heads & ((2u << rowbeg) - 1u)) - 1;
    const double m0 = act ? Bc[v.wcol[e0]] : 0.0;
    const double m1 = (act && has1) ? Bc[v.wcol[e0 + 1]] : 0.0;
    const double wh0 = act ? what[e0] : 0.0;
    const double wh1 = (act && has1) ? what[e0 + 1] : 0.0;
    s_m[wib][2 * lane] = m0 * m0;
    s_m[wib][2 * lane + 1] = m1 * m1;
    s_w[wib][2 * lane] = m0 * wh0;
    s_w[wib][2 * lane + 1] = m1 * wh1;
    __syncwarp();
    double smm = 0.0, smw = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
      if (p < rowlen) { smm += s_m[wib][2 * rowbeg + p]; smw += s_w[wib][2 * rowbeg + p]; }
    __syncwarp();
    if (act) {
      const double rv = B[frow[i]] - smw;
      const double R = sqrt(smm);
      int k = 0;
      double q0 = 0.0, q1 = 0.0, dl0 = 0.0, dl1 = 0.0;
      if (R > 0.0) {
        const double rr = rv / R;
        q0 = m0 / R; q1 = m1 / R;
        dl0 = q0 * rr; dl1 = q1 * rr;
        k = 1;
      }
      Qout[e0] = q0;
      w0[e0] = wh0 + dl0;
      if (has1) { Qout[e0 + 1] = q1; w0[e0 + 1] = wh1 + dl1; }
      if (p0 == 0) {
        n_svd += (k == 0);
        n_frozen += (rowlen == k);
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

// k_spgemm_wd's setup / energy modes (the same records and lookahead loop;
// the lane's row from the window's first row and the head lanes):
//   MM_R0      r0 = -Pi Pi (A P0)|F, the C-identity term A(i, c_j) added  (A1/A2)
//   MM_ENERGY  partial W . (A_FF W + 2 A_FC), W = X + X2 (or X)           (Eq. trInc)
//   MM_R0E     both (setup: they share A P0)
template <int MODE, int NT = WD_NT>
__global__ void __launch_bounds__(NT, 2048 / NT)
k_spgemm_wdm(DevView v, const SpEnt* __restrict__ A, const int4* __restrict__ whdr, const uint32_t* __restrict__ wdesc,
             int32_t nwin, const double* __restrict__ X, const double* __restrict__ X2, double* __restrict__ out,
             double* __restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double s_qa[NT / 32][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const bool two = MODE == MM_ENERGY && X2 != nullptr;
  auto xval = [&](int idx) -> double { return two ? X[idx] + X2[idx] : X[idx]; };
  const int2* I2 = reinterpret_cast<const int2*>(A);
  const double* Ad = reinterpret_cast<const double*>(A);
  double part = 0.0;
  for (int w = gw; w < nwin; w += nw) {
    const int4 h = __ldg(whdr + w);
    const int nent = h.z;
    if (nent == 0) continue;                           // warp-uniform
    const bool act = lane < nent;
    const int e = h.x + lane;
    const uint32_t dsc = act ? __ldg(wdesc + e) : 0u;
    const int rowbeg = (int)(dsc & 31u);
    const int rowlen = (int)((dsc >> 5) & 7u) + 1;
    const int qb = h.y + (int)(dsc >> 16);
    const int qe = qb + (int)((dsc >> 8) & 255u);
    const int pos = lane - rowbeg;
    const unsigned heads = __ballot_sync(0xffffffffu, act && pos == 0);
    const int i = h.w + __popc(heads & ((2u << rowbeg) - 1u)) - 1;
    double acc = 0.0, fc = 0.0, xo = 0.0;
    if (act) {
      xo = xval(e);
      acc = Ad[2 * qb] * xo;                           // diagonal record first
      const unsigned sh4 = 4u * (unsigned)pos;
      int q = qb + 1;
      int2 la0 = (q < qe) ? __ldg(I2 + 2 * q + 1) : make_int2(0, -1);
      int2 la1 = (q + 1 < qe) ? __ldg(I2 + 2 * (q + 1) + 1) : make_int2(0, -1);
#pragma unroll 2
      for (; q < qe; ++q) {
        const int2 cur = la0;
        la0 = la1;
        la1 = (q + 2 < qe) ? __ldg(I2 + 2 * (q + 2) + 1) : make_int2(0, -1);
        const unsigned sidx = ((unsigned)cur.y >> sh4) & 0xFu;
        if (sidx != 0xFu) acc = fma(__ldg(Ad + 2 * q), xval(cur.x + (int)sidx), acc);
      }
      const int32_t j = v.wcol[e];                    // A(i, c_j): search the short A_FC row
      for (int64_t qq = v.afcptr[i]; qq < v.afcptr[i + 1]; ++qq)
        if (v.afccol[qq] == j) { fc = v.afcval[qq]; break; }
    }
    if (MODE == MM_ENERGY || MODE == MM_R0E)
      if (act) part = fma(xo, acc + 2.0 * fc, part);
    if (MODE == MM_ENERGY) continue;                  // warp-uniform (MODE)
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

// k_alg2_nv1 on the window descriptors (k_spgemm_wd's plan): the same
// windows, lanes and sums (bitwise the same Q and W0), without the run-time
// window decode
__global__ void __launch_bounds__(256)
k_alg2_nv1_wd(DevView v, const int4* __restrict__ whdr, const uint32_t* __restrict__ wdesc, int32_t nwin,
              const double* __restrict__ Bc, const double* __restrict__ B, const int64_t* __restrict__ frow,
              const double* __restrict__ what, double* __restrict__ Qout, double* __restrict__ w0,
              unsigned long long* counters) {
  __shared__ unsigned long long cnt[2];
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  unsigned n_svd = 0, n_frozen = 0;
  for (int w = gw; w < nwin; w += nw) {
    const int4 h = __ldg(whdr + w);
    if (h.z == 0) continue;                            // warp-uniform
    WinLane L;
    L.base = h.x;
    L.nent = h.z;
    L.act = lane < h.z;
    const uint32_t dsc = L.act ? __ldg(wdesc + h.x + lane) : 0u;
    L.rowbeg = (int)(dsc & 31u);
    L.rowlen = (int)((dsc >> 5) & 7u) + 1;
    L.pos = lane - L.rowbeg;
    const unsigned heads = __ballot_sync(0xffffffffu, L.act && L.pos == 0);
    L.rloc = __popc(heads & ((2u << L.rowbeg) - 1u)) - 1;
    const int64_t e = L.base + lane;
    const int64_t i = (int64_t)h.w + L.rloc;
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
            const double* __restrict__ dw, const int64_t* __restrict__ pofs, double* __restrict__ out,
            const double* __restrict__ srow) {
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
      // dW = S dW~ under the symmetric scaling
      out[pofs[r0 + L.rloc] + L.pos] = w0[e] + (srow ? srow[r0 + L.rloc] * dw[e] : dw[e]);
    }
  }
}

// ---------------------------------------------------------------------------
// Tiled kernel: one CTA per tile of consecutive rows whose first entry lies
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

constexpr int TILE_SMEM_CAP = 160 * 1024;   // dynamic shared memory of the tile kernel, at most

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

// window headers and lane descriptors of k_spgemm_wd, one thread per window;
// a window whose counts do not fit the descriptor clears *ok
__global__ void k_plan_wdesc(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr,
                             const int32_t* __restrict__ rowstart, int64_t nwin, int4* __restrict__ whdr,
                             uint32_t* __restrict__ wdesc, int32_t* ok) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = rowstart[w], r1 = rowstart[w + 1];
    const int64_t base = wptr[r0], rec = affptr[r0];
    whdr[w] = make_int4((int)base, (int)rec, (int)(wptr[r1] - base), r0);
    for (int i = r0; i < r1; ++i) {
      const int64_t b = wptr[i], len = wptr[i + 1] - b;
      const int64_t rc = affptr[i + 1] - affptr[i], rs = affptr[i] - rec;
      if (len > 8 || rc < 1 || rc > (int64_t)WD_MAXREC || rs > (int64_t)WD_MAXREL) { *ok = 0; continue; }
      const uint32_t d = (uint32_t)(b - base) | ((uint32_t)(len - 1) << 5) | ((uint32_t)rc << 8) | ((uint32_t)rs << 16);
      for (int64_t e = b; e < b + len; ++e) wdesc[e] = d;
    }
  }
}

// one group of 8 lanes per F row, lane per A_FF entry (setup only)
__global__ void k_plan_entries(DevView v, const int32_t* __restrict__ adiag, SpEnt* __restrict__ ent,
                               const double* __restrict__ srow, SpEnt* __restrict__ entS) {
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
    const int64_t qd = qb + adiag[i];             // (k_fill; validation ensures the diagonal)
    for (int64_t q = qb + lg; q < qe; q += 8) {
      const int64_t dst = (q == qd) ? qb : (q < qd ? q + 1 : q);
      const int32_t k = v.affcol[q];
      const int64_t kb = v.wptr[k];
      const int nk = (int)(v.wptr[k + 1] - kb);
      int32_t jk[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) jk[s] = (s < nk) ? v.wcol[kb + s] : -2;
      // nibble t = position of J_i[t] in J_k (0xF absent); the lists hold
      // distinct columns, so at most one s matches a t
      uint32_t pm = 0u;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        uint32_t nib = 0xFu;
#pragma unroll
        for (int s = 0; s < 8; ++s) nib = (ji[t] == jk[s]) ? (uint32_t)s : nib;
        pm |= nib << (4 * t);
      }
      SpEnt e;
      e.a = v.affval[q];
      e.ybase = (int32_t)kb;
      e.pm = pm;
      ent[dst] = e;
      if (entS && q != qd) {          // a~(i,k) = (A(i,k) s_i) s_k, the diagonal left out
        e.a = (e.a * srow[i]) * srow[k];
        entS[dst - i - 1] = e;        // row i's records start at affptr[i] - i
      }
    }
  }
}

// k_spgemm_wp's plan: lane slots per row, ceil(|J_r| / E), and the longest
// record run (the descriptor holds <= WD_MAXREC records per row)
__global__ void k_plan_lane_count(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr, int64_t nF,
                                  int32_t E, int64_t* __restrict__ lcnt, int32_t* __restrict__ maxrc) {
  int32_t m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nF; i += (int64_t)gridDim.x * blockDim.x) {
    lcnt[i] = (wptr[i + 1] - wptr[i] + E - 1) / E;
    const int64_t rc = affptr[i + 1] - affptr[i];
    m = max(m, (int32_t)min(rc, (int64_t)INT32_MAX));
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(maxrc, m);
}
// pair-window headers, one thread per window
// (compact: the record offsets of the diagonal-free records, row i's at
// affptr[i] - i, k_spgemm_wp<SYM>)
__global__ void k_plan_phdr(const int64_t* __restrict__ affptr, const int64_t* __restrict__ lptr,
                            const int32_t* __restrict__ rowstart, int64_t nwin, int32_t compact,
                            int4* __restrict__ phdr) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = rowstart[w], r1 = rowstart[w + 1];
    const int64_t lb = lptr[r0];
    phdr[w] = make_int4((int)lb, (int)(affptr[r0] - (compact ? r0 : 0)), (int)(lptr[r1] - lb), r0);
  }
}
// lane-slot descriptors, one thread per row (row i lies in window
// lptr[i] / S2: rows whose first lane slot lies in [w S2, (w+1) S2)); the
// counts fit: <= 8 entries and <= WD_MAXREC records per row, and <= 31 rows
// per window keep the first record relative to the window below WD_MAXREL
__global__ void k_plan_pdesc(const int64_t* __restrict__ wptr, const int64_t* __restrict__ affptr,
                             const int64_t* __restrict__ lptr, const int32_t* __restrict__ rowstart, int64_t nF,
                             int32_t S2, int32_t E, int32_t compact, int2* __restrict__ pdesc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nF; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l0 = lptr[i], l1 = lptr[i + 1];
    const int r0 = rowstart[l0 / S2];
    const int64_t lb = lptr[r0], rec = affptr[r0] - (compact ? r0 : 0);
    const int64_t len = wptr[i + 1] - wptr[i];
    const int64_t rc = affptr[i + 1] - affptr[i] - (compact ? 1 : 0);
    const int64_t rs = affptr[i] - (compact ? i : 0) - rec;
    const uint32_t d = (uint32_t)(l0 - lb) | ((uint32_t)(len - 1) << 5) | ((uint32_t)rc << 8) | ((uint32_t)rs << 16);
    for (int64_t l = l0; l < l1; ++l) pdesc[l] = make_int2((int)(wptr[i] + E * (l - l0)), (int)d);
  }
}

// s_i = 1 / sqrt(A(i,i)) (symmetric Jacobi scaling)
__global__ void k_rsqrt(const double* __restrict__ d, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = 1.0 / sqrt(d[i]);
}

// x_e = d(row(e)) over the owned W entries, thread per row
__global__ void k_spread_rows(const int64_t* __restrict__ wptr, const double* __restrict__ d, int64_t nF,
                              double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nF; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = wptr[i]; e < wptr[i + 1]; ++e) x[e] = d[i];
}
// s of the halo rows [nF, nFh) from their exchanged first W entry
__global__ void k_halo_rsqrt(const int64_t* __restrict__ wptr, const double* __restrict__ dW, int64_t nF,
                             int64_t nFh, double* __restrict__ srow) {
  for (int64_t i = nF + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nFh; i += (int64_t)gridDim.x * blockDim.x)
    srow[i] = 1.0 / sqrt(dW[wptr[i]]);
}

// ---- host side ------------------------------------------------------------
// S = A(i,i)^-1/2 of the owned F rows and, on several GPUs, of the halo rows
// (their A(i,i) live on the owners: spread over the owned W entries, sent by
// the W-value halo exchange -- collective -- and read back at each halo
// row's first entry)
static emin_status emin_build_srow(emin_ctx c) {
  cudaStream_t s = c->stream;
  const int SM = emin_num_sms();
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&c->srow, sizeof(double) * std::max<int64_t>(c->nFh, 1), s));
  k_rsqrt<<<SM * 4, 256, 0, s>>>(c->d, c->nF, c->srow);
  c->launches += 1;
  if (c->dist) {
    double* dW = nullptr;
    EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&dW, sizeof(double) * std::max<int64_t>(c->nnzWh, 1), s));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));       // the peers copy into it from their streams
    k_spread_rows<<<SM * 8, 256, 0, s>>>(c->wptr, c->d, c->nF, dW);
    const emin_status st = emin_dist_halo_values(c, dW, s);
    if (st != EMIN_OK) return st;
    k_halo_rsqrt<<<SM * 4, 256, 0, s>>>(c->wptr, dW, c->nF, c->nFh, c->srow);
    cudaFreeAsync(dW, s);
    c->launches += 2;
  }
  return cudaGetLastError() == cudaSuccess ? EMIN_OK : EMIN_ERR_CUDA;
}

struct FastPaths {
  ScalarPlan sc;
};
static FastPaths* fast_of(emin_ctx c) { return reinterpret_cast<FastPaths*>(c->fast); }

static inline int select_fast_path(emin_ctx c) {
  if (c->nv != 1 || c->max_row > 8 || c->nnzWh >= INT32_MAX || c->nF >= INT32_MAX || c->nnzAFF >= INT32_MAX ||
      c->nF == 0)
    return 0;
  if (c->opts.debug_flags & EMIN_DBG_FORCE_GENERIC) return 0;
  FastPaths* f = new FastPaths();
  c->fast = f;
  ScalarPlan& p = f->sc;
  p.S = std::min(31, 33 - c->max_row);   // <= 31 rows per window (lane nrows loads the end)
  p.nwin = (c->nnzW + p.S - 1) / p.S;
  cudaStream_t s = c->stream;
  if (emin_mallocAsync((void**)&p.rowstart, sizeof(int32_t) * (p.nwin + 1), s) != cudaSuccess) return 0;
  if (emin_mallocAsync((void**)&p.ent, sizeof(SpEnt) * (size_t)(c->nnzAFF + WP_PAD), s) != cudaSuccess) return 0;
  cudaMemsetAsync(p.ent + c->nnzAFF, 0, sizeof(SpEnt) * WP_PAD, s);
  const int SM = emin_num_sms();
  k_plan_rowstart<<<SM * 8, 256, 0, s>>>(c->wptr, c->nF, p.S, p.nwin, p.rowstart);
  // lane slots of the pair-lane kernel (k_spgemm_wp) and the longest record run
  int64_t* lscr = nullptr;
  int32_t* dmaxrc = nullptr;
  if (emin_mallocAsync((void**)&p.lptr, sizeof(int64_t) * (c->nF + 1), s) != cudaSuccess ||
      emin_mallocAsync((void**)&lscr, sizeof(int64_t) * emin_scan_scratch_elems(c->nF + 1), s) != cudaSuccess ||
      emin_mallocAsync((void**)&dmaxrc, sizeof(int32_t), s) != cudaSuccess)
    return 0;
  cudaMemsetAsync(dmaxrc, 0, sizeof(int32_t), s);
  k_plan_lane_count<<<SM * 8, 256, 0, s>>>(c->wptr, c->affptr, c->nF, 2, p.lptr, dmaxrc);   // two entries per lane
  if (emin_scan_i64(p.lptr, p.lptr, c->nF, p.lptr + c->nF, lscr, s) != cudaSuccess) return 0;
  c->launches += 5;
  // several GPUs: every rank takes the same branch below (collectives follow)
  if (c->dist && emin_dist_allreduce_max_i32(c, dmaxrc, s) != EMIN_OK) return 0;
  int64_t hL = 0;
  int32_t hmaxrc = 0;
  cudaMemcpyAsync(&hmaxrc, dmaxrc, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hL, p.lptr + c->nF, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaFreeAsync(lscr, s);
  cudaFreeAsync(dmaxrc, s);
  const bool pair_ok = hmaxrc <= (int32_t)WD_MAXREC;
  // symmetric Jacobi scaling of the CG (see emin_ctx_s::sym): one GPU,
  // Jacobi without the post-projection, on the pair-lane kernel; its records
  // of S A_FF S leave out the diagonal ((S A S)_ii = 1: s_i = A(i,i)^-1/2)
  c->sym = (pair_ok && c->opts.precond == EMIN_PREC_JACOBI && !c->opts.project_after_jacobi &&
            !(c->opts.debug_flags & (EMIN_DBG_UNSCALED | EMIN_DBG_AB2))) ? 1 : 0;
  if (c->sym) {
    const int64_t nS = c->nnzAFF - c->nF;
    if (emin_mallocAsync((void**)&p.entS, sizeof(SpEnt) * (size_t)(nS + WP_PAD), s) != cudaSuccess) return 0;
    cudaMemsetAsync(p.entS + nS, 0, sizeof(SpEnt) * WP_PAD, s);
    if (emin_build_srow(c) != EMIN_OK) return 0;
  }
  // short in-order CTAs (kernel-plan phase 0.45 -> 0.37 ms on config 3)
  k_plan_entries<<<SM * 32, 256, 0, s>>>(c->view(), c->adiag, p.ent, c->srow, p.entS);
  c->launches += 1;
  if (hmaxrc <= (int32_t)WD_MAXREC) {
    // pair windows: rows whose first lane slot lies in [w S2, (w+1) S2)
    const int32_t S2 = std::min(31, 33 - (c->max_row + 1) / 2);
    p.npwin = (hL + S2 - 1) / S2;
    if (emin_mallocAsync((void**)&p.prowstart, sizeof(int32_t) * (p.npwin + 1), s) != cudaSuccess ||
        emin_mallocAsync((void**)&p.phdr, sizeof(int4) * std::max<int64_t>(p.npwin, 1), s) != cudaSuccess ||
        emin_mallocAsync((void**)&p.pdesc, sizeof(int2) * std::max<int64_t>(hL, 1), s) != cudaSuccess)
      return 0;
    k_plan_rowstart<<<SM * 8, 256, 0, s>>>(p.lptr, c->nF, S2, p.npwin, p.prowstart);
    k_plan_phdr<<<SM * 4, 256, 0, s>>>(c->affptr, p.lptr, p.prowstart, p.npwin, c->sym, p.phdr);
    k_plan_pdesc<<<SM * 8, 256, 0, s>>>(c->wptr, c->affptr, p.lptr, p.prowstart, c->nF, S2, 2, c->sym, p.pdesc);
    c->launches += 3;
    if (c->opts.debug_flags & EMIN_DBG_AB2) {
      // window headers + lane descriptors of k_spgemm_wd, the one-entry-per-
      // lane reference (its counts fit whenever the pair plan's do)
      int32_t* dok = nullptr;
      if (emin_mallocAsync((void**)&p.whdr, sizeof(int4) * std::max<int64_t>(p.nwin, 1), s) != cudaSuccess ||
          emin_mallocAsync((void**)&p.wdesc, sizeof(uint32_t) * std::max<int64_t>(c->nnzW, 1), s) != cudaSuccess ||
          emin_mallocAsync((void**)&dok, sizeof(int32_t), s) != cudaSuccess)
        return 0;
      k_plan_wdesc<<<SM * 8, 256, 0, s>>>(c->wptr, c->affptr, p.rowstart, p.nwin, p.whdr, p.wdesc, dok);
      cudaFreeAsync(dok, s);
      c->launches += 1;
    }
  }
  // the staged tile kernel (setup / energy modes) is needed only without the
  // window descriptors (or as the test reference, debug bit 256)
  if ((p.phdr || p.whdr) && !(c->opts.debug_flags & 256)) return 1;
  // tile plan for the staged setup / energy kernel
  const int ST = TILE_E - c->max_row + 1;
  p.ntiles = (c->nnzW + ST - 1) / ST;
  int32_t* trow = nullptr;
  int32_t* dmax = nullptr;
  int32_t hmax[2] = {0, 0};
  if (emin_mallocAsync((void**)&trow, sizeof(int32_t) * (p.ntiles + 1), s) != cudaSuccess ||
      emin_mallocAsync((void**)&p.hdr, sizeof(TileHdr) * std::max<int64_t>(p.ntiles, 1), s) != cudaSuccess ||
      emin_mallocAsync((void**)&dmax, sizeof(int32_t) * 2, s) != cudaSuccess)
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
  if (p.tile_smem <= TILE_SMEM_CAP) {
    p.use_tiles = 1;
    // the attribute is per kernel and process-wide: always the cap, never the
    // size of this context's tiles (contexts set up concurrently by several
    // threads must not lower it under each other's launches)
    cudaFuncSetAttribute(k_spgemm_tile<MM_R0>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM_CAP);
    cudaFuncSetAttribute(k_spgemm_tile<MM_ENERGY>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM_CAP);
    cudaFuncSetAttribute(k_spgemm_tile<MM_R0E>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM_CAP);
  }
  return 1;
}

// grid of the window kernels: short in-order CTAs, 8 per SM (one wave at
// the 256-thread launch bound)
static inline int scalar_grid(emin_ctx c) {
  const int SM = emin_num_sms();
  const int64_t nwin = fast_of(c)->sc.nwin;
  return (int)std::max<int64_t>(1, std::min<int64_t>((nwin + 7) / 8, (int64_t)SM * 8));
}
// grid of the per-iteration masked launch (MM_ITER)
// (k_spgemm_wd: 1024-thread CTAs, 2 per SM -- a CTA's 32 consecutive
// windows share neighbour y rows in its SM's L1: 114.7 vs 116.8 us with
// 256-thread CTAs, config 3)
static inline int scalar_iter_grid(emin_ctx c) {
  const ScalarPlan& p = fast_of(c)->sc;
  if (!p.whdr) return scalar_grid(c);
  const int per = 2048 / WD_NT;
  return (int)std::max<int64_t>(1, std::min<int64_t>((p.nwin + WD_NT / 32 - 1) / (WD_NT / 32),
                                                     (int64_t)emin_num_sms() * per));
}
// grid of the per-iteration launch (the kernel launch_scalar_masked picks)
static inline int scalar_iter_launch_grid(emin_ctx c) {
  const ScalarPlan& p = fast_of(c)->sc;
  if (!(p.phdr && !(c->opts.debug_flags & EMIN_DBG_AB2))) return scalar_iter_grid(c);
  if (c->sym)
    return (int)std::max<int64_t>(1, std::min<int64_t>((p.npwin + WPS_NT / 32 - 1) / (WPS_NT / 32),
                                                       (int64_t)emin_num_sms() * WPS_MINB));
  return (int)std::max<int64_t>(1, std::min<int64_t>((p.npwin + WP_NT / 32 - 1) / (WP_NT / 32),
                                                     (int64_t)emin_num_sms() * WP_MINB));
}
// the per-iteration kernel's units (windows): pair windows unless wd runs
static inline const int32_t* scalar_iter_windows(emin_ctx c, int64_t* nwin) {
  const ScalarPlan& p = fast_of(c)->sc;
  if (p.phdr && !(c->opts.debug_flags & EMIN_DBG_AB2)) { *nwin = p.npwin; return p.prowstart; }
  *nwin = p.nwin;
  return p.rowstart;
}

// grid of the setup-time masked launches (MM_R0, MM_R0E, MM_ENERGY): the
// window-descriptor kernel's, else the tile kernel's (or win2m's)
static inline int scalar_spgemm_grid(emin_ctx c) {
  const ScalarPlan& p = fast_of(c)->sc;
  if (p.phdr && !(c->opts.debug_flags & (256 | EMIN_DBG_AB2)))      // k_spgemm_wpm: 512 x 3 per SM
    return (int)std::max<int64_t>(1, std::min<int64_t>((p.npwin + WP_NT / 32 - 1) / (WP_NT / 32),
                                                       (int64_t)emin_num_sms() * WP_MINB));
  if (p.whdr && !(c->opts.debug_flags & 256)) return scalar_iter_grid(c);
  return p.use_tiles ? (int)std::max<int64_t>(1, p.ntiles) : scalar_grid(c);
}
static inline bool launch_scalar_masked(emin_ctx c, int mode, const double* X, const double* X2, double* out,
                                        cudaStream_t s) {
  const ScalarPlan& p = fast_of(c)->sc;
  const DevView v = c->view();
  if (mode == MM_ITER) {
    // two W entries per lane on precomputed pair windows (config 3: 91.4 us
    // vs wd's 110.6 and win2's 120.2, profiles/r02/spgemm_ab_c3.txt); wd is
    // the A/B reference (EMIN_DBG_AB2); win2 when a window's counts overflow
    // the lane descriptor
    if (c->sym)          // S A_FF S (unit diagonal) on the pair windows
      k_spgemm_wp<WPS_NT, WPS_MINB, WPS_UNR, 2, true><<<scalar_iter_launch_grid(c), WPS_NT, 0, s>>>(
          v, p.entS, p.phdr, p.pdesc, (int32_t)p.npwin, X, out, c->partials);
    else if (p.phdr && !(c->opts.debug_flags & EMIN_DBG_AB2))
      k_spgemm_wp<WP_NT, WP_MINB, WP_UNR, 2><<<scalar_iter_launch_grid(c), WP_NT, 0, s>>>(
          v, p.ent, p.phdr, p.pdesc, (int32_t)p.npwin, X, out, c->partials);
    else if (p.whdr)
      k_spgemm_wd<WD_NT, WD_LA, true><<<scalar_iter_grid(c), WD_NT, 0, s>>>(v, p.ent, p.whdr, p.wdesc,
                                                                          (int32_t)p.nwin, X, out, c->partials);
    else
      k_spgemm_win2<2><<<scalar_grid(c), 256, 0, s>>>(v, p.ent, p.rowstart, p.nwin, X, out, c->partials);
    return true;
  }
  if (p.phdr && !(c->opts.debug_flags & (256 | EMIN_DBG_AB2))) {
    const int g = scalar_spgemm_grid(c);
    const int np = (int)p.npwin;
    if (mode == MM_R0E)
      k_spgemm_wpm<MM_R0E><<<g, WP_NT, 0, s>>>(v, p.ent, p.phdr, p.pdesc, np, X, X2, out, c->partials,
                                              c->sym);
    else if (mode == MM_R0)
      k_spgemm_wpm<MM_R0><<<g, WP_NT, 0, s>>>(v, p.ent, p.phdr, p.pdesc, np, X, X2, out, c->partials,
                                              c->sym);
    else
      k_spgemm_wpm<MM_ENERGY><<<g, WP_NT, 0, s>>>(v, p.ent, p.phdr, p.pdesc, np, X, X2, out, c->partials,
                                              c->sym);
    return true;
  }
  if (p.whdr && !(c->opts.debug_flags & 256)) {
    const int g = scalar_iter_grid(c);
    if (mode == MM_R0E)
      k_spgemm_wdm<MM_R0E><<<g, WD_NT, 0, s>>>(v, p.ent, p.whdr, p.wdesc, (int32_t)p.nwin, X, X2, out, c->partials);
    else if (mode == MM_R0)
      k_spgemm_wdm<MM_R0><<<g, WD_NT, 0, s>>>(v, p.ent, p.whdr, p.wdesc, (int32_t)p.nwin, X, X2, out, c->partials);
    else
      k_spgemm_wdm<MM_ENERGY><<<g, WD_NT, 0, s>>>(v, p.ent, p.whdr, p.wdesc, (int32_t)p.nwin, X, X2, out,
                                                  c->partials);
    return true;
  }
  if (mode == MM_R0E) {                      // fused r0 + E0: the tile kernel only
    if (!p.use_tiles) return false;
    k_spgemm_tile<MM_R0E><<<(int)std::max<int64_t>(1, p.ntiles), TILE_T, p.tile_smem, s>>>(v, p.ent, p.hdr, X, X2,
                                                                                         out, c->partials);
    return true;
  }
  if (!p.use_tiles) {
    // a tile's records exceed shared memory: win2's window kernel (measured
    // slower than the tile kernel on config 3: emin_energy 0.34 vs 0.28 ms)
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
  if (p.phdr && !(c->opts.debug_flags & EMIN_DBG_AB2))
    k_alg2_nv1_wp<<<(int)std::max<int64_t>(1, std::min<int64_t>((p.npwin + 7) / 8, (int64_t)emin_num_sms() * 8)), 256,
                    0, s>>>(c->view(), p.phdr, p.pdesc, (int32_t)p.npwin, Bc, B, frow, what, c->Q, c->w0, counters);
  else if (p.whdr)
    k_alg2_nv1_wd<<<scalar_grid(c), 256, 0, s>>>(c->view(), p.whdr, p.wdesc, (int32_t)p.nwin, Bc, B, frow, what,
                                                 c->Q, c->w0, counters);
  else
    k_alg2_nv1<<<scalar_grid(c), 256, 0, s>>>(c->view(), p.rowstart, p.nwin, Bc, B, frow, what, c->Q, c->w0,
                                              counters);
}
static inline void launch_scalar_get_P(emin_ctx c, double* out, cudaStream_t s) {
  const ScalarPlan& p = fast_of(c)->sc;
  k_get_P_win<<<scalar_grid(c), 256, 0, s>>>(c->view(), p.rowstart, p.nwin, c->w0, c->dw, c->pofs, out,
                                             c->sym ? c->srow : nullptr);
}

static inline void free_fast_path(emin_ctx c) {
  FastPaths* f = fast_of(c);
  if (!f) return;
  if (f->sc.rowstart) cudaFreeAsync(f->sc.rowstart, c->stream);
  if (f->sc.whdr) cudaFreeAsync(f->sc.whdr, c->stream);
  if (f->sc.wdesc) cudaFreeAsync(f->sc.wdesc, c->stream);
  if (f->sc.lptr) cudaFreeAsync(f->sc.lptr, c->stream);
  if (f->sc.prowstart) cudaFreeAsync(f->sc.prowstart, c->stream);
  if (f->sc.phdr) cudaFreeAsync(f->sc.phdr, c->stream);
  if (f->sc.pdesc) cudaFreeAsync(f->sc.pdesc, c->stream);
  if (f->sc.ent) cudaFreeAsync(f->sc.ent, c->stream);
  if (f->sc.entS) cudaFreeAsync(f->sc.entS, c->stream);
  if (f->sc.hdr) cudaFreeAsync(f->sc.hdr, c->stream);
  delete f;
  c->fast = nullptr;
}
