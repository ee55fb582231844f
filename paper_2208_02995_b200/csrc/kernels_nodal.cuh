// kernels_nodal.cuh -- nodal (3x3 block) path for vector problems
// (elasticity, configs 4-5; kernel_path 2), selected when emin_opts.block_size
// = 3 and the structure checks pass.
//
// Rows 3n..3n+2 of an F node n share the pattern J_n (blockwise: columns
// 3c, 3c+1, 3c+2 for every C node c in J_n) and hence the same M_i =
// B_c(J_i,:) and the same Q_i; A_FF is made of dense 3x3 blocks (I,K).  The
// masked product of node I is then
//     Yb(I,d; c,b) = sum_K sum_d' A_IK[d][d'] Y(K,d'; c,b),  c in J_I n J_K
// computed by one warp per node: lane t owns the pattern positions t and
// t+32 (t = 3 s + b: C node s of J_I, component b) for all three output rows
// d, so each matched (block, position) costs 3 gathers and 9 FMAs and the
// node-level match (s in J_I -> s_K in J_K) is read once per block and lane
// from a byte map built at setup.  Q is read once per node (row 3I) instead
// of three times.
#pragma once
#include "emin_internal.cuh"
#include "masked.cuh"

struct NodalBlk {      // one per A_FF 3x3 block (I,K)
  int32_t ybase;       // wptr[3K]: first W entry of the neighbour node
  int32_t nK3;         // 3 |J_K|: row length of the neighbour node
};

struct NodalPlan {
  int64_t nFn = 0;            // owned F nodes
  NodalBlk* blk = nullptr;    // [nblk]
  int64_t* bptr = nullptr;    // [nFn+1] block offset of node n (= affptr[3n] / 9)
  uint8_t* pm8 = nullptr;     // [sum_n nblk_n |J_n|] position of J_I[s] in J_K, 0xFF absent
  int64_t* pmoff = nullptr;   // [nFn+1]
  int64_t nblk = 0, npm = 0;
  int32_t max_nb = 0;         // most blocks of one node (> ND_MAXB: v2 stages in chunks; SGS goes generic)
};

// structure checks, one warp per F node (lanes over pattern positions and A
// entries, coalesced); any violation clears *ok
__global__ void k_nodal_check(DevView v, int64_t nFn, int32_t* ok, int64_t* pm_len, int32_t* max_nb) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = gw; n < nFn; n += nw) {
    const int64_t r = 3 * n;
    const int64_t wb = v.wptr[r];
    const int64_t len = v.wptr[r + 1] - wb;
    bool good = (len % 3 == 0) && len > 0 && len <= 64;     // two 32-lane chunks per node
    for (int d = 1; d < 3 && good; ++d) good = (v.wptr[r + d + 1] - v.wptr[r + d]) == len;
    bool lg = true;
    if (good)
      for (int64_t t = lane; t < len; t += 32) {
        const int32_t c = v.wcol[wb + t];
        if ((t % 3 == 0 && c % 3 != 0) || (t % 3 != 0 && c != v.wcol[wb + t - 1] + 1)) lg = false;
        for (int d = 1; d < 3; ++d) lg = lg && v.wcol[v.wptr[r + d] + t] == c;
      }
    const int64_t ab = v.affptr[r];
    const int64_t alen = v.affptr[r + 1] - ab;
    good = good && (alen % 3 == 0);
    for (int d = 1; d < 3 && good; ++d) good = (v.affptr[r + d + 1] - v.affptr[r + d]) == alen;
    if (good)
      for (int64_t q = lane; q < alen; q += 32) {
        const int32_t k = v.affcol[ab + q];
        if ((q % 3 == 0 && k % 3 != 0) || (q % 3 != 0 && k != v.affcol[ab + q - 1] + 1)) lg = false;
        for (int d = 1; d < 3; ++d) lg = lg && v.affcol[v.affptr[r + d] + q] == k;
      }
    good = __all_sync(0xffffffffu, good && lg);
    if (lane == 0) {
      if (!good) atomicExch(ok, 0);
      else atomicMax(max_nb, (int32_t)(alen / 3));
      // (each node's byte map starts 16-byte aligned: staged with 16-byte loads)
      pm_len[n] = good ? (((alen / 3) * (len / 3) + 15) & ~(int64_t)15) : 0;
    }
  }
}

// per node: block records and the byte position map, one warp per node
// (lane per block: the merge of the sorted node lists J_I and J_K)
__global__ void k_nodal_build(DevView v, int64_t nFn, const int64_t* __restrict__ pmoff, NodalBlk* __restrict__ blk,
                              int64_t* __restrict__ bptr, uint8_t* __restrict__ pm8) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = gw; n < nFn; n += nw) {
    const int64_t r = 3 * n;
    const int64_t wb = v.wptr[r];
    const int nJ = (int)((v.wptr[r + 1] - wb) / 3);
    const int64_t ab = v.affptr[r];
    const int nb = (int)((v.affptr[r + 1] - ab) / 3);
    const int64_t b0 = ab / 9;
    if (lane == 0) {
      bptr[n] = b0;
      if (n == nFn - 1) bptr[nFn] = v.affptr[3 * nFn] / 9;
    }
    const int64_t po = pmoff[n];
    for (int b = lane; b < nb; b += 32) {
      const int32_t K = v.affcol[ab + 3 * b] / 3;
      const int64_t kb = v.wptr[3 * (int64_t)K];
      const int nK = (int)((v.wptr[3 * (int64_t)K + 1] - kb) / 3);
      NodalBlk nbk;
      nbk.ybase = (int32_t)kb;
      nbk.nK3 = 3 * nK;
      blk[b0 + b] = nbk;
      int sK = 0;
      for (int s = 0; s < nJ; ++s) {
        const int32_t c = v.wcol[wb + 3 * s];
        while (sK < nK && v.wcol[kb + 3 * sK] < c) ++sK;
        pm8[po + (int64_t)b * nJ + s] = (sK < nK && v.wcol[kb + 3 * sK] == c) ? (uint8_t)sK : (uint8_t)0xFF;
      }
    }
  }
}

constexpr int ND_WARPS = 8;
constexpr int ND_MAXB = 27;      // blocks per node (27-point node stencil)
constexpr int ND_MAXJ = 32;      // C nodes per pattern row (3|J| <= 96 entries -> 2 chunks of 32 needs |J| <= 21)

// ---------------------------------------------------------------------------
// v2: the round-1 staged kernel (k_spgemm_nodal_s, profiles/ab_r01/), cut down to
// what the L1 data pipe must carry (profiles/r01: the staged kernel was
// bound by L1/shared wavefronts, 74 % of peak, not by DRAM):
//  * the 3x3 block is read ONCE per block for both lane chunks, as five
//    16-byte shared loads (block-major, 10-double stride) instead of 2 x 9
//    8-byte loads;
//  * Pi_B's nv dots of each of the 3 rows are reduced by a recursive-halving
//    butterfly (a lane ends owning one dot; 8 doubles exchanged per row for
//    nv = 6) and broadcast through shared memory, instead of nv full
//    warp_sum butterflies per row (30 doubles);
//  * 32-bit entry indices (nnz(W) < 2^31 is checked at plan time).
// The per-entry arithmetic (block order, 9 FMAs in (d, e) order per block)
// is unchanged, so y^ is bitwise equal to the staged kernel's except for the
// order of the nv-dot sums.
// ---------------------------------------------------------------------------
constexpr int ND2_AST = 10;      // doubles per staged block (9 + pad, 16-byte aligned)

// recursive-halving reduce-scatter of N values over the 32 lanes.  The N
// values are padded to P = 2^ceil(log2 N); each halving stage splits a
// lane's index range with its xor partner (disjoint ranges), and once a
// range is a single index the remaining stages are plain xor adds (the two
// partners compute a + b and b + a: bitwise equal).  On return the lane
// holds in v[0] the full 32-lane sum of value index *own (valid iff
// *own < N; a valid index may be held, bitwise equal, by several lanes).
template <int S, int OFF>
struct Nd2Rs {
  static __device__ __forceinline__ void run(double* a, int lane, int& lo) {
    if constexpr (OFF > 0) {
      if constexpr (S > 1) {
        constexpr int H = S / 2;
        const bool lower = !(lane & OFF);
#pragma unroll
        for (int i = 0; i < H; ++i) {
          const double send = lower ? a[H + i] : a[i];
          const double recv = __shfl_xor_sync(0xffffffffu, send, OFF);
          a[i] = (lower ? a[i] : a[H + i]) + recv;
        }
        if (!lower) lo += H;
        Nd2Rs<H, OFF / 2>::run(a, lane, lo);
      } else {
        a[0] += __shfl_xor_sync(0xffffffffu, a[0], OFF);
        Nd2Rs<1, OFF / 2>::run(a, lane, lo);
      }
    }
  }
};

template <int N>
__device__ __forceinline__ void nd2_reduce_scatter(double (&v)[N], int lane, int* own) {
  constexpr int P = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : 32;
  static_assert(N <= 32, "N <= 32");
  double a[P];
#pragma unroll
  for (int i = 0; i < P; ++i) a[i] = i < N ? v[i] : 0.0;
  int lo = 0;
  Nd2Rs<P, 16>::run(a, lane, lo);
  v[0] = a[0];
  *own = lo;
}

// masked-product sums of one pattern position (C node s, component bc) over
// the staged blocks bstart, bstart + bstep, ... < cb of a node: GRP blocks per
// round, the (3 GRP) gathers of the round issued before its FMAs, which run
// in ascending block order, 9 per matched block in (d, e) order.  Lanes of
// a warp may take different blocks (the second chunk's groups).
template <int GRP, typename XV>
__device__ __forceinline__ void nd2_accum(const double* __restrict__ sa, const uint8_t* __restrict__ spm, int nJ, int cb, int bstart, int bstep,
                                          int s, int bc, bool act, XV xval, double (&acc)[3]) {
  for (int b = bstart; b < cb; b += GRP * bstep) {
    double y[GRP][3], a8[GRP];
    bool m[GRP];
#pragma unroll
    for (int g = 0; g < GRP; ++g) {
      const int bg = b + g * bstep;
      const bool has = act && bg < cb;
      const double2 t = reinterpret_cast<const double2*>(sa + (has ? bg : b) * ND2_AST)[4];
      a8[g] = t.x;
      const NodalBlk k{(int32_t)__double2loint(t.y), (int32_t)__double2hiint(t.y)};
      const int p = has ? spm[bg * nJ + s] : 0xFF;
      m[g] = p != 0xFF;
      const int i = k.ybase + 3 * (m[g] ? p : 0) + bc;
#pragma unroll
      for (int e = 0; e < 3; ++e) y[g][e] = m[g] ? xval(i + e * k.nK3) : 0.0;
    }
#pragma unroll
    for (int g = 0; g < GRP; ++g) {
      if (m[g]) {
        const double2* a2 = reinterpret_cast<const double2*>(sa + (b + g * bstep) * ND2_AST);
        const double2 a01 = a2[0], a23 = a2[1], a45 = a2[2], a67 = a2[3];
        const double a[9] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y, a8[g]};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          acc[d] = fma(a[d * 3 + 0], y[g][0], acc[d]);
          acc[d] = fma(a[d * 3 + 1], y[g][1], acc[d]);
          acc[d] = fma(a[d * 3 + 2], y[g][2], acc[d]);
        }
      }
    }
  }
}

template <int NV, int MODE, bool CS = false, bool WIDE = false, int GRP = 1, int MINB = 4>
__global__ void __launch_bounds__(ND_WARPS * 32, MINB)
k_spgemm_nodal_v2(DevView v, const NodalBlk* __restrict__ blk, const int64_t* __restrict__ bptr,
                  const uint8_t* __restrict__ pm8, const int64_t* __restrict__ pmoff, int64_t nFn,
                  const double* __restrict__ X, const double* __restrict__ X2, double* __restrict__ out,
                  double* __restrict__ partials) {
  __shared__ double sh[32];
  // per warp: the A chunk block-major at a 10-double stride with the block
  // record {ybase, 3|J_K|} in each block's 10th slot (read with a8 by one
  // 16-byte load), and the byte map
  __shared__ __align__(16) double s_a[ND_WARPS][ND_MAXB * ND2_AST];
  __shared__ __align__(16) uint8_t s_pm[ND_WARPS][ND_MAXB * ND_MAXJ];
  __shared__ __align__(16) double s_dot[ND_WARPS][3 * NV + 1];
  if (MODE == MM_ITER && v.st->stopped) { iter_stopped(v); return; }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // MM_ENERGY: W = X + X2, or X alone when the caller summed it (X2 null)
  const bool two = MODE == MM_ENERGY && X2 != nullptr;
  auto xval = [&](int idx) -> double { return two ? X[idx] + X2[idx] : X[idx]; };
  const int t0 = lane, t1 = lane + 32;
  const int s0 = t0 / 3, b0 = t0 - 3 * s0;
  double part = 0.0;
  const int64_t ncnt = unit_count(v, nFn);
  for (int64_t n1 = gw; n1 < ncnt; n1 += nw) {
    const int64_t n = unit_of(v, n1);
    const int64_t r = 3 * n;
    const int wb = (int)v.wptr[r];
    const int n3 = (int)v.wptr[r + 1] - wb;
    const int nJ = n3 / 3;
    const int64_t ab = v.affptr[r];
    const int64_t bb = bptr[n];
    const int nb = (int)(bptr[n + 1] - bb);
    const int64_t po = pmoff[n];
    const int rs = 3 * nb;
    const bool act0 = t0 < n3, act1 = t1 < n3;
    const bool any1 = n3 > 32;                          // warp-uniform
    // lanes per position of the second chunk: 32 / 2^ceil(log2(n3 - 32))
    const int l1sh = any1 ? __clz(n3 - 33) - 27 : 0;    // log2 L1 (n3 - 32 in [1, 32])
    const int L1 = 1 << l1sh;
    double acc0[3] = {0.0, 0.0, 0.0}, acc1[3] = {0.0, 0.0, 0.0};
    // nodes with more than ND_MAXB blocks (Galerkin operators of coarse
    // levels, NEXT-4) are staged ND_MAXB blocks at a time, same block order
    // (template WIDE; otherwise the one chunk is the whole node, c0 = 0)
    for (int cl = 0; cl < nb; cl += WIDE ? ND_MAXB : nb) {
    const int c0 = WIDE ? cl : 0;
    const int cb = WIDE ? min(ND_MAXB, nb - c0) : nb, cs = 3 * cb;
    if (WIDE && c0) __syncwarp();
    // ---- stage the chunk (A row by row, re-ordered block-major)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double* srow = v.affval + ab + (int64_t)d * rs + 3 * c0;
      for (int j = lane; j < cs; j += 32) {
        const int b = j / 3, e = j - 3 * b;
        s_a[wib][b * ND2_AST + d * 3 + e] = CS ? __ldcs(srow + j) : __ldg(srow + j);
      }
    }
    for (int k = lane; k < cb; k += 32) {
      const int2 t = CS ? __ldcs(reinterpret_cast<const int2*>(blk + bb + c0 + k))
                        : *reinterpret_cast<const int2*>(blk + bb + c0 + k);
      *reinterpret_cast<int2*>(&s_a[wib][k * ND2_AST + 9]) = t;
    }
    if (!WIDE) {
      // 16-byte loads (the node's map is 16-byte aligned, padded)
      const uint4* src4 = reinterpret_cast<const uint4*>(pm8 + po);
      uint4* dst4 = reinterpret_cast<uint4*>(&s_pm[wib][0]);
      for (int k = lane; k < ((cb * nJ + 15) >> 4); k += 32) dst4[k] = CS ? __ldcs(src4 + k) : src4[k];
    } else
      for (int k = lane; k < cb * nJ; k += 32) {
        const int64_t src = po + (int64_t)c0 * nJ + k;
        s_pm[wib][k] = CS ? (uint8_t)__ldcs(reinterpret_cast<const char*>(pm8 + src)) : pm8[src];
      }
    __syncwarp();
    // positions 0..31: one lane per position, every block of the chunk
    nd2_accum<GRP>(&s_a[wib][0], &s_pm[wib][0], nJ, cb, 0, 1, s0, b0, act0, xval, acc0);
    // positions 32..n3-1 (n3 <= 64): L1 lanes per position, lane sub of a
    // group taking blocks sub, sub + L1, ...; the group's partial sums are
    // combined after the last chunk (elasticity: n3 = 36, 4 positions x 8
    // lanes, 4 rounds per node instead of 27 with 28 of 32 lanes idle)
    if (any1) {
      const int h = lane >> l1sh, sub = lane & (L1 - 1);
      const int t = 32 + h, s = t / 3;
      nd2_accum<GRP>(&s_a[wib][0], &s_pm[wib][0], nJ, cb, sub, L1, s, t - 3 * s, t < n3, xval, acc1);
    }
    }  // chunks of ND_MAXB blocks
    if (any1) {
      // sum each group's L1 partials (xor butterfly inside the aligned group),
      // lane h < n3 - 32 takes group h's sum for position 32 + h
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        for (int o = L1 >> 1; o > 0; o >>= 1) acc1[d] += __shfl_xor_sync(0xffffffffu, acc1[d], o);
        const double gs = __shfl_sync(0xffffffffu, acc1[d], act1 ? lane << l1sh : 0);
        acc1[d] = act1 ? gs : 0.0;
      }
    }
    double g0[3], g1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) { g0[d] = acc0[d]; g1[d] = acc1[d]; }
    if (MODE != MM_ITER) {            // C-identity term A(i, c_j) (setup / energy only)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int64_t fb = v.afcptr[r + d], fe = v.afcptr[r + d + 1];
        const int ro = wb + d * n3;
        double f0 = 0.0, f1 = 0.0;
        if (act0) {
          const int32_t j = v.wcol[ro + t0];
          for (int64_t q = fb; q < fe; ++q) if (v.afccol[q] == j) { f0 = v.afcval[q]; break; }
        }
        if (act1) {
          const int32_t j = v.wcol[ro + t1];
          for (int64_t q = fb; q < fe; ++q) if (v.afccol[q] == j) { f1 = v.afcval[q]; break; }
        }
        if (MODE == MM_ENERGY || MODE == MM_R0E) {
          if (act0) part = fma(xval(ro + t0), g0[d] + 2.0 * f0, part);
          if (act1) part = fma(xval(ro + t1), g1[d] + 2.0 * f1, part);
        }
        if (MODE != MM_ENERGY) {
          g0[d] += f0;
          g1[d] += f1;
        }
      }
    }
    if (MODE != MM_ENERGY) {
      // Q of the node (row 3n, shared by its 3 rows): 16-byte loads
      double q0[NV], q1[NV];
#pragma unroll
      for (int m = 0; m < NV; ++m) { q0[m] = 0.0; q1[m] = 0.0; }
      if ((NV & 1) == 0) {
        if (act0) {
          const double2* qp = reinterpret_cast<const double2*>(v.Q + (int64_t)(wb + t0) * NV);
#pragma unroll
          for (int m = 0; m < NV / 2; ++m) { const double2 t = CS ? __ldcs(qp + m) : __ldg(qp + m); q0[2 * m] = t.x; q0[2 * m + 1] = t.y; }
        }
        if (act1) {
          const double2* qp = reinterpret_cast<const double2*>(v.Q + (int64_t)(wb + t1) * NV);
#pragma unroll
          for (int m = 0; m < NV / 2; ++m) { const double2 t = CS ? __ldcs(qp + m) : __ldg(qp + m); q1[2 * m] = t.x; q1[2 * m + 1] = t.y; }
        }
      } else {
#pragma unroll
        for (int m = 0; m < NV; ++m) {
          q0[m] = act0 ? __ldg(v.Q + (int64_t)(wb + t0) * NV + m) : 0.0;
          q1[m] = act1 ? __ldg(v.Q + (int64_t)(wb + t1) * NV + m) : 0.0;
        }
      }
      // Pi_B (twice for r0, see masked.cuh)
#pragma unroll
      for (int pass = 0; pass < ((MODE == MM_R0 || MODE == MM_R0E) ? 2 : 1); ++pass) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double dv[NV];
#pragma unroll
          for (int m = 0; m < NV; ++m) dv[m] = fma(q0[m], g0[d], q1[m] * g1[d]);
          int own;
          nd2_reduce_scatter<NV>(dv, lane, &own);
          if (own < NV) s_dot[wib][d * NV + own] = dv[0];
        }
        __syncwarp();
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double s0v = 0.0, s1v = 0.0;
#pragma unroll
          for (int m = 0; m < NV; ++m) {
            const double dm = s_dot[wib][d * NV + m];
            s0v = fma(q0[m], dm, s0v);
            s1v = fma(q1[m], dm, s1v);
          }
          g0[d] -= s0v;
          g1[d] -= s1v;
        }
        __syncwarp();
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int ro = wb + d * n3;
        if (act0) {
          if (MODE == MM_ITER) { if (CS) __stcs(out + ro + t0, g0[d]); else out[ro + t0] = g0[d]; part = fma(X[ro + t0], g0[d], part); }
          else out[ro + t0] = -g0[d];
        }
        if (act1) {
          if (MODE == MM_ITER) { if (CS) __stcs(out + ro + t1, g1[d]); else out[ro + t1] = g1[d]; part = fma(X[ro + t1], g1[d], part); }
          else out[ro + t1] = -g1[d];
        }
      }
    }
    __syncwarp();
  }
  const double tot = block_sum(part, sh);
  block_partial_out(v, partials, tot, sh, MODE == MM_ITER ? 1 : -1);
}

// ---- host side ------------------------------------------------------------
template <typename T>
static cudaError_t nd_alloc(T** p, int64_t n, cudaStream_t s) {
  return emin_mallocAsync((void**)p, sizeof(T) * (size_t)(n > 0 ? n : 1), s);
}

// returns true if the nodal path was built
static inline bool select_nodal_path(emin_ctx c, NodalPlan*& out) {
  out = nullptr;
  if (c->opts.block_size != 3 || c->nF % 3 != 0 || c->nF == 0 || c->nv > 8 || c->nnzWh >= INT32_MAX) return false;
  if (c->opts.debug_flags & EMIN_DBG_FORCE_GENERIC) return false;
  cudaStream_t s = c->stream;
  const int SM = emin_num_sms();
  const int64_t nFn = c->nF / 3;
  int32_t* ok;
  int64_t *pmlen, *scratch, *tot;
  if (nd_alloc(&ok, 2, s) || nd_alloc(&pmlen, nFn + 1, s) || nd_alloc(&scratch, emin_scan_scratch_elems(nFn + 1), s) ||
      nd_alloc(&tot, 1, s))
    return false;
  const int32_t init[2] = {1, 0};
  cudaMemcpyAsync(ok, init, sizeof(int32_t) * 2, cudaMemcpyHostToDevice, s);
  k_nodal_check<<<SM * 8, 256, 0, s>>>(c->view(), nFn, ok, pmlen, ok + 1);
  int32_t h_ok2[2] = {0, 0};
  cudaMemcpyAsync(h_ok2, ok, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const int32_t h_ok = h_ok2[0];
  c->launches += 1;
  if (!h_ok) {
    cudaFreeAsync(ok, s); cudaFreeAsync(pmlen, s); cudaFreeAsync(scratch, s); cudaFreeAsync(tot, s);
    return false;
  }
  NodalPlan* p = new NodalPlan();
  p->nFn = nFn;
  p->max_nb = h_ok2[1];
  p->nblk = c->nnzAFF / 9;
  emin_scan_i64(pmlen, pmlen, nFn, tot, scratch, s);     // exclusive -> offsets
  cudaMemcpyAsync(pmlen + nFn, tot, sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(&p->npm, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  p->pmoff = pmlen;
  if (nd_alloc(&p->blk, p->nblk, s) || nd_alloc(&p->bptr, nFn + 1, s) || nd_alloc(&p->pm8, p->npm, s)) {
    delete p;
    return false;
  }
  k_nodal_build<<<SM * 8, 256, 0, s>>>(c->view(), nFn, p->pmoff, p->blk, p->bptr, p->pm8);
  c->launches += 4;
  cudaFreeAsync(ok, s); cudaFreeAsync(scratch, s); cudaFreeAsync(tot, s);
  out = p;
  return true;
}

// Grid of the nodal kernels: ~12 nodes per warp, between 32 and 256 CTAs
// per SM.  Many short CTAs dispatched in order keep the resident warps on a
// narrow, advancing window of nodes, so neighbour rows of y stay in L2
// (config 5: SM x 16 CTAs 15.27 ms, x 64 14.76, x 256 14.33; config 4 is
// best at x 32: 396 vs 404 us at x 16).
static inline int nodal_grid(emin_ctx c, const NodalPlan* p) {
  const int SM = emin_num_sms();
  int64_t per_sm = std::min<int64_t>(256, std::max<int64_t>(32, p->nFn / (8 * 12) / SM));
  return (int)std::max<int64_t>(1, std::min<int64_t>((p->nFn + 7) / 8, (int64_t)SM * per_sm));
}

// one v2 configuration for every mode: CS = evict-first hints (iteration
// only), WIDE = chunked staging (> ND_MAXB blocks per node), GRP = blocks per
// round
template <int NV, bool CS, bool WIDE, int GRP, int MINB = 4>
static inline void nd_v2(int mode, const DevView& v, const NodalPlan* p, int g, const double* X, const double* X2,
                         double* out, double* partials, cudaStream_t s) {
#define ND_ARGS <<<g, ND_WARPS * 32, 0, s>>>(v, p->blk, p->bptr, p->pm8, p->pmoff, p->nFn, X, X2, out, partials)
  if (mode == MM_ITER) k_spgemm_nodal_v2<NV, MM_ITER, CS, WIDE, GRP, MINB> ND_ARGS;
  else if (mode == MM_R0) k_spgemm_nodal_v2<NV, MM_R0, false, WIDE, GRP> ND_ARGS;
  else if (mode == MM_R0E) k_spgemm_nodal_v2<NV, MM_R0E, false, WIDE, GRP> ND_ARGS;
  else k_spgemm_nodal_v2<NV, MM_ENERGY, false, WIDE, GRP> ND_ARGS;
#undef ND_ARGS
}

template <bool CS, bool WIDE, int GRP, int MINB = 4>
static inline void nd_v2_nv(int nv, int mode, const DevView& v, const NodalPlan* p, int g, const double* X,
                            const double* X2, double* out, double* partials, cudaStream_t s) {
  switch (nv) {
#define NV_CASE(N) case N: nd_v2<N, CS, WIDE, GRP, MINB>(mode, v, p, g, X, X2, out, partials, s); break;
    NV_CASE(1) NV_CASE(2) NV_CASE(3) NV_CASE(4) NV_CASE(5) NV_CASE(6) NV_CASE(7) NV_CASE(8)
#undef NV_CASE
  }
}

static inline bool launch_nodal(emin_ctx c, const NodalPlan* p, int mode, const double* X, const double* X2,
                                double* out, cudaStream_t s) {
  DevView v = c->view();
  if (mode == MM_ITER && c->sym) v.affval = c->affvalS;   // S A_FF S (symmetric Jacobi scaling)
  const int g = nodal_grid(c, p);
  // v2 with two blocks per round (all gathers of both issued before the
  // FMAs; config 5 20.7 -> 15.9 ms, config 4 471 -> 420 us; three or four per
  // round spill or lose occupancy: 16.6 / 21.0+ ms) and, in the iteration,
  // evict-first hints on the streamed data (A chunk, block records, position
  // bytes, Q, y^) so the L2 keeps the gathered y rows.  Galerkin levels
  // (NEXT-4, > ND_MAXB blocks per node): the same, staged in chunks.
  if (p->max_nb > ND_MAXB)
    nd_v2_nv<true, true, 2>(c->nv, mode, v, p, g, X, X2, out, c->partials, s);
  else
    nd_v2_nv<true, false, 3>(c->nv, mode, v, p, g, X, X2, out, c->partials, s);
  return true;
}

static inline void free_nodal_path(emin_ctx c, NodalPlan*& p) {
  if (!p) return;
  void* ptrs[] = {p->blk, p->bptr, p->pm8, p->pmoff};
  for (void* q : ptrs) if (q) cudaFreeAsync(q, c->stream);
  delete p;
  p = nullptr;
}
