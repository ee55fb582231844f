// galerkin_bsr.cuh -- the 3x3-block (node-level) path of emin_galerkin, used
// when A and P have the structure of the vector (elasticity) problems: A's
// rows 3I..3I+2 list the same nodes K in full 3x3 blocks, P's F-node rows
// the same C nodes in full 3x3 blocks and P's C-node rows the single entry
// P(3K+e, 3c+e).  Then T = A P and A_c = P^T T are made of full 3x3 blocks
// and the products can be formed per (block, block) pair: one hash probe per
// pair instead of 27, the 3 output rows of a pair on 3 lanes (10 pairs per
// round), each lane adding <= 3 terms to each of its 3 elements.
//
// Same sums as the point path and the oracle, term by term: an output element
// (d, b) of a node row collects the terms of its pairs in X order (A's blocks /
// P^T's node rows ascending) and, inside a pair, in ascending inner index e
// (A's column 3K+e / P^T's row 3I+d), one __dmul_rn and one __dadd_rn per term;
// lanes that hit the same element in one round are added by the lowest of
// them in lane (= pair) order.  So the result is bitwise the point path's.
#pragma once

// T = A P, node level
struct BsrAP {
  const int64_t* Arp;
  const int32_t* Acol;
  const double* Aval;
  const int64_t* Prp;
  const int32_t* Pcol;
  const double* Pval;
  __device__ __forceinline__ int64_t nx(int64_t R) const { return (Arp[3 * R + 1] - Arp[3 * R]) / 3; }
  __device__ __forceinline__ int32_t xrow(int64_t R, int64_t m) const { return Acol[Arp[3 * R] + 3 * m] / 3; }
  __device__ __forceinline__ int64_t ny(int32_t K) const {
    const int64_t l = Prp[3 * (int64_t)K + 1] - Prp[3 * (int64_t)K];
    return l == 1 ? 1 : l / 3;
  }
  __device__ __forceinline__ int32_t ycol(int32_t K, int64_t s) const {
    const int64_t b = Prp[3 * (int64_t)K];
    return Pcol[b + (Prp[3 * (int64_t)K + 1] - b == 1 ? 0 : 3 * s)] / 3;
  }
  // the stored terms X[d][e] * Y[e][bb], e ascending
  __device__ __forceinline__ int terms(int64_t R, int64_t m, int32_t K, int64_t s, int d, int bb, double* t) const {
    const double* a = Aval + Arp[3 * R + d] + 3 * m;
    const int64_t p0 = Prp[3 * (int64_t)K];
    if (Prp[3 * (int64_t)K + 1] - p0 == 1) {      // C node K: only P(3K+bb, 3c+bb)
      t[0] = __dmul_rn(a[bb], Pval[Prp[3 * (int64_t)K + bb]]);
      return 1;
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) t[e] = __dmul_rn(a[e], Pval[Prp[3 * (int64_t)K + e] + 3 * s + bb]);
    return 3;
  }
};

// A_c = P^T T, node level; P^T as sorted (c, I) node entries with the
// position s of c in J_I (-1: I is c's own C node)
struct BsrPtT {
  const int64_t* Ptnp;
  const int32_t* PtI;
  const int32_t* PtS;
  const int64_t* Prp;
  const double* Pval;
  const int64_t* Tnp;
  const int32_t* Tnc;
  const double* Tv;
  __device__ __forceinline__ int64_t nx(int64_t c) const { return Ptnp[c + 1] - Ptnp[c]; }
  __device__ __forceinline__ int32_t xrow(int64_t c, int64_t m) const { return PtI[Ptnp[c] + m]; }
  __device__ __forceinline__ int64_t ny(int32_t I) const { return Tnp[I + 1] - Tnp[I]; }
  __device__ __forceinline__ int32_t ycol(int32_t I, int64_t t) const { return Tnc[Tnp[I] + t]; }
  __device__ __forceinline__ int terms(int64_t c, int64_t m, int32_t I, int64_t t, int dp, int bb, double* o) const {
    const int32_t S = PtS[Ptnp[c] + m];
    const double* y = Tv + 9 * (Tnp[I] + t);
    if (S < 0) {                                      // C node I: only P(3I+dp, 3c+dp)
      o[0] = __dmul_rn(Pval[Prp[3 * (int64_t)I + dp]], y[3 * dp + bb]);
      return 1;
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) o[d] = __dmul_rn(Pval[Prp[3 * (int64_t)I + d] + 3 * S + dp], y[3 * d + bb]);
    return 3;
  }
};

// pairs of output node row R, PPR per round with LPP lanes each (32 x 1:
// lane per pair; 10 x 3: elem = lane % 3 = the output row d of the pair);
// f(act, m, K, s, elem) returns false to stop
template <int PPR, int LPP, class OP, class F>
__device__ __forceinline__ void bsr_pairs(const OP& op, int64_t R, int lane, F&& f) {
  const int64_t nxr = op.nx(R);
  const int pl = LPP == 1 ? lane : (lane < LPP * PPR ? lane / LPP : -1);
  const int elem = LPP == 1 ? 0 : lane - LPP * (lane / LPP);
  for (int64_t xb = 0; xb < nxr; xb += 32) {
    const int64_t xi = xb + lane;
    const int nx = (int)(nxr - xb < 32 ? nxr - xb : 32);
    int32_t K = 0;
    int64_t len = 0;
    if (xi < nxr) { K = op.xrow(R, xi); len = op.ny(K); }
    int64_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t excl = incl - len;
    const int64_t tot = __shfl_sync(0xffffffffu, incl, 31);
    for (int64_t pb = 0; pb < tot; pb += PPR) {
      const int64_t p = pb + (pl < 0 ? 0 : pl);
      int lo = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int cand = lo + step;
        const int64_t e = __shfl_sync(0xffffffffu, excl, cand & 31);
        if (cand < nx && e <= p) lo = cand;
      }
      const int64_t eb = __shfl_sync(0xffffffffu, excl, lo);
      const int32_t Kl = __shfl_sync(0xffffffffu, K, lo);
      const bool act = pl >= 0 && p < tot;
      if (!f(act, xb + lo, Kl, p - eb, elem)) return;
    }
  }
}

constexpr int BS_TIERS = 4;
constexpr int BS_LOG[BS_TIERS] = {7, 8, 10, 11};    // node slots 128 / 256 / 1024 / 2048
constexpr int BS_WARPS[BS_TIERS] = {8, 4, 1, 1};
__device__ __forceinline__ int bs_tier(int64_t c) { return c <= 64 ? 0 : c <= 128 ? 1 : c <= 512 ? 2 : 3; }

struct BsrOut {
  int64_t nrows;           // output node rows
  int64_t* cnt;            // distinct node columns per node row (symbolic; -1 - tier on overflow)
  const int64_t* Onp;      // T: block row pointers (numeric)
  int32_t* Onc;            // T: block node columns
  double* Ov;              // T: 9 values per block (d-major)
  const int64_t* Crp;      // A_c: point row pointers
  int32_t* Ccol;
  double* Cval;
  int32_t* err;            // bit 2: a node row wider than the largest table
};

template <int T, class OP>
__global__ void __launch_bounds__(BS_WARPS[T] * 32) k_bsr_symbolic(OP op, BsrOut o) {
  constexpr int LOG = BS_LOG[T], CAP = 1 << LOG, W = BS_WARPS[T];
  extern __shared__ int32_t bs_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* keys = bs_smem + w * CAP;
  for (int s = lane; s < CAP; s += 32) keys[s] = -1;
  __syncwarp();
  for (int64_t R = (int64_t)blockIdx.x * W + w; R < o.nrows; R += (int64_t)gridDim.x * W) {
    if (T > 0 && o.cnt[R] != -T) continue;
    int64_t count = 0;
    bsr_pairs<32, 1>(op, R, lane, [&](bool act, int64_t m, int32_t K, int64_t s, int) {
      bool fresh = false;
      if (act) gk_insert(keys, LOG, op.ycol(K, s), &fresh);
      count += __popc(__ballot_sync(0xffffffffu, fresh));
      __syncwarp();
      return count <= CAP / 2;
    });
    if (lane == 0) {
      if (count <= CAP / 2) o.cnt[R] = count;
      else if (T == BS_TIERS - 1) { o.cnt[R] = 0; atomicOr(o.err, 4); }
      else o.cnt[R] = -(T + 1);
    }
    for (int s = lane; s < CAP; s += 32) keys[s] = -1;
    __syncwarp();
  }
}

// numeric: OUT 0 = T (BSR, slot order), OUT 1 = A_c (point CSR, node columns ascending)
template <int T, int OUT, class OP>
__global__ void __launch_bounds__(BS_WARPS[T] * 32) k_bsr_numeric(OP op, BsrOut o) {
  constexpr int LOG = BS_LOG[T], CAP = 1 << LOG, W = BS_WARPS[T];
  extern __shared__ double bs_smemd[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* vals = bs_smemd + (size_t)w * (9 * CAP + 288);
  double* contrib = vals + 9 * CAP;                        // [32][3 bb][3 terms]
  int32_t* keys = reinterpret_cast<int32_t*>(bs_smemd + (size_t)W * (9 * CAP + 288)) + w * (CAP + 32);
  int32_t* ncontrib = keys + CAP;                          // [32]
  for (int s = lane; s < CAP; s += 32) keys[s] = -1;
  for (int s = lane; s < 9 * CAP; s += 32) vals[s] = 0.0;
  __syncwarp();
  for (int64_t R = (int64_t)blockIdx.x * W + w; R < o.nrows; R += (int64_t)gridDim.x * W) {
    const int64_t mR = o.cnt[R];
    if (bs_tier(mR) != T || mR == 0) continue;
    // 10 pairs per round, 3 lanes per pair: lane d computes the output row d
    // of its pair (3 elements, <= 3 terms each)
    bsr_pairs<10, 3>(op, R, lane, [&](bool act, int64_t m, int32_t K, int64_t s, int d) {
      int slot = 0;
      if (act && d == 0) {
        bool fresh;
        slot = gk_insert(keys, LOG, op.ycol(K, s), &fresh);
      }
      slot = __shfl_sync(0xffffffffu, slot, lane - d);
      int nt = 0;
      if (act) {
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) nt = op.terms(R, m, K, s, d, bb, contrib + 9 * lane + 3 * bb);
      }
      ncontrib[lane] = nt;
      __syncwarp();
      const int key = act ? slot * 3 + d : -1 - lane;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (act && (__ffs(peers) - 1) == lane) {
        double acc[3];
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) acc[bb] = vals[9 * slot + 3 * d + bb];
        for (unsigned pm = peers; pm; pm &= pm - 1) {
          const int q = __ffs(pm) - 1;
          const int nq = ncontrib[q];
#pragma unroll
          for (int bb = 0; bb < 3; ++bb)
            for (int k = 0; k < nq; ++k) acc[bb] = __dadd_rn(acc[bb], contrib[9 * q + 3 * bb + k]);
        }
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) vals[9 * slot + 3 * d + bb] = acc[bb];
      }
      __syncwarp();
      return true;
    });
    if (OUT == 0) {
      int64_t pos = o.Onp[R];
      for (int s0 = 0; s0 < CAP; s0 += 32) {
        const int32_t k = keys[s0 + lane];
        const unsigned used = __ballot_sync(0xffffffffu, k >= 0);
        if (k >= 0) {
          const int64_t q = pos + __popc(used & ((1u << lane) - 1));
          o.Onc[q] = k;
#pragma unroll
          for (int e = 0; e < 9; ++e) o.Ov[9 * q + e] = vals[9 * (s0 + lane) + e];
        }
        pos += __popc(used);
      }
    } else {
      const int64_t r0 = o.Crp[3 * R], r1 = o.Crp[3 * R + 1], r2 = o.Crp[3 * R + 2];
      for (int s = lane; s < CAP; s += 32) {
        const int32_t k = keys[s];
        if (k < 0) continue;
        int r = 0;
        for (int t2 = 0; t2 < CAP; ++t2) r += (uint32_t)keys[t2] < (uint32_t)k;
#pragma unroll
        for (int dp = 0; dp < 3; ++dp) {
          const int64_t base = (dp == 0 ? r0 : dp == 1 ? r1 : r2) + 3 * r;
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            o.Ccol[base + bb] = 3 * k + bb;
            o.Cval[base + bb] = vals[9 * s + 3 * dp + bb];
          }
        }
      }
    }
    __syncwarp();
    for (int s = lane; s < CAP; s += 32) keys[s] = -1;
    for (int s = lane; s < 9 * CAP; s += 32) vals[s] = 0.0;
    __syncwarp();
  }
}

// structure check, thread per node: bit 0 A not 3x3-blocked, bit 1 P not
// blockwise (F nodes) / not the identity (C nodes)
__global__ void k_bsr_check(int64_t nn, const int64_t* __restrict__ Arp, const int32_t* __restrict__ Acol,
                            const int64_t* __restrict__ Prp, const int32_t* __restrict__ Pcol, int32_t* __restrict__ bad) {
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < nn; I += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = 3 * I;
    bool okA = true;
    const int64_t la = Arp[r + 1] - Arp[r];
    for (int d = 1; d < 3; ++d) okA = okA && (Arp[r + d + 1] - Arp[r + d] == la);
    okA = okA && (la % 3 == 0);
    for (int64_t m = 0; okA && m < la / 3; ++m) {
      const int32_t k3 = Acol[Arp[r] + 3 * m];
      okA = (k3 % 3 == 0);
      for (int d = 0; d < 3 && okA; ++d)
        for (int e = 0; e < 3 && okA; ++e) okA = Acol[Arp[r + d] + 3 * m + e] == k3 + e;
    }
    bool okP = true;
    const int64_t lp = Prp[r + 1] - Prp[r];
    for (int d = 1; d < 3; ++d) okP = okP && (Prp[r + d + 1] - Prp[r + d] == lp);
    if (okP && lp == 1) {
      const int32_t c3 = Pcol[Prp[r]];
      okP = (c3 % 3 == 0) && Pcol[Prp[r + 1]] == c3 + 1 && Pcol[Prp[r + 2]] == c3 + 2;
    } else if (okP) {
      okP = (lp % 3 == 0) && lp > 0;
      for (int64_t s = 0; okP && s < lp / 3; ++s) {
        const int32_t c3 = Pcol[Prp[r] + 3 * s];
        okP = (c3 % 3 == 0);
        for (int d = 0; d < 3 && okP; ++d)
          for (int b = 0; b < 3 && okP; ++b) okP = Pcol[Prp[r + d] + 3 * s + b] == c3 + b;
      }
    }
    if (!okA) atomicOr(bad, 1);
    if (!okP) atomicOr(bad, 2);
  }
}

// node-level transpose keys of P: (c * nn + I, s), s = -1 for a C node row
__global__ void k_bsr_tkeys(int64_t nn, const int64_t* __restrict__ Prp, const int32_t* __restrict__ Pcol,
                            const int64_t* __restrict__ nofs, uint64_t* __restrict__ key, int32_t* __restrict__ sv,
                            int64_t* __restrict__ ccount) {
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < nn; I += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = Prp[3 * I], l = Prp[3 * I + 1] - b;
    const int64_t o = nofs[I];
    if (l == 1) {
      const uint64_t c = (uint64_t)(Pcol[b] / 3);
      key[o] = c * (uint64_t)nn + (uint64_t)I;
      sv[o] = -1;
      atomicAdd(reinterpret_cast<unsigned long long*>(&ccount[c]), 1ull);
    } else {
      for (int64_t s = 0; s < l / 3; ++s) {
        const uint64_t c = (uint64_t)(Pcol[b + 3 * s] / 3);
        key[o + s] = c * (uint64_t)nn + (uint64_t)I;
        sv[o + s] = (int32_t)s;
        atomicAdd(reinterpret_cast<unsigned long long*>(&ccount[c]), 1ull);
      }
    }
  }
}

__global__ void k_bsr_nodelen(int64_t nn, const int64_t* __restrict__ Prp, int64_t* __restrict__ len) {
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < nn; I += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = Prp[3 * I + 1] - Prp[3 * I];
    len[I] = l == 1 ? 1 : l / 3;
  }
}

__global__ void k_bsr_trows(int64_t m, int64_t nn, const uint64_t* __restrict__ key, int32_t* __restrict__ I) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    I[q] = (int32_t)(key[q] % (uint64_t)nn);
}

// A_c point row pointers from the node counts (exclusive node-block offsets nb)
__global__ void k_bsr_crp(int64_t nnc, const int64_t* __restrict__ nb, const int64_t* __restrict__ cnt,
                          int64_t* __restrict__ crp) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nnc; c += (int64_t)gridDim.x * blockDim.x) {
    for (int dp = 0; dp < 3; ++dp) crp[3 * c + dp] = 9 * nb[c] + 3 * cnt[c] * dp;
    if (c == nnc - 1) crp[3 * nnc] = 9 * (nb[c] + cnt[c]);
  }
}

template <int T>
size_t bs_smem_numeric() { return (size_t)BS_WARPS[T] * ((9 * (1 << BS_LOG[T]) + 288) * 8 + ((1 << BS_LOG[T]) + 32) * 4); }
template <int T>
size_t bs_smem_symbolic() { return (size_t)BS_WARPS[T] * (1 << BS_LOG[T]) * 4; }

template <int T, int OUT, class OP>
cudaError_t bs_launch(bool numeric, const OP& op, const BsrOut& o, int SM, cudaStream_t s) {
  const size_t sm = numeric ? bs_smem_numeric<T>() : bs_smem_symbolic<T>();
  cudaError_t e = numeric
      ? cudaFuncSetAttribute(k_bsr_numeric<T, OUT, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)
      : cudaFuncSetAttribute(k_bsr_symbolic<T, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(2048 / (BS_WARPS[T] * 32), (220u << 10) / sm));
  const int64_t want = (o.nrows + BS_WARPS[T] - 1) / BS_WARPS[T];
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)SM * per_sm));
  if (numeric) k_bsr_numeric<T, OUT, OP><<<g, BS_WARPS[T] * 32, sm, s>>>(op, o);
  else k_bsr_symbolic<T, OP><<<g, BS_WARPS[T] * 32, sm, s>>>(op, o);
  return cudaGetLastError();
}

template <int OUT, class OP>
cudaError_t bs_launch_all(bool numeric, const OP& op, const BsrOut& o, int SM, cudaStream_t s) {
  cudaError_t e = bs_launch<0, OUT>(numeric, op, o, SM, s);
  if (e == cudaSuccess) e = bs_launch<1, OUT>(numeric, op, o, SM, s);
  if (e == cudaSuccess) e = bs_launch<2, OUT>(numeric, op, o, SM, s);
  if (e == cudaSuccess) e = bs_launch<3, OUT>(numeric, op, o, SM, s);
  return e;
}
