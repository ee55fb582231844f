// galerkin.cu -- the next level's operator A_c = P^T A P on the GPU (SURVEY
// §8f NEXT-4, reading A26): emin_galerkin().
//
// A_c is the matrix whose trace is the energy the method minimises (Eq.
// trace); the paper forms it with the "sparse matrix-matrix
// product" of its coarse grid construction and re-runs the
// prolongation construction on it level by level (T_p sums levels).
// Two row-wise (Gustavson) products with the same kernel:
//   T   = A P      rows of A    x rows of P      (n  x nc, unsorted rows)
//   A_c = P^T T    rows of P^T  x rows of T      (nc x nc, columns ascending)
// P^T comes from one 64-bit-key radix sort (col * n + row) of P's entries.
//
// One warp per output row.  The (X entry, Y entry) pairs of a row are
// enumerated 32 at a time over chunks of 32 X entries (warp scan of the Y
// row lengths, shuffle binary search), the column goes into a per-warp
// open-addressing table in shared memory (atomicCAS claims a slot).  Two
// passes: symbolic (distinct columns -> row pointers), numeric (values).
// Deterministic and bitwise equal to the oracle's definition: every output
// entry is the sum of its product terms in X order with one rounding per
// multiply and per add (__dmul_rn / __dadd_rn) -- within a round the lanes
// that hit the same slot (__match_any_sync) are added by the lowest of them
// in lane order, i.e. in X order, and rounds run in X order.  A row goes to
// the smallest of four table sizes (256 / 512 / 2048 / 16384 slots) that
// keeps the load factor <= 1/2 (the small tables keep 32-64 warps per SM);
// wider rows are an error.
#include <cub/device/device_radix_sort.cuh>

#include <string>
#include <vector>

#include "emin_internal.cuh"

namespace {

constexpr int GK_TIERS = 4;
constexpr int GK_LOG[GK_TIERS] = {8, 9, 11, 14};   // table slots 256 / 512 / 2048 / 16384
constexpr int GK_WARPS[GK_TIERS] = {8, 8, 4, 1};   // warps per CTA

struct GkArgs {
  int64_t nrows;
  const int64_t* Xrp;
  const int32_t* Xcol;                        // Y row of each X entry
  const double* Xval;
  const int64_t* Yrp;
  const int32_t* Ycol;
  const double* Yval;
  int64_t* cnt;                               // distinct columns per row; symbolic marks -1 - tier on overflow
  const int64_t* Orp;                         // numeric output row pointers
  int32_t* Ocol;
  double* Oval;
  int sort;                                   // numeric: columns ascending
  int32_t* err;                               // bit 1: a row wider than the largest table
};

__device__ __forceinline__ int gk_hash(int32_t key, int log) {
  return (int)(((uint32_t)key * 2654435761u) >> (32 - log));
}

// claim or find the slot of key (the table is never more than half full + 32)
__device__ __forceinline__ int gk_insert(int32_t* keys, int log, int32_t key, bool* fresh) {
  int h = gk_hash(key, log);
  const int mask = (1 << log) - 1;
  while (true) {
    const int32_t prev = atomicCAS(&keys[h], -1, key);
    if (prev == -1) { *fresh = true; return h; }
    if (prev == key) { *fresh = false; return h; }
    h = (h + 1) & mask;
  }
}

// Enumerate the pairs of row `row`, 32 per round; f(active, key, xval, yval)
// returns false to stop early (uniform across the warp).
template <class F>
__device__ __forceinline__ void gk_pairs(const GkArgs& a, int64_t row, int lane, F&& f) {
  const int64_t x0 = a.Xrp[row], x1 = a.Xrp[row + 1];
  for (int64_t xb = x0; xb < x1; xb += 32) {
    const int64_t xi = xb + lane;
    const int nx = (int)(x1 - xb < 32 ? x1 - xb : 32);
    int64_t ybeg = 0, len = 0;
    double xv = 0.0;
    if (xi < x1) {
      const int32_t k = a.Xcol[xi];
      ybeg = a.Yrp[k];
      len = a.Yrp[k + 1] - ybeg;
      xv = a.Xval ? a.Xval[xi] : 0.0;
    }
    int64_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t excl = incl - len;
    const int64_t tot = __shfl_sync(0xffffffffu, incl, 31);
    for (int64_t pb = 0; pb < tot; pb += 32) {
      const int64_t p = pb + lane;
      // largest x < nx with excl_x <= p (skips X entries with empty Y rows)
      int lo = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int cand = lo + step;
        const int64_t e = __shfl_sync(0xffffffffu, excl, cand & 31);
        if (cand < nx && e <= p) lo = cand;
      }
      const int64_t eb = __shfl_sync(0xffffffffu, excl, lo);
      const int64_t yb = __shfl_sync(0xffffffffu, ybeg, lo);
      const double xvl = __shfl_sync(0xffffffffu, xv, lo);
      const bool act = p < tot;
      int32_t key = -1;
      double yv = 0.0;
      if (act) {
        const int64_t y = yb + (p - eb);
        key = a.Ycol[y];
        if (a.Yval) yv = a.Yval[y];
      }
      if (!f(act, key, xvl, yv)) return;
    }
  }
}

// symbolic: distinct columns per row into cnt (tier 0: every row; tier t > 0:
// the rows tier t - 1 marked -t)
template <int T>
__global__ void __launch_bounds__(GK_WARPS[T] * 32) k_gk_symbolic(GkArgs a) {
  constexpr int LOG = GK_LOG[T], CAP = 1 << LOG, W = GK_WARPS[T];
  extern __shared__ int32_t gk_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* keys = gk_smem + w * CAP;
  for (int s = lane; s < CAP; s += 32) keys[s] = -1;
  __syncwarp();
  for (int64_t row = (int64_t)blockIdx.x * W + w; row < a.nrows; row += (int64_t)gridDim.x * W) {
    if (T > 0 && a.cnt[row] != -T) continue;
    int64_t count = 0;
    gk_pairs(a, row, lane, [&](bool act, int32_t key, double, double) {
      bool fresh = false;
      if (act) gk_insert(keys, LOG, key, &fresh);
      count += __popc(__ballot_sync(0xffffffffu, fresh));
      __syncwarp();
      return count <= CAP / 2;
    });
    if (lane == 0) {
      if (count <= CAP / 2) a.cnt[row] = count;
      else if (T == GK_TIERS - 1) { a.cnt[row] = 0; atomicOr(a.err, 2); }
      else a.cnt[row] = -(T + 1);
    }
    for (int s = lane; s < CAP; s += 32) keys[s] = -1;
    __syncwarp();
  }
}

// the table a row of c distinct columns goes to (load factor <= 1/2)
__device__ __forceinline__ int gk_tier(int64_t c) { return c <= 128 ? 0 : c <= 256 ? 1 : c <= 1024 ? 2 : 3; }

template <int T>
__global__ void __launch_bounds__(GK_WARPS[T] * 32) k_gk_numeric(GkArgs a) {
  constexpr int LOG = GK_LOG[T], CAP = 1 << LOG, W = GK_WARPS[T];
  extern __shared__ double gk_smemd[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* vals = gk_smemd + (size_t)w * (CAP + 32);
  double* contrib = vals + CAP;
  int32_t* keys = reinterpret_cast<int32_t*>(gk_smemd + (size_t)W * (CAP + 32)) + w * CAP;
  for (int s = lane; s < CAP; s += 32) { keys[s] = -1; vals[s] = 0.0; }
  __syncwarp();
  for (int64_t row = (int64_t)blockIdx.x * W + w; row < a.nrows; row += (int64_t)gridDim.x * W) {
    const int64_t m = a.cnt[row];
    if (gk_tier(m) != T || m == 0) continue;
    gk_pairs(a, row, lane, [&](bool act, int32_t key, double xv, double yv) {
      bool fresh = false;
      int slot = -1 - lane;
      double v = 0.0;
      if (act) {
        slot = gk_insert(keys, LOG, key, &fresh);
        v = __dmul_rn(xv, yv);
      }
      contrib[lane] = v;
      __syncwarp();
      const unsigned peers = __match_any_sync(0xffffffffu, slot);
      if (act && (__ffs(peers) - 1) == lane) {
        double acc = vals[slot];
        for (unsigned pm = peers; pm; pm &= pm - 1) acc = __dadd_rn(acc, contrib[__ffs(pm) - 1]);
        vals[slot] = acc;
      }
      __syncwarp();
      return true;
    });
    const int64_t base = a.Orp[row];
    if (a.sort) {
      for (int s = lane; s < CAP; s += 32) {
        const int32_t k = keys[s];
        if (k < 0) continue;
        int r = 0;
        for (int t = 0; t < CAP; ++t) r += (uint32_t)keys[t] < (uint32_t)k;
        a.Ocol[base + r] = k;
        a.Oval[base + r] = vals[s];
      }
    } else {
      int64_t pos = base;
      for (int s0 = 0; s0 < CAP; s0 += 32) {
        const int32_t k = keys[s0 + lane];
        const unsigned used = __ballot_sync(0xffffffffu, k >= 0);
        if (k >= 0) {
          const int64_t q = pos + __popc(used & ((1u << lane) - 1));
          a.Ocol[q] = k;
          a.Oval[q] = vals[s0 + lane];
        }
        pos += __popc(used);
      }
    }
    __syncwarp();
    for (int s = lane; s < CAP; s += 32) { keys[s] = -1; vals[s] = 0.0; }
    __syncwarp();
  }
}

__global__ void k_gk_check(int64_t nrows, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                           int64_t ncols, int32_t* __restrict__ err) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rp[r], e = rp[r + 1];
    if (e < b) { atomicOr(err, 1); continue; }
    for (int64_t q = b; q < e; ++q)
      if (col[q] < 0 || col[q] >= ncols) { atomicOr(err, 1); break; }
  }
}

__global__ void k_gk_keys(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                          uint64_t* __restrict__ key, int64_t* __restrict__ ccount) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
      key[q] = (uint64_t)col[q] * (uint64_t)n + (uint64_t)i;
      atomicAdd(reinterpret_cast<unsigned long long*>(&ccount[col[q]]), 1ull);
    }
}

__global__ void k_gk_rows(int64_t nnz, int64_t n, const uint64_t* __restrict__ key, int32_t* __restrict__ row) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x)
    row[q] = (int32_t)(key[q] % (uint64_t)n);
}

template <int T>
size_t gk_smem_numeric() { return (size_t)GK_WARPS[T] * ((1 << GK_LOG[T]) * 12 + 32 * 8); }
template <int T>
size_t gk_smem_symbolic() { return (size_t)GK_WARPS[T] * (1 << GK_LOG[T]) * 4; }

template <int T>
cudaError_t gk_launch(bool numeric, const GkArgs& a, int SM, cudaStream_t s) {
  const size_t sm = numeric ? gk_smem_numeric<T>() : gk_smem_symbolic<T>();
  cudaError_t e = numeric ? cudaFuncSetAttribute(k_gk_numeric<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)
                          : cudaFuncSetAttribute(k_gk_symbolic<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(2048 / (GK_WARPS[T] * 32), (220u << 10) / sm));
  const int64_t want = (a.nrows + GK_WARPS[T] - 1) / GK_WARPS[T];
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)SM * per_sm));
  if (numeric) k_gk_numeric<T><<<g, GK_WARPS[T] * 32, sm, s>>>(a);
  else k_gk_symbolic<T><<<g, GK_WARPS[T] * 32, sm, s>>>(a);
  return cudaGetLastError();
}

#include "galerkin_bsr.cuh"

// every tier in order (symbolic: tier t > 0 re-counts the rows tier t - 1 overflowed)
cudaError_t gk_launch_all(bool numeric, const GkArgs& a, int SM, cudaStream_t s) {
  cudaError_t e = gk_launch<0>(numeric, a, SM, s);
  if (e == cudaSuccess) e = gk_launch<1>(numeric, a, SM, s);
  if (e == cudaSuccess) e = gk_launch<2>(numeric, a, SM, s);
  if (e == cudaSuccess) e = gk_launch<3>(numeric, a, SM, s);
  return e;
}

}  // namespace

static thread_local std::string g_galerkin_error;
static thread_local int32_t g_galerkin_path = 0;

extern "C" emin_status emin_galerkin(int64_t n, int64_t nc, const int64_t* A_rowptr, const int32_t* A_col,
                                     const double* A_val, const int64_t* P_rowptr, const int32_t* P_col,
                                     const double* P_val, int64_t* Ac_rowptr, int32_t* Ac_col, double* Ac_val,
                                     int64_t Ac_cap, int64_t* nnz_out, int32_t flags, void* stream) {
  const bool inputs_on_device = (flags & EMIN_GALERKIN_DEVICE) != 0;
  g_galerkin_error.clear();
  g_galerkin_path = 0;
  if (n <= 0 || nc <= 0 || n >= INT32_MAX || nc >= INT32_MAX || !A_rowptr || !A_col || !A_val || !P_rowptr ||
      !P_col || !P_val || !Ac_rowptr || !nnz_out || (Ac_col && !Ac_val)) {
    g_galerkin_error = "bad argument";
    return EMIN_ERR_ARG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int SM = emin_num_sms();
  const int G = SM * 4;
  std::vector<void*> tmp;
  auto dal = [&](void** p, size_t bytes) -> cudaError_t {
    cudaError_t e = emin_mallocAsync(p, bytes + 64, s);
    if (e == cudaSuccess) tmp.push_back(*p);
    return e;
  };
  auto done = [&](emin_status st, const char* msg) {
    for (void* p : tmp) cudaFreeAsync(p, s);
    emin_pool_trim(s);   // the temporaries are large and one-off: back to the driver
    if (msg) g_galerkin_error = msg;
    return st;
  };
#define GK_TRY(x) do { if ((x) != cudaSuccess) return done(EMIN_ERR_CUDA, #x); } while (0)
  const cudaMemcpyKind h2d = cudaMemcpyHostToDevice;
  const int64_t *dArp = A_rowptr, *dPrp = P_rowptr;
  const int32_t *dAcol = A_col, *dPcol = P_col;
  const double *dAval = A_val, *dPval = P_val;
  int64_t nnzA = 0, nnzP = 0;
  if (inputs_on_device) {
    GK_TRY(cudaMemcpyAsync(&nnzA, A_rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GK_TRY(cudaMemcpyAsync(&nnzP, P_rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GK_TRY(cudaStreamSynchronize(s));
  } else {
    nnzA = A_rowptr[n];
    nnzP = P_rowptr[n];
    int64_t *a1, *p1; int32_t *a2, *p2; double *a3, *p3;
    GK_TRY(dal((void**)&a1, sizeof(int64_t) * (n + 1)));
    GK_TRY(dal((void**)&a2, sizeof(int32_t) * std::max<int64_t>(nnzA, 1)));
    GK_TRY(dal((void**)&a3, sizeof(double) * std::max<int64_t>(nnzA, 1)));
    GK_TRY(dal((void**)&p1, sizeof(int64_t) * (n + 1)));
    GK_TRY(dal((void**)&p2, sizeof(int32_t) * std::max<int64_t>(nnzP, 1)));
    GK_TRY(dal((void**)&p3, sizeof(double) * std::max<int64_t>(nnzP, 1)));
    GK_TRY(cudaMemcpyAsync(a1, A_rowptr, sizeof(int64_t) * (n + 1), h2d, s));
    GK_TRY(cudaMemcpyAsync(a2, A_col, sizeof(int32_t) * nnzA, h2d, s));
    GK_TRY(cudaMemcpyAsync(a3, A_val, sizeof(double) * nnzA, h2d, s));
    GK_TRY(cudaMemcpyAsync(p1, P_rowptr, sizeof(int64_t) * (n + 1), h2d, s));
    GK_TRY(cudaMemcpyAsync(p2, P_col, sizeof(int32_t) * nnzP, h2d, s));
    GK_TRY(cudaMemcpyAsync(p3, P_val, sizeof(double) * nnzP, h2d, s));
    dArp = a1; dAcol = a2; dAval = a3; dPrp = p1; dPcol = p2; dPval = p3;
  }
  if (nnzA < 0 || nnzP < 0 || nnzP >= INT32_MAX) return done(EMIN_ERR_ARG, "nnz out of range");
  int32_t* err;
  int64_t *tot, *scratch;
  GK_TRY(dal((void**)&err, sizeof(int32_t)));
  GK_TRY(dal((void**)&tot, sizeof(int64_t) * 2));
  GK_TRY(dal((void**)&scratch, sizeof(int64_t) * emin_scan_scratch_elems(std::max(n, nc) + 1)));
  GK_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), s));
  k_gk_check<<<G, 256, 0, s>>>(n, dArp, dAcol, n, err);
  k_gk_check<<<G, 256, 0, s>>>(n, dPrp, dPcol, nc, err);
  int32_t h_err = 0;
  GK_TRY(cudaMemcpyAsync(&h_err, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  GK_TRY(cudaStreamSynchronize(s));
  if (h_err) return done(EMIN_ERR_CSR, "row pointers decrease or column ids out of range");

  // ---- 3x3-block path (elasticity-structured A and P; same sums, bitwise)
  if (!(flags & EMIN_GALERKIN_POINT) && n % 3 == 0 && nc % 3 == 0) {
    const int64_t nn = n / 3, nnc = nc / 3;
    GK_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), s));
    k_bsr_check<<<G, 256, 0, s>>>(nn, dArp, dAcol, dPrp, dPcol, err);
    GK_TRY(cudaMemcpyAsync(&h_err, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    GK_TRY(cudaStreamSynchronize(s));
    // (a node row wider than the largest table: fall back to the point path)
    if (!h_err) do {
      auto sync_err = [&]() -> int32_t {
        int32_t h = 0;
        cudaMemcpyAsync(&h, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        return h;
      };
      // T = A P (BSR)
      BsrAP opT{dArp, dAcol, dAval, dPrp, dPcol, dPval};
      int64_t *cntT, *Tnp, nbT = 0;
      GK_TRY(dal((void**)&cntT, sizeof(int64_t) * (nn + 1)));
      GK_TRY(dal((void**)&Tnp, sizeof(int64_t) * (nn + 1)));
      BsrOut oT{};
      oT.nrows = nn; oT.cnt = cntT; oT.err = err;
      GK_TRY((bs_launch_all<0>(false, opT, oT, SM, s)));
      if (sync_err()) break;
      GK_TRY(emin_scan_i64(cntT, Tnp, nn, tot, scratch, s));
      GK_TRY(cudaMemcpyAsync(Tnp + nn, tot, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
      GK_TRY(cudaMemcpyAsync(&nbT, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      GK_TRY(cudaStreamSynchronize(s));
      int32_t* Tnc;
      double* Tv;
      if (dal((void**)&Tnc, sizeof(int32_t) * std::max<int64_t>(nbT, 1)) != cudaSuccess ||
          dal((void**)&Tv, sizeof(double) * 9 * std::max<int64_t>(nbT, 1)) != cudaSuccess)
        return done(EMIN_ERR_OOM, "A P: out of memory");
      oT.Onp = Tnp; oT.Onc = Tnc; oT.Ov = Tv;
      GK_TRY((bs_launch_all<0>(true, opT, oT, SM, s)));
      // P^T at node level: (c, I) entries sorted, with the position s of c in J_I
      int64_t *nlen, *nofs, *ccount, *Ptnp, M = 0;
      GK_TRY(dal((void**)&nlen, sizeof(int64_t) * (nn + 1)));
      GK_TRY(dal((void**)&nofs, sizeof(int64_t) * (nn + 1)));
      GK_TRY(dal((void**)&ccount, sizeof(int64_t) * (nnc + 1)));
      GK_TRY(dal((void**)&Ptnp, sizeof(int64_t) * (nnc + 1)));
      k_bsr_nodelen<<<G, 256, 0, s>>>(nn, dPrp, nlen);
      GK_TRY(emin_scan_i64(nlen, nofs, nn, tot + 1, scratch, s));
      GK_TRY(cudaMemcpyAsync(&M, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      GK_TRY(cudaStreamSynchronize(s));
      if (M >= INT32_MAX) return done(EMIN_ERR_ARG, "P: too many node entries");
      uint64_t *kin, *kout;
      int32_t *sin, *sout, *PtI;
      GK_TRY(dal((void**)&kin, sizeof(uint64_t) * std::max<int64_t>(M, 1)));
      GK_TRY(dal((void**)&kout, sizeof(uint64_t) * std::max<int64_t>(M, 1)));
      GK_TRY(dal((void**)&sin, sizeof(int32_t) * std::max<int64_t>(M, 1)));
      GK_TRY(dal((void**)&sout, sizeof(int32_t) * std::max<int64_t>(M, 1)));
      GK_TRY(dal((void**)&PtI, sizeof(int32_t) * std::max<int64_t>(M, 1)));
      GK_TRY(cudaMemsetAsync(ccount, 0, sizeof(int64_t) * (nnc + 1), s));
      k_bsr_tkeys<<<G, 256, 0, s>>>(nn, dPrp, dPcol, nofs, kin, sin, ccount);
      int eb = 1;
      while (eb < 64 && (((unsigned __int128)1) << eb) < (unsigned __int128)nnc * (unsigned __int128)nn) ++eb;
      size_t tb = 0;
      GK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, sin, sout, (int)M, 0, eb, s));
      void* ct;
      GK_TRY(dal(&ct, tb));
      GK_TRY(cub::DeviceRadixSort::SortPairs(ct, tb, kin, kout, sin, sout, (int)M, 0, eb, s));
      k_bsr_trows<<<G, 256, 0, s>>>(M, nn, kout, PtI);
      GK_TRY(emin_scan_i64(ccount, Ptnp, nnc, tot + 1, scratch, s));
      GK_TRY(cudaMemcpyAsync(Ptnp + nnc, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
      // A_c = P^T T: node counts, point row pointers, values
      BsrPtT opC{Ptnp, PtI, sout, dPrp, dPval, Tnp, Tnc, Tv};
      int64_t *cntC, *nbC, NB = 0;
      GK_TRY(dal((void**)&cntC, sizeof(int64_t) * (nnc + 1)));
      GK_TRY(dal((void**)&nbC, sizeof(int64_t) * (nnc + 1)));
      BsrOut oC{};
      oC.nrows = nnc; oC.cnt = cntC; oC.err = err;
      GK_TRY((bs_launch_all<1>(false, opC, oC, SM, s)));
      if (sync_err()) break;
      GK_TRY(emin_scan_i64(cntC, nbC, nnc, tot, scratch, s));
      GK_TRY(cudaMemcpyAsync(&NB, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      int64_t* Crp = Ac_rowptr;
      if (!inputs_on_device) GK_TRY(dal((void**)&Crp, sizeof(int64_t) * (nc + 1)));
      k_bsr_crp<<<G, 256, 0, s>>>(nnc, nbC, cntC, Crp);
      GK_TRY(cudaStreamSynchronize(s));
      const int64_t nnzC = 9 * NB;
      *nnz_out = nnzC;
      if (!inputs_on_device)
        GK_TRY(cudaMemcpyAsync(Ac_rowptr, Crp, sizeof(int64_t) * (nc + 1), cudaMemcpyDeviceToHost, s));
      if (Ac_col) {
        if (Ac_cap < nnzC) return done(EMIN_ERR_ARG, "Ac_cap < nnz (call again with a larger buffer)");
        int32_t* Ccol = Ac_col;
        double* Cval = Ac_val;
        if (!inputs_on_device) {
          GK_TRY(dal((void**)&Ccol, sizeof(int32_t) * std::max<int64_t>(nnzC, 1)));
          GK_TRY(dal((void**)&Cval, sizeof(double) * std::max<int64_t>(nnzC, 1)));
        }
        oC.Crp = Crp; oC.Ccol = Ccol; oC.Cval = Cval;
        GK_TRY((bs_launch_all<1>(true, opC, oC, SM, s)));
        if (!inputs_on_device) {
          GK_TRY(cudaMemcpyAsync(Ac_col, Ccol, sizeof(int32_t) * nnzC, cudaMemcpyDeviceToHost, s));
          GK_TRY(cudaMemcpyAsync(Ac_val, Cval, sizeof(double) * nnzC, cudaMemcpyDeviceToHost, s));
        }
      }
      GK_TRY(cudaGetLastError());
      g_galerkin_path = 1;
      return done(EMIN_OK, nullptr);
    } while (0);
    GK_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), s));
  }

  // one product X * Y -> O (symbolic, row pointers, numeric)
  auto product = [&](int64_t nrows, const int64_t* Xrp, const int32_t* Xcol, const double* Xval,
                     const int64_t* Yrp, const int32_t* Ycol, const double* Yval, int64_t* cnt, int64_t* Orp,
                     int64_t* nnz, int32_t** Ocol, double** Oval, bool sort, bool alloc) -> emin_status {
    GkArgs a{};
    a.nrows = nrows; a.Xrp = Xrp; a.Xcol = Xcol; a.Xval = Xval; a.Yrp = Yrp; a.Ycol = Ycol; a.Yval = Yval;
    a.cnt = cnt; a.sort = sort; a.err = err;
    if (gk_launch_all(false, a, SM, s) != cudaSuccess) return EMIN_ERR_CUDA;
    int32_t h = 0;
    if (cudaMemcpyAsync(&h, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return EMIN_ERR_CUDA;
    if (h) return EMIN_ERR_ARG;
    if (emin_scan_i64(cnt, Orp, nrows, tot, scratch, s) != cudaSuccess) return EMIN_ERR_CUDA;
    if (cudaMemcpyAsync(Orp + nrows, tot, sizeof(int64_t), cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(nnz, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return EMIN_ERR_CUDA;
    if (alloc) {
      if (dal((void**)Ocol, sizeof(int32_t) * std::max<int64_t>(*nnz, 1)) != cudaSuccess ||
          dal((void**)Oval, sizeof(double) * std::max<int64_t>(*nnz, 1)) != cudaSuccess)
        return EMIN_ERR_OOM;
    }
    if (!*Ocol) return EMIN_OK;
    a.Orp = Orp; a.Ocol = *Ocol; a.Oval = *Oval;
    if (gk_launch_all(true, a, SM, s) != cudaSuccess) return EMIN_ERR_CUDA;
    return EMIN_OK;
  };

  // T = A P
  int64_t *cntT, *Trp, nnzT = 0;
  int32_t* Tcol = nullptr;
  double* Tval = nullptr;
  GK_TRY(dal((void**)&cntT, sizeof(int64_t) * (n + 1)));
  GK_TRY(dal((void**)&Trp, sizeof(int64_t) * (n + 1)));
  emin_status st = product(n, dArp, dAcol, dAval, dPrp, dPcol, dPval, cntT, Trp, &nnzT, &Tcol, &Tval, false, true);
  if (st != EMIN_OK) return done(st, "A P: product failed (a row wider than 8192 columns, or out of memory)");

  // P^T: sort (col * n + row) keys with P's values
  uint64_t *kin, *kout;
  double* vout;
  int64_t *ccount, *Ptp;
  int32_t* Ptrow;
  GK_TRY(dal((void**)&kin, sizeof(uint64_t) * std::max<int64_t>(nnzP, 1)));
  GK_TRY(dal((void**)&kout, sizeof(uint64_t) * std::max<int64_t>(nnzP, 1)));
  GK_TRY(dal((void**)&vout, sizeof(double) * std::max<int64_t>(nnzP, 1)));
  GK_TRY(dal((void**)&ccount, sizeof(int64_t) * (nc + 1)));
  GK_TRY(dal((void**)&Ptp, sizeof(int64_t) * (nc + 1)));
  GK_TRY(dal((void**)&Ptrow, sizeof(int32_t) * std::max<int64_t>(nnzP, 1)));
  GK_TRY(cudaMemsetAsync(ccount, 0, sizeof(int64_t) * (nc + 1), s));
  k_gk_keys<<<G, 256, 0, s>>>(n, dPrp, dPcol, kin, ccount);
  int end_bit = 1;
  while (end_bit < 64 && (((unsigned __int128)1) << end_bit) < (unsigned __int128)nc * (unsigned __int128)n) ++end_bit;
  size_t tbytes = 0;
  GK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, kin, kout, dPval, vout, (int)nnzP, 0, end_bit, s));
  void* ctemp;
  GK_TRY(dal(&ctemp, tbytes));
  GK_TRY(cub::DeviceRadixSort::SortPairs(ctemp, tbytes, kin, kout, dPval, vout, (int)nnzP, 0, end_bit, s));
  k_gk_rows<<<G, 256, 0, s>>>(nnzP, n, kout, Ptrow);
  GK_TRY(emin_scan_i64(ccount, Ptp, nc, tot + 1, scratch, s));
  GK_TRY(cudaMemcpyAsync(Ptp + nc, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));

  // A_c = P^T T
  int64_t *cntC, *Crp, nnzC = 0;
  GK_TRY(dal((void**)&cntC, sizeof(int64_t) * (nc + 1)));
  Crp = Ac_rowptr;
  if (!inputs_on_device) GK_TRY(dal((void**)&Crp, sizeof(int64_t) * (nc + 1)));
  int32_t* Ccol = nullptr;
  double* Cval = nullptr;
  // count first (no output columns), then fill the caller's (or staging) buffers
  st = product(nc, Ptp, Ptrow, vout, Trp, Tcol, Tval, cntC, Crp, &nnzC, &Ccol, &Cval, true, false);
  if (st != EMIN_OK) return done(st, "P^T (A P): product failed (a row wider than 8192 columns)");
  *nnz_out = nnzC;
  if (!inputs_on_device)
    GK_TRY(cudaMemcpyAsync(Ac_rowptr, Crp, sizeof(int64_t) * (nc + 1), cudaMemcpyDeviceToHost, s));
  if (Ac_col) {
    if (Ac_cap < nnzC) return done(EMIN_ERR_ARG, "Ac_cap < nnz (call again with a larger buffer)");
    if (inputs_on_device) { Ccol = Ac_col; Cval = Ac_val; }
    else {
      GK_TRY(dal((void**)&Ccol, sizeof(int32_t) * std::max<int64_t>(nnzC, 1)));
      GK_TRY(dal((void**)&Cval, sizeof(double) * std::max<int64_t>(nnzC, 1)));
    }
    GkArgs a{};
    a.nrows = nc; a.Xrp = Ptp; a.Xcol = Ptrow; a.Xval = vout; a.Yrp = Trp; a.Ycol = Tcol; a.Yval = Tval;
    a.cnt = cntC; a.Orp = Crp; a.Ocol = Ccol; a.Oval = Cval; a.sort = 1; a.err = err;
    GK_TRY(gk_launch_all(true, a, SM, s));
    if (!inputs_on_device) {
      GK_TRY(cudaMemcpyAsync(Ac_col, Ccol, sizeof(int32_t) * nnzC, cudaMemcpyDeviceToHost, s));
      GK_TRY(cudaMemcpyAsync(Ac_val, Cval, sizeof(double) * nnzC, cudaMemcpyDeviceToHost, s));
    }
  }
  GK_TRY(cudaGetLastError());
  return done(EMIN_OK, nullptr);
#undef GK_TRY
}

extern "C" const char* emin_galerkin_error() { return g_galerkin_error.c_str(); }
extern "C" int32_t emin_galerkin_path() { return g_galerkin_path; }
