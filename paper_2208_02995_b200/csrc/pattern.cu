// pattern.cu -- Alg. 1's pattern growth on the GPU (PTent_SetUp, P:527-540,
// with the distance-l pattern of Eq. enlPatt):
// emin_pattern().
//
// The graph: an edge i ~ k for every off-diagonal nonzero of A (reading A12,
// no strength threshold); with block_size 3 the node graph (node I ~ K if the
// 3x3 block (I,K) holds a nonzero, read from row 3I) and the pattern applied
// blockwise.  For every F node: N_l = the C nodes within graph distance l,
// l = l0, l0 + 1, ... until the Gram matrix G = M^T M of M = V_c(J,:) (J = the
// dofs of N_l) has lambda_min > 1e-10 lambda_max, unconditionally at l =
// lmax (reading A25, the input generator's criterion).  Columns ascending.
//
// One warp per F node: breadth-first layers in shared memory -- a
// generation-tagged open-addressing set of visited nodes (no clearing between
// nodes), the current / next frontier, the list of C nodes reached; the Gram
// matrix by a warp reduction, its extreme eigenvalues by cyclic Jacobi in one
// lane; the list sorted by ranks.  Two launches: counts, then columns.
#include <algorithm>
#include <cstring>
#include <vector>

#include "emin_internal.cuh"

namespace {

// two tiers of per-warp sets: every node first runs with the small sets (4
// warps per CTA, ~7.7 KB each -> 32 warps per SM); the nodes whose
// neighbourhood overflows them are flagged and re-run with the large sets
// (one warp per CTA, 28 KB).  Static shared memory stays <= 48 KB per CTA.
constexpr int PT_WARPS = 1;       // large tier
constexpr int PT_HASH = 2048;     // visited-set slots per warp
constexpr int PT_FRONT = 1024;    // frontier capacity
constexpr int PT_CLIST = 1024;    // C nodes reached
constexpr int PS_WARPS = 4;       // small tier
constexpr int PS_HASH = 512;
constexpr int PS_FRONT = 256;
constexpr int PS_CLIST = 256;

struct PtArgs {
  int64_t nn;                     // nodes (= n / bs)
  int bs, nv, l0, lmax;
  const int64_t* Arp;
  const int32_t* Acol;
  const int64_t* cid;             // coarse node id or -1
  const double* Bc;               // [nc x nv] point-level coarse near kernel
  const int64_t* fnode;           // F node list
  int64_t nfn;
  int64_t* cnt;                   // [nfn] C nodes per F node (count pass)
  const int64_t* colofs;          // [nfn] first column slot of the node's first row (fill pass)
  int32_t* col;                   // fill pass output (P_col)
  const int64_t* rowofs;          // [nn * bs + 1] row pointers (fill pass)
  int32_t* overflow;
  uint8_t* big;                   // [nfn] node overflowed the small sets
};

// extreme eigenvalues of the symmetric N x N matrix a (row-major, destroyed)
// by cyclic Jacobi rotations, fully unrolled (registers); stops when the
// off-diagonal mass is below (1e-16 trace)^2 (the oracle's criterion)
template <int N>
__device__ void pt_jacobi_minmax(double* a, double* mn, double* mx) {
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0, tr = 0.0;
#pragma unroll
    for (int p = 0; p < N; ++p) {
      tr += fabs(a[p * N + p]);
#pragma unroll
      for (int q = p + 1; q < N; ++q) off += a[p * N + q] * a[p * N + q];
    }
    if (off <= 1e-32 * tr * tr) break;
#pragma unroll
    for (int p = 0; p < N; ++p)
#pragma unroll
      for (int q = p + 1; q < N; ++q) {
        const double apq = a[p * N + q];
        if (apq == 0.0) continue;
        const double theta = (a[q * N + q] - a[p * N + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double akp = a[k * N + p], akq = a[k * N + q];
          a[k * N + p] = c * akp - s * akq;
          a[k * N + q] = s * akp + c * akq;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double apk = a[p * N + k], aqk = a[q * N + k];
          a[p * N + k] = c * apk - s * aqk;
          a[q * N + k] = s * apk + c * aqk;
        }
      }
  }
  double lo = a[0], hi = a[0];
#pragma unroll
  for (int k = 1; k < N; ++k) { lo = fmin(lo, a[k * N + k]); hi = fmax(hi, a[k * N + k]); }
  *mn = lo;
  *mx = hi;
}

template <int N>
__device__ bool pt_full_rank(const double* G) {
  double a[N * N], mn, mx;
#pragma unroll
  for (int k = 0; k < N * N; ++k) a[k] = G[k];
  pt_jacobi_minmax<N>(a, &mn, &mx);
  return mn > 1e-10 * fmax(mx, 0.0);
}

__device__ bool pt_full_rank_nv(int nv, const double* G) {
  switch (nv) {
    case 1: return pt_full_rank<1>(G);
    case 2: return pt_full_rank<2>(G);
    case 3: return pt_full_rank<3>(G);
    case 4: return pt_full_rank<4>(G);
    case 5: return pt_full_rank<5>(G);
    case 6: return pt_full_rank<6>(G);
    case 7: return pt_full_rank<7>(G);
    default: return pt_full_rank<8>(G);
  }
}

template <bool FILL, bool BIG, int WARPS, int HASH, int FRONT, int CLIST>
__global__ void __launch_bounds__(WARPS * 32)
k_pattern(PtArgs a) {
  __shared__ unsigned long long s_hash[WARPS][HASH];   // (generation << 32) | node
  __shared__ int32_t s_front[WARPS][2][FRONT];
  __shared__ int32_t s_cl[WARPS][CLIST];
  __shared__ int32_t s_n[WARPS][3];                       // frontier size, next size, C count
  __shared__ double s_G[WARPS][EMIN_NV_MAX * EMIN_NV_MAX];
  __shared__ int s_ok[WARPS];
  __shared__ int s_ovf[WARPS];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int k = lane; k < HASH; k += 32) s_hash[wib][k] = ~0ull;
  __syncwarp();
  const int nv = a.nv, bs = a.bs;
  // small tier: an overflow flags the node (re-run by the large tier);
  // large tier: only flagged nodes, an overflow is an error
  auto overflow = [&]() { if (BIG) atomicExch(a.overflow, 1); else s_ovf[wib] = 1; };
  for (int64_t f = gw; f < a.nfn; f += nw) {
    if (BIG ? !a.big[f] : (FILL && a.big[f])) continue;     // warp-uniform
    if (lane == 0) s_ovf[wib] = 0;
    const unsigned long long gen = (unsigned long long)(f + 1) << 32;   // this node's tag (never ~0)
    const int32_t I = (int32_t)a.fnode[f];
    auto insert = [&](int32_t w) -> bool {      // true if w was not yet visited for this node
      unsigned h = ((unsigned)w * 2654435761u) & (HASH - 1);
      const unsigned long long key = gen | (unsigned)w;
      for (int probe = 0; probe < HASH; ++probe) {
        const unsigned long long cur = s_hash[wib][h];
        if (cur == key) return false;
        if ((cur >> 32) != (gen >> 32)) {      // stale or empty slot: claim it
          const unsigned long long prev = atomicCAS(&s_hash[wib][h], cur, key);
          if (prev == cur) return true;
          if (prev == key) return false;
          continue;                            // lost the race to another key: re-read
        }
        h = (h + 1) & (HASH - 1);
      }
      overflow();
      return false;
    };
    // s_cl[0 .. ncl) ascending (the coarse ids are distinct: rank = position)
    auto sort_clist = [&](int ncl, int32_t* tmpbuf) {
      __syncwarp();
      for (int t = lane; t < ncl; t += 32) {
        const int32_t c = s_cl[wib][t];
        int rk = 0;
        for (int u = 0; u < ncl; ++u) rk += s_cl[wib][u] < c;
        tmpbuf[rk] = c;
      }
      __syncwarp();
      for (int t = lane; t < ncl; t += 32) s_cl[wib][t] = tmpbuf[t];
      __syncwarp();
    };
    if (lane == 0) {
      s_n[wib][0] = 1;
      s_n[wib][2] = 0;
      s_front[wib][0][0] = I;
    }
    if (lane == 0) insert(I);
    __syncwarp();
    int cur = 0;
    for (int l = 1; l <= a.lmax; ++l) {
      if (lane == 0) s_n[wib][1] = 0;
      __syncwarp();
      const int nf = s_n[wib][0];
      for (int x = lane; x < nf; x += 32) {
        const int64_t r = (int64_t)s_front[wib][cur][x] * bs;
        int32_t prevw = -1;
        for (int64_t q = a.Arp[r]; q < a.Arp[r + 1]; ++q) {
          const int32_t w = a.Acol[q] / bs;
          if (w == prevw) continue;               // the other dofs of the same node (3x3 blocks)
          prevw = w;
          if (!insert(w)) continue;
          const int pos = atomicAdd(&s_n[wib][1], 1);
          if (pos < FRONT) s_front[wib][cur ^ 1][pos] = w; else overflow();
          const int64_t c = a.cid[w];
          if (c >= 0) {
            const int cp = atomicAdd(&s_n[wib][2], 1);
            if (cp < CLIST) s_cl[wib][cp] = (int32_t)c; else overflow();
          }
        }
      }
      __syncwarp();
      if (lane == 0) s_n[wib][0] = min(s_n[wib][1], FRONT);
      cur ^= 1;
      __syncwarp();
      if (l < a.l0) continue;
      if (l == a.lmax) break;
      if (!BIG && s_ovf[wib]) break;          // flagged: the large tier redoes this node
      const int ncl = min(s_n[wib][2], CLIST);
      if (ncl == 0) continue;
      sort_clist(ncl, s_front[wib][cur ^ 1]);   // deterministic Gram summation order
      // Gram matrix of M = V_c(J,:), J = the dofs of the C nodes reached
      for (int pq = 0; pq < nv * nv; ++pq) {
        const int p = pq / nv, q2 = pq - p * nv;
        double sum = 0.0;
        for (int t = lane; t < ncl; t += 32)
          for (int b = 0; b < bs; ++b) {
            const double* row = a.Bc + ((int64_t)bs * s_cl[wib][t] + b) * nv;
            sum += row[p] * row[q2];
          }
        sum = warp_sum(sum);
        if (lane == 0) s_G[wib][pq] = sum;
      }
      __syncwarp();
      if (lane == 0) s_ok[wib] = pt_full_rank_nv(nv, s_G[wib]);
      __syncwarp();
      if (s_ok[wib]) break;
    }
    __syncwarp();
    if (!BIG && s_ovf[wib]) {                   // (count pass only: fill skips flagged nodes)
      if (lane == 0) a.big[f] = 1;
      __syncwarp();
      continue;
    }
    const int ncl = min(s_n[wib][2], CLIST);
    if (!FILL) {
      if (lane == 0) a.cnt[f] = ncl;
    } else {
      sort_clist(ncl, s_front[wib][cur ^ 1]);
      const int64_t node_row0 = (int64_t)I * bs;
      for (int t = lane; t < ncl; t += 32) {
        const int32_t c = s_cl[wib][t];
        for (int d = 0; d < bs; ++d) {
          int32_t* dst = a.col + a.rowofs[node_row0 + d];
          for (int b = 0; b < bs; ++b) dst[(int64_t)t * bs + b] = bs * c + b;
        }
      }
    }
    __syncwarp();
  }
}

__global__ void k_pt_nodes(int64_t nn, int bs, const uint8_t* __restrict__ isc, int64_t* __restrict__ cflag) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nn; u += (int64_t)gridDim.x * blockDim.x)
    cflag[u] = isc[u * bs] ? 1 : 0;
}

// row lengths: C rows 1, F rows bs * (C nodes of the node)
__global__ void k_pt_rowlen(int64_t nn, int bs, const int64_t* __restrict__ cid, const int64_t* __restrict__ fpos,
                            const int64_t* __restrict__ cnt, int64_t* __restrict__ rowlen) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nn; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = cid[u] >= 0 ? 1 : bs * cnt[fpos[u]];
    for (int d = 0; d < bs; ++d) rowlen[u * bs + d] = len;
  }
}

__global__ void k_pt_crows(int64_t nn, int bs, const int64_t* __restrict__ cid, const int64_t* __restrict__ rowofs,
                           int32_t* __restrict__ col) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nn; u += (int64_t)gridDim.x * blockDim.x)
    if (cid[u] >= 0)
      for (int d = 0; d < bs; ++d) col[rowofs[u * bs + d]] = (int32_t)(bs * cid[u] + d);
}

__global__ void k_pt_index(int64_t nn, const int64_t* __restrict__ cflag, const int64_t* __restrict__ cscan,
                           int64_t* __restrict__ cid, int64_t* __restrict__ fpos, int64_t* __restrict__ fnode) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nn; u += (int64_t)gridDim.x * blockDim.x) {
    if (cflag[u]) { cid[u] = cscan[u]; fpos[u] = -1; }
    else { cid[u] = -1; const int64_t fp = u - cscan[u]; fpos[u] = fp; fnode[fp] = u; }
  }
}

}  // namespace

static thread_local std::string g_pattern_error;

extern "C" emin_status emin_pattern(int64_t n, const int64_t* A_rowptr, const int32_t* A_col, const uint8_t* is_coarse,
                                    int32_t block_size, int32_t nv, const double* Bc, int64_t nc, int32_t l0,
                                    int32_t lmax, int64_t* P_rowptr, int32_t* P_col, int64_t P_col_cap,
                                    int64_t* nnz_out, int32_t inputs_on_device, void* stream) {
  g_pattern_error.clear();
  if (n <= 0 || !A_rowptr || !A_col || !is_coarse || !Bc || !P_rowptr || !nnz_out || nv < 1 || nv > EMIN_NV_MAX ||
      (block_size != 1 && block_size != 3) || n % block_size || l0 < 1 || lmax < l0 || nc < 0) {
    g_pattern_error = "bad argument";
    return EMIN_ERR_ARG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int bs = block_size;
  const int64_t nn = n / bs;
  const int SM = emin_num_sms();
  std::vector<void*> tmp;
  auto dal = [&](void** p, size_t bytes) -> cudaError_t {
    cudaError_t e = emin_mallocAsync(p, bytes + 64, s);
    if (e == cudaSuccess) tmp.push_back(*p);
    return e;
  };
  auto done = [&](emin_status st, const char* msg) {
    for (void* p : tmp) cudaFreeAsync(p, s);
    emin_pool_trim(s);   // the temporaries are large and one-off: back to the driver
    if (msg) g_pattern_error = msg;
    return st;
  };
#define PT_TRY(x) do { if ((x) != cudaSuccess) return done(EMIN_ERR_CUDA, #x); } while (0)
  const int64_t* dArp = A_rowptr;
  const int32_t* dAcol = A_col;
  const uint8_t* dIsc = is_coarse;
  const double* dBc = Bc;
  int64_t nnzA = 0;
  if (!inputs_on_device) {
    nnzA = A_rowptr[n];
    int64_t* a1; int32_t* a2; uint8_t* a3; double* a4;
    PT_TRY(dal((void**)&a1, sizeof(int64_t) * (n + 1)));
    PT_TRY(cudaMemcpyAsync(a1, A_rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    PT_TRY(dal((void**)&a2, sizeof(int32_t) * std::max<int64_t>(nnzA, 1)));
    PT_TRY(cudaMemcpyAsync(a2, A_col, sizeof(int32_t) * nnzA, cudaMemcpyHostToDevice, s));
    PT_TRY(dal((void**)&a3, n));
    PT_TRY(cudaMemcpyAsync(a3, is_coarse, n, cudaMemcpyHostToDevice, s));
    PT_TRY(dal((void**)&a4, sizeof(double) * std::max<int64_t>(nc * nv, 1)));
    PT_TRY(cudaMemcpyAsync(a4, Bc, sizeof(double) * nc * nv, cudaMemcpyHostToDevice, s));
    dArp = a1; dAcol = a2; dIsc = a3; dBc = a4;
  }
  int64_t *cflag, *cscan, *cid, *fpos, *fnode, *cnt, *rowlen, *rowofs, *tot, *scratch;
  int32_t* ovf;
  PT_TRY(dal((void**)&cflag, sizeof(int64_t) * (nn + 1)));
  PT_TRY(dal((void**)&cscan, sizeof(int64_t) * (nn + 1)));
  PT_TRY(dal((void**)&cid, sizeof(int64_t) * nn));
  PT_TRY(dal((void**)&fpos, sizeof(int64_t) * nn));
  PT_TRY(dal((void**)&fnode, sizeof(int64_t) * nn));
  PT_TRY(dal((void**)&tot, sizeof(int64_t) * 2));
  PT_TRY(dal((void**)&scratch, sizeof(int64_t) * emin_scan_scratch_elems(n + 1)));
  PT_TRY(dal((void**)&ovf, sizeof(int32_t)));
  PT_TRY(cudaMemsetAsync(ovf, 0, sizeof(int32_t), s));
  k_pt_nodes<<<SM * 4, 256, 0, s>>>(nn, bs, dIsc, cflag);
  PT_TRY(emin_scan_i64(cflag, cscan, nn, tot, scratch, s));
  int64_t h_nc = 0;
  PT_TRY(cudaMemcpyAsync(&h_nc, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  k_pt_index<<<SM * 4, 256, 0, s>>>(nn, cflag, cscan, cid, fpos, fnode);
  PT_TRY(cudaStreamSynchronize(s));
  if (h_nc * bs != nc) return done(EMIN_ERR_ARG, "sum(is_coarse) != nc");
  const int64_t nfn = nn - h_nc;
  PT_TRY(dal((void**)&cnt, sizeof(int64_t) * std::max<int64_t>(nfn, 1)));
  PT_TRY(dal((void**)&rowlen, sizeof(int64_t) * (n + 1)));
  PT_TRY(dal((void**)&rowofs, sizeof(int64_t) * (n + 1)));
  PtArgs pa;
  pa.nn = nn; pa.bs = bs; pa.nv = nv; pa.l0 = l0; pa.lmax = lmax;
  pa.Arp = dArp; pa.Acol = dAcol; pa.cid = cid; pa.Bc = dBc; pa.fnode = fnode; pa.nfn = nfn;
  pa.cnt = cnt; pa.colofs = nullptr; pa.col = nullptr; pa.rowofs = nullptr; pa.overflow = ovf;
  uint8_t* big;
  PT_TRY(dal((void**)&big, std::max<int64_t>(nfn, 1)));
  PT_TRY(cudaMemsetAsync(big, 0, std::max<int64_t>(nfn, 1), s));
  pa.big = big;
  const int gs = (int)std::max<int64_t>(1, std::min<int64_t>((nfn + PS_WARPS - 1) / PS_WARPS, (int64_t)SM * 8));
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nfn + PT_WARPS - 1) / PT_WARPS, (int64_t)SM * 8));
  if (nfn) {
    k_pattern<false, false, PS_WARPS, PS_HASH, PS_FRONT, PS_CLIST><<<gs, PS_WARPS * 32, 0, s>>>(pa);
    k_pattern<false, true, PT_WARPS, PT_HASH, PT_FRONT, PT_CLIST><<<g, PT_WARPS * 32, 0, s>>>(pa);
  }
  k_pt_rowlen<<<SM * 4, 256, 0, s>>>(nn, bs, cid, fpos, cnt, rowlen);
  PT_TRY(emin_scan_i64(rowlen, rowofs, n, tot + 1, scratch, s));
  PT_TRY(cudaMemcpyAsync(rowofs + n, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  int64_t h_nnz = 0;
  int32_t h_ovf = 0;
  PT_TRY(cudaMemcpyAsync(&h_nnz, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  PT_TRY(cudaMemcpyAsync(&h_ovf, ovf, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  PT_TRY(cudaStreamSynchronize(s));
  if (h_ovf) return done(EMIN_ERR_PATTERN, "neighbourhood larger than the kernel's shared-memory sets");
  *nnz_out = h_nnz;
  PT_TRY(cudaMemcpyAsync(P_rowptr, rowofs, sizeof(int64_t) * (n + 1),
                         inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (P_col) {
    if (P_col_cap < h_nnz) return done(EMIN_ERR_ARG, "P_col_cap < nnz (call again with a larger buffer)");
    int32_t* dcol = P_col;
    if (!inputs_on_device) PT_TRY(dal((void**)&dcol, sizeof(int32_t) * std::max<int64_t>(h_nnz, 1)));
    pa.col = dcol;
    pa.rowofs = rowofs;
    if (nfn) {
      k_pattern<true, false, PS_WARPS, PS_HASH, PS_FRONT, PS_CLIST><<<gs, PS_WARPS * 32, 0, s>>>(pa);
      k_pattern<true, true, PT_WARPS, PT_HASH, PT_FRONT, PT_CLIST><<<g, PT_WARPS * 32, 0, s>>>(pa);
    }
    k_pt_crows<<<SM * 4, 256, 0, s>>>(nn, bs, cid, rowofs, dcol);
    if (!inputs_on_device) PT_TRY(cudaMemcpyAsync(P_col, dcol, sizeof(int32_t) * h_nnz, cudaMemcpyDeviceToHost, s));
  }
  PT_TRY(cudaGetLastError());
  return done(EMIN_OK, nullptr);
#undef PT_TRY
}

extern "C" const char* emin_pattern_error() { return g_pattern_error.c_str(); }
