// dist.cu -- row-partitioned multi-GPU plumbing (NCCL over NVLink).
//
// P:980-986 [§4]: "the sparsity pattern adjacency information of P can be
// communicated only once before entering PCG, then for all the successive
// A P products only the entries of P are exchanged ... buffers ... allocated
// and set-up only once".  P:988-993: Pi_B needs no communication.
//
// Each rank owns a contiguous block of global rows (z-slabs for the
// lexicographic grids), hence a contiguous range of global F ids.  At setup
// the F rows referenced by the owned A_FF rows but owned elsewhere (the halo)
// are found, requested from their owners (global F ids), and their pattern
// rows (lengths, then coarse column ids) are received once and appended
// after the owned rows in the W layout (local ids nF .. nF+nH-1, ordered by
// global id, hence grouped by owner).  Per iteration only the values of the
// search direction y on those rows are exchanged (ncclSend/ncclRecv grouped,
// received in place into the halo tail of y); the two CG scalars are
// combined by ncclAllReduce of one double each.
#include <algorithm>
#include <cstring>
#include <vector>

#include "emin_internal.cuh"
#include "dist.cuh"

#ifdef EMIN_WITH_NCCL
#include <nccl.h>
#endif

namespace {

__global__ void k_mark_halo(int64_t m, int64_t row_begin, int64_t fbegin, int64_t fend,
                            const int64_t* __restrict__ Arp, const int32_t* __restrict__ Acol,
                            const uint8_t* __restrict__ isc, const int64_t* __restrict__ cidx,
                            int64_t* __restrict__ flag) {
  for (int64_t rl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rl < m; rl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row_begin + rl;
    if (isc[r]) continue;
    for (int64_t q = Arp[rl] - Arp[0]; q < Arp[rl + 1] - Arp[0]; ++q) {
      const int32_t c = Acol[q];
      if (isc[c]) continue;
      const int64_t g = (int64_t)c - cidx[c];
      if (g < fbegin || g >= fend) flag[g] = 1;
    }
  }
}

__global__ void k_halo_list(const int64_t* __restrict__ flag, const int64_t* __restrict__ pos, int64_t nFg,
                            int64_t* __restrict__ hlist) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nFg; g += (int64_t)gridDim.x * blockDim.x)
    if (flag[g]) hlist[pos[g]] = g;
}

__global__ void k_to_local(const int64_t* __restrict__ gids, int64_t n, int64_t fbegin, int32_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (int32_t)(gids[t] - fbegin);
}

__global__ void k_row_lengths(const int32_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ wptr,
                              int64_t* __restrict__ len) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    len[t] = wptr[rows[t] + 1] - wptr[rows[t]];
}

// send entry list: entries of the requested rows, concatenated
__global__ void k_send_entries(const int32_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ wptr,
                               const int64_t* __restrict__ off, int64_t* __restrict__ eidx) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = wptr[rows[t]], l = wptr[rows[t] + 1] - b, o = off[t];
    for (int64_t p = 0; p < l; ++p) eidx[o + p] = b + p;
  }
}

// halo wptr tail: wptr[nF + 1 + h] = nnzW + inclusive prefix of halo lengths
__global__ void k_halo_wptr(const int64_t* __restrict__ excl, const int64_t* __restrict__ len, int64_t nH,
                            int64_t nnzW, int64_t* __restrict__ wptr_tail) {
  for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nH; h += (int64_t)gridDim.x * blockDim.x)
    wptr_tail[h] = nnzW + excl[h] + len[h];
}

template <typename T>
__global__ void k_pack(const T* __restrict__ src, const int64_t* __restrict__ idx, int64_t n, T* __restrict__ dst) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[idx[t]];
}

}  // namespace

#ifdef EMIN_WITH_NCCL
#define NCCL_TRY(ctx, call)                                                                   \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) {                                                                  \
      (ctx)->last_error = std::string(#call) + ": " + ncclGetErrorString(r_);                 \
      return EMIN_ERR_NCCL;                                                                   \
    }                                                                                         \
  } while (0)

static ncclComm_t comm_of(emin_ctx c) { return (ncclComm_t)c->comm; }

template <typename T> static ncclDataType_t nccl_type();
template <> ncclDataType_t nccl_type<double>() { return ncclFloat64; }
template <> ncclDataType_t nccl_type<int64_t>() { return ncclInt64; }
template <> ncclDataType_t nccl_type<int32_t>() { return ncclInt32; }

// grouped point-to-point: send[p] (count, offset in sendbuf) / recv[p]
template <typename T>
static emin_status exchange(emin_ctx c, const T* sendbuf, const std::vector<int64_t>& scnt,
                            const std::vector<int64_t>& soff, T* recvbuf, const std::vector<int64_t>& rcnt,
                            const std::vector<int64_t>& roff, cudaStream_t s) {
  NCCL_TRY(c, ncclGroupStart());
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank) continue;
    if (scnt[p]) NCCL_TRY(c, ncclSend(sendbuf + soff[p], (size_t)scnt[p], nccl_type<T>(), p, comm_of(c), s));
    if (rcnt[p]) NCCL_TRY(c, ncclRecv(recvbuf + roff[p], (size_t)rcnt[p], nccl_type<T>(), p, comm_of(c), s));
  }
  NCCL_TRY(c, ncclGroupEnd());
  return EMIN_OK;
}
#endif

emin_status emin_dist_attach(emin_ctx c, void* comm) {
#ifdef EMIN_WITH_NCCL
  c->comm = comm;
  int n = 1, r = 0;
  NCCL_TRY(c, ncclCommCount(comm_of(c), &n));
  NCCL_TRY(c, ncclCommUserRank(comm_of(c), &r));
  c->nranks = n;
  c->rank = r;
  c->dist = new DistPlan();
  return EMIN_OK;
#else
  (void)comm;
  c->last_error = "libemin was built without NCCL";
  return EMIN_ERR_NCCL;
#endif
}

// Gather every rank's F range; find, request and receive the halo rows'
// pattern.  Fills c->dist, sets nFh / nnzWh, extends wptr / wcol (caller
// allocated them with room: see emin_dist_halo_sizes).
emin_status emin_dist_find_halo(emin_ctx c, int64_t fbegin, int64_t nF, int64_t nFg, int64_t m,
                                const int64_t* Arp, const int32_t* Acol, const uint8_t* isc,
                                const int64_t* cidx, int64_t* scratch) {
#ifdef EMIN_WITH_NCCL
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  const int R = c->nranks;
  const int SM = emin_num_sms();
  // ---- all F ranges
  int64_t* buf;
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&buf, sizeof(int64_t) * (2 + 2 * R), s));
  int64_t mine[2] = {fbegin, nF};
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(buf, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
  NCCL_TRY(c, ncclAllGather(buf, buf + 2, 2, ncclInt64, comm_of(c), s));
  std::vector<int64_t> all(2 * R);
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(all.data(), buf + 2, sizeof(int64_t) * 2 * R, cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  cudaFreeAsync(buf, s);
  d.fbeg.resize(R);
  d.fcnt.resize(R);
  for (int p = 0; p < R; ++p) { d.fbeg[p] = all[2 * p]; d.fcnt[p] = all[2 * p + 1]; }
  // ---- halo rows: F columns of owned rows outside [fbegin, fbegin + nF)
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&d.hflag, sizeof(int64_t) * std::max<int64_t>(nFg, 1), s));
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&d.hpos, sizeof(int64_t) * std::max<int64_t>(nFg + 1, 1), s));
  EMIN_CUDA_TRY(c, cudaMemsetAsync(d.hflag, 0, sizeof(int64_t) * std::max<int64_t>(nFg, 1), s));
  k_mark_halo<<<SM * 8, 256, 0, s>>>(m, c->opts.row_begin, fbegin, fbegin + nF, Arp, Acol, isc, cidx, d.hflag);
  int64_t* tot;
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&tot, sizeof(int64_t), s));
  EMIN_CUDA_TRY(c, emin_scan_i64(d.hflag, d.hpos, nFg, tot, scratch, s));
  int64_t nH = 0;
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(&nH, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  cudaFreeAsync(tot, s);
  d.nH = nH;
  int64_t* hlist;
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&hlist, sizeof(int64_t) * std::max<int64_t>(nH, 1), s));
  k_halo_list<<<SM * 8, 256, 0, s>>>(d.hflag, d.hpos, nFg, hlist);
  std::vector<int64_t> h_hlist(nH);
  if (nH) EMIN_CUDA_TRY(c, cudaMemcpyAsync(h_hlist.data(), hlist, sizeof(int64_t) * nH, cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  // ---- rows to receive per owner (hlist is sorted, owners own contiguous ranges)
  d.rrow.assign(R, 0);
  d.rrow_off.assign(R, 0);
  for (int64_t h = 0, p = 0; h < nH; ++h) {
    while (p < R && h_hlist[h] >= d.fbeg[p] + d.fcnt[p]) ++p;
    if (p >= R || h_hlist[h] < d.fbeg[p]) { c->last_error = "halo row owned by no rank"; return EMIN_ERR_ARG; }
    d.rrow[p]++;
  }
  for (int p = 1; p < R; ++p) d.rrow_off[p] = d.rrow_off[p - 1] + d.rrow[p - 1];
  // ---- counts matrix -> rows to send per requester
  int64_t* cm;
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&cm, sizeof(int64_t) * (R + R * R), s));
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(cm, d.rrow.data(), sizeof(int64_t) * R, cudaMemcpyHostToDevice, s));
  NCCL_TRY(c, ncclAllGather(cm, cm + R, R, ncclInt64, comm_of(c), s));
  std::vector<int64_t> M(R * R);
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(M.data(), cm + R, sizeof(int64_t) * R * R, cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  cudaFreeAsync(cm, s);
  d.srow.assign(R, 0);
  d.srow_off.assign(R, 0);
  for (int p = 0; p < R; ++p) d.srow[p] = M[(int64_t)p * R + c->rank];   // rank p wants this many of mine
  for (int p = 1; p < R; ++p) d.srow_off[p] = d.srow_off[p - 1] + d.srow[p - 1];
  d.nS = d.srow_off[R - 1] + d.srow[R - 1];
  // ---- the requests themselves (global F ids) -> local ids of rows to send
  int64_t* req;
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&req, sizeof(int64_t) * std::max<int64_t>(d.nS, 1), s));
  {
    emin_status st = exchange<int64_t>(c, hlist, d.rrow, d.rrow_off, req, d.srow, d.srow_off, s);
    if (st != EMIN_OK) return st;
  }
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&d.send_rows, sizeof(int32_t) * std::max<int64_t>(d.nS, 1), s));
  k_to_local<<<SM * 4, 256, 0, s>>>(req, d.nS, fbegin, d.send_rows);
  cudaFreeAsync(req, s);
  cudaFreeAsync(hlist, s);
  c->launches += 4;
  return EMIN_OK;
#else
  (void)fbegin; (void)nF; (void)nFg; (void)m; (void)Arp; (void)Acol; (void)isc; (void)cidx; (void)scratch;
  return EMIN_ERR_NCCL;
#endif
}

// After the owned wptr is known: exchange the lengths of the halo rows,
// extend wptr, build the send-entry list; returns the halo entry count.
emin_status emin_dist_halo_pattern_sizes(emin_ctx c, int64_t* scratch) {
#ifdef EMIN_WITH_NCCL
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  const int R = c->nranks;
  const int SM = emin_num_sms();
  int64_t *slen, *rlen, *excl, *tot;
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&slen, sizeof(int64_t) * (d.nS + 1), s));
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&rlen, sizeof(int64_t) * (d.nH + 1), s));
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&excl, sizeof(int64_t) * (std::max(d.nS, d.nH) + 1), s));
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&tot, sizeof(int64_t) * 2, s));
  k_row_lengths<<<SM * 4, 256, 0, s>>>(d.send_rows, d.nS, c->wptr, slen);
  {
    emin_status st = exchange<int64_t>(c, slen, d.srow, d.srow_off, rlen, d.rrow, d.rrow_off, s);
    if (st != EMIN_OK) return st;
  }
  // halo wptr tail
  EMIN_CUDA_TRY(c, emin_scan_i64(rlen, excl, d.nH, tot, scratch, s));
  k_halo_wptr<<<SM * 4, 256, 0, s>>>(excl, rlen, d.nH, c->nnzW, c->wptr + c->nF + 1);
  int64_t nHW = 0;
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(&nHW, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  // per-peer received entry counts: prefix sums of halo lengths at the peer boundaries
  std::vector<int64_t> h_excl(d.nH + 1, 0);
  if (d.nH) EMIN_CUDA_TRY(c, cudaMemcpyAsync(h_excl.data(), excl, sizeof(int64_t) * d.nH, cudaMemcpyDeviceToHost, s));
  // send entry list
  EMIN_CUDA_TRY(c, emin_scan_i64(slen, excl, d.nS, tot + 1, scratch, s));
  int64_t nSE = 0;
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(&nSE, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> h_sexcl(d.nS + 1, 0);
  if (d.nS) EMIN_CUDA_TRY(c, cudaMemcpyAsync(h_sexcl.data(), excl, sizeof(int64_t) * d.nS, cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  h_excl[d.nH] = nHW;
  h_sexcl[d.nS] = nSE;
  d.nHW = nHW;
  d.nSE = nSE;
  d.rent.assign(R, 0); d.rent_off.assign(R, 0); d.sent.assign(R, 0); d.sent_off.assign(R, 0);
  for (int p = 0; p < R; ++p) {
    d.rent_off[p] = h_excl[d.rrow_off[p]];
    d.rent[p] = h_excl[d.rrow_off[p] + d.rrow[p]] - d.rent_off[p];
    d.sent_off[p] = h_sexcl[d.srow_off[p]];
    d.sent[p] = h_sexcl[d.srow_off[p] + d.srow[p]] - d.sent_off[p];
  }
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&d.send_eidx, sizeof(int64_t) * std::max<int64_t>(nSE, 1), s));
  k_send_entries<<<SM * 4, 256, 0, s>>>(d.send_rows, d.nS, c->wptr, excl, d.send_eidx);
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&d.sendbuf, sizeof(double) * std::max<int64_t>(nSE, 1), s));
  cudaFreeAsync(slen, s); cudaFreeAsync(rlen, s); cudaFreeAsync(excl, s); cudaFreeAsync(tot, s);
  c->launches += 3 + 6;
  return EMIN_OK;
#else
  (void)scratch;
  return EMIN_ERR_NCCL;
#endif
}

// pattern (coarse ids) of the halo rows, once
emin_status emin_dist_halo_wcol(emin_ctx c) {
#ifdef EMIN_WITH_NCCL
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  int32_t* sb;
  EMIN_CUDA_TRY(c, cudaMallocAsync((void**)&sb, sizeof(int32_t) * std::max<int64_t>(d.nSE, 1), s));
  k_pack<int32_t><<<emin_num_sms() * 4, 256, 0, s>>>(c->wcol, d.send_eidx, d.nSE, sb);
  emin_status st = exchange<int32_t>(c, sb, d.sent, d.sent_off, c->wcol + c->nnzW, d.rent, d.rent_off, s);
  cudaFreeAsync(sb, s);
  c->launches += 1;
  return st;
#else
  return EMIN_ERR_NCCL;
#endif
}

// values of a W-layout vector on the halo rows (per iteration for y)
emin_status emin_dist_halo_values(emin_ctx c, double* vec, cudaStream_t s) {
#ifdef EMIN_WITH_NCCL
  DistPlan& d = *c->dist;
  if (d.nSE) k_pack<double><<<emin_num_sms() * 2, 256, 0, s>>>(vec, d.send_eidx, d.nSE, d.sendbuf);
  c->launches += d.nSE ? 1 : 0;
  return exchange<double>(c, d.sendbuf, d.sent, d.sent_off, vec + c->nnzW, d.rent, d.rent_off, s);
#else
  (void)vec; (void)s;
  return EMIN_ERR_NCCL;
#endif
}

// in-place sum of n doubles over the ranks
emin_status emin_dist_allreduce(emin_ctx c, double* dev, int n, cudaStream_t s) {
#ifdef EMIN_WITH_NCCL
  NCCL_TRY(c, ncclAllReduce(dev, dev, (size_t)n, ncclFloat64, ncclSum, comm_of(c), s));
  return EMIN_OK;
#else
  (void)dev; (void)n; (void)s;
  return EMIN_ERR_NCCL;
#endif
}

emin_status emin_dist_allreduce_max_i32(emin_ctx c, int32_t* dev, cudaStream_t s) {
#ifdef EMIN_WITH_NCCL
  NCCL_TRY(c, ncclAllReduce(dev, dev, 1, ncclInt32, ncclMax, comm_of(c), s));
  return EMIN_OK;
#else
  (void)dev; (void)s;
  return EMIN_ERR_NCCL;
#endif
}

void emin_dist_free(emin_ctx c) {
  if (!c->dist) return;
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  void* ptrs[] = {d.hflag, d.hpos, d.send_rows, d.send_eidx, d.sendbuf};
  for (void* p : ptrs) if (p) cudaFreeAsync(p, s);
  delete c->dist;
  c->dist = nullptr;
}

// ---------------------------------------------------------------- NCCL helpers (ABI)
extern "C" emin_status emin_nccl_unique_id(uint8_t* id128) {
#ifdef EMIN_WITH_NCCL
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return EMIN_ERR_NCCL;
  std::memcpy(id128, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  return EMIN_OK;
#else
  (void)id128;
  return EMIN_ERR_NCCL;
#endif
}

extern "C" emin_status emin_nccl_comm_init(void** comm, int32_t nranks, const uint8_t* id128, int32_t rank) {
#ifdef EMIN_WITH_NCCL
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t cm;
  if (ncclCommInitRank(&cm, nranks, id, rank) != ncclSuccess) return EMIN_ERR_NCCL;
  *comm = cm;
  return EMIN_OK;
#else
  (void)comm; (void)nranks; (void)id128; (void)rank;
  return EMIN_ERR_NCCL;
#endif
}

extern "C" emin_status emin_nccl_comm_destroy(void* comm) {
#ifdef EMIN_WITH_NCCL
  if (comm) ncclCommDestroy((ncclComm_t)comm);
  return EMIN_OK;
#else
  (void)comm;
  return EMIN_ERR_NCCL;
#endif
}
