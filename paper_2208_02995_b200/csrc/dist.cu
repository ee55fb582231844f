// dist.cu -- row-partitioned multi-GPU plumbing: the halo plan, and the two
// transports behind it (NCCL over NVLink; the in-process loopback group).
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
//
// The same plan runs over either transport (dist.cuh::Transport): NCCL, one
// process per GPU; or the loopback group, R contexts in one process driven
// by R host threads, whose exchange is one cudaMemcpyAsync per (sender,
// receiver) pair ordered by CUDA events and whose sums add the R rank-local
// values in rank order -- so the halo plan, the halo tail of the W layout
// and the per-iteration exchange run (and are tested) with R > 1 ranks on a
// single device.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
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

__global__ void k_sum_ranks(const double* __restrict__ g, int R, int n, double* __restrict__ out) {
  const int j = threadIdx.x;
  if (j < n) {
    double t = g[j];
    for (int p = 1; p < R; ++p) t += g[p * n + j];   // rank order
    out[j] = t;
  }
}

#ifdef EMIN_WITH_NCCL
#define NCCL_TRY(ctx, call)                                                                   \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) {                                                                  \
      (ctx)->last_error = std::string(#call) + ": " + ncclGetErrorString(r_);                 \
      return EMIN_ERR_NCCL;                                                                   \
    }                                                                                         \
  } while (0)

// ---------------------------------------------------------------- NCCL
struct NcclTransport final : Transport {
  ncclComm_t comm;
  explicit NcclTransport(ncclComm_t cm) : comm(cm) {}
  emin_status allgather_i64(emin_ctx c, const int64_t* mine, int n, int64_t* all) override {
    cudaStream_t s = c->stream;
    int64_t* buf;
    EMIN_CUDA_TRY(c, emin_mallocAsync(&buf, sizeof(int64_t) * n * (1 + c->nranks), s));
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(buf, mine, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    NCCL_TRY(c, ncclAllGather(buf, buf + n, (size_t)n, ncclInt64, comm, s));
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(all, buf + n, sizeof(int64_t) * n * c->nranks, cudaMemcpyDeviceToHost, s));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
    cudaFreeAsync(buf, s);
    return EMIN_OK;
  }
  emin_status exchange(emin_ctx c, const void* sendbuf, size_t esz, const std::vector<int64_t>& scnt,
                       const std::vector<int64_t>& soff, void* recvbuf, const std::vector<int64_t>& rcnt,
                       const std::vector<int64_t>& roff, cudaStream_t s) override {
    const char* sb = static_cast<const char*>(sendbuf);
    char* rb = static_cast<char*>(recvbuf);
    NCCL_TRY(c, ncclGroupStart());
    for (int p = 0; p < c->nranks; ++p) {
      if (p == c->rank) continue;
      if (scnt[p]) NCCL_TRY(c, ncclSend(sb + soff[p] * esz, (size_t)scnt[p] * esz, ncclInt8, p, comm, s));
      if (rcnt[p]) NCCL_TRY(c, ncclRecv(rb + roff[p] * esz, (size_t)rcnt[p] * esz, ncclInt8, p, comm, s));
    }
    NCCL_TRY(c, ncclGroupEnd());
    return EMIN_OK;
  }
  emin_status allreduce_sum(emin_ctx c, const double* in, double* out, int n, cudaStream_t s) override {
    NCCL_TRY(c, ncclAllReduce(in, out, (size_t)n, ncclFloat64, ncclSum, comm, s));
    return EMIN_OK;
  }
  emin_status allreduce_max_i32(emin_ctx c, int32_t* inout, cudaStream_t s) override {
    NCCL_TRY(c, ncclAllReduce(inout, inout, 1, ncclInt32, ncclMax, comm, s));
    return EMIN_OK;
  }
  bool capturable() const override { return true; }
};
#endif

// ---------------------------------------------------------------- loopback
// Shared by the R contexts of one group.  A generation barrier on the host
// orders the publication of each rank's buffers and events; the device-side
// order is carried by the events (stream waits, copies on the waiting
// rank's stream): nothing on the device waits for another rank's kernel.
struct LoopbackGroup {
  int R;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  struct Slot {
    const void* buf = nullptr;
    size_t esz = 0;
    std::vector<int64_t> scnt, soff;
    std::vector<int64_t> host;
    cudaEvent_t ready = nullptr, done = nullptr;
    double* gbuf = nullptr;     // [R * 4] gathered rank-local sums (device of the rank)
  };
  std::vector<Slot> slot;
  bool aborted = false;
  std::string why;
  explicit LoopbackGroup(int r) : R(r), slot(r) {}
  // false if the group was aborted (a rank failed) or a peer did not arrive
  // within 300 s: no rank is left waiting for a peer that is gone
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const int64_t g = gen;
    if (++arrived == R) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g || aborted; })) {
      aborted = true;
      why = "a peer rank did not reach the collective within 300 s";
      cv.notify_all();
    }
    return !aborted;
  }
  void abort(const std::string& w) {
    std::lock_guard<std::mutex> lk(mu);
    if (!aborted) { aborted = true; why = w; }
    cv.notify_all();
  }
};

struct LoopbackTransport final : Transport {
  LoopbackGroup* G;
  int r;
  LoopbackTransport(LoopbackGroup* g, int rank) : G(g), r(rank) {}
  LoopbackGroup::Slot& me() { return G->slot[r]; }
  emin_status gone(emin_ctx c) {
    c->last_error = "loopback group aborted: " + G->why;
    return EMIN_ERR_CUDA;
  }
  void abort(const std::string& why) override { G->abort("rank " + std::to_string(r) + ": " + why); }
  emin_status allgather_i64(emin_ctx c, const int64_t* mine, int n, int64_t* all) override {
    me().host.assign(mine, mine + n);
    if (!G->barrier()) return gone(c);
    for (int p = 0; p < G->R; ++p)
      for (int j = 0; j < n; ++j) all[(int64_t)p * n + j] = G->slot[p].host[j];
    if (!G->barrier()) return gone(c);
    return EMIN_OK;
  }
  emin_status exchange(emin_ctx c, const void* sendbuf, size_t esz, const std::vector<int64_t>& scnt,
                       const std::vector<int64_t>& soff, void* recvbuf, const std::vector<int64_t>& rcnt,
                       const std::vector<int64_t>& roff, cudaStream_t s) override {
    {
      const cudaError_t e0 = cudaGetLastError();
      if (e0 != cudaSuccess) {
        c->last_error = std::string("loopback exchange: error pending before the collective: ") +
                        cudaGetErrorString(e0);
        G->abort(c->last_error);
        return EMIN_ERR_CUDA;
      }
    }
    me().buf = sendbuf;
    me().esz = esz;
    me().scnt = scnt;
    me().soff = soff;
    cudaError_t e = cudaEventRecord(me().ready, s);
    if (!G->barrier()) return gone(c);
    // pull every peer's slice for me (one copy per sender)
    for (int p = 0; p < G->R && e == cudaSuccess; ++p) {
      if (p == r || !rcnt[p]) continue;
      const LoopbackGroup::Slot& q = G->slot[p];
      if (q.esz != esz || q.scnt[r] != rcnt[p]) {
        c->last_error = "loopback exchange: rank " + std::to_string(r) + " expects " + std::to_string(rcnt[p]) +
                        " elements of " + std::to_string(esz) + " bytes from rank " + std::to_string(p) +
                        ", which sends " + std::to_string(q.scnt[r]) + " of " + std::to_string(q.esz);
        e = cudaErrorInvalidValue;
        break;
      }
      e = cudaStreamWaitEvent(s, q.ready, 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(static_cast<char*>(recvbuf) + roff[p] * esz,
                            static_cast<const char*>(q.buf) + q.soff[r] * esz, (size_t)rcnt[p] * esz,
                            cudaMemcpyDeviceToDevice, s);
    }
    if (e == cudaSuccess) e = cudaEventRecord(me().done, s);
    if (e != cudaSuccess) {
      if (c->last_error.empty()) c->last_error = std::string("loopback exchange: ") + cudaGetErrorString(e);
      G->abort(c->last_error);
      return EMIN_ERR_CUDA;
    }
    if (!G->barrier()) return gone(c);
    // the peers that read my buffer are done before my stream may touch it
    for (int p = 0; p < G->R && e == cudaSuccess; ++p)
      if (p != r && scnt[p]) e = cudaStreamWaitEvent(s, G->slot[p].done, 0);
    if (!G->barrier()) return gone(c);
    if (e != cudaSuccess) {
      c->last_error = std::string("loopback exchange: ") + cudaGetErrorString(e);
      G->abort(c->last_error);
      return EMIN_ERR_CUDA;
    }
    return EMIN_OK;
  }
  emin_status allreduce_sum(emin_ctx c, const double* in, double* out, int n, cudaStream_t s) override {
    const char* where = "";
    auto fail = [&](cudaError_t e) {
      c->last_error = std::string("loopback allreduce (") + where + "): " + cudaGetErrorString(e);
      G->abort(c->last_error);
      return EMIN_ERR_CUDA;
    };
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { where = "error pending before the collective"; return fail(e); }
    me().buf = in;
    where = "record ready";
    e = cudaEventRecord(me().ready, s);
    if (e != cudaSuccess) return fail(e);
    if (!G->barrier()) return gone(c);
    for (int p = 0; p < G->R; ++p) {
      if (p != r) {
        where = "wait ready";
        e = cudaStreamWaitEvent(s, G->slot[p].ready, 0);
        if (e != cudaSuccess) return fail(e);
      }
      where = "gather copy";
      e = cudaMemcpyAsync(me().gbuf + p * n, G->slot[p].buf, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return fail(e);
    }
    where = "record done";
    e = cudaEventRecord(me().done, s);
    if (e != cudaSuccess) return fail(e);
    if (!G->barrier()) return gone(c);
    for (int p = 0; p < G->R; ++p)
      if (p != r) {
        where = "wait done";
        e = cudaStreamWaitEvent(s, G->slot[p].done, 0);
        if (e != cudaSuccess) return fail(e);
      }
    if (!G->barrier()) return gone(c);
    k_sum_ranks<<<1, 32, 0, s>>>(me().gbuf, G->R, n, out);
    c->launches += 1;
    where = "rank-sum kernel";
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(e);
    return EMIN_OK;
  }
  emin_status allreduce_max_i32(emin_ctx c, int32_t* inout, cudaStream_t s) override {
    int32_t v = 0;
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(&v, inout, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
    int64_t mine = v;
    std::vector<int64_t> all(G->R);
    {
      emin_status st = allgather_i64(c, &mine, 1, all.data());
      if (st != EMIN_OK) return st;
    }
    v = (int32_t)*std::max_element(all.begin(), all.end());
    EMIN_CUDA_TRY(c, cudaMemcpyAsync(inout, &v, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
    return EMIN_OK;
  }
  bool capturable() const override { return false; }
  ~LoopbackTransport() override {
    if (me().ready) cudaEventDestroy(me().ready);
    if (me().done) cudaEventDestroy(me().done);
    if (me().gbuf) cudaFree(me().gbuf);
    me() = LoopbackGroup::Slot();
  }
};

extern "C" emin_status emin_loopback_create(void** out, int32_t nranks) {
  if (!out || nranks < 1 || nranks > 64) return EMIN_ERR_ARG;
  *out = new LoopbackGroup(nranks);
  return EMIN_OK;
}

extern "C" void emin_loopback_destroy(void* lb) { delete static_cast<LoopbackGroup*>(lb); }

emin_status emin_dist_attach(emin_ctx c, void* nccl_comm, void* loopback, int32_t loopback_rank) {
  if (loopback) {
    LoopbackGroup* G = static_cast<LoopbackGroup*>(loopback);
    if (loopback_rank < 0 || loopback_rank >= G->R) {
      c->last_error = "loopback_rank out of range";
      return EMIN_ERR_ARG;
    }
    c->nranks = G->R;
    c->rank = loopback_rank;
    c->dist = new DistPlan();
    LoopbackGroup::Slot& sl = G->slot[loopback_rank];
    EMIN_CUDA_TRY(c, cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
    EMIN_CUDA_TRY(c, cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    EMIN_CUDA_TRY(c, cudaMalloc((void**)&sl.gbuf, sizeof(double) * 4 * G->R));
    c->dist->tp = new LoopbackTransport(G, loopback_rank);
    return EMIN_OK;
  }
#ifdef EMIN_WITH_NCCL
  ncclComm_t cm = (ncclComm_t)nccl_comm;
  int n = 1, r = 0;
  NCCL_TRY(c, ncclCommCount(cm, &n));
  NCCL_TRY(c, ncclCommUserRank(cm, &r));
  c->comm = nccl_comm;
  c->nranks = n;
  c->rank = r;
  c->dist = new DistPlan();
  c->dist->tp = new NcclTransport(cm);
  return EMIN_OK;
#else
  (void)nccl_comm;
  c->last_error = "libemin was built without NCCL";
  return EMIN_ERR_NCCL;
#endif
}

bool emin_dist_capturable(emin_ctx c) { return !c->dist || c->dist->tp->capturable(); }

void emin_dist_abort(emin_ctx c, const std::string& why) {
  if (c && c->dist && c->dist->tp) c->dist->tp->abort(why);
}

// Gather every rank's F range; find, request and receive the halo rows'
// pattern.  Fills c->dist, sets nFh / nnzWh, extends wptr / wcol (caller
// allocated them with room: see emin_dist_halo_sizes).
emin_status emin_dist_find_halo(emin_ctx c, int64_t fbegin, int64_t nF, int64_t nFg, int64_t m,
                                const int64_t* Arp, const int32_t* Acol, const uint8_t* isc,
                                const int64_t* cidx, int64_t* scratch) {
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  const int R = c->nranks;
  const int SM = emin_num_sms();
  // ---- all F ranges
  const int64_t mine[2] = {fbegin, nF};
  std::vector<int64_t> all(2 * R);
  {
    emin_status st = d.tp->allgather_i64(c, mine, 2, all.data());
    if (st != EMIN_OK) return st;
  }
  d.fbeg.resize(R);
  d.fcnt.resize(R);
  for (int p = 0; p < R; ++p) { d.fbeg[p] = all[2 * p]; d.fcnt[p] = all[2 * p + 1]; }
  // ---- halo rows: F columns of owned rows outside [fbegin, fbegin + nF)
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&d.hflag, sizeof(int64_t) * std::max<int64_t>(nFg, 1), s));
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&d.hpos, sizeof(int64_t) * std::max<int64_t>(nFg + 1, 1), s));
  EMIN_CUDA_TRY(c, cudaMemsetAsync(d.hflag, 0, sizeof(int64_t) * std::max<int64_t>(nFg, 1), s));
  k_mark_halo<<<SM * 8, 256, 0, s>>>(m, c->opts.row_begin, fbegin, fbegin + nF, Arp, Acol, isc, cidx, d.hflag);
  int64_t* tot;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&tot, sizeof(int64_t), s));
  EMIN_CUDA_TRY(c, emin_scan_i64(d.hflag, d.hpos, nFg, tot, scratch, s));
  int64_t nH = 0;
  EMIN_CUDA_TRY(c, cudaMemcpyAsync(&nH, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  cudaFreeAsync(tot, s);
  d.nH = nH;
  int64_t* hlist;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&hlist, sizeof(int64_t) * std::max<int64_t>(nH, 1), s));
  k_halo_list<<<SM * 8, 256, 0, s>>>(d.hflag, d.hpos, nFg, hlist);
  std::vector<int64_t> h_hlist(nH);
  if (nH) EMIN_CUDA_TRY(c, cudaMemcpyAsync(h_hlist.data(), hlist, sizeof(int64_t) * nH, cudaMemcpyDeviceToHost, s));
  EMIN_CUDA_TRY(c, cudaStreamSynchronize(s));
  // ---- rows to receive per owner (hlist is sorted, owners own contiguous ranges)
  d.rrow.assign(R, 0);
  d.rrow_off.assign(R, 0);
  bool orphan = false;   // (reported after the collective below, so no rank is left waiting)
  for (int64_t h = 0, p = 0; h < nH; ++h) {
    while (p < R && h_hlist[h] >= d.fbeg[p] + d.fcnt[p]) ++p;
    if (p >= R || h_hlist[h] < d.fbeg[p]) { orphan = true; break; }
    d.rrow[p]++;
  }
  for (int p = 1; p < R; ++p) d.rrow_off[p] = d.rrow_off[p - 1] + d.rrow[p - 1];
  // ---- counts matrix -> rows to send per requester
  std::vector<int64_t> M(R * R);
  {
    emin_status st = d.tp->allgather_i64(c, d.rrow.data(), R, M.data());
    if (st != EMIN_OK) return st;
  }
  if (orphan) { c->last_error = "halo row owned by no rank"; return EMIN_ERR_ARG; }
  d.srow.assign(R, 0);
  d.srow_off.assign(R, 0);
  for (int p = 0; p < R; ++p) d.srow[p] = M[(int64_t)p * R + c->rank];   // rank p wants this many of mine
  for (int p = 1; p < R; ++p) d.srow_off[p] = d.srow_off[p - 1] + d.srow[p - 1];
  d.nS = d.srow_off[R - 1] + d.srow[R - 1];
  // ---- the requests themselves (global F ids) -> local ids of rows to send
  int64_t* req;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&req, sizeof(int64_t) * std::max<int64_t>(d.nS, 1), s));
  {
    emin_status st = d.tp->exchange(c, hlist, sizeof(int64_t), d.rrow, d.rrow_off, req, d.srow, d.srow_off, s);
    if (st != EMIN_OK) return st;
  }
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&d.send_rows, sizeof(int32_t) * std::max<int64_t>(d.nS, 1), s));
  k_to_local<<<SM * 4, 256, 0, s>>>(req, d.nS, fbegin, d.send_rows);
  cudaFreeAsync(req, s);
  cudaFreeAsync(hlist, s);
  c->launches += 4;
  return EMIN_OK;
}

// After the owned wptr is known: exchange the lengths of the halo rows,
// extend wptr, build the send-entry list; returns the halo entry count.
emin_status emin_dist_halo_pattern_sizes(emin_ctx c, int64_t* scratch) {
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  const int R = c->nranks;
  const int SM = emin_num_sms();
  int64_t *slen, *rlen, *excl, *tot;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&slen, sizeof(int64_t) * (d.nS + 1), s));
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&rlen, sizeof(int64_t) * (d.nH + 1), s));
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&excl, sizeof(int64_t) * (std::max(d.nS, d.nH) + 1), s));
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&tot, sizeof(int64_t) * 2, s));
  k_row_lengths<<<SM * 4, 256, 0, s>>>(d.send_rows, d.nS, c->wptr, slen);
  {
    emin_status st = d.tp->exchange(c, slen, sizeof(int64_t), d.srow, d.srow_off, rlen, d.rrow, d.rrow_off, s);
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
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&d.send_eidx, sizeof(int64_t) * std::max<int64_t>(nSE, 1), s));
  k_send_entries<<<SM * 4, 256, 0, s>>>(d.send_rows, d.nS, c->wptr, excl, d.send_eidx);
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&d.sendbuf, sizeof(double) * std::max<int64_t>(nSE, 1), s));
  cudaFreeAsync(slen, s); cudaFreeAsync(rlen, s); cudaFreeAsync(excl, s); cudaFreeAsync(tot, s);
  c->launches += 3 + 6;
  return EMIN_OK;
}

// pattern (coarse ids) of the halo rows, once
emin_status emin_dist_halo_wcol(emin_ctx c) {
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  int32_t* sb;
  EMIN_CUDA_TRY(c, emin_mallocAsync((void**)&sb, sizeof(int32_t) * std::max<int64_t>(d.nSE, 1), s));
  if (d.nSE) k_pack<int32_t><<<emin_num_sms() * 4, 256, 0, s>>>(c->wcol, d.send_eidx, d.nSE, sb);
  emin_status st = d.tp->exchange(c, sb, sizeof(int32_t), d.sent, d.sent_off, c->wcol + c->nnzW, d.rent,
                                  d.rent_off, s);
  cudaFreeAsync(sb, s);
  c->launches += d.nSE ? 1 : 0;
  return st;
}

// values of a W-layout vector on the halo rows (per iteration for y)
emin_status emin_dist_halo_values(emin_ctx c, double* vec, cudaStream_t s) {
  DistPlan& d = *c->dist;
  if (d.nSE) k_pack<double><<<emin_num_sms() * 2, 256, 0, s>>>(vec, d.send_eidx, d.nSE, d.sendbuf);
  c->launches += d.nSE ? 1 : 0;
  return d.tp->exchange(c, d.sendbuf, sizeof(double), d.sent, d.sent_off, vec + c->nnzW, d.rent, d.rent_off, s);
}

// out = sum over the ranks of in (n <= 4 doubles, device, in != out)
emin_status emin_dist_allreduce(emin_ctx c, const double* in, double* out, int n, cudaStream_t s) {
  return c->dist->tp->allreduce_sum(c, in, out, n, s);
}

emin_status emin_dist_allreduce_max_i32(emin_ctx c, int32_t* dev, cudaStream_t s) {
  return c->dist->tp->allreduce_max_i32(c, dev, s);
}

void emin_dist_free(emin_ctx c) {
  if (!c->dist) return;
  DistPlan& d = *c->dist;
  cudaStream_t s = c->stream;
  void* ptrs[] = {d.hflag, d.hpos, d.send_rows, d.send_eidx, d.sendbuf};
  for (void* p : ptrs) if (p) cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  delete d.tp;
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
