// dist.cuh -- halo plan and transports of the row-partitioned path (see dist.cu).
#pragma once
#include <vector>
#include "emin_internal.cuh"

// The data movement of the row-partitioned path, behind one interface:
// NCCL (one process per GPU) or the in-process loopback group (R contexts
// driven by R host threads, on one or several devices).  Every call is
// collective over the group.
struct Transport {
  virtual ~Transport() {}
  // host in / host out: all[p * n + j] = rank p's mine[j]   (setup only)
  virtual emin_status allgather_i64(emin_ctx c, const int64_t* mine, int n, int64_t* all) = 0;
  // grouped point-to-point, bytes: rank p receives scnt[q] elements of esz
  // bytes from sendbuf + soff[q] for every q it names in rcnt / roff
  virtual emin_status exchange(emin_ctx c, const void* sendbuf, size_t esz, const std::vector<int64_t>& scnt,
                               const std::vector<int64_t>& soff, void* recvbuf, const std::vector<int64_t>& rcnt,
                               const std::vector<int64_t>& roff, cudaStream_t s) = 0;
  // out[j] = sum over ranks of in[j] (device pointers, in != out), n <= 4
  virtual emin_status allreduce_sum(emin_ctx c, const double* in, double* out, int n, cudaStream_t s) = 0;
  // in place max of one device int32 (setup only)
  virtual emin_status allreduce_max_i32(emin_ctx c, int32_t* inout, cudaStream_t s) = 0;
  // may the per-iteration calls be captured into a CUDA graph?
  virtual bool capturable() const = 0;
  // a rank failed between collectives: release the peers waiting for it
  virtual void abort(const std::string& why) { (void)why; }
};

struct DistPlan {
  Transport* tp = nullptr;
  std::vector<int64_t> fbeg, fcnt;           // F range of every rank (global F ids)
  int64_t nH = 0, nHW = 0;                   // halo rows / halo W entries received
  int64_t nS = 0, nSE = 0;                   // rows / W entries sent
  int64_t* hflag = nullptr;                  // [nF_global] 1 if the global F row is a halo row
  int64_t* hpos = nullptr;                   // [nF_global] exclusive scan of hflag (halo slot)
  int32_t* send_rows = nullptr;              // [nS] local F ids requested by the peers
  int64_t* send_eidx = nullptr;              // [nSE] W entries to pack
  double* sendbuf = nullptr;                 // [nSE]
  std::vector<int64_t> rrow, rrow_off, srow, srow_off;   // rows per peer
  std::vector<int64_t> rent, rent_off, sent, sent_off;   // W entries per peer
};

emin_status emin_dist_attach(emin_ctx c, void* nccl_comm, void* loopback, int32_t loopback_rank);
emin_status emin_dist_find_halo(emin_ctx c, int64_t fbegin, int64_t nF, int64_t nFg, int64_t m,
                                const int64_t* Arp, const int32_t* Acol, const uint8_t* isc,
                                const int64_t* cidx, int64_t* scratch);
emin_status emin_dist_halo_pattern_sizes(emin_ctx c, int64_t* scratch);
emin_status emin_dist_halo_wcol(emin_ctx c);
emin_status emin_dist_halo_values(emin_ctx c, double* vec, cudaStream_t s);
emin_status emin_dist_allreduce(emin_ctx c, const double* in, double* out, int n, cudaStream_t s);
emin_status emin_dist_allreduce_max_i32(emin_ctx c, int32_t* dev, cudaStream_t s);
bool emin_dist_capturable(emin_ctx c);
void emin_dist_abort(emin_ctx c, const std::string& why);
void emin_dist_free(emin_ctx c);
