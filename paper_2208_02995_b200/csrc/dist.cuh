// dist.cuh -- halo plan of the row-partitioned path (see dist.cu).
#pragma once
#include <vector>
#include "emin_internal.cuh"

struct DistPlan {
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

emin_status emin_dist_attach(emin_ctx c, void* comm);
emin_status emin_dist_find_halo(emin_ctx c, int64_t fbegin, int64_t nF, int64_t nFg, int64_t m,
                                const int64_t* Arp, const int32_t* Acol, const uint8_t* isc,
                                const int64_t* cidx, int64_t* scratch);
emin_status emin_dist_halo_pattern_sizes(emin_ctx c, int64_t* scratch);
emin_status emin_dist_halo_wcol(emin_ctx c);
emin_status emin_dist_halo_values(emin_ctx c, double* vec, cudaStream_t s);
emin_status emin_dist_allreduce(emin_ctx c, double* dev, int n, cudaStream_t s);
emin_status emin_dist_allreduce_max_i32(emin_ctx c, int32_t* dev, cudaStream_t s);
void emin_dist_free(emin_ctx c);
