// util.cu -- device-wide exclusive scan (setup-time index preparation) and
// small host helpers.
#include <mutex>

#include "emin_internal.cuh"

namespace {
constexpr int SCAN_T = 256;
constexpr int SCAN_IPT = 4;
constexpr int SCAN_TILE = SCAN_T * SCAN_IPT;

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
  const int l = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += t;
  }
  return v;
}

// exclusive scan of one value per thread over the block; *total = block sum
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total) {
  __shared__ int64_t sh[33];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t inc = warp_incl_scan(v);
  if (l == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int nw = (int)(blockDim.x >> 5);
    const int64_t s = (l < nw) ? sh[l] : 0;
    const int64_t si = warp_incl_scan(s);
    sh[l] = si - s;
    if (l == 31) sh[32] = si;
  }
  __syncthreads();
  const int64_t excl = sh[w] + inc - v;
  if (total) *total = sh[32];
  __syncthreads();
  return excl;
}

__global__ void k_tile_sums(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ bs) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t i = base + (int64_t)k * SCAN_T + threadIdx.x;
    if (i < n) s += in[i];
  }
  __shared__ int64_t sh[SCAN_T / 32];
  s = warp_incl_scan(s);  // lane 31 holds warp total
  if ((threadIdx.x & 31) == 31) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < SCAN_T / 32; ++w) t += sh[w];
    bs[blockIdx.x] = t;
  }
}

// single block: exclusive scan of bs[0..nb) in place, total to *total
__global__ void k_scan_tile_sums(int64_t* bs, int64_t nb, int64_t* total) {
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = (i < nb) ? bs[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, &tot);
    const int64_t c = carry;
    if (i < nb) bs[i] = c + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_scan_apply(const int64_t* in, int64_t* out, int64_t n, const int64_t* __restrict__ bs) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  // each thread owns SCAN_IPT consecutive items
  int64_t v[SCAN_IPT];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t i = base + (int64_t)threadIdx.x * SCAN_IPT + k;
    v[k] = (i < n) ? in[i] : 0;
    s += v[k];
  }
  const int64_t ex = block_excl_scan(s, nullptr);
  int64_t run = bs[blockIdx.x] + ex;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t i = base + (int64_t)threadIdx.x * SCAN_IPT + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
}
}  // namespace

int64_t emin_scan_scratch_elems(int64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE + 1; }

cudaError_t emin_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total_dev,
                          int64_t* scratch, cudaStream_t s) {
  if (n <= 0) {
    if (total_dev) return cudaMemsetAsync(total_dev, 0, sizeof(int64_t), s);
    return cudaSuccess;
  }
  const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  k_tile_sums<<<(unsigned)nb, SCAN_T, 0, s>>>(in, n, scratch);
  k_scan_tile_sums<<<1, 1024, 0, s>>>(scratch, nb, total_dev);
  k_scan_apply<<<(unsigned)nb, SCAN_T, 0, s>>>(in, out, n, scratch);
  return cudaGetLastError();
}

// Library-owned stream-ordered memory pool, one per device (the
// release threshold of the device's DEFAULT pool is process-wide state and
// must not be changed by a library).  Freed blocks stay cached in this pool
// (repeated emin_setup calls reuse them) and are returned to the driver by
// emin_release_memory(), and at the end of emin_galerkin / emin_pattern.
static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[64] = {};

cudaMemPool_t emin_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    g_pool[dev] = p;
  }
  return g_pool[dev];
}

cudaError_t emin_mallocAsync(void** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = emin_pool();
  if (!pool) return cudaMallocAsync(p, bytes, s);
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

void emin_pool_trim(cudaStream_t s) {
  cudaMemPool_t pool = emin_pool();
  if (!pool) return;
  cudaStreamSynchronize(s);
  cudaMemPoolTrimTo(pool, 0);
}

extern "C" void emin_release_memory(void) {
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (cudaMemPool_t p : g_pool)
    if (p) cudaMemPoolTrimTo(p, 0);
}

int emin_num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

extern "C" const char* emin_status_str(emin_status s) {
  switch (s) {
    case EMIN_OK: return "EMIN_OK";
    case EMIN_ERR_ARG: return "EMIN_ERR_ARG";
    case EMIN_ERR_CSR: return "EMIN_ERR_CSR";
    case EMIN_ERR_PATTERN: return "EMIN_ERR_PATTERN";
    case EMIN_ERR_BC: return "EMIN_ERR_BC";
    case EMIN_ERR_DIAG: return "EMIN_ERR_DIAG";
    case EMIN_ERR_NONFINITE: return "EMIN_ERR_NONFINITE";
    case EMIN_ERR_BREAKDOWN: return "EMIN_ERR_BREAKDOWN";
    case EMIN_ERR_CUDA: return "EMIN_ERR_CUDA";
    case EMIN_ERR_NCCL: return "EMIN_ERR_NCCL";
    case EMIN_ERR_OOM: return "EMIN_ERR_OOM";
    case EMIN_ERR_STATE: return "EMIN_ERR_STATE";
  }
  return "EMIN_ERR_UNKNOWN";
}
