// sa_twiddles.cu -- device twiddle sets built from the host reference table
// (transforms.py:108-146).  The host computes cos/sin exactly as the reference
// does (quadrant entries exact); the device only casts, splits and re-packs.
#include "sa_common.cuh"
#include "sa_internal.h"

template <typename T>
__global__ void k_tw_raw_quad(const double2 *__restrict__ host_tab, int64_t n,
                              typename SaVec<T>::c2 *raw, typename SaVec<T>::c4 *quad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 w = host_tab[i];
  T wr = (T)w.x, wi = (T)w.y;  // round-to-nearest cast (numpy astype(complex64))
  raw[i] = {wr, wi};
  quad[i] = {wr, wi, sa_sgn_np(wr), sa_sgn_np(wi)};
}

// entry e of the stage-packed table: stage s = floor(log2(e+1)) + 1, j = e+1-2^(s-1),
// value table[j * n / 2^s]  (transforms.py:295: entries[arange(h) * (n // m)])
template <typename T>
__global__ void k_tw_stage(const typename SaVec<T>::c2 *__restrict__ raw, int64_t n,
                           typename SaVec<T>::c4 *stage, typename SaVec<T>::c2 *stage2) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n - 1) return;
  int s = 63 - __clzll(e + 1) + 1;
  int64_t j = e + 1 - (1LL << (s - 1));
  auto w = raw[j * (n >> s)];
  stage[e] = {fabs(w.x), fabs(w.y), sa_sgn_np(w.x), sa_sgn_np(w.y)};
  stage2[e] = w;
}

int sa_twiddles_build(SaTwiddles *tw, const double *host_table, cudaStream_t s) {
  int64_t n = tw->n;
  size_t c2 = tw->dtype == SA_C64 ? sizeof(float2) : sizeof(double2);
  size_t c4 = tw->dtype == SA_C64 ? sizeof(float4) : sizeof(double4);
  bool pow2 = n >= 2 && (n & (n - 1)) == 0;
  double2 *d_host = nullptr;
  SA_CUDA_TRY(cudaMallocAsync((void **)&d_host, sizeof(double2) * n, s));
  SA_CUDA_TRY(cudaMemcpyAsync(d_host, host_table, sizeof(double2) * n, cudaMemcpyHostToDevice, s));
  SA_CUDA_TRY(cudaMalloc(&tw->raw, c2 * n));
  SA_CUDA_TRY(cudaMalloc(&tw->quad, c4 * n));
  tw->stage = nullptr;
  tw->stage2 = nullptr;
  if (pow2) SA_CUDA_TRY(cudaMalloc(&tw->stage, c4 * (n - 1)));
  if (pow2) SA_CUDA_TRY(cudaMalloc(&tw->stage2, c2 * (n - 1)));
  int g = (int)((n + 255) / 256);
  if (tw->dtype == SA_C64) {
    k_tw_raw_quad<float><<<g, 256, 0, s>>>(d_host, n, (float2 *)tw->raw, (float4 *)tw->quad);
    if (pow2) k_tw_stage<float><<<g, 256, 0, s>>>((const float2 *)tw->raw, n, (float4 *)tw->stage,
                                                  (float2 *)tw->stage2);
  } else {
    k_tw_raw_quad<double><<<g, 256, 0, s>>>(d_host, n, (double2 *)tw->raw, (double4 *)tw->quad);
    if (pow2)
      k_tw_stage<double><<<g, 256, 0, s>>>((const double2 *)tw->raw, n, (double4 *)tw->stage,
                                                   (double2 *)tw->stage2);
  }
  SA_LAUNCH_CHECK();
  SA_CUDA_TRY(cudaFreeAsync(d_host, s));
  // the host buffer may be released by the caller right after return
  SA_CUDA_TRY(cudaStreamSynchronize(s));
  return SA_OK;
}

// Stream-ordered scratch from a library-owned pool per device that keeps its
// memory (release threshold = max): repeated calls reuse it with no driver
// allocation (the default pool hands memory back at every synchronisation).
#include <mutex>
namespace {
std::mutex g_pool_mutex;
cudaMemPool_t g_pools[64] = {};
}  // namespace

int sa_scratch_alloc(void **p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> g(g_pool_mutex);
    if (dev < 64 && g_pools[dev]) {
      pool = g_pools[dev];
    } else {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      SA_CUDA_TRY(cudaMemPoolCreate(&pool, &props));
      uint64_t keep = ~0ull;
      SA_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      if (dev < 64) g_pools[dev] = pool;
    }
  }
  SA_CUDA_TRY(cudaMallocFromPoolAsync(p, bytes, pool, s));
  return SA_OK;
}
