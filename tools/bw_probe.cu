// HBM copy bandwidth vs access granularity (tile of TCOLS complex64 columns x 256 rows
// of a [rows][256] matrix), to size the NL-FFT tiles.  Dev tool, not part of the library.
#include <cstdio>
#include <cuda_runtime.h>
template <int TCOLS>
__global__ void copy_tiles(const float2* __restrict__ x, float2* __restrict__ y, long long ntiles) {
  const int tpr = 256 / TCOLS;  // tiles per 256x256 signal
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    long long sig = t / tpr; int c0 = (int)(t % tpr) * TCOLS;
    const float2* xs = x + sig * 65536; float2* ys = y + sig * 65536;
    for (int e = threadIdx.x; e < 256 * TCOLS; e += blockDim.x) {
      int r = e / TCOLS, c = e % TCOLS;
      ys[r * 256 + c0 + c] = __ldcs(&xs[r * 256 + c0 + c]);
    }
  }
}
__global__ void copy_contig(const float4* __restrict__ x, float4* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __ldcs(&x[i]);
}
template <typename F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a); for (int i = 0; i < 10; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10;
}
int main() {
  long long nsig = 4096, n = nsig * 65536;
  float2 *x, *y; cudaMalloc(&x, n * 8); cudaMalloc(&y, n * 8); cudaMemset(x, 0, n * 8);
  double gb = 2.0 * n * 8 / 1e9;
  float ms = timeit([&] { copy_contig<<<148 * 8, 256>>>((float4*)x, (float4*)y, n / 2); });
  printf("contig      %.3f ms %.0f GB/s\n", ms, gb / ms * 1e3);
#define T(TC) { long long nt = nsig * (256 / TC); float m = timeit([&] { copy_tiles<TC><<<148 * 8, 256>>>(x, y, nt); }); printf("tiles TC=%3d %.3f ms %.0f GB/s\n", TC, m, gb / m * 1e3); }
  T(8) T(16) T(32) T(64) T(128) T(256)
  return 0;
}
