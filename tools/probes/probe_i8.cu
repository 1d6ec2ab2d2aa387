// Probe: tcgen05.mma.cta_group::1.kind::i8 instruction descriptor (s8 x s8 -> s32), M = 128, N = 16, K = 32.
// A[r][k] = (k - 16) * (r % 7 - 3), B[n][k] = ((n + k) % 5) - 2: D[r][n] = sum_k A[r][k] B[n][k] (checked on host).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
__host__ __device__ int aval(int r, int k) { return (k - 16) * (r % 7 - 3); }
__host__ __device__ int bval(int n, int k) { return ((n + k) % 5) - 2; }
__global__ void k(int *out, uint32_t dfmt, uint32_t afmt, uint32_t bfmt) {
  __shared__ __align__(1024) int8_t A[128 * 32];
  __shared__ __align__(1024) int8_t B[16 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int tid = threadIdx.x, warp = tid >> 5;
  // no-swizzle K-major: core matrix 8 rows x 16 B (16 int8); core (i, kc) at i*256 + kc*128 bytes (K = 32 -> 2 kc)
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    int r = e / 32, kx = e % 32;
    A[(r / 8) * 256 + (kx / 16) * 128 + (r % 8) * 16 + (kx % 16)] = (int8_t)aval(r, kx);
  }
  for (int e = tid; e < 16 * 32; e += blockDim.x) {
    int n = e / 32, kx = e % 32;
    B[(n / 8) * 256 + (kx / 16) * 128 + (n % 8) * 16 + (kx % 16)] = (int8_t)bval(n, kx);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = holder;
  if (tid == 0) {
    uint32_t id = (dfmt << 4) | (afmt << 7) | (bfmt << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint64_t da = desc(su32(A), 128, 256), db = desc(su32(B), 128, 256);
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tm), "l"(da), "l"(db), "r"(id));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(tm + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int c = 0; c < 16; ++c) out[tid * 16 + c] = (int)v[c];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}
int main() {
  int *d, h[128 * 16];
  cudaMalloc(&d, sizeof(h));
  for (uint32_t dfmt = 2; dfmt <= 2; ++dfmt)
    for (uint32_t af = 0; af <= 1; ++af) {
      cudaMemset(d, 0, sizeof(h));
      k<<<1, 128>>>(d, dfmt, af, af);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int r = 0; r < 128; ++r)
        for (int n = 0; n < 16; ++n) {
          int s = 0;
          for (int kx = 0; kx < 32; ++kx) s += aval(r, kx) * bval(n, kx);
          bad += h[r * 16 + n] != s;
        }
      printf("dfmt=%u ab=%u err=%s mismatches=%d  D[5][3]=%d\n", dfmt, af, cudaGetErrorString(e), bad, h[5 * 16 + 3]);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
