// Probe: where does tcgen05.mma.cta_group::1 M=64 put accumulator row r in TMEM?
// A[r][0] = r, A[r][1] = 100 + r, B = identity (N = 16): D[r][n] = A[r][n].
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
template <int M>
__global__ void k(float *out) {
  __shared__ __align__(1024) __nv_bfloat16 A[M * 16];
  __shared__ __align__(1024) __nv_bfloat16 B[16 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int tid = threadIdx.x, warp = tid >> 5;
  // core (i, kc) at i*256 + kc*128 bytes; element (r, k) -> i = r/8, rr = r%8, kc = k/8, kk = k%8
  for (int e = tid; e < M * 16; e += blockDim.x) {
    int r = e / 16, kx = e % 16;
    float v = kx == 0 ? r : (kx == 1 ? 100 + r : 0);
    int off = (r / 8) * 128 + (kx / 8) * 64 + (r % 8) * 8 + (kx % 8);  // in elements
    A[off] = __float2bfloat16(v);
  }
  for (int e = tid; e < 256; e += blockDim.x) {
    int n = e / 16, kx = e % 16;
    int off = (n / 8) * 128 + (kx / 8) * 64 + (n % 8) * 8 + (kx % 8);
    B[off] = __float2bfloat16(n == kx ? 1.f : 0.f);
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
    uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint64_t da = desc(su32(A), 128, 256), db = desc(su32(B), 128, 256);
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tm), "l"(da), "l"(db), "r"(id));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(tm + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int c = 0; c < 4; ++c) out[tid * 4 + c] = __uint_as_float(v[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}
int main() {
  float *d, h[512];
  cudaMalloc(&d, 512 * 4);
  for (int m : {128, 64}) {
    cudaMemset(d, 0xff, 512 * 4);
    if (m == 128) k<128><<<1, 128>>>(d); else k<64><<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 512 * 4, cudaMemcpyDeviceToHost);
    printf("M=%d err=%s\n", m, cudaGetErrorString(e));
    for (int lane = 0; lane < 128; ++lane) {
      printf("lane %3d: %6.1f %6.1f %6.1f %6.1f%s", lane, h[lane * 4], h[lane * 4 + 1], h[lane * 4 + 2], h[lane * 4 + 3],
             lane % 2 ? "\n" : "   |   ");
    }
  }
  return 0;
}
