// MEASURED ALTERNATIVE, NOT BUILT: moved here from csrc/ after the A/B; to try it, copy
// into csrc/, add it to the Makefile and dispatch sa_launch_nlfft64k_l2 from sa_nlfft.cu.
// sa_nlfft64k_l2.cu -- NL-FFT for N = 2^16 (BASELINE config C3), one SM per
// signal at a time, the 256 x 256 transpose through an L2-resident scratch.
//
// DIT, value-identical to transforms.py:254-298 (same butterflies, twiddles and
// evaluation order as sa_nlfft64k.cu; only where the intermediate lives differs):
//   A-items (8 per signal): TMA-load column tile t of X[i][c] = x[256 i + c]
//     (32 columns x 256 rows), global stages 1..8 in two register radix-16 rounds
//     (stage 1 = the 2-point NDFT bottom), store node rows R = rev8(c) to this
//     CTA's 512-KB scratch (row-major [R][q], coalesced, stays in L2).
//   B-items (8 per signal): TMA-load node columns q of the scratch, stages 9..16
//     along R (twiddle j = (R mod 2^(t-1)) 256 + q), store y[256 R + q].
// Each CTA (one per SM, persistent) walks its signals' items in order through a
// ring of three 64-KB tile buffers; the load of item it + 3 is issued when item
// it is done, except that the B-items of a signal wait for its last A-item's
// stores (fence.proxy.async.global + CTA barrier).  In-order processing makes
// scratch reuse safe: A-items of signal s + 1 come after every B-item of s.
// No cluster, no cross-SM waits: the lock-step of the cluster kernel (DESIGN
// §5.2) is gone; HBM traffic is x once + y once, the scratch round trip is L2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

constexpr int NN = 1 << 16;
#ifndef SA_L2_TC
#define SA_L2_TC 32
#endif
#ifndef SA_L2_NR
#define SA_L2_NR 3
#endif
constexpr int TC = SA_L2_TC;       // columns per tile
constexpr int THREADS = 16 * TC;   // 16 elements per thread
constexpr int NR = SA_L2_NR;       // ring depth
constexpr int NT = 256 / TC;       // tiles per pass per signal

struct Lay {
  static constexpr size_t TILE = sizeof(float2) * 256 * TC;
  static constexpr size_t OFF_TWA = NR * TILE;
  static constexpr size_t OFF_BAR = OFF_TWA + ((sizeof(float4) * 255 + 15) & ~(size_t)15);
  static constexpr size_t SMEM = OFF_BAR + 8 * NR + 64;
};

SA_HD int rev4(int v) { return (int)(__brev((unsigned)v) >> 28); }
SA_HD int rev8(int v) { return (int)(__brev((unsigned)v) >> 24); }
constexpr int crev4(int v) { return ((v & 1) << 3) | ((v & 2) << 1) | ((v & 4) >> 1) | ((v & 8) >> 3); }

// twiddles of global stages 9..16 for node column q (sa_nlfft64k.cu load_wf)
SA_HD void load_wf(float2 (&wf)[30], const float2 *__restrict__ stage2, int q, int g) {
#pragma unroll
  for (int t = 1; t <= 4; ++t)
#pragma unroll
    for (int a = 0; a < (1 << (t - 1)); ++a) wf[(1 << (t - 1)) - 1 + a] = sa_ldg(&stage2[(1 << (7 + t)) - 1 + a * 256 + q]);
#pragma unroll
  for (int t = 5; t <= 8; ++t)
#pragma unroll
    for (int a = 0; a < (1 << (t - 5)); ++a)
      wf[15 + (1 << (t - 5)) - 1 + a] = sa_ldg(&stage2[(1 << (7 + t)) - 1 + (g + 16 * a) * 256 + q]);
}
SA_HD float4 c4of(const float2 &w) { return {fabsf(w.x), fabsf(w.y), sa_sgn(w.x), sa_sgn(w.y)}; }
SA_HD bool special_column(int q) { return __any_sync(0xffffffffu, q == 0 || q == 128); }
SA_HD void tma_hint(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(sa_smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(sa_smem_u32(bar)), "l"(pol)
      : "memory");
}
SA_HD void st_keep(float2 *p, float2 v, uint64_t pol) {  // scratch store, L2 evict_last
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
               : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    k_nlfft64k_l2_dit(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmi,
                      float2 *__restrict__ y, float2 *__restrict__ scratch, int64_t batch,
                      const float4 *__restrict__ stage, const float2 *__restrict__ stage2, float gain, int use_gain) {
  using A = Ar<float>;
  using V = A::V;
  extern __shared__ __align__(128) unsigned char smem[];
  float4 *twA = reinterpret_cast<float4 *>(smem + Lay::OFF_TWA);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + Lay::OFF_BAR);
  const int tid = threadIdx.x;
  const int m1_cc = tid % TC, m1_g = tid / TC;
  const int m2_g = tid & 15, m2_cc = tid >> 4;
  float2 *inter = scratch + (int64_t)blockIdx.x * NN;
  const int64_t nsig = blockIdx.x < batch ? (batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nitems = 2 * NT * nsig;
  uint64_t keep, drop;  // scratch stores stay in L2; x tiles and scratch reads go first
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(drop));

  for (int e = tid; e < 255; e += THREADS) twA[e] = stage[e];  // global stages 1..8
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) sa_mbar_init(&bar[i], 1);
    sa_fence_mbar_init();
  }
  __syncthreads();

  // ---- producer state (thread 0): items are issued in order; B-items of signal i
  // only once its A-phase stores are done (a_done > i) ----
  int64_t next_issue = 0, a_done = 0;
  auto issue = [&](int64_t it) {
    const int slot = (int)(it % NR);
    const int64_t i = it / (2 * NT);
    const int j = (int)(it % (2 * NT));
    sa_fence_proxy_async();
    sa_mbar_expect_tx(&bar[slot], (uint32_t)Lay::TILE);
    float2 *dst = reinterpret_cast<float2 *>(smem + slot * Lay::TILE);
    if (j < NT) tma_hint(dst, &tmx, j * TC, (int)((blockIdx.x + i * gridDim.x) * 256), &bar[slot], drop);
    else tma_hint(dst, &tmi, (j - NT) * TC, (int)(blockIdx.x * 256), &bar[slot], drop);
  };
  auto pump = [&](int64_t it_done) {  // after item it_done: fill the ring up to it_done + NR
    while (next_issue < nitems && next_issue <= it_done + NR) {
      const int64_t i = next_issue / (2 * NT);
      const int j = (int)(next_issue % (2 * NT));
      if (j >= NT && a_done <= i) break;
      issue(next_issue++);
    }
  };
  if (tid == 0) pump(-1);

  for (int64_t it = 0; it < nitems; ++it) {
    const int slot = (int)(it % NR);
    const int64_t i = it / (2 * NT);
    const int j = (int)(it % (2 * NT));
    const int64_t sig = blockIdx.x + i * gridDim.x;
    sa_mbar_wait(&bar[slot], (uint32_t)((it / NR) & 1));
    float2 *wk = reinterpret_cast<float2 *>(smem + slot * Lay::TILE);
    V v[16];
    if (j < NT) {
      // ---- A-item: columns c = j TC + cc of X[i][c], stages 1..8 ----
      {
        const int rg = rev4(m1_g);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          V x = A::from(wk[(crev4(k) * 16 + rg) * TC + m1_cc]);
          v[k] = use_gain ? A::scale(x, gain) : x;
        }
#pragma unroll
        for (int k = 0; k < 16; k += 2) r_two_point<float>(v[k], v[k + 1]);  // stage 1
#pragma unroll
        for (int k = 0; k < 16; ++k)  // stage 2: j = k & 1
          if (!(k & 2)) {
            if (k & 1) r_dit_mj<float>(v[k], v[k + 2]);
            else r_dit_one<float>(v[k], v[k + 2]);
          }
#pragma unroll
        for (int k = 0; k < 16; ++k)  // stage 3: j = k & 3
          if (!(k & 4)) {
            const int jj = k & 3;
            if (jj == 0) r_dit_one<float>(v[k], v[k + 4]);
            else if (jj == 2) r_dit_mj<float>(v[k], v[k + 4]);
            else r_dit<float>(v[k], v[k + 4], twA[3 + jj]);
          }
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // stage 4: j = k
          if (k == 0) r_dit_one<float>(v[k], v[k + 8]);
          else if (k == 4) r_dit_mj<float>(v[k], v[k + 8]);
          else r_dit<float>(v[k], v[k + 8], twA[7 + k]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k)  // exchange: node q = 16g+k, column swizzled by k
        wk[(m1_g * 16 + k) * TC + (m1_cc ^ k)] = A::to(v[k]);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k)  // round 2: node g + 16k of sub-transform cc
        v[k] = A::from(wk[(m2_g + 16 * k) * TC + (m2_cc ^ m2_g)]);
#pragma unroll
      for (int t = 5; t <= 8; ++t) {
        const int hr = 1 << (t - 5), h = 1 << (t - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & hr)) r_dit<float>(v[k], v[k + hr], twA[(h - 1) + m2_g + 16 * (k & (hr - 1))]);
      }
      // node row R = rev8(c), q = g + 16 k: two 128-B row segments per warp store
      float2 *row = inter + rev8(j * TC + m2_cc) * 256 + m2_g;
#pragma unroll
      for (int k = 0; k < 16; ++k) st_keep(row + 16 * k, A::to(v[k]), keep);
      if (j == NT - 1) asm volatile("fence.proxy.async.global;" ::: "memory");  // scratch -> the B-items' TMA
    } else {
      // ---- B-item: node columns q = (j - NT) TC + cc, stages 9..16 along R ----
      const int q = (j - NT) * TC + m1_cc;
      const bool gen = special_column(q);
      float2 wf[30];
      load_wf(wf, stage2, q, m1_g);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(wk[(m1_g * 16 + k) * TC + m1_cc]);
      if (gen) {  // warps with column 0 / 128: general product (twiddles with zero components)
#pragma unroll
        for (int t = 1; t <= 4; ++t) {
          const int h = 1 << (t - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dit<float>(v[k], v[k + h], c4of(wf[h - 1 + (k & (h - 1))]));
        }
      } else {
#pragma unroll
        for (int t = 1; t <= 4; ++t) {
          const int h = 1 << (t - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dit_fast<float>(v[k], v[k + h], wf[h - 1 + (k & (h - 1))]);
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) wk[(m1_g * 16 + k) * TC + m1_cc] = A::to(v[k]);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(wk[(m1_g + 16 * k) * TC + m1_cc]);
      if (gen) {
#pragma unroll
        for (int t = 5; t <= 8; ++t) {
          const int hr = 1 << (t - 5);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dit<float>(v[k], v[k + hr], c4of(wf[15 + hr - 1 + (k & (hr - 1))]));
        }
      } else {
#pragma unroll
        for (int t = 5; t <= 8; ++t) {
          const int hr = 1 << (t - 5);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dit_fast<float>(v[k], v[k + hr], wf[15 + hr - 1 + (k & (hr - 1))]);
        }
      }
      float2 *ysig = y + sig * NN;
#pragma unroll
      for (int k = 0; k < 16; ++k) __stcs(&ysig[(m1_g + 16 * k) * 256 + q], A::to(v[k]));
    }
    __syncthreads();  // tile consumed (and, after the last A-item, the scratch stores fenced)
    if (tid == 0) {
      if (j == NT - 1) a_done = i + 1;
      pump(it);
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

int encode_rows(CUtensorMap *map, const void *base, int64_t rows) {  // [rows][256] float2, box TC x 256
  auto enc = encode_fn();
  if (!enc) {
    sa_set_error("cuTensorMapEncodeTiled unavailable");
    return SA_ERR_CUDA;
  }
  cuuint64_t dims[2] = {256, (cuuint64_t)rows};
  cuuint64_t strides[1] = {256 * sizeof(float2)};
  cuuint32_t box[2] = {(cuuint32_t)TC, 256};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    sa_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SA_ERR_CUDA;
  }
  return SA_OK;
}

}  // namespace

// complex64 DIT only (SA_ERR_UNSUPPORTED otherwise: the caller uses the cluster kernel)
int sa_launch_nlfft64k_l2(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
                          const SaTwiddles *tw, double gain, cudaStream_t s) {
  if (n != NN || batch < 1 || dtype != SA_C64 || variant != SA_DIT) return SA_ERR_UNSUPPORTED;
  if (((uintptr_t)x & 15) != 0) return SA_ERR_UNSUPPORTED;
  int dev = 0, sms = 148;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  SA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t grid = std::min<int64_t>(batch, sms);
  float2 *scratch = nullptr;
  {
    const int rc_ = sa_scratch_alloc((void **)&scratch, (size_t)grid * NN * sizeof(float2), s);
    if (rc_ != SA_OK) return rc_;
  }
  CUtensorMap mx, mi;
  int rc = encode_rows(&mx, x, batch * 256);
  if (rc == SA_OK) rc = encode_rows(&mi, scratch, grid * 256);
  if (rc == SA_OK) {
    static bool attr_set[64] = {};
    if (dev >= 64 || !attr_set[dev]) {
      SA_CUDA_TRY(cudaFuncSetAttribute(k_nlfft64k_l2_dit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Lay::SMEM));
      if (dev < 64) attr_set[dev] = true;
    }
    k_nlfft64k_l2_dit<<<(unsigned)grid, THREADS, Lay::SMEM, s>>>(mx, mi, (float2 *)y, scratch, batch,
                                                                (const float4 *)tw->stage, (const float2 *)tw->stage2,
                                                                (float)gain, (int)(gain != 1.0));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      sa_set_error("k_nlfft64k_l2_dit launch failed: %s", cudaGetErrorString(e));
      rc = SA_ERR_CUDA;
    }
  }
  SA_CUDA_TRY(cudaFreeAsync(scratch, s));
  return rc;
}
