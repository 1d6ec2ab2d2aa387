// sa_nlfft64k.cu -- single-HBM-pass NL-FFT for N = 2^16 (BASELINE config C3).
//
// One signal per thread-block cluster, entirely on chip:
//   c64 : cluster of 4 CTAs x 128 KiB of node storage (512 KiB signal)
//   c128: cluster of 8 CTAs x 128 KiB                 (1 MiB signal)
// N = 256 x 256.  DIT (value-identical to transforms.py:254-298):
//   phase A: CTA r takes columns c of X[i][c] = x[256 i + c] (the reference's
//     bit-reversed blocks, SURVEY §7 hard part 4), in TMA-loaded tiles of TC
//     columns x 256 rows, runs global stages 1..8 in two register radix-16
//     rounds (stage 1 = the 2-point NDFT bottom), and scatters node row
//     R = rev8(c) over the cluster through DSMEM: q-columns [r*COLS, (r+1)*COLS)
//     of every row live in CTA r.
//   cluster barrier
//   phase B: CTA r runs global stages 9..16 along R for its COLS columns
//     (twiddle j = (R mod 2^(t-1))*256 + q) and writes y[256 R + q] (coalesced).
//   cluster barrier (node storage reusable), next signal.
// HBM traffic = one read + one write of the signal.  The next tile's TMA load
// is issued before the current tile is processed (double buffer, mbarriers).
#include <algorithm>
#include <cooperative_groups.h>
#include <cudaTypedefs.h>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int LOGN = 16;
constexpr int NN = 1 << LOGN;

template <typename T> struct K64;
template <> struct K64<float> {
  static constexpr int TC = 16;  // columns per tile
  static constexpr int CL = 4;   // cluster size
};
template <> struct K64<double> {
  static constexpr int TC = 8;
  static constexpr int CL = 8;
};

template <typename T> struct L64 {
  static constexpr int TC = K64<T>::TC, CL = K64<T>::CL;
  static constexpr int THREADS = 16 * TC;
  static constexpr int COLS = 256 / CL;  // node columns owned per CTA
  static constexpr int TILES = COLS / TC;
  using C2 = typename Ar<T>::C2;
  using C4 = typename Ar<T>::C4;
  static constexpr size_t INTER = sizeof(C2) * 256 * COLS;
  static constexpr size_t WORK = sizeof(C2) * 256 * TC;
  static constexpr size_t TWA = sizeof(C4) * 255;
  static constexpr size_t SMEM = INTER + 2 * WORK + TWA + 16;
  static constexpr int EW = sizeof(C2) / 8;  // 8-byte TMA elements per complex
};

SA_HD int rev4(int v) { return (int)(__brev((unsigned)v) >> 28); }
SA_HD int rev8(int v) { return (int)(__brev((unsigned)v) >> 24); }
constexpr int crev4(int v) { return ((v & 1) << 3) | ((v & 2) << 1) | ((v & 4) >> 1) | ((v & 8) >> 3); }

template <typename T>
__global__ void __launch_bounds__(L64<T>::THREADS, 1)
    k_nlfft64k_dit(const __grid_constant__ CUtensorMap tmx, typename Ar<T>::C2 *__restrict__ y,
                   int64_t batch, const typename Ar<T>::C4 *__restrict__ stage, T gain,
                   int use_gain) {
  using P = L64<T>;
  using A = Ar<T>;
  using V = typename A::V;
  using C2 = typename P::C2;
  using C4 = typename P::C4;
  constexpr int TC = P::TC, COLS = P::COLS, TILES = P::TILES;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  C2 *inter = reinterpret_cast<C2 *>(smem_raw);
  C2 *work = reinterpret_cast<C2 *>(smem_raw + P::INTER);
  C4 *twA = reinterpret_cast<C4 *>(smem_raw + P::INTER + 2 * P::WORK);
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem_raw + P::INTER + 2 * P::WORK + P::TWA);

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int64_t cid = blockIdx.x / P::CL;
  const int64_t ncl = gridDim.x / P::CL;
  const int tid = threadIdx.x;
  // mapping M1: cc fastest ; mapping M2: g fastest
  const int m1_cc = tid % TC, m1_g = tid / TC;
  const int m2_g = tid & 15, m2_cc = tid >> 4;

  for (int e = tid; e < 255; e += P::THREADS) twA[e] = stage[e];  // global stages 1..8
  if (tid == 0) {
    sa_mbar_init(&mbar[0], 1);
    sa_mbar_init(&mbar[1], 1);
    sa_fence_mbar_init();
  }
  __syncthreads();
  cluster.sync();

  C2 *inter_rank[P::CL];
#pragma unroll
  for (int r = 0; r < P::CL; ++r) inter_rank[r] = cluster.map_shared_rank(inter, r);

  auto issue = [&](int64_t sig, int tt, int buf) {
    if (tid == 0) {
      sa_fence_proxy_async();
      sa_mbar_expect_tx(&mbar[buf], (uint32_t)P::WORK);
      sa_tma_load_2d(work + buf * 256 * TC, &tmx, (rank * COLS + tt * TC) * P::EW, (int)(sig * 256),
                     &mbar[buf]);
    }
  };

  int64_t it = 0;  // global tile counter (buffer / parity)
  if (cid < batch) issue(cid, 0, 0);

  for (int64_t sig = cid; sig < batch; sig += ncl) {
    // ------------------------------------------------------------- phase A
    for (int tt = 0; tt < TILES; ++tt, ++it) {
      const int buf = (int)(it & 1);
      if (tt + 1 < TILES) issue(sig, tt + 1, buf ^ 1);
      else if (sig + ncl < batch) issue(sig + ncl, 0, buf ^ 1);
      sa_mbar_wait(&mbar[buf], (uint32_t)((it >> 1) & 1));
      C2 *wk = work + buf * 256 * TC;
      V v[16];
      // round 1 (M1): v[k] = node 16g+k of sub-transform cc = X[rev8(16g+k)][cc]
      {
        const int rg = rev4(m1_g);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          V x = A::from(wk[(crev4(k) * 16 + rg) * TC + m1_cc]);
          v[k] = use_gain ? A::scale(x, gain) : x;
        }
#pragma unroll
        for (int k = 0; k < 16; k += 2) r_two_point<T>(v[k], v[k + 1]);  // stage 1
#pragma unroll
        for (int k = 0; k < 16; ++k)  // stage 2: j = k & 1
          if (!(k & 2)) {
            if (k & 1) r_dit_mj<T>(v[k], v[k + 2]);
            else r_dit_one<T>(v[k], v[k + 2]);
          }
#pragma unroll
        for (int k = 0; k < 16; ++k)  // stage 3: j = k & 3
          if (!(k & 4)) {
            const int j = k & 3;
            if (j == 0) r_dit_one<T>(v[k], v[k + 4]);
            else if (j == 2) r_dit_mj<T>(v[k], v[k + 4]);
            else r_dit<T>(v[k], v[k + 4], twA[3 + j]);
          }
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // stage 4: j = k
          if (k == 0) r_dit_one<T>(v[k], v[k + 8]);
          else if (k == 4) r_dit_mj<T>(v[k], v[k + 8]);
          else r_dit<T>(v[k], v[k + 8], twA[7 + k]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k)  // exchange: node q = 16g+k, column swizzled by q & (TC-1)
        wk[(m1_g * 16 + k) * TC + (m1_cc ^ (k & (TC - 1)))] = A::to(v[k]);
      __syncthreads();
      // round 2 (M2): v[k] = node g + 16k of sub-transform cc ; global stages 5..8
#pragma unroll
      for (int k = 0; k < 16; ++k)
        v[k] = A::from(wk[(m2_g + 16 * k) * TC + (m2_cc ^ (m2_g & (TC - 1)))]);
#pragma unroll
      for (int t = 5; t <= 8; ++t) {
        const int hr = 1 << (t - 5), h = 1 << (t - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & hr)) r_dit<T>(v[k], v[k + hr], twA[(h - 1) + m2_g + 16 * (k & (hr - 1))]);
      }
      // scatter node row R = rev8(c) over the cluster: column q lives in CTA q / COLS
      {
        const int c = rank * COLS + tt * TC + m2_cc;
        const int R = rev8(c);
        constexpr int KPC = COLS / 16;  // registers per owner CTA
#pragma unroll
        for (int k = 0; k < 16; ++k)
          inter_rank[k / KPC][R * COLS + m2_g + 16 * (k % KPC)] = A::to(v[k]);
      }
      __syncthreads();  // work[buf] fully consumed before it is re-armed
    }
    cluster.sync();
    // ------------------------------------------------------------- phase B
    C2 *ysig = y + sig * NN;
    for (int tt = 0; tt < TILES; ++tt) {
      const int lq = tt * TC + m1_cc;
      const int q = rank * COLS + lq;
      V v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(inter[(m1_g * 16 + k) * COLS + lq]);
#pragma unroll
      for (int t = 1; t <= 4; ++t) {  // global stage s = 8 + t, pairs along R bits 0..3
        const int h = 1 << (t - 1);
        const int off = (1 << (7 + t)) - 1;
        C4 w[8];
#pragma unroll
        for (int a = 0; a < h; ++a) w[a] = sa_ldg(&stage[off + a * 256 + q]);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & h)) r_dit<T>(v[k], v[k + h], w[k & (h - 1)]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) inter[(m1_g * 16 + k) * COLS + lq] = A::to(v[k]);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(inter[(m1_g + 16 * k) * COLS + lq]);
#pragma unroll
      for (int t = 5; t <= 8; ++t) {  // global stage s = 8 + t, pairs along R bits 4..7
        const int hr = 1 << (t - 5);
        const int off = (1 << (7 + t)) - 1;
        C4 w[8];
#pragma unroll
        for (int a = 0; a < hr; ++a) w[a] = sa_ldg(&stage[off + (m1_g + 16 * a) * 256 + q]);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & hr)) r_dit<T>(v[k], v[k + hr], w[k & (hr - 1)]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) __stcs(&ysig[(m1_g + 16 * k) * 256 + q], A::to(v[k]));
    }
    cluster.sync();
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

template <typename T>
int launch64k(const void *x, void *y, int64_t batch, const SaTwiddles *tw, double gain,
              cudaStream_t s) {
  using P = L64<T>;
  auto enc = encode_fn();
  if (!enc) {
    sa_set_error("cuTensorMapEncodeTiled unavailable");
    return SA_ERR_CUDA;
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)(256 * P::EW), (cuuint64_t)(batch * 256)};
  cuuint64_t strides[1] = {(cuuint64_t)(256 * sizeof(typename P::C2))};
  cuuint32_t box[2] = {(cuuint32_t)(P::TC * P::EW), 256};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    sa_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SA_ERR_CUDA;
  }
  auto kern = k_nlfft64k_dit<T>;
  SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(P::THREADS);
  cfg.dynamicSmemBytes = P::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  cfg.gridDim = dim3(P::CL * (sms / P::CL));
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    max_clusters = sms / P::CL;
  int64_t ncl = std::min<int64_t>(batch, max_clusters);
  cfg.gridDim = dim3((unsigned)(ncl * P::CL));
  SA_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, map, (typename P::C2 *)y, batch,
                                 (const typename P::C4 *)tw->stage, (T)gain, (int)(gain != 1.0)));
  return SA_OK;
}

}  // namespace

// Returns SA_ERR_UNSUPPORTED when the fused path does not apply (caller falls back).
int sa_launch_nlfft64k(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
                       const SaTwiddles *tw, double gain, cudaStream_t s) {
  if (n != NN || variant != SA_DIT || batch < 1) return SA_ERR_UNSUPPORTED;
  if (((uintptr_t)x & 15) != 0) return SA_ERR_UNSUPPORTED;
  if (dtype == SA_C64) return launch64k<float>(x, y, batch, tw, gain, s);
  return launch64k<double>(x, y, batch, tw, gain, s);
}
