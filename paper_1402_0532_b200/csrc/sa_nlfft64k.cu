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
  static constexpr size_t SMEM = INTER + 2 * WORK + TWA + 32;
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
    sa_mbar_init(&mbar[2], 1);  // "node storage full": expect_tx(INTER) per signal
    sa_fence_mbar_init();
  }
  __syncthreads();
  cluster.sync();

  // cluster-window addresses of every peer's node storage and "full" mbarrier
  uint32_t inter_rank[P::CL], full_rank[P::CL];
#pragma unroll
  for (int r = 0; r < P::CL; ++r) {
    inter_rank[r] = sa_mapa(sa_smem_u32(inter), r);
    full_rank[r] = sa_mapa(sa_smem_u32(&mbar[2]), r);
  }
  uint32_t sig_iter = 0;

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
  sa_cluster_arrive_relaxed();  // "node storage free" for the first signal

  for (int64_t sig = cid; sig < batch; sig += ncl, ++sig_iter) {
    if (tid == 0) sa_mbar_expect_tx(&mbar[2], (uint32_t)P::INTER);
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
      // scatter node row R = rev8(c) over the cluster: column q lives in CTA q / COLS.
      // Before the first scatter of a signal, every CTA must be done reading its
      // node storage for the previous signal (arrived after its last phase-B read).
      if (tt == 0) sa_cluster_wait();
      {
        const int c = rank * COLS + tt * TC + m2_cc;
        const int R = rev8(c);
        constexpr int KPC = COLS / 16;  // registers per owner CTA
#pragma unroll
        for (int k = 0; k < 16; ++k)
          sa_st_async(inter_rank[k / KPC] + (uint32_t)(sizeof(C2) * (R * COLS + m2_g + 16 * (k % KPC))),
                      A::to(v[k]), full_rank[k / KPC]);
      }
      __syncthreads();  // work[buf] fully consumed before it is re-armed
    }
    // ------------------------------------------------------------- phase B
    C2 *ysig = y + sig * NN;
    // twiddles: round 1 (stages 9..12) w1[h-1+a] = stage[off(t) + a*256 + q];
    //           round 2 (stages 13..16) w2[hr-1+a] = stage[off(t) + (g+16a)*256 + q].
    // Software-pipelined: w2 of tile tt and w1 of tile tt+1 are in flight while
    // the other round computes, so L2 latency is hidden.
    C4 w1[15], w2[15];
    auto load_w1 = [&](int q) {
#pragma unroll
      for (int t = 1; t <= 4; ++t)
#pragma unroll
        for (int a = 0; a < (1 << (t - 1)); ++a)
          w1[(1 << (t - 1)) - 1 + a] = sa_ldg(&stage[(1 << (7 + t)) - 1 + a * 256 + q]);
    };
    auto load_w2 = [&](int q) {
#pragma unroll
      for (int t = 5; t <= 8; ++t)
#pragma unroll
        for (int a = 0; a < (1 << (t - 5)); ++a)
          w2[(1 << (t - 5)) - 1 + a] = sa_ldg(&stage[(1 << (7 + t)) - 1 + (m1_g + 16 * a) * 256 + q]);
    };
    // fp64 keeps one twiddle set in flight (register budget); fp32 pipelines both.
    constexpr bool PREF = sizeof(T) == 4;
    load_w1(rank * COLS + m1_cc);
    sa_mbar_wait_cluster(&mbar[2], sig_iter & 1);  // all INTER bytes of this signal landed
    for (int tt = 0; tt < TILES; ++tt) {
      const int lq = tt * TC + m1_cc;
      const int q = rank * COLS + lq;
      if (PREF) load_w2(q);
      else if (tt > 0) load_w1(q);
      V v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(inter[(m1_g * 16 + k) * COLS + lq]);
#pragma unroll
      for (int t = 1; t <= 4; ++t) {  // global stage s = 8 + t, pairs along R bits 0..3
        const int h = 1 << (t - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & h)) r_dit<T>(v[k], v[k + h], w1[h - 1 + (k & (h - 1))]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) inter[(m1_g * 16 + k) * COLS + lq] = A::to(v[k]);
      __syncthreads();
      if (PREF && tt + 1 < TILES) load_w1(q + TC);
      if (!PREF) load_w2(q);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(inter[(m1_g + 16 * k) * COLS + lq]);
#pragma unroll
      for (int t = 5; t <= 8; ++t) {  // global stage s = 8 + t, pairs along R bits 4..7
        const int hr = 1 << (t - 5);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & hr)) r_dit<T>(v[k], v[k + hr], w2[hr - 1 + (k & (hr - 1))]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) __stcs(&ysig[(m1_g + 16 * k) * 256 + q], A::to(v[k]));
    }
    // Every value this CTA loaded from its node storage has been consumed by the
    // stores above (in-order issue), so a relaxed arrive is enough to let the
    // other CTAs start scattering the next signal into it.
    sa_cluster_arrive_relaxed();
  }
  sa_cluster_wait();  // pairs the last arrive; no CTA leaves while others may still read
}

// DIF (DESIGN.md convention): stages s = 16..2 with top = a + b, bot = W ⊙ (a − b),
// final 2-point NDFT, bit-reversed output.  Mirror image of the DIT kernel:
//   phase 1: CTA r takes node columns q in [r*COLS, (r+1)*COLS) of x[256 R + q]
//     (TMA tiles), runs stages 16..9 along R (j = (R mod 2^(t-1))*256 + q), and
//     sends row R to the CTA owning c = rev8(R) (DSMEM), stored q-swizzled;
//   phase 2: CTA r' runs stages 8..2 + the 2-point stage along q for its rows
//     and writes out[rev8(q)*256 + c] (coalesced over c).
template <typename T>
__global__ void __launch_bounds__(L64<T>::THREADS, 1)
    k_nlfft64k_dif(const __grid_constant__ CUtensorMap tmx, typename Ar<T>::C2 *__restrict__ y,
                   int64_t batch, const typename Ar<T>::C4 *__restrict__ stage, T gain,
                   int use_gain) {
  using P = L64<T>;
  using A = Ar<T>;
  using V = typename A::V;
  using C2 = typename P::C2;
  using C4 = typename P::C4;
  constexpr int TC = P::TC, COLS = P::COLS, TILES = P::TILES;
  constexpr bool PREF = sizeof(T) == 4;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  C2 *inter = reinterpret_cast<C2 *>(smem_raw);  // [COLS local rows][256 q], q ^ (lr & 15)
  C2 *work = reinterpret_cast<C2 *>(smem_raw + P::INTER);
  C4 *twA = reinterpret_cast<C4 *>(smem_raw + P::INTER + 2 * P::WORK);
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem_raw + P::INTER + 2 * P::WORK + P::TWA);

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int64_t cid = blockIdx.x / P::CL;
  const int64_t ncl = gridDim.x / P::CL;
  const int tid = threadIdx.x;
  const int m1_cc = tid % TC, m1_g = tid / TC;
  const int m2_g = tid & 15, m2_cc = tid >> 4;

  for (int e = tid; e < 255; e += P::THREADS) twA[e] = stage[e];
  if (tid == 0) {
    sa_mbar_init(&mbar[0], 1);
    sa_mbar_init(&mbar[1], 1);
    sa_mbar_init(&mbar[2], 1);
    sa_fence_mbar_init();
  }
  __syncthreads();
  cluster.sync();

  uint32_t inter_rank[P::CL], full_rank[P::CL];
#pragma unroll
  for (int r = 0; r < P::CL; ++r) {
    inter_rank[r] = sa_mapa(sa_smem_u32(inter), r);
    full_rank[r] = sa_mapa(sa_smem_u32(&mbar[2]), r);
  }

  auto issue = [&](int64_t sig, int tt, int buf) {
    if (tid == 0) {
      sa_fence_proxy_async();
      sa_mbar_expect_tx(&mbar[buf], (uint32_t)P::WORK);
      sa_tma_load_2d(work + buf * 256 * TC, &tmx, (rank * COLS + tt * TC) * P::EW, (int)(sig * 256),
                     &mbar[buf]);
    }
  };
  // phase-1 twiddles: wa (stages 16..13, R bits 7..4): stage[off(t) + (g+16a)*256 + q], t=5..8
  //                   wb (stages 12..9,  R bits 3..0): stage[off(t) + a*256 + q],      t=1..4
  C4 wa[15], wb[15];
  auto load_wa = [&](int q) {
#pragma unroll
    for (int t = 5; t <= 8; ++t)
#pragma unroll
      for (int a = 0; a < (1 << (t - 5)); ++a)
        wa[(1 << (t - 5)) - 1 + a] = sa_ldg(&stage[(1 << (7 + t)) - 1 + (m1_g + 16 * a) * 256 + q]);
  };
  auto load_wb = [&](int q) {
#pragma unroll
    for (int t = 1; t <= 4; ++t)
#pragma unroll
      for (int a = 0; a < (1 << (t - 1)); ++a)
        wb[(1 << (t - 1)) - 1 + a] = sa_ldg(&stage[(1 << (7 + t)) - 1 + a * 256 + q]);
  };

  int64_t it = 0;
  uint32_t sig_iter = 0;
  if (cid < batch) issue(cid, 0, 0);
  sa_cluster_arrive_relaxed();  // node storage free for the first signal
  const int rg1 = rev4(m1_g);

  for (int64_t sig = cid; sig < batch; sig += ncl, ++sig_iter) {
    if (tid == 0) sa_mbar_expect_tx(&mbar[2], (uint32_t)P::INTER);
    // ------------------------------------------------------------- phase 1
    for (int tt = 0; tt < TILES; ++tt, ++it) {
      const int buf = (int)(it & 1);
      const int q = rank * COLS + tt * TC + m1_cc;
      load_wa(q);
      if (PREF) load_wb(q);
      if (tt + 1 < TILES) issue(sig, tt + 1, buf ^ 1);
      else if (sig + ncl < batch) issue(sig + ncl, 0, buf ^ 1);
      sa_mbar_wait(&mbar[buf], (uint32_t)((it >> 1) & 1));
      C2 *wk = work + buf * 256 * TC;
      V v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {  // R = g + 16k
        V x = A::from(wk[(m1_g + 16 * k) * TC + m1_cc]);
        v[k] = use_gain ? A::scale(x, gain) : x;
      }
#pragma unroll
      for (int t = 8; t >= 5; --t) {  // global stage s = 8 + t, R bits 7..4
        const int hr = 1 << (t - 5);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & hr)) r_dif<T>(v[k], v[k + hr], wa[hr - 1 + (k & (hr - 1))]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) wk[(m1_g + 16 * k) * TC + m1_cc] = A::to(v[k]);
      __syncthreads();
      if (!PREF) load_wb(q);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(wk[(m1_g * 16 + k) * TC + m1_cc]);  // R = 16g + k
#pragma unroll
      for (int t = 4; t >= 1; --t) {  // R bits 3..0
        const int h = 1 << (t - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & h)) r_dif<T>(v[k], v[k + h], wb[h - 1 + (k & (h - 1))]);
      }
      // row R = 16g + k goes to the CTA owning c = rev8(R): local row lr = c mod COLS
      if (tt == 0) sa_cluster_wait();  // peers are done reading their node storage
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int c = crev4(k) * 16 + rg1;
        const int lr = c % COLS;
        sa_st_async(inter_rank[c / COLS] + (uint32_t)(sizeof(C2) * (lr * 256 + (q ^ (lr & 15)))),
                    A::to(v[k]), full_rank[c / COLS]);
      }
      __syncthreads();  // work[buf] consumed before it is re-armed
    }
    sa_mbar_wait_cluster(&mbar[2], sig_iter & 1);
    // ------------------------------------------------------------- phase 2
    C2 *ysig = y + sig * NN;
    for (int tt = 0; tt < TILES; ++tt) {
      V v[16];
      {  // round 1 (M2: g fastest): q = g + 16k ; stages 8..5
        const int lr = tt * TC + m2_cc;
        C2 *row = inter + lr * 256;
        const int sw = lr & 15;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = A::from(row[(m2_g + 16 * k) ^ sw]);
#pragma unroll
        for (int s = 8; s >= 5; --s) {
          const int hr = 1 << (s - 5), h = 1 << (s - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dif<T>(v[k], v[k + hr], twA[(h - 1) + m2_g + 16 * (k & (hr - 1))]);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) row[(m2_g + 16 * k) ^ sw] = A::to(v[k]);
      }
      __syncthreads();
      {  // round 2 (M1: cc fastest): q = 16g + k ; stages 4..2 + 2-point ; bit-reversed store
        const int lr = tt * TC + m1_cc;
        const C2 *row = inter + lr * 256;
        const int sw = lr & 15;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = A::from(row[(m1_g * 16 + k) ^ sw]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // s = 4: j = k
          if (k == 0) r_dif_one<T>(v[k], v[k + 8]);
          else if (k == 4) r_dif_mj<T>(v[k], v[k + 8]);
          else r_dif<T>(v[k], v[k + 8], twA[7 + k]);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)  // s = 3: j = k & 3
          if (!(k & 4)) {
            const int j = k & 3;
            if (j == 0) r_dif_one<T>(v[k], v[k + 4]);
            else if (j == 2) r_dif_mj<T>(v[k], v[k + 4]);
            else r_dif<T>(v[k], v[k + 4], twA[3 + j]);
          }
#pragma unroll
        for (int k = 0; k < 16; ++k)  // s = 2: j = k & 1
          if (!(k & 2)) {
            if (k & 1) r_dif_mj<T>(v[k], v[k + 2]);
            else r_dif_one<T>(v[k], v[k + 2]);
          }
#pragma unroll
        for (int k = 0; k < 16; k += 2) r_two_point<T>(v[k], v[k + 1]);
        const int c = rank * COLS + lr;
        const int rg = rev4(m1_g);
#pragma unroll
        for (int k = 0; k < 16; ++k) __stcs(&ysig[(crev4(k) * 16 + rg) * 256 + c], A::to(v[k]));
      }
    }
    sa_cluster_arrive_relaxed();  // all node-storage reads consumed (stores issued)
  }
  sa_cluster_wait();
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
int launch64k(int variant, const void *x, void *y, int64_t batch, const SaTwiddles *tw, double gain,
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
  auto kern = variant == SA_DIT ? k_nlfft64k_dit<T> : k_nlfft64k_dif<T>;
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
  if (n != NN || batch < 1) return SA_ERR_UNSUPPORTED;
  if (((uintptr_t)x & 15) != 0) return SA_ERR_UNSUPPORTED;
  if (dtype == SA_C64) return launch64k<float>(variant, x, y, batch, tw, gain, s);
  return launch64k<double>(variant, x, y, batch, tw, gain, s);
}
