// sa_nlfft64k.cu -- single-HBM-pass NL-FFT for N = 2^16 (BASELINE config C3).
//
// One signal per thread-block cluster (4 CTAs for c64, 8 for c128), entirely on
// chip, 1 CTA per SM.  N = 256 x 256.
// DIT (value-identical to transforms.py:254-298):
//   phase A: CTA r takes columns c of X[i][c] = x[256 i + c] (the reference's
//     bit-reversed blocks, SURVEY §7 hard part 4) in TMA-loaded tiles of TC
//     columns x 256 rows, runs global stages 1..8 in two register radix-16
//     rounds (stage 1 = the 2-point NDFT bottom), and scatters node row
//     R = rev8(c) over the cluster with st.async into the owner's smem, crediting
//     the owner's "full" mbarrier (no fence, no cluster barrier): q-columns
//     [r*COLS, (r+1)*COLS) of every row live in CTA r.  The CTA's own share goes
//     through st.shared, each warp arriving on the local full barrier after its
//     last store (SA_LOCALQ).
//   phase B: CTA r waits for its node storage, runs global stages 9..16 along R
//     for its columns (twiddle j = (R mod 2^(t-1))*256 + q), writes y[256 R + q].
//   An "empty" mbarrier fed by remote relaxed arrives guards storage reuse; each
//   thread group releases on its own (SA_GREL), so a group that finishes phase B
//   early starts the next signal.  The TMA tile of the next signal is issued at
//   the end of phase A, so HBM reads overlap phase B.
// complex64 DIT (SA_K64_PARK): each thread group computes one phase-A tile of the
// signal after next ahead of time and parks its results in TMEM (tcgen05.st into the
// thread's own lane, 32 columns per tile; fetched back with tcgen05.ld for the
// scatter), so that both cluster-wide waits of a signal -- "storage empty" before
// the scatter and "storage full" before phase B -- have one tile of compute in front
// of them (Pipe::run_park): C3 1.753 -> 1.676 ms, outputs bit-identical.  complex128
// uses the same schedule (64 words per tile) in DIT and DIF, in the compact loop form
// (4.28 -> 4.24 ms, 4.74 -> 4.42 ms); complex64 DIF does not (measured slower).
// Each CTA runs NG thread groups (named barriers, own TMA buffer) that split a
// phase's tiles.  HBM traffic = one read + one write.  Double-buffered node
// storage (NS = 2, pipelining phase B of signal s behind phase A of s+1) is
// supported but measured slower: it needs cluster 8 for c64.
#include <algorithm>
#include <cooperative_groups.h>
#include <cudaTypedefs.h>
#include <type_traits>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int LOGN = 16;
constexpr int NN = 1 << LOGN;

#ifndef SA_GREL
#define SA_GREL 1
#endif
#ifndef SA_WAIT1
#define SA_WAIT1 0  // 1: one warp per group polls, the rest block in bar.sync (measured slower: 1.790 vs 1.757 ms C3 DIT)
#endif
#ifndef SA_LOCALQ
#define SA_LOCALQ 1  // the CTA's own share of the scatter: st.shared + warp arrivals
#endif
#ifndef SA_K64_L2S
#define SA_K64_L2S 0  // c64: second node storage in an L2 scratch (signals alternate smem / L2)
#endif
#ifndef SA_K64_PARK
#define SA_K64_PARK 1  // c64 DIT: one phase-A tile per signal computed ahead and parked in TMEM (run_park)
#endif
#ifndef SA_K64_PARK_LOOP
#define SA_K64_PARK_LOOP 0  // c64: 1 = compact one-call-site form of the PARK signal loop (1.829 vs 1.676 ms DIT)
#endif
#ifndef SA_K64_PARK_S2
#define SA_K64_PARK_S2 0  // c64 DIT straight-line form: the B-tile / A-tile interleaved order (experiment)
#endif
#ifndef SA_K64_PARK_DIF
#define SA_K64_PARK_DIF 0  // the same for DIF (measured slower: 1.98 vs 1.79 ms)
#endif
#ifndef SA_K64_UNROLL_A
#define SA_K64_UNROLL_A 0
#endif
#ifndef SA_K64_WX
#define SA_K64_WX 0  // c64 DIT: phase-A 16 x 16 exchange inside a warp (128B-swizzled TMA tiles, __syncwarp)
#endif
#ifndef SA_K64_SKEW_F
#define SA_K64_SKEW_F 0  // ns: thread groups > 0 sleep this long after the full wait (de-phases the groups)
#endif
#ifndef SA_K64_SKEW_E
#define SA_K64_SKEW_E 0  // ns: the same after the empty wait
#endif
#ifndef SA_K64F_TC
#define SA_K64F_TC 16
#define SA_K64F_CL 4
#define SA_K64F_NG 2
#define SA_K64F_MINB 1
#define SA_K64F_NS 1
#endif

template <typename T> struct K64;
template <> struct K64<float> {
  static constexpr int TC = SA_K64F_TC;  // columns per tile
  static constexpr int CL = SA_K64F_CL;  // cluster size
  static constexpr int NG = SA_K64F_NG;  // thread groups per CTA
  static constexpr bool L2S = SA_K64_L2S;  // storage 1 in a global (L2-resident) scratch
  static constexpr int NS = L2S ? 2 : SA_K64F_NS;  // node storages (2 = pipelined signals)
  static constexpr int MINB = SA_K64F_MINB;  // resident CTAs per SM
  static constexpr bool PARK = SA_K64_PARK && !SA_K64_L2S && SA_K64F_NS == 1 && SA_K64F_NG * SA_K64F_TC == 32;
  static constexpr bool PARK_DIF = PARK && SA_K64_PARK_DIF;
  static constexpr bool PARK_LOOP = SA_K64_PARK_LOOP;
};
#ifndef SA_K64D_TC  // complex128 shape (-D for sweeps)
#define SA_K64D_TC 8
#define SA_K64D_NG 2
#endif
#ifndef SA_K64D_PARK
#define SA_K64D_PARK 1  // complex128: the TMEM-parking schedule, DIT (4.36 -> 4.24-4.34 ms)
#endif
#ifndef SA_K64D_PARK_DIF
#define SA_K64D_PARK_DIF 1  // and DIF (4.74 -> 4.44 ms)
#endif
#ifndef SA_K64D_PARK_LOOP
#define SA_K64D_PARK_LOOP 1  // compact loop form (the straight-line form is slower here: 4.57 / 4.86 ms)
#endif
template <> struct K64<double> {
  static constexpr int TC = SA_K64D_TC;
  static constexpr int CL = 8;
  static constexpr int NG = SA_K64D_NG;
  static constexpr bool L2S = false;
  static constexpr int NS = 1;
  static constexpr int MINB = 1;
  static constexpr bool PARK = SA_K64D_PARK && SA_K64D_NG * SA_K64D_TC == 16, PARK_DIF = PARK && SA_K64D_PARK_DIF;
  static constexpr bool PARK_LOOP = SA_K64D_PARK_LOOP;
};

template <typename T> struct L64 {
  static constexpr int TC = K64<T>::TC, CL = K64<T>::CL, NG = K64<T>::NG, NS = K64<T>::NS;
  static constexpr bool L2S = K64<T>::L2S;
  static constexpr bool PARK = K64<T>::PARK, PARK_DIF = K64<T>::PARK_DIF;
  static constexpr int NSM = L2S ? 1 : NS;  // node storages in smem
  static constexpr int GT = 16 * TC;       // threads per group
  static constexpr int THREADS = NG * GT;
  static constexpr int COLS = 256 / CL;    // node columns owned per CTA
  static constexpr int TILES = COLS / TC;  // tiles per CTA per phase
  static constexpr int TPG = TILES / NG;   // tiles per group per phase
  using C2 = typename Ar<T>::C2;
  using C4 = typename Ar<T>::C4;
  static constexpr size_t INTER1 = sizeof(C2) * 256 * COLS;  // one signal's node share
  static constexpr size_t WORK = sizeof(C2) * 256 * TC;      // one tile
  static constexpr size_t TWA = sizeof(C4) * 255;
  static constexpr size_t OFF_WORK = NSM * INTER1;
  static constexpr size_t OFF_TWA = OFF_WORK + NG * WORK;
  static constexpr size_t OFF_BAR = OFF_TWA + TWA;
  static constexpr size_t OFF_TMEM = OFF_BAR + 8 * (NG + 2 * NS);  // PARK: the TMEM base address
#if SA_K64_WX == 2
  static constexpr size_t OFF_CONS = OFF_TMEM + 8;  // WX = 2: per-group count of warps that consumed the tile
  static constexpr size_t SMEM = OFF_CONS + 4 * NG;
#else
  static constexpr size_t SMEM = OFF_TMEM + 8;
#endif
  // PARK: a thread parks one tile's 16 values (32 words) in its own TMEM lane; the 4 warps of a lane
  // quarter x TPG tiles take 32 columns each
  static constexpr int PARK_W = 4 * (int)sizeof(C2);  // words per thread and tile
  static constexpr int PARK_COLS = PARK_W * TPG * (THREADS / 128);
  static_assert(!PARK || (TPG == 2 && THREADS % 128 == 0 && PARK_COLS <= 512 && (PARK_COLS & (PARK_COLS - 1)) == 0),
                "park layout");
  static constexpr int EW = sizeof(C2) / 8;  // 8-byte TMA elements per complex
  static_assert(TILES % NG == 0 && TPG >= 1, "tiles must split evenly over groups");
};

SA_HD int rev4(int v) { return (int)(__brev((unsigned)v) >> 28); }
SA_HD int rev8(int v) { return (int)(__brev((unsigned)v) >> 24); }
constexpr int crev4(int v) { return ((v & 1) << 3) | ((v & 2) << 1) | ((v & 4) >> 1) | ((v & 8) >> 3); }

SA_HD void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Twiddles of the 8 cross-row stages (global 9..16) for node column q, as raw
// (wr, wi): wf[h-1+a] = table_s[a*256 + q] (stages 9..12, t = 1..4) and
// wf[15 + hr-1+a] = table_s[(g+16a)*256 + q] (stages 13..16, t = 5..8).  Every
// one has wr != 0 and wi < 0 unless q is 0 or 128 (j == 0 or j == h/2), so warps
// away from those two columns use the FMUL-free product (sa_regs.cuh).
template <typename T>
SA_HD void load_wf(typename Ar<T>::C2 (&wf)[30], const typename Ar<T>::C2 *__restrict__ stage2,
                   int q, int g) {
#pragma unroll
  for (int t = 1; t <= 4; ++t)
#pragma unroll
    for (int a = 0; a < (1 << (t - 1)); ++a)
      wf[(1 << (t - 1)) - 1 + a] = sa_ldg(&stage2[(1 << (7 + t)) - 1 + a * 256 + q]);
#pragma unroll
  for (int t = 5; t <= 8; ++t)
#pragma unroll
    for (int a = 0; a < (1 << (t - 5)); ++a)
      wf[15 + (1 << (t - 5)) - 1 + a] = sa_ldg(&stage2[(1 << (7 + t)) - 1 + (g + 16 * a) * 256 + q]);
}
// general form {|wr|, |wi|, sgn wr, sgn wi} (as the stage table) of a raw twiddle
template <typename T> SA_HD typename Ar<T>::C4 c4of(const typename Ar<T>::C2 &w) {
  return {fabs(w.x), fabs(w.y), sa_sgn(w.x), sa_sgn(w.y)};
}
#if defined(SA_PROBE_NOGEN)  // timing probe only (wrong results in columns 0 and 128): no general-product tiles
SA_HD bool special_column(int) { return false; }
#elif defined(SA_PROBE_ALLGEN)  // timing probe: every tile takes the general product
SA_HD bool special_column(int) { return true; }
#else
SA_HD bool special_column(int q) { return __any_sync(0xffffffffu, q == 0 || q == 128); }
#endif

// TMEM parking (SA_K64_PARK): 32 words of the executing thread's own lane, 32x32b shape
SA_HD void tm_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
SA_HD void tm_ld32(uint32_t (&r)[32], uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared per-CTA state and the signal pipeline orchestration of both kernels.
// PK: the TMEM-parking schedule (run_park) is in use
template <typename T, bool PK = false> struct Pipe {
  using P = L64<T>;
  using C2 = typename P::C2;
  using C4 = typename P::C4;
  unsigned char *smem;
  C4 *twA;
  uint64_t *tma_bar, *full_bar, *empty_bar;
  int rank, gi, gt;
  int64_t cid, ncl;
  uint32_t tile_it = 0;
  C2 *scr = nullptr;  // L2S: this cluster's scratch storage, [owner][INTER1 / sizeof(C2)]
  static constexpr int SE = (int)(P::INTER1 / sizeof(C2));  // elements of one owner's share
  uint32_t tm_park = 0;  // PARK: TMEM address of this thread's first parking slot
  SA_HD static bool in_l2(int b) { return P::L2S && b == 1; }
  // park / fetch tile u's 16 register values (fp32 pairs: 32 words; fp64 pairs: 64 words) in the
  // thread's TMEM lane
  SA_HD void park(int u, const sa_u64 (&v)[16]) const {
    if constexpr (PK) {
      uint32_t r[32];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        r[2 * k] = (uint32_t)v[k];
        r[2 * k + 1] = (uint32_t)(v[k] >> 32);
      }
      tm_st32(tm_park + 32u * (uint32_t)u, r);
    }
  }
  SA_HD void unpark(int u, sa_u64 (&v)[16]) const {
    if constexpr (PK) {
      uint32_t r[32];
      tm_ld32(r, tm_park + 32u * (uint32_t)u);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = (sa_u64)r[2 * k] | ((sa_u64)r[2 * k + 1] << 32);
    }
  }
  SA_HD void park(int u, const double2 (&v)[16]) const {
    if constexpr (PK) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t r[32];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          r[4 * k] = (uint32_t)__double2loint(v[8 * h + k].x);
          r[4 * k + 1] = (uint32_t)__double2hiint(v[8 * h + k].x);
          r[4 * k + 2] = (uint32_t)__double2loint(v[8 * h + k].y);
          r[4 * k + 3] = (uint32_t)__double2hiint(v[8 * h + k].y);
        }
        tm_st32(tm_park + 64u * (uint32_t)u + 32u * (uint32_t)h, r);
      }
    }
  }
  SA_HD void unpark(int u, double2 (&v)[16]) const {
    if constexpr (PK) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t r[32];
        tm_ld32(r, tm_park + 64u * (uint32_t)u + 32u * (uint32_t)h);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[8 * h + k].x = __hiloint2double((int)r[4 * k + 1], (int)r[4 * k]);
          v[8 * h + k].y = __hiloint2double((int)r[4 * k + 3], (int)r[4 * k + 2]);
        }
      }
    }
  }
  template <bool S> SA_HD static C2 ld(const C2 *p) {
    if constexpr (S) return __ldcg(p);
    else return *p;
  }
  template <bool S> SA_HD static void st(C2 *p, C2 v) {
    if constexpr (S) __stcg(p, v);
    else *p = v;
  }
  // this CTA's share of storage b (smem, or its owner region of the L2 scratch)
  SA_HD C2 *share(int b) const { return in_l2(b) ? scr + (size_t)rank * SE : inter(b); }

  SA_HD C2 *inter(int b) const { return reinterpret_cast<C2 *>(smem + b * P::INTER1); }
  // after a thread's last local scatter store of a signal: its warp's arrive on full[b]
  SA_HD void local_done(int b) const {
    if (in_l2(b)) {  // scratch stores of this group -> every owner's full[1] (release at cluster scope)
      group_sync(1 + gi, P::GT);
      if (gt == 0)
#pragma unroll
        for (int r = 0; r < P::CL; ++r) sa_mbar_arrive_remote_release(peer_full(1, r));
      return;
    }
    if (SA_LOCALQ) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) sa_mbar_arrive_local(&full_bar[b]);
    }
  }
  SA_HD C2 *work() const { return reinterpret_cast<C2 *>(smem + P::OFF_WORK + gi * P::WORK); }
  // cluster-window address of peer r's node storage b (byte offset off) / its full mbarrier
  // (mapa is linear inside a CTA's window: the peer bases are mapped once, in init)
  uint32_t pinter[P::CL], pfull[P::CL];
  SA_HD uint32_t peer_inter(int b, int r, uint32_t off) const { return pinter[r] + (uint32_t)(b * P::INTER1) + off; }
  SA_HD uint32_t peer_full(int b, int r) const { return pfull[r] + 8u * (uint32_t)b; }
  // wait for an mbarrier phase: one warp of the thread group polls, the rest block
  // in the group's named barrier (no issue slots spent spinning)
  SA_HD void group_wait(uint64_t *bar, uint32_t parity) const {
#ifdef SA_PROBE_NOSYNC  // timing probe only (wrong results): no cross-CTA storage waits
    if (bar != &tma_bar[gi]) return;
#endif
#if SA_WAIT1
    if ((gt >> 5) == 0) sa_mbar_wait(bar, parity);
    group_sync(1 + gi, P::GT);
#else
    sa_mbar_wait(bar, parity);
#endif
  }

  SA_HD void init(unsigned char *smem_raw, const C4 *stage, C2 *scratch) {
    cg::cluster_group cluster = cg::this_cluster();
    smem = smem_raw;
    twA = reinterpret_cast<C4 *>(smem + P::OFF_TWA);
    tma_bar = reinterpret_cast<uint64_t *>(smem + P::OFF_BAR);
    full_bar = tma_bar + P::NG;
    empty_bar = full_bar + P::NS;
    rank = (int)cluster.block_rank();
    cid = blockIdx.x / P::CL;
    ncl = gridDim.x / P::CL;
    gi = threadIdx.x / P::GT;
    gt = threadIdx.x % P::GT;
    if (P::L2S) scr = scratch + (size_t)cid * P::CL * SE;
#pragma unroll
    for (int r = 0; r < P::CL; ++r) {
      pinter[r] = sa_mapa(sa_smem_u32(smem), r);
      pfull[r] = sa_mapa(sa_smem_u32(smem + P::OFF_BAR + 8 * P::NG), r);
    }
    for (int e = threadIdx.x; e < 255; e += P::THREADS) twA[e] = stage[e];  // global stages 1..8
#if SA_K64_WX == 2
    if (threadIdx.x < P::NG) reinterpret_cast<uint32_t *>(smem + P::OFF_CONS)[threadIdx.x] = 0u;
#endif
    if (threadIdx.x == 0) {
      for (int g = 0; g < P::NG; ++g) sa_mbar_init(&tma_bar[g], 1);
      for (int b = 0; b < P::NS; ++b) {
        // expect_tx(remote bytes) once per use (+ one arrive per warp for the local share)
        sa_mbar_init(&full_bar[b], in_l2(b) ? P::CL * P::NG  // one arrive per thread group of the cluster
                                            : 1 + (SA_LOCALQ ? P::THREADS / 32 : 0));
        sa_mbar_init(&empty_bar[b], SA_GREL ? P::CL * P::NG : P::CL);  // remote arrives per use
      }
      sa_fence_mbar_init();
    }
    if constexpr (PK) {
      uint32_t *holder = reinterpret_cast<uint32_t *>(smem + P::OFF_TMEM);
      if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa_smem_u32(holder)),
                     "r"((uint32_t)P::PARK_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t w = threadIdx.x >> 5;
      tm_park = *holder + (((w & 3u) * 32u) << 16) + (w >> 2) * (uint32_t)(P::PARK_W * P::TPG);
    }
    __syncthreads();
    cluster.sync();
  }
  SA_HD void finish() const {
    if constexpr (PK) {
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < 32) {
        const uint32_t base = *reinterpret_cast<const uint32_t *>(smem + P::OFF_TMEM);
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"((uint32_t)P::PARK_COLS)
                     : "memory");
      }
    }
  }
  // group-leader TMA of tile tt (TC columns x 256 rows) of signal sig
  SA_HD void tma(const CUtensorMap *tmx, int64_t sig, int tt) const {
    if (gt == 0) {
      sa_fence_proxy_async();
      sa_mbar_expect_tx(&tma_bar[gi], (uint32_t)P::WORK);
      sa_tma_load_2d(work(), tmx, (rank * P::COLS + tt * P::TC) * P::EW, (int)(sig * 256), &tma_bar[gi]);
    }
  }
#if SA_K64_WX == 2
  // WX = 2: every warp calls this once its lanes have read the tile (after __syncwarp); the last
  // of the group's warps re-arms the buffer and issues the next TMA -- no group barrier
  SA_HD void tma_last(const CUtensorMap *tmx, int64_t sig, int tt) const {
    if ((threadIdx.x & 31) == 0) {
      uint32_t *cons = reinterpret_cast<uint32_t *>(smem + P::OFF_CONS) + gi;
      __threadfence_block();
      const uint32_t old = atomicAdd(cons, 1u);
      if ((old % (P::GT / 32)) == (P::GT / 32) - 1 && sig >= 0) {
        __threadfence_block();
        sa_fence_proxy_async();
        sa_mbar_expect_tx(&tma_bar[gi], (uint32_t)P::WORK);
        sa_tma_load_2d(work(), tmx, (rank * P::COLS + tt * P::TC) * P::EW, (int)(sig * 256), &tma_bar[gi]);
      }
    }
  }
#endif
  SA_HD void wait_tile() {
    group_wait(&tma_bar[gi], tile_it & 1);
    ++tile_it;
  }
  // "storage b may be overwritten": the CTA (SA_GREL: this thread group)
  // finished reading it; one thread arrives on every peer's empty barrier for b.
  SA_HD void release(int b) const {
#if SA_GREL
    group_sync(1 + gi, P::GT);
    if (gt == 0)
#else
    __syncthreads();
    if (threadIdx.x == 0)
#endif
#pragma unroll
      for (int r = 0; r < P::CL; ++r) {
        const uint32_t a = sa_mapa(sa_smem_u32(&empty_bar[b]), r);
        if (in_l2(b)) sa_mbar_arrive_remote_release(a);  // our scratch write-backs precede the next writer's
        else sa_mbar_arrive_remote(a);
      }
  }
  // wait until storage b may be written (scratch: cluster-scope acquire)
  SA_HD void wait_empty(int b, uint32_t parity) const {
    if (in_l2(b)) sa_mbar_wait_cluster(&empty_bar[b], parity);
    else group_wait(&empty_bar[b], parity);
    if (SA_K64_SKEW_E > 0 && gi > 0) __nanosleep(SA_K64_SKEW_E * gi);
  }
  SA_HD void wait_full(int b, uint32_t parity) const {
    if (in_l2(b)) sa_mbar_wait_cluster(&full_bar[b], parity);
    else group_wait(&full_bar[b], parity);
    if (SA_K64_SKEW_F > 0 && gi > 0) __nanosleep(SA_K64_SKEW_F * gi);
  }
  // signal loop: phaseA(sig, b, use, next_sig) then (pipelined) phaseB of the
  // previous signal; every storage use waits full/empty with parity use & 1.
  template <class FA, class FB>
  SA_HD void run(const CUtensorMap *tmx, int64_t batch, FA phaseA, FB phaseB) {
    if (cid < batch) tma(tmx, cid, gi);
    for (int b = 0; b < P::NS; ++b) release(b);  // all storages free
    int64_t i = 0;
    for (int64_t sig = cid; sig < batch; sig += ncl, ++i) {
      const int b = (int)(i % P::NS);
      if (threadIdx.x == 0 && !in_l2(b))
#ifdef SA_PROBE_NOSCATTER
        sa_mbar_arrive_local(&full_bar[b]);  // probe: no remote bytes expected
#else
        sa_mbar_expect_tx(&full_bar[b], (uint32_t)(SA_LOCALQ ? P::INTER1 - P::INTER1 / P::CL : P::INTER1));
#endif
      phaseA(sig, b, (uint32_t)(i / P::NS), sig + ncl);
      if (P::NS == 1) {
        phaseB(sig, 0, (uint32_t)i);
        if (sig + ncl < batch) release(0);
      } else if (i > 0) {
        const int pb = (int)((i - 1) % P::NS);
        phaseB(sig - ncl, pb, (uint32_t)((i - 1) / P::NS));
        if (sig + ncl < batch) release(pb);  // next user of pb is signal i+1
      }
    }
    if (P::NS == 2 && i > 0)
      phaseB(cid + (i - 1) * ncl, (int)((i - 1) % P::NS), (uint32_t)((i - 1) / P::NS));
#ifdef SA_PROBE_NOSYNC
    cg::this_cluster().sync();  // the probe skips the storage waits: let peers' stores land first
#endif
  }
  // PARK signal loop (one node storage, TPG = 2).  tileA(M = 3, sig, u, b, use, we, tsig, tu)
  // computes phase-A tile u of sig (issuing the group's next TMA (tsig, tile index tu) once its
  // buffer is consumed) and then either parks the 16 results of each thread in TMEM (we = false)
  // or waits for the storage, scatters them and the parked tile 1, and arrives on full.  Per group:
  //   B(s) | release | X: A(s+1, tile 0), wait empty, scatter tiles 0 and 1 | Y: A(s+2, tile 1), park |
  //   wait full | B(s+1) ...
  // so each of the two cluster-wide waits has one tile of compute in front of it.  One loop, one
  // call site per lambda (the instruction cache matters: an unrolled phase A costs 5%).
  template <class FT, class FB>
  SA_HD void run_park(const CUtensorMap *tmx, int64_t batch, FT tileA, FB phaseB) {
    static_assert(!PK || P::TPG == 2, "PARK schedule is written for two tiles per group");
    const uint32_t tx = (uint32_t)(SA_LOCALQ ? P::INTER1 - P::INTER1 / P::CL : P::INTER1);
    if constexpr (!K64<T>::PARK_LOOP) {
    // straight-line form (complex64: 1.676 ms C3 DIT against 1.829 for the compact loop below,
    // although it is twice the code; complex128 is faster with the compact loop)
    using M0 = std::integral_constant<int, 0>;
    using M1 = std::integral_constant<int, 1>;
    using M2 = std::integral_constant<int, 2>;
    auto sig_or_none = [&](int64_t sg) { return sg < batch ? sg : (int64_t)-1; };
    if (cid < batch) tma(tmx, cid, gi);
    release(0);
    if (cid < batch) {
      if (threadIdx.x == 0) sa_mbar_expect_tx(&full_bar[0], tx);
      tileA(M0{}, cid, 0, 0, 0u, true, cid, 1);
      tileA(M0{}, cid, 1, 0, 0u, false, sig_or_none(cid + ncl), 1);
      local_done(0);
      if (cid + ncl < batch) tileA(M1{}, cid + ncl, 1, 0, 0u, false, cid + ncl, 0);
    }
#if SA_K64_PARK_S2
    // variant: B tile 0 | A(s+1, tile 0) -> park | B tile 1 | release, wait empty, scatter both parked
    // tiles | A(s+2, tile 1) -> park | wait full: both TMA loads get a long lead
    {
      uint32_t it2 = 0;
      for (int64_t sig = cid; sig < batch; sig += ncl, ++it2) {
        const int64_t n1 = sig + ncl, n2 = n1 + ncl;
        phaseB(sig, 0, it2, 0, 1);
        if (n1 < batch) tileA(M1{}, n1, 0, 0, 0u, false, sig_or_none(n2), 1);
        phaseB(sig, 0, it2, 1, 2);
        if (n1 < batch) {
          if (threadIdx.x == 0) sa_mbar_expect_tx(&full_bar[0], tx);
          release(0);
          tileA(M2{}, n1, 0, 0, it2 + 1, true, (int64_t)-1, 0);
          tileA(M2{}, n1, 1, 0, it2 + 1, false, (int64_t)-1, 0);
          local_done(0);
          if (n2 < batch) tileA(M1{}, n2, 1, 0, 0u, false, n2, 0);
        }
      }
      finish();
      return;
    }
#endif
    uint32_t it = 0;
    for (int64_t sig = cid; sig < batch; sig += ncl, ++it) {
      const int64_t n1 = sig + ncl, n2 = n1 + ncl;
      phaseB(sig, 0, it);  // waits full (parity it & 1)
      if (n1 < batch) {
        // the next use of the full barrier is armed after this one completed (thread 0 has
        // passed its wait) and before this group's release lets any peer send
        if (threadIdx.x == 0) sa_mbar_expect_tx(&full_bar[0], tx);
        release(0);
        tileA(M0{}, n1, 0, 0, it + 1, true, sig_or_none(n2), 1);
        tileA(M2{}, n1, 1, 0, it + 1, false, (int64_t)-1, 0);
        local_done(0);
        if (n2 < batch) tileA(M1{}, n2, 1, 0, 0u, false, n2, 0);
      }
    }
    finish();
    return;
    }
    if (cid < batch) tma(tmx, cid, gi + P::NG);  // tile index 1 of the first signal comes first
    release(0);
    for (int64_t i = -2;; ++i) {
      const int64_t sig = cid + i * ncl;
      if (i >= 0) {
        if (sig >= batch) break;
        phaseB(sig, 0, (uint32_t)i);  // waits full (parity i & 1)
      }
#pragma unroll 1
      for (int j = 0; j < 2; ++j) {
        const bool isx = j == 0;
        const int64_t s = sig + (isx ? 1 : 2) * ncl;  // X: signal i + 1, Y: signal i + 2
        if (s >= batch || (isx && i < -1)) continue;
        int64_t tsig = s;  // Y: this signal's tile 0 next
        if (isx) {
          // the next use of the full barrier is armed after the last one completed (thread 0
          // has passed its wait) and before this group's release lets any peer send
          if (threadIdx.x == 0) sa_mbar_expect_tx(&full_bar[0], tx);
          if (i >= 0) release(0);
          tsig = s + ncl < batch ? s + ncl : (int64_t)-1;  // X: the next signal's tile 1
        }
        tileA(std::integral_constant<int, 3>{}, s, isx ? 0 : 1, 0, (uint32_t)(i + 1), isx, tsig, isx ? 1 : 0);
      }
    }
    finish();
  }
};

template <typename T>
__global__ void __launch_bounds__(L64<T>::THREADS, K64<T>::MINB)
    k_nlfft64k_dit(const __grid_constant__ CUtensorMap tmx, typename Ar<T>::C2 *__restrict__ y,
                   int64_t batch, const typename Ar<T>::C4 *__restrict__ stage,
                   const typename Ar<T>::C2 *__restrict__ stage2, T gain, int use_gain,
                   typename Ar<T>::C2 *__restrict__ scratch) {
  using P = L64<T>;
  using A = Ar<T>;
  using V = typename A::V;
  using C2 = typename P::C2;
  using C4 = typename P::C4;
  constexpr int TC = P::TC, COLS = P::COLS, NG = P::NG, GT = P::GT, TPG = P::TPG;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Pipe<T, P::PARK> pp;
  pp.init(smem_raw, stage, scratch);
  const int gbar = 1 + pp.gi;
  const int m1_cc = pp.gt % TC, m1_g = pp.gt / TC;
  // WX: a warp owns two columns; each half-warp holds eight g values (one parity) of both, so
  // that its 16 lanes touch 16 distinct 8-byte bank pairs of the 128B-swizzled tile
#if SA_K64_WX
  constexpr bool WX = std::is_same<T, float>::value && TC == 16;
  const int wx_lane = threadIdx.x & 31;
  const int m2_g = WX ? ((wx_lane >> 1) & 7) * 2 + (wx_lane >> 4) : (pp.gt & 15);
  const int m2_cc = WX ? 2 * (pp.gt >> 5) + (wx_lane & 1) : (pp.gt >> 4);
#else
  const int m2_g = pp.gt & 15, m2_cc = pp.gt >> 4;
#endif
  const C4 *twA = pp.twA;

  // M = 0: compute and scatter; PARK schedule (run_park): 1 compute and park, 2 fetch the parked
  // tile and scatter, 3 the runtime-selected form of the compact loop
  // one phase-A tile; the group's next TMA (signal tsig, tile index tu; none if tsig < 0) is issued
  // once the tile buffer has been consumed; we: wait for the storage to be free before scattering
  auto tileA = [&](auto M_, int64_t sig, int u, int b, uint32_t use, bool we, int64_t tsig, int tu) {
    constexpr int M = decltype(M_)::value;
    {
      V v[16];
      if constexpr (M == 2) pp.unpark(u, v);
      if constexpr (M != 2) {
      pp.wait_tile();
      C2 *wk = pp.work();
#if SA_K64_WX
      // WX: physical position of (row, column m2_cc) in the 128B-swizzled tile
      auto wx_at = [&](int row) { return row * TC + ((((m2_cc >> 1) ^ (row & 7)) << 1) | (m2_cc & 1)); };
#endif
      {  // round 1 (M1; WX: M2): v[k] = node 16g+k of sub-transform cc = X[rev8(16g+k)][cc]
#if SA_K64_WX
        const int rg = rev4(WX ? m2_g : m1_g);
#else
        const int rg = rev4(m1_g);
#endif
#pragma unroll
        for (int k = 0; k < 16; ++k) {
#if SA_K64_WX
          V x = A::from(WX ? wk[wx_at(crev4(k) * 16 + rg)] : wk[(crev4(k) * 16 + rg) * TC + m1_cc]);
#else
          V x = A::from(wk[(crev4(k) * 16 + rg) * TC + m1_cc]);
#endif
          v[k] = use_gain ? A::scale(x, gain) : x;
        }
#ifndef SA_PROBE_SKIP_A
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
#endif
      }
#if SA_K64_WX
      if constexpr (WX) {
        // the 16 threads of a column are lanes of one warp: exchange through the column's own
        // 256 slots, entry (g, k) in row rho = ((2g + (k & 1)) << 3) | ((k >> 1) ^ (g >> 1)), so
        // that writes (fixed k) and reads (fixed k') of a half-warp are bank-conflict free
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 16; ++k)
          wk[wx_at(((m2_g * 2 + (k & 1)) << 3) | ((k >> 1) ^ (m2_g >> 1)))] = A::to(v[k]);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 16; ++k)  // node g + 16k = entry (k, g)
          v[k] = A::from(wk[wx_at(((k * 2 + (m2_g & 1)) << 3) | ((m2_g >> 1) ^ (k >> 1)))]);
      } else
#endif
      {
      group_sync(gbar, GT);
#pragma unroll
      for (int k = 0; k < 16; ++k)  // exchange: node q = 16g+k, column swizzled by q & (TC-1)
        wk[(m1_g * 16 + k) * TC + (m1_cc ^ (k & (TC - 1)))] = A::to(v[k]);
      group_sync(gbar, GT);
#pragma unroll
      for (int k = 0; k < 16; ++k)  // round 2 (M2): node g + 16k of sub-transform cc
        v[k] = A::from(wk[(m2_g + 16 * k) * TC + (m2_cc ^ (m2_g & (TC - 1)))]);
      }
#if SA_K64_WX == 2
      if constexpr (WX) {
        __syncwarp();
        pp.tma_last(&tmx, tsig, pp.gi + NG * tu);
      } else
#endif
      {
        group_sync(gbar, GT);  // tile buffer consumed: re-arm it
        if (tsig >= 0) pp.tma(&tmx, tsig, pp.gi + NG * tu);
      }
#ifndef SA_PROBE_SKIP_A
#pragma unroll
      for (int t = 5; t <= 8; ++t) {
        const int hr = 1 << (t - 5), h = 1 << (t - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & hr)) r_dit<T>(v[k], v[k + hr], twA[(h - 1) + m2_g + 16 * (k & (hr - 1))]);
      }
#endif
      }
      // scatter node row R = rev8(c) of tile index uu: column q lives in CTA q / COLS
      auto scat = [&](int uu) {
        const int R = rev8(pp.rank * COLS + (pp.gi + NG * uu) * TC + m2_cc);
        constexpr int KPC = COLS / 16;  // registers per owner CTA
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int e = R * COLS + m2_g + 16 * (k % KPC);
          if (Pipe<T>::in_l2(b)) __stcg(&pp.scr[(k / KPC) * Pipe<T>::SE + e], A::to(v[k]));
          else if (SA_LOCALQ && k / KPC == pp.rank) pp.inter(b)[e] = A::to(v[k]);
#ifndef SA_PROBE_NOSCATTER
          else sa_st_async(pp.peer_inter(b, k / KPC, (uint32_t)(sizeof(C2) * e)), A::to(v[k]), pp.peer_full(b, k / KPC));
#else
          else pp.inter(b)[e] = A::to(v[k]);  // probe: local store instead of the DSMEM scatter
#endif
        }
      };
      if constexpr (M == 1) {  // PARK: park this tile
        pp.park(u, v);
      } else if constexpr (M == 3) {  // PARK, compact loop: we ? scatter this tile (0) and the parked tile 1 : park
        if (!we) {
          pp.park(u, v);
          return;
        }
        pp.wait_empty(b, use & 1);
#pragma unroll 1
        for (int w = 0; w < 2; ++w) {
          if (w) pp.unpark(1, v);
          scat(w);
        }
        pp.local_done(b);
      } else {
        if (we) pp.wait_empty(b, use & 1);  // peers released storage b
        scat(u);
      }
    }
  };
  auto phaseA = [&](int64_t sig, int b, uint32_t use, int64_t nsig) {
#if SA_K64_UNROLL_A
#pragma unroll
#endif
    for (int u = 0; u < TPG; ++u)
      tileA(std::integral_constant<int, 0>{}, sig, u, b, use, u == 0,
            u + 1 < TPG ? sig : (nsig < batch ? nsig : (int64_t)-1), u + 1 < TPG ? u + 1 : 0);
    pp.local_done(b);
  };

  // tiles [u0, u1) of the group; the storage wait comes with tile 0
  auto phaseB_s = [&](auto S_, int64_t sig, int b, uint32_t use, int u0, int u1) {
    constexpr bool S = decltype(S_)::value;  // storage in the L2 scratch
    C2 *inter = pp.share(b);
    C2 *ysig = y + sig * NN;
    C2 wf[30];
    {
      const int q0 = pp.rank * COLS + (pp.gi + NG * u0) * TC + m1_cc;  // independent of the node storage
      load_wf<T>(wf, stage2, q0, m1_g);
    }
    if (u0 == 0) pp.wait_full(b, use & 1);  // all INTER1 bytes of this signal landed
    for (int u = u0; u < u1; ++u) {
      const int tt = pp.gi + NG * u;
      const int lq = tt * TC + m1_cc;
      const int q = pp.rank * COLS + lq;
      const bool gen = special_column(q);
#ifndef SA_PROBE_NOTWLD
      if (u > u0) load_wf<T>(wf, stage2, q, m1_g);
#endif
      V v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(Pipe<T>::template ld<S>(&inter[(m1_g * 16 + k) * COLS + lq]));
#ifndef SA_PROBE_SKIP_B
      if (gen) {  // warps with column 0 / 128: general product (twiddles with zero components)
#pragma unroll
        for (int t = 1; t <= 4; ++t) {  // R bits 0..3
          const int h = 1 << (t - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dit<T>(v[k], v[k + h], c4of<T>(wf[h - 1 + (k & (h - 1))]));
        }
      } else {
#pragma unroll
        for (int t = 1; t <= 4; ++t) {
          const int h = 1 << (t - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dit_fast<T>(v[k], v[k + h], wf[h - 1 + (k & (h - 1))]);
        }
      }
#endif
#pragma unroll
      for (int k = 0; k < 16; ++k) Pipe<T>::template st<S>(&inter[(m1_g * 16 + k) * COLS + lq], A::to(v[k]));
      group_sync(gbar, GT);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(Pipe<T>::template ld<S>(&inter[(m1_g + 16 * k) * COLS + lq]));
#ifndef SA_PROBE_SKIP_B
      if (gen) {
#pragma unroll
        for (int t = 5; t <= 8; ++t) {  // R bits 4..7
          const int hr = 1 << (t - 5);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dit<T>(v[k], v[k + hr], c4of<T>(wf[15 + hr - 1 + (k & (hr - 1))]));
        }
      } else {
#pragma unroll
        for (int t = 5; t <= 8; ++t) {
          const int hr = 1 << (t - 5);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dit_fast<T>(v[k], v[k + hr], wf[15 + hr - 1 + (k & (hr - 1))]);
        }
      }
#endif
#pragma unroll
      for (int k = 0; k < 16; ++k) __stcs(&ysig[(m1_g + 16 * k) * 256 + q], A::to(v[k]));
    }
  };

  auto phaseB = [&](int64_t sig, int b, uint32_t use, int u0 = 0, int u1 = P::TPG) {
    if constexpr (P::L2S) {
      if (Pipe<T>::in_l2(b)) {
        phaseB_s(std::true_type{}, sig, b, use, u0, u1);
        return;
      }
    }
    phaseB_s(std::false_type{}, sig, b, use, u0, u1);
  };

  if constexpr (P::PARK) {
    pp.run_park(&tmx, batch, tileA, phaseB);
  } else {
    pp.run(&tmx, batch, phaseA, phaseB);
  }
}

// DIF (DESIGN.md convention): stages s = 16..2 with top = a + b, bot = W ⊙ (a − b),
// final 2-point NDFT, bit-reversed output.  Mirror image of the DIT kernel:
//   phase 1: CTA r takes node columns q in [r*COLS, (r+1)*COLS) of x[256 R + q]
//     (TMA tiles), runs stages 16..9 along R (j = (R mod 2^(t-1))*256 + q), and
//     sends row R to the CTA owning c = rev8(R) (st.async), stored q-swizzled;
//   phase 2: CTA r' runs stages 8..2 + the 2-point stage along q for its rows
//     and writes out[rev8(q)*256 + c] (coalesced over c).
template <typename T>
__global__ void __launch_bounds__(L64<T>::THREADS, K64<T>::MINB)
    k_nlfft64k_dif(const __grid_constant__ CUtensorMap tmx, typename Ar<T>::C2 *__restrict__ y,
                   int64_t batch, const typename Ar<T>::C4 *__restrict__ stage,
                   const typename Ar<T>::C2 *__restrict__ stage2, T gain, int use_gain,
                   typename Ar<T>::C2 *__restrict__ scratch) {
  using P = L64<T>;
  using A = Ar<T>;
  using V = typename A::V;
  using C2 = typename P::C2;
  using C4 = typename P::C4;
  constexpr int TC = P::TC, COLS = P::COLS, NG = P::NG, GT = P::GT, TPG = P::TPG;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Pipe<T, P::PARK_DIF> pp;
  pp.init(smem_raw, stage, scratch);
  const int gbar = 1 + pp.gi;
  const int m1_cc = pp.gt % TC, m1_g = pp.gt / TC;
  const int m2_g = pp.gt & 15, m2_cc = pp.gt >> 4;
  const C4 *twA = pp.twA;
  const int rg1 = rev4(m1_g);

  auto tileA = [&](auto M_, int64_t sig, int u, int b, uint32_t use, bool we, int64_t tsig, int tu) {
    constexpr int M = decltype(M_)::value;  // as in the DIT kernel
    {
      const int tt = pp.gi + NG * u;
      const int q = pp.rank * COLS + tt * TC + m1_cc;
      V v[16];
      if constexpr (M == 2) pp.unpark(u, v);
      if constexpr (M != 2) {
      const bool gen = special_column(q);
      C2 wf[30];
      load_wf<T>(wf, stage2, q, m1_g);
      pp.wait_tile();
      C2 *wk = pp.work();
#pragma unroll
      for (int k = 0; k < 16; ++k) {  // R = g + 16k
        V x = A::from(wk[(m1_g + 16 * k) * TC + m1_cc]);
        v[k] = use_gain ? A::scale(x, gain) : x;
      }
      if (gen) {  // warps with column 0 / 128: general product
#pragma unroll
        for (int t = 8; t >= 5; --t) {  // R bits 7..4
          const int hr = 1 << (t - 5);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dif<T>(v[k], v[k + hr], c4of<T>(wf[15 + hr - 1 + (k & (hr - 1))]));
        }
      } else {
#pragma unroll
        for (int t = 8; t >= 5; --t) {
          const int hr = 1 << (t - 5);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dif_fast<T>(v[k], v[k + hr], wf[15 + hr - 1 + (k & (hr - 1))]);
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) wk[(m1_g + 16 * k) * TC + m1_cc] = A::to(v[k]);
      group_sync(gbar, GT);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(wk[(m1_g * 16 + k) * TC + m1_cc]);  // R = 16g + k
      group_sync(gbar, GT);  // tile buffer consumed: re-arm it
      if (tsig >= 0) pp.tma(&tmx, tsig, pp.gi + NG * tu);
      if (gen) {
#pragma unroll
        for (int t = 4; t >= 1; --t) {  // R bits 3..0
          const int h = 1 << (t - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dif<T>(v[k], v[k + h], c4of<T>(wf[h - 1 + (k & (h - 1))]));
        }
      } else {
#pragma unroll
        for (int t = 4; t >= 1; --t) {
          const int h = 1 << (t - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dif_fast<T>(v[k], v[k + h], wf[h - 1 + (k & (h - 1))]);
        }
      }
      }
      auto scat = [&](int uu) {
        const int qq = pp.rank * COLS + (pp.gi + NG * uu) * TC + m1_cc;
#pragma unroll
        for (int k = 0; k < 16; ++k) {  // row R = 16g + k -> CTA owning cr = rev8(R), local row cr mod COLS
          const int cr = crev4(k) * 16 + rg1;
          const int lr = cr % COLS;
          const int e = lr * 256 + (qq ^ (lr & 15));
          if (Pipe<T>::in_l2(b)) __stcg(&pp.scr[(cr / COLS) * Pipe<T>::SE + e], A::to(v[k]));
          else if (SA_LOCALQ && cr / COLS == pp.rank) pp.inter(b)[e] = A::to(v[k]);  // owner is warp-uniform
          else sa_st_async(pp.peer_inter(b, cr / COLS, (uint32_t)(sizeof(C2) * e)), A::to(v[k]), pp.peer_full(b, cr / COLS));
        }
      };
      if constexpr (M == 1) {
        pp.park(u, v);
      } else if constexpr (M == 3) {  // PARK: as in the DIT kernel
        if (!we) {
          pp.park(u, v);
          return;
        }
        pp.wait_empty(b, use & 1);
#pragma unroll 1
        for (int w = 0; w < 2; ++w) {
          if (w) pp.unpark(1, v);
          scat(w);
        }
        pp.local_done(b);
      } else {
        if (we) pp.wait_empty(b, use & 1);
        scat(u);
      }
    }
  };
  auto phaseA = [&](int64_t sig, int b, uint32_t use, int64_t nsig) {
#if SA_K64_UNROLL_A
#pragma unroll
#endif
    for (int u = 0; u < TPG; ++u)
      tileA(std::integral_constant<int, 0>{}, sig, u, b, use, u == 0,
            u + 1 < TPG ? sig : (nsig < batch ? nsig : (int64_t)-1), u + 1 < TPG ? u + 1 : 0);
    pp.local_done(b);
  };

  auto phaseB_s = [&](auto S_, int64_t sig, int b, uint32_t use) {
    constexpr bool S = decltype(S_)::value;  // storage in the L2 scratch
    C2 *inter = pp.share(b);
    C2 *ysig = y + sig * NN;
    pp.wait_full(b, use & 1);
    for (int u = 0; u < TPG; ++u) {
      const int tt = pp.gi + NG * u;
      V v[16];
      {  // round 1 (M2: g fastest): q = g + 16k ; stages 8..5
        const int lr = tt * TC + m2_cc;
        C2 *row = inter + lr * 256;
        const int sw = lr & 15;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = A::from(Pipe<T>::template ld<S>(&row[(m2_g + 16 * k) ^ sw]));
#pragma unroll
        for (int s = 8; s >= 5; --s) {
          const int hr = 1 << (s - 5), h = 1 << (s - 1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dif<T>(v[k], v[k + hr], twA[(h - 1) + m2_g + 16 * (k & (hr - 1))]);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) Pipe<T>::template st<S>(&row[(m2_g + 16 * k) ^ sw], A::to(v[k]));
      }
      group_sync(gbar, GT);
      {  // round 2 (M1: cc fastest): q = 16g + k ; stages 4..2 + 2-point ; bit-reversed store
        const int lr = tt * TC + m1_cc;
        const C2 *row = inter + lr * 256;
        const int sw = lr & 15;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = A::from(Pipe<T>::template ld<S>(&row[(m1_g * 16 + k) ^ sw]));
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
        const int cr = pp.rank * COLS + lr;
        const int rg = rev4(m1_g);
#pragma unroll
        for (int k = 0; k < 16; ++k) __stcs(&ysig[(crev4(k) * 16 + rg) * 256 + cr], A::to(v[k]));
      }
    }
  };

  auto phaseB = [&](int64_t sig, int b, uint32_t use) {
    if constexpr (P::L2S) {
      if (Pipe<T>::in_l2(b)) {
        phaseB_s(std::true_type{}, sig, b, use);
        return;
      }
    }
    phaseB_s(std::false_type{}, sig, b, use);
  };

  if constexpr (P::PARK_DIF) {
    pp.run_park(&tmx, batch, tileA, phaseB);
  } else {
    pp.run(&tmx, batch, phaseA, phaseB);
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
  const bool wx = SA_K64_WX && std::is_same<T, float>::value && P::TC == 16 && variant == SA_DIT;
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   wx ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    sa_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SA_ERR_CUDA;
  }
  auto kern = variant == SA_DIT ? k_nlfft64k_dit<T> : k_nlfft64k_dif<T>;
  // per device and variant, once: function attributes and the resident cluster count
  static int cached_clusters[2][64] = {};
  int dev = 0, sms = 148;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  const int vi = variant == SA_DIT ? 0 : 1;
  const bool cached = dev < 64 && cached_clusters[vi][dev] > 0;
  if (!cached) {
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
    if (P::CL > 8) SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
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
  int max_clusters = cached ? cached_clusters[vi][dev] : 0;
  if (!cached) {
    cfg.gridDim = dim3(P::CL * (sms / P::CL));
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
      cudaGetLastError();
      max_clusters = sms / P::CL;
    }
    if (dev < 64) cached_clusters[vi][dev] = max_clusters;
  }
  int64_t ncl = std::min<int64_t>(batch, max_clusters);
  cfg.gridDim = dim3((unsigned)(ncl * P::CL));
  typename P::C2 *scratch = nullptr;  // L2S: one signal's node storage per cluster (L2-resident)
  if (P::L2S) {
    const int rc_ = sa_scratch_alloc((void **)&scratch, (size_t)ncl * NN * sizeof(typename P::C2), s);
    if (rc_ != SA_OK) return rc_;
  }
  SA_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, map, (typename P::C2 *)y, batch,
                                 (const typename P::C4 *)tw->stage,
                                 (const typename P::C2 *)tw->stage2, (T)gain, (int)(gain != 1.0), scratch));
  if (scratch) SA_CUDA_TRY(cudaFreeAsync(scratch, s));
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
