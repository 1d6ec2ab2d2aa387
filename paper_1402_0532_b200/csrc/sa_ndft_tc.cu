// sa_ndft_tc.cu -- fast-mode NDFT (transforms.py:223-251, regrouped) on the
// 5th-generation tensor cores: tcgen05.mma with TMEM accumulators, TMA-loaded
// twiddle operands and CUDA-core warps that build the signal operand in smem.
//
// Fast mode already evaluates every complex ⊙ as four exact sign products
// (sa_ndft.cu):
//   Re X_k = Σ_n sgn(xr) Wr + sgn(Wr) xr − sgn(xi) Wi − sgn(Wi) xi
//   Im X_k = Σ_n sgn(xr) Wi + sgn(Wi) xr + sgn(xi) Wr + sgn(Wr) xi ,  W = W^(kn mod N)
// which is one real GEMM per batch of vectors, D[v, o] = Σ_K A[v, K] B[o, K], with
// o = 2k + (re|im) (so D rows are complex64 spectra as stored) and K = 2n + (re|im):
//   D = S · Wv^T + X · sgn(Wv)^T,   S = sgn(x) (exact in bf16),  Wv = [[Wr, −Wi], [Wi, Wr]].
// The non-sign operands are split into two bf16 terms (Wv = W0 + W1, x = X0 + X1,
// each residual exact in fp32), so every product the tensor core forms is a
// sign times a 16-bit-mantissa piece, and the four GEMM terms
//   S·W0 + S·W1 + X0·sgn(Wv) + X1·sgn(Wv)
// accumulate in fp32 in TMEM.  Error vs the fp64 oracle: ≤ 2^-17 relative per
// term from the splits plus fp32 accumulation (tests: ≤ 1e-4 of ‖y‖₁, the
// north-star fp32 bound; measured 8.2e-7 on C2).  Multiplication-free in the ⊙ sense:
// one factor of every product is a sign.
//
// Kernel (persistent, 1 CTA per SM, 448 threads, CTA pairs: cluster of 2):
//   warp 0      TMA producer: this CTA's 128 rows of the W0 / W1 / sgn(Wv) tiles
//               (256 outputs x 16 samples per pair), completing on the leader's barrier
//   warp 1      TMEM allocator; in the leader CTA the single-thread MMA issuer:
//               tcgen05.mma.cta_group::2, M = 256 (128 vectors per CTA), N = 256, K = 16
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> fp32 rows of y
// A tile is 256 vectors x 512 outputs (two N = 256 MMAs per A tile, the whole of
// TMEM as one accumulator) when 2n % 512 == 0, else 256 outputs with two
// double-buffered accumulators.
//   warps 6-13  converters: x (c64, gain applied) -> S, X0, X1 bf16 tiles in the
//               SWIZZLE_64B K-major layout, fence.proxy.async, arrive on the leader
// Three smem slots of 72 KB per CTA (3 A tiles of 8 KB + 3 x 2 half-B tiles of 8 KB).
// Measured C2 (65536 x 1024 c64): 1.34 ms = 1.64 PFLOP/s of bf16 MMA (256-output
// tiles: 1.59 ms).  Dead ends: single-CTA M = 128 (1.71 ms),
// TMA-staged x (1.73-1.76 ms: fewer slots fit), 16 converter warps (1.61 ms),
// cluster-scope release/acquire on the pair barriers (MEMBAR.GPU per arrive: 2.8 ms).
#include <cuda.h>

#include <map>
#include <tuple>
#include <cudaTypedefs.h>

#include <mutex>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

constexpr int BM = 128;          // vectors per CTA per tile (TMEM lanes)
constexpr int BN = 256;          // outputs per MMA (128 bins x {re, im}; TMEM columns)
constexpr int KC = 16;           // samples per slot
constexpr int KS = 2 * KC;       // bf16 per operand row per slot = 64 B (SWIZZLE_64B)
constexpr int A_TILE = BM * KS * 2;  // 8 KB
#ifndef SA_TC_CONV_WARPS
#define SA_TC_CONV_WARPS 8
#endif
constexpr int CONV_WARPS = SA_TC_CONV_WARPS;
constexpr int CROWS = CONV_WARPS * 4;   // rows covered per pass (8 threads per row)
constexpr int RPT = BM / CROWS;         // rows per converter thread
constexpr int THREADS = 32 * (6 + CONV_WARPS);
constexpr int TMEM_COLS = 512;   // all of TMEM: 512 / TN accumulators of TN columns

// CG = CTAs per MMA (tcgen05 cta_group).  CG = 2: a CTA pair (cluster of 2) issues
// M = 256 MMAs from the leader; each CTA holds its 128 vector rows of A and half
// (128 rows) of every twiddle tile, so each SM streams half the B bytes.
// TN = outputs per tile (256 or 512): a 512-output tile issues two N = 256 MMAs per
// A tile, so each converted x tile feeds twice the outputs (half the x loads and
// conversions per step) at the price of one TMEM accumulator instead of two.
template <int CG, int TN> struct TcCfg {
  static constexpr int NH = TN / BN;                  // N = 256 halves per tile
  static constexpr int BROWS = BN / CG;               // twiddle rows per CTA per half
  static constexpr int B_TILE = NH * BROWS * KS * 2;  // per piece: 16 KB (CG 1) / 8 KB (CG 2) per half
  static constexpr int SLOT = 3 * A_TILE + 3 * B_TILE;
  static constexpr int NSLOT = (227 * 1024 - 2048) / SLOT < 4 ? (227 * 1024 - 2048) / SLOT : 4;
  static constexpr int NACC = TMEM_COLS / TN;
  static constexpr int SMEM = NSLOT * SLOT + 1024 + 256;
  // instruction descriptor: kind::f16, A = B = bf16, D = f32, both K-major, M = 128 CG, N = 256
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)((BM * CG) >> 4) << 24);
};

// smem matrix descriptor, K-major SWIZZLE_64B: rows of 64 B, 8-row atoms 512 B apart
SA_HD uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

SA_HD void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SA_HD void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// MMA completion -> mbarrier (CG 2: the barrier at the same offset in both CTAs)
template <int CG> SA_HD void tc_commit(uint64_t *bar) {
  if (CG == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     sa_smem_u32(bar))
                 : "memory");
  else
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            sa_smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
template <int CG> SA_HD void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  if (CG == 1)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(TcCfg<1, 256>::IDESC), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(TcCfg<2, 256>::IDESC), "r"(acc)
        : "memory");
}
SA_HD void mbar_init(uint64_t *bar, uint32_t count) { sa_mbar_init(bar, count); }
// arrive on a barrier given by its shared::cluster address (own or the leader's)
SA_HD void mbar_arrive_cl(uint32_t cl_addr) {
  // default .release.cta semantics, as CUTLASS's ClusterBarrier::arrive(cta_id): the
  // .cluster-scope form costs a MEMBAR.GPU per arrive (measured: 2.8 vs 1.7 ms)
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
// twiddle operand tiles are re-read by every vector tile: keep them in L2 (evict_last)
SA_HD void tma_load_2d_cg2(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t lead_bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(lead_bar), "l"(pol)
      : "memory");
}
SA_HD uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SA_HD uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SA_HD void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

SA_HD uint32_t bf2(float hi, float lo) {  // {lo -> bits 0..15, hi -> bits 16..31}, RN
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

#define SA_LD32(v, taddr)                                                                                  \
  asm volatile(                                                                                            \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"     \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                           \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),           \
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),         \
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),         \
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                              \
      : "r"(taddr))

template <int CG, int TN>
__global__ void __launch_bounds__(THREADS, 1)
    k_ndft_tc(const __grid_constant__ CUtensorMap wmap, const float4 *__restrict__ x, float *__restrict__ y,
              int64_t batch, int n, float gain, int use_gain) {
  using C = TcCfg<CG, TN>;
  constexpr int NH = C::NH, NACC = C::NACC;
  constexpr int NSLOT = C::NSLOT, SLOT = C::SLOT, B_TILE = C::B_TILE;
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + NSLOT * SLOT);
  uint64_t *empty = full + NSLOT;
  uint64_t *tfull = empty + NSLOT;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = (uint32_t *)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 1 ? 0 : cluster_rank();
  const int64_t cl = blockIdx.x / CG, ncl = gridDim.x / CG;
  const int ot_count = (2 * n) / TN;
  const int64_t vt_count = (batch + BM * CG - 1) / (BM * CG);
  const int64_t ntiles = vt_count * ot_count;
  const int kslots = n / KC;
  // the leader CTA's full / tempty barriers as shared::cluster addresses
  auto lead = [&](uint64_t *bar) { return CG == 1 ? sa_smem_u32(bar) : sa_mapa(sa_smem_u32(bar), 0); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&full[s], 1 + CG * CONV_WARPS);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * CG);
    }
    sa_fence_mbar_init();
  }
  if (warp == 1) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       sa_smem_u32(tmem_holder)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       sa_smem_u32(tmem_holder)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (CG == 1) __syncthreads();
  else cluster_sync_all();  // barrier inits + TMEM allocation visible pair-wide
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // this CTA's slots: it -> (tile cl + (it / kslots) ncl, K chunk it % kslots)
  const int64_t my_tiles = cl < ntiles ? (ntiles - 1 - cl) / ncl + 1 : 0;
  const int64_t total = my_tiles * kslots;

  if (warp == 0) {
    // ---- TMA producer: this CTA's rows of the twiddle operand tiles ----
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&wmap) : "memory");
      const uint64_t wpol = l2_policy_evict_last();
      for (int64_t it = 0; it < total; ++it) {
        const int64_t lt = it / kslots;
        const int kc = (int)(it - lt * kslots);
        const int o0 = (int)((cl + lt * ncl) % ot_count) * TN + (int)rank * C::BROWS;
        const int s = (int)(it % NSLOT);
        sa_mbar_wait(&empty[s], ((it / NSLOT) & 1) ^ 1);
        unsigned char *b = smem + s * SLOT + 3 * A_TILE;
        if (rank == 0) sa_mbar_expect_tx(&full[s], CG * 3 * B_TILE);
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int hh = 0; hh < NH; ++hh) {
            unsigned char *dst = b + p * B_TILE + hh * C::BROWS * KS * 2;
            const int row = p * 2 * n + o0 + hh * BN;
            if (CG == 1) sa_tma_load_2d(dst, &wmap, kc * KS, row, &full[s]);
            else tma_load_2d_cg2(sa_smem_u32(dst), &wmap, kc * KS, row, lead(&full[s]), wpol);
          }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (the leader CTA) ----
    if (lane == 0 && rank == 0) {
      uint32_t it = 0, lt = 0;
      for (int64_t t = cl; t < ntiles; t += ncl, ++lt) {
        const uint32_t acc = lt % NACC;
        sa_mbar_wait(&tempty[acc], ((lt / NACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * TN;
        for (int kc = 0; kc < kslots; ++kc, ++it) {
          const int s = it % NSLOT;
          sa_mbar_wait(&full[s], (it / NSLOT) & 1);
          tc_fence_after();
          const uint32_t base = sa_smem_u32(smem + s * SLOT);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t off = ks * 32;  // 16 bf16 along K inside the 64-B swizzled row
            const uint64_t aS = sdesc(base + off), aX0 = sdesc(base + A_TILE + off),
                           aX1 = sdesc(base + 2 * A_TILE + off);
#pragma unroll
            for (int hh = 0; hh < NH; ++hh) {
              const uint32_t bb = base + 3 * A_TILE + hh * C::BROWS * KS * 2 + off;
              const uint64_t bW0 = sdesc(bb), bW1 = sdesc(bb + B_TILE), bWs = sdesc(bb + 2 * B_TILE);
              const uint32_t dh = d + hh * BN;
              tc_mma<CG>(dh, aS, bW0, (kc | ks) != 0);
              tc_mma<CG>(dh, aS, bW1, 1);
              tc_mma<CG>(dh, aX0, bWs, 1);
              tc_mma<CG>(dh, aX1, bWs, 1);
            }
          }
          tc_commit<CG>(&empty[s]);
        }
        tc_commit<CG>(&tfull[acc]);
      }
    }
  } else if (warp < 6) {
    // ---- epilogue: this CTA's 128 TMEM lanes -> y ----
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    uint32_t lt = 0;
    for (int64_t t = cl; t < ntiles; t += ncl, ++lt) {
      const uint32_t acc = lt % NACC;
      const int64_t v = (t / ot_count) * (BM * CG) + rank * BM + q * 32 + lane;
      const int o0 = (int)(t % ot_count) * TN;
      sa_mbar_wait(&tfull[acc], (lt / NACC) & 1);
      tc_fence_after();
      float4 *dst = (float4 *)(y + v * 2 * n + o0);
#pragma unroll 1
      for (int c = 0; c < TN / 32; ++c) {
        uint32_t r[32];
        SA_LD32(r, tmem + ((uint32_t)(q * 32) << 16) + acc * TN + c * 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v < batch) {
#pragma unroll
          for (int j = 0; j < 8; ++j)  // streaming stores (evict-first): keep x, re-read by the
            __stcs(&dst[c * 8 + j],      // other output tiles of this vector tile, in L2
                   make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cl(lead(&tempty[acc]));
    }
  } else {
    // ---- converters: x -> S, X0, X1 (bf16, SWIZZLE_64B K-major) ----
    // Each thread owns sample pair h of rows r0 + 32 i.  x for slot it+3 is in
    // flight (three register sets) while slot it is converted.  Loads are
    // unconditional (row and slot clamped) so no select waits on them; rows
    // >= batch convert a copy of the last row, whose outputs are never stored.
    const int ct = threadIdx.x - 6 * 32;  // 0..32 CONV_WARPS - 1
    const int h = ct & 7;                 // sample pair 2h, 2h+1 of the slot
    const int r0 = ct >> 3;               // rows r0 + CROWS i
    const uint32_t sbase = sa_smem_u32(smem);
    auto load = [&](float4(&b)[RPT], int64_t it) {
      if (it >= total) it = total > 0 ? total - 1 : 0;
      const int64_t lt = it / kslots;
      const int kc = (int)(it - lt * kslots);
      const int64_t vbase = ((cl + lt * ncl) / ot_count) * (BM * CG) + rank * BM;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t v = vbase + r0 + CROWS * i;
        b[i] = __ldg(&x[((v < batch ? v : batch - 1) * n + (int64_t)kc * KC) / 2 + h]);
      }
    };
    auto convert = [&](const float4(&b)[RPT], int64_t it) {
      const int s = (int)(it % NSLOT);
      sa_mbar_wait(&empty[s], ((it / NSLOT) & 1) ^ 1);
      const uint32_t a = sbase + s * SLOT;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = r0 + CROWS * i;
        float4 f = b[i];
        if (use_gain) f = make_float4(sa_mul(gain, f.x), sa_mul(gain, f.y), sa_mul(gain, f.z), sa_mul(gain, f.w));
        const uint32_t s01 = bf2(sa_sgn(f.y), sa_sgn(f.x)), s23 = bf2(sa_sgn(f.w), sa_sgn(f.z));
        const uint32_t h01 = bf2(f.y, f.x), h23 = bf2(f.w, f.z);
        const float e0 = sa_sub(f.x, __uint_as_float(h01 << 16)), e1 = sa_sub(f.y, __uint_as_float(h01 & 0xFFFF0000u));
        const float e2 = sa_sub(f.z, __uint_as_float(h23 << 16)), e3 = sa_sub(f.w, __uint_as_float(h23 & 0xFFFF0000u));
        const uint32_t l01 = bf2(e1, e0), l23 = bf2(e3, e2);
        const uint32_t off = a + r * 64 + ((((h >> 1) ^ (r >> 1)) & 3) << 4) + (h & 1) * 8;
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(off), "r"(s01), "r"(s23) : "memory");
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(off + A_TILE), "r"(h01), "r"(h23) : "memory");
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(off + 2 * A_TILE), "r"(l01), "r"(l23) : "memory");
      }
      sa_fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05.mma
      __syncwarp();
      if (lane == 0) mbar_arrive_cl(lead(&full[s]));
    };
    float4 b0[RPT], b1[RPT], b2[RPT];
    load(b0, 0);
    load(b1, 1);
    load(b2, 2);
    for (int64_t it = 0; it < total; it += 3) {
      convert(b0, it);
      load(b0, it + 3);
      if (it + 1 < total) {
        convert(b1, it + 1);
        load(b1, it + 4);
      }
      if (it + 2 < total) {
        convert(b2, it + 2);
        load(b2, it + 5);
      }
    }
  }

  tc_fence_before();
  if (CG == 1) __syncthreads();
  else cluster_sync_all();  // no CTA leaves while its pair may still signal it
  if (warp == 1) {
    tc_fence_after();
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

// Twiddle operands [W0; W1; sgn(Wv)], each 2n x 2n bf16, row o = 2k + c_out, column K = 2m + c_in:
// Wv = [[Wr, -Wi], [Wi, Wr]] of W = raw[(k m) mod n] (the fp32 table, as the FFMA2 kernels use).
__global__ void k_tc_wbuild(const float2 *__restrict__ raw, int n, uint16_t *__restrict__ w) {
  const int64_t nn = 2LL * n, total = nn * nn;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / nn, kk = i % nn;
    const int64_t k = o >> 1, m = kk >> 1;
    const int co = (int)(o & 1), ci = (int)(kk & 1);
    const float2 tw = raw[(k * m) % n];
    const float val = co == ci ? tw.x : (co == 0 ? -tw.y : tw.y);
    const uint32_t hi = bf2(0.f, val);
    const uint32_t lo = bf2(0.f, sa_sub(val, __uint_as_float(hi << 16)));
    const uint32_t sg = bf2(0.f, sa_sgn(val));
    w[i] = (uint16_t)hi;
    w[total + i] = (uint16_t)lo;
    w[2 * total + i] = (uint16_t)sg;
  }
}

std::mutex g_tc_mutex;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_tc() {
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

// Tensor maps of the twiddle operands, encoded once per (operand buffer, n, box rows).
std::map<std::tuple<const void *, int64_t, int>, CUtensorMap> g_tc_maps;

template <int CG, int TN>
int launch_tc(const void *x, void *y, int64_t batch, int64_t n, SaTwiddles *tw, double gain, cudaStream_t s) {
  using Cf = TcCfg<CG, TN>;
  CUtensorMap map;
  {
    std::lock_guard<std::mutex> g(g_tc_mutex);
    const auto key = std::make_tuple((const void *)tw->tcw, n, (int)Cf::BROWS);
    auto it = g_tc_maps.find(key);
    if (it == g_tc_maps.end()) {
      auto enc = encode_fn_tc();
      cuuint64_t dims[2] = {(cuuint64_t)(2 * n), (cuuint64_t)(6 * n)};
      cuuint64_t strides[1] = {(cuuint64_t)(2 * n * 2)};
      cuuint32_t box[2] = {(cuuint32_t)KS, (cuuint32_t)Cf::BROWS};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tw->tcw, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        sa_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return SA_ERR_CUDA;
      }
      g_tc_maps.emplace(key, map);
    } else {
      map = it->second;
    }
  }
  static bool smem_set[64] = {};
  int dev = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64 || !smem_set[dev]) {
    SA_CUDA_TRY(cudaFuncSetAttribute(k_ndft_tc<CG, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    if (dev < 64) smem_set[dev] = true;
  }
  int sms = 0;
  SA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t ntiles = ((batch + BM * CG - 1) / (BM * CG)) * ((2 * n) / TN);
  const int64_t units = ntiles < sms / CG ? ntiles : sms / CG;  // persistent: one CTA group per SM group
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * CG));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_ndft_tc<CG, TN>, map, (const float4 *)x, (float *)y, batch, (int)n,
                                 (float)gain, (int)(gain != 1.0)));
  SA_LAUNCH_CHECK();
  return SA_OK;
}

}  // namespace

bool sa_ndft_tc_supported(int dtype, int64_t n) {
  return dtype == SA_C64 && n >= 128 && n <= 4096 && n % 128 == 0;
}

int64_t sa_ndft_tc_wbytes(int64_t n) { return 3 * (2 * n) * (2 * n) * 2; }

int sa_launch_ndft_tc(const void *x, void *y, int64_t batch, int64_t n, const SaTwiddles *tw_c, double gain,
                      cudaStream_t s) {
  if (!sa_ndft_tc_supported(tw_c->dtype, n)) return SA_ERR_UNSUPPORTED;
  if (((uintptr_t)x | (uintptr_t)y) & 15) return SA_ERR_UNSUPPORTED;  // TMA / float4 epilogue alignment
  if (batch == 0) return SA_OK;
  SaTwiddles *tw = const_cast<SaTwiddles *>(tw_c);
  {
    // operands built once per twiddle set, stream-ordered (no host sync): on the
    // first caller's stream, with an event every later launch's stream waits on
    std::lock_guard<std::mutex> g(g_tc_mutex);
    if (!tw->tcw) {
      void *w = nullptr;
      cudaEvent_t ev = nullptr;
      SA_CUDA_TRY(cudaMalloc(&w, sa_ndft_tc_wbytes(n)));
      k_tc_wbuild<<<1184, 256, 0, s>>>((const float2 *)tw->raw, (int)n, (uint16_t *)w);
      SA_LAUNCH_CHECK();
      SA_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      SA_CUDA_TRY(cudaEventRecord(ev, s));
      tw->tcw = w;
      tw->tcw_ready = ev;
    }
  }
  if (tw->tcw_ready) SA_CUDA_TRY(cudaStreamWaitEvent(s, (cudaEvent_t)tw->tcw_ready, 0));
  auto enc = encode_fn_tc();
  if (!enc) {
    sa_set_error("cuTensorMapEncodeTiled unavailable");
    return SA_ERR_CUDA;
  }
#ifndef SA_NDFT_TC_CG
#define SA_NDFT_TC_CG 2
#endif
  constexpr int CG = SA_NDFT_TC_CG;
#ifndef SA_NDFT_TC_TN
#define SA_NDFT_TC_TN 512
#endif
  return (2 * n) % SA_NDFT_TC_TN == 0 ? launch_tc<CG, SA_NDFT_TC_TN>(x, y, batch, n, tw, gain, s)
                                      : launch_tc<CG, 256>(x, y, batch, n, tw, gain, s);
}

