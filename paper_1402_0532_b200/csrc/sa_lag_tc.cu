// sa_lag_tc.cu -- block-integrated ⊙ lag products (the range-Doppler map's lag
// stage, sa_ambiguity.cu) on the tcgen05 tensor cores, fast mode, complex64.
//
//   z_l[q] = Σ_{t<T} s[qT+t] ⊙ c[qT+t-l],   c = conj(ref) (ref[<0] = 0)
//
// Fast mode evaluates each ⊙ through the sign-split identity (sa_ambiguity.cu):
//   Re = Σ sgn(sr) cr + sr sgn(cr) − sgn(si) ci − si sgn(ci)
//   Im = Σ sgn(si) cr + si sgn(cr) + sgn(sr) ci + sr sgn(ci)
// so for one block q every real term is a correlation Σ_t a[t] b[t − l].  With
// lag l = lbase + 8 l1 + l0 (l1 < 128, l0 < 8) and u = t − 8 l1 it is a GEMM
//   Z[l1, l0] = Σ_u A[l1, u] B[l0, u],   A[l1, u] = a[u + 8 l1],  B[l0, u] = b[u − l0]
// over u in [−1024, T).  A is a Hankel matrix: in the K-major no-swizzle UMMA
// layout the 8 rows of a core matrix sit 16 B (= 8 bf16 = one l1 step) apart, so
// the descriptor (LBO 16 B, SBO 128 B) reads A straight out of one zero-padded
// linear array per operand kind -- nothing is materialised.  B (8 shifts x 2
// components x pieces) is built per K chunk of 128 u.  As in sa_ndft_tc.cu the
// non-sign operands are split in two bf16 pieces (hi + lo) and one factor of
// every product is a sign; accumulation is fp32 in TMEM.
//
// Per K step (16 u) six MMAs, M = 128 (l1) x K = 16:
//   D1 (32 cols: Re_hi, Im_hi, Re_lo, Im_lo x 8 l0) += sgn(sr) x B1 + sgn(si) x B2   (N = 32)
//   D2 (16 cols: Re, Im x 8 l0)                    += sr_hi x B3 + sr_lo x B3 + si_hi x B4 + si_lo x B4
//   B1 = [cr_hi, ci_hi, cr_lo, ci_lo], B2 = [−ci_hi, cr_hi, −ci_lo, cr_lo],
//   B3 = [sgn cr, sgn ci], B4 = [−sgn ci, sgn cr]   (each block of 8 rows = l0 0..7)
// Epilogue: Re = D1[l0] + D1[16+l0] + D2[l0], Im = D1[8+l0] + D1[24+l0] + D2[8+l0].
//
// One CTA per integration block q (256 threads, 2 CTAs per SM), looping over
// groups of 1024 lags aligned to lag multiples of 16; rows outside the call's
// lag range are dropped.
#include <cuda.h>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

// A lag group is MR rows l1 (MMA M = 128, or 64 for short lag ranges: half the
// A-operand bytes per MMA, twice the groups stacked along N) x 8 l0: 8 MR lags;
// the A arrays carry 8 MR zeros on each side (u >= -8 MR).
constexpr int NKIND = 6;         // A kinds: sgn sr, sgn si, sr_hi, sr_lo, si_hi, si_lo
constexpr int BROWS = 96;        // B rows per lag group: B1 32 + B2 32 + B3 16 + B4 16
constexpr int B_BYTES = BROWS * 128 * 2;  // 24 KB per buffer: G groups x 128 / G u per K chunk
constexpr int BUILDERS = 256;    // warps 0-7 build the operands (warps 0-3 also drain TMEM)
constexpr int THREADS = BUILDERS + 32;  // warp 8 issues the MMAs

__host__ __device__ inline int a_len(int tb, int mr) { return tb + 16 * mr; }  // u + 8 l1 in [-8 MR, T + 8 MR), padded
__host__ __device__ inline size_t a_bytes(int tb, int mr) { return ((size_t)NKIND * a_len(tb, mr) * 2 + 1023) & ~(size_t)1023; }
__host__ __device__ inline size_t smem_bytes(int tb, int mr) { return a_bytes(tb, mr) + 2 * B_BYTES + 1024 + 64; }
constexpr int tmem_cols(int g) { return g == 1 ? 64 : (g == 2 ? 128 : 256); }  // >= 48 G, power of 2

// instruction descriptor: kind::f16, bf16 x bf16 -> f32, K-major, M = mr, N = n
constexpr uint32_t idesc(int n, int mr) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(mr >> 4) << 24);
}
// K-major, no swizzle: core matrices of 8 rows x 16 B; LBO = next 8 K elements, SBO = next 8 rows
SA_HD uint64_t sdesc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46);
}
SA_HD void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
SA_HD void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   sa_smem_u32(bar))
               : "memory");
}
SA_HD void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SA_HD void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SA_HD uint32_t bf2(float hi, float lo) {  // {lo -> bits 0..15, hi -> bits 16..31}, RN
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

#define SA_LD16(v, taddr)                                                                                  \
  asm volatile(                                                                                            \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"    \
      " [%16];"                                                                                            \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),           \
        "=r"(v[15])                                                                                        \
      : "r"(taddr))

// the 8 conj-ref values a B-builder thread needs: c[g0 .. g0+7] (0 before the signal start)
// and from ref_len on: lags below the call's range (groups start at multiples of 16)
// reach past the end, and 0 x NaN in the MMA would poison the kept rows
SA_HD void load_c(float2 (&cv)[8], const float2 *__restrict__ ref, int64_t g0, int64_t ref_len, float csign) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int64_t g = g0 + e;
    float2 v = (g >= 0 && g < ref_len) ? __ldg(&ref[g]) : make_float2(0.f, 0.f);
    cv[e] = make_float2(v.x, csign * v.y);
  }
}

// Where row `lag` of z goes: the local (l_count x m) z, or -- block-sharded
// multi-GPU maps (sharded.py) -- the z rows of the rank that owns the lag
// (shard_rows partition: the first `extra` owners hold base + 1 rows), written
// over NVLink/NVSwitch peer memory.
// Blocked layout (sa_doppler.cu): tiles of 16 consecutive lags counted from the
// call's 16-aligned base lalign; element q of a tile's 16 rows is one 128-B line
//   zb[(k * m + q) * 16 + j] = z[lalign + 16 k + j][q]
// Peer owners then hold `base` rows each (16-aligned shards, l0 = 0, extra = 0).
struct LagDst {
  float2 *const *ptr;  // device array of per-owner row-block bases (null: local z)
  int64_t base, extra;
  SA_HD float2 *row(float2 *z, int64_t lag, int64_t m, int64_t q) const {
    if (!ptr) return z + lag * m + q;
    const int64_t big = extra * (base + 1);
    const int64_t o = lag < big ? lag / (base + 1) : extra + (lag - big) / base;
    const int64_t first = o * base + (o < extra ? o : extra);
    return ptr[o] + (lag - first) * m + q;
  }
  SA_HD float2 *line(float2 *z, int64_t k, int64_t m, int64_t q) const {
    if (!ptr) return z + (k * m + q) * 16;
    const int64_t o = (16 * k) / base;
    return ptr[o] + ((k - o * (base >> 4)) * m + q) * 16;
  }
};

// G lag groups share each A read (one pass): the MMAs widen to N = 32 G / 16 G.
// MR = 64: accumulator row r sits in TMEM lane 32 (r / 16) + r % 16 (the lower
// half of each warp's sub-partition; measured, tools/probes/probe_m64.cu).
template <int G, bool BLK, int MR>
__global__ void __launch_bounds__(THREADS, 2)
    k_lag_tc(const float2 *__restrict__ surv, const float2 *__restrict__ ref, int64_t ref_len, int64_t l0g, int64_t l_count,
             int64_t m, int tb, float csign, float2 *__restrict__ z, int64_t q0, LagDst dst) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int LGRP = 8 * MR, PAD = 8 * MR;
  const int al = a_len(tb, MR);
  uint16_t *A = (uint16_t *)smem;                      // NKIND x al bf16
  unsigned char *Bb = smem + a_bytes(tb, MR);          // 2 x B_BYTES (1024-aligned)
  uint64_t *bar = (uint64_t *)(Bb + 2 * B_BYTES);      // "empty": MMAs that read B buffer b are done
  uint64_t *full = bar + 2;                            // B buffer b built (one arrive per builder warp)
  uint64_t *dempty = full + 2;                         // TMEM drained by the epilogue warps
  uint32_t *tmem_holder = (uint32_t *)(dempty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t q = q0 + blockIdx.x;
  constexpr int KCH = 128 / G;          // u per K chunk (B buffer stays 24 KB)
  constexpr int SBO = (KCH / 8) * 128;    // bytes per 8-row block of a B buffer
  constexpr int TMEM_COLS = tmem_cols(G);
  const int nch = (tb + PAD) / KCH;

  if (tid == 0) {
    sa_mbar_init(&bar[0], 1);
    sa_mbar_init(&bar[1], 1);
    sa_mbar_init(&full[0], BUILDERS / 32);
    sa_mbar_init(&full[1], BUILDERS / 32);
    sa_mbar_init(dempty, 4);
    sa_fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa_smem_u32(tmem_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // A: the surveillance block as six zero-padded linear bf16 arrays, a[t] at PAD + t
  for (int j = 2 * tid; j < al; j += 2 * THREADS) {  // (the MMA warp helps here)
    const int t = j - PAD;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t >= 0 && t < tb) v = __ldg((const float4 *)&surv[q * tb + t]);  // t even, tb even: 16-B aligned
    const uint32_t sr = bf2(sa_sgn(v.z), sa_sgn(v.x)), si = bf2(sa_sgn(v.w), sa_sgn(v.y));
    const uint32_t rh = bf2(v.z, v.x), ih = bf2(v.w, v.y);
    const uint32_t rl = bf2(sa_sub(v.z, __uint_as_float(rh & 0xFFFF0000u)), sa_sub(v.x, __uint_as_float(rh << 16)));
    const uint32_t il = bf2(sa_sub(v.w, __uint_as_float(ih & 0xFFFF0000u)), sa_sub(v.y, __uint_as_float(ih << 16)));
    const uint32_t w[NKIND] = {sr, si, rh, rl, ih, il};
#pragma unroll
    for (int k = 0; k < NKIND; ++k) *(uint32_t *)&A[(size_t)k * al + j] = w[k];
  }
  sa_fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t abase = sa_smem_u32(A), bbase = sa_smem_u32(Bb);

  // Groups start at lag multiples of 16, so every (lag, t) product lands in the
  // same row parity, column and K-step position whatever l0 the call starts at:
  // lag shards (sharded.py) reproduce the single-call rows bit for bit.
  const int64_t lalign = l0g - (l0g & 15);
  const int ngrp = (int)((l0g - lalign + l_count + LGRP - 1) / LGRP);
  const int npass = (ngrp + G - 1) / G;

  if (warp == BUILDERS / 32) {
    // ---- MMA issuer: one thread, six MMAs per 16 u, commit frees the B buffer ----
    if (lane == 0) {
      uint32_t cc = 0;
      for (int pi = 0; pi < npass; ++pi) {
        if (pi > 0) sa_mbar_wait(dempty, (pi - 1) & 1);  // epilogue has read the previous pass's D
        for (int ch = 0; ch < nch; ++ch, ++cc) {
          const int b = cc & 1;
          sa_mbar_wait(&full[b], (cc >> 1) & 1);
          fence_after();
          const uint32_t bb = bbase + b * B_BYTES;
#pragma unroll
          for (int ks = 0; ks < KCH / 16; ++ks) {
            const uint32_t ua = (uint32_t)(ch * KCH + ks * 16) * 2;  // byte offset of u0 + PAD in the A arrays
            const uint32_t bo = bb + ks * 256;                      // 16 u = two 128-B core columns
            const uint32_t acc = (ch | ks) != 0;
            const uint64_t b1 = sdesc_ns(bo, 128, SBO), b2 = sdesc_ns(bo + 4 * G * SBO, 128, SBO),
                           b3 = sdesc_ns(bo + 8 * G * SBO, 128, SBO), b4 = sdesc_ns(bo + 10 * G * SBO, 128, SBO);
            auto ad = [&](int k) { return sdesc_ns(abase + (uint32_t)k * al * 2 + ua, 16, 128); };
            mma(tmem, ad(0), b1, idesc(32 * G, MR), acc);
            mma(tmem, ad(1), b2, idesc(32 * G, MR), 1);
            mma(tmem + 32 * G, ad(2), b3, idesc(16 * G, MR), acc);
            mma(tmem + 32 * G, ad(3), b3, idesc(16 * G, MR), 1);
            mma(tmem + 32 * G, ad(4), b4, idesc(16 * G, MR), 1);
            mma(tmem + 32 * G, ad(5), b4, idesc(16 * G, MR), 1);
          }
          commit(&bar[b]);
        }
      }
    }
  } else {
    // ---- builders: thread (l0, octet of the chunk, group of the pass, half) ----
    const int bl0 = tid & 7, boct = (tid >> 3) % (KCH / 8), bg = ((tid >> 3) / (KCH / 8)) % G, bhalf = tid >> 7;
    uint32_t cc = 0;  // chunk counter across passes (B buffer = cc & 1)
    for (int pi = 0; pi < npass; ++pi) {
      const int64_t lpass = lalign + (int64_t)pi * G * LGRP;
      // c index of (u, l0) for this thread's group: q T - lbase + u - l0
      const int64_t cbase = q * tb - (lpass + (int64_t)bg * LGRP) - PAD - bl0 + boct * 8;
      float2 cv[8];
      load_c(cv, ref, cbase, ref_len, csign);
      for (int ch = 0; ch < nch; ++ch, ++cc) {
        const int b = cc & 1;
        if (cc >= 2) sa_mbar_wait(&bar[b], ((cc >> 1) - 1) & 1);  // MMAs that read this buffer are done
        // build chunk ch of B into buffer b: rows (block of 8 = one component, row = l0), octet boct
        {
          unsigned char *B = Bb + b * B_BYTES;
          float cr[8], ci[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) cr[e] = cv[e].x, ci[e] = cv[e].y;
          const uint32_t o = (uint32_t)boct * 128 + (uint32_t)bl0 * 16;  // (row l0, octet) inside an 8-row block
          // matrix at row offset mrow0 (B1 0, B2 32 G, B3 64 G, B4 80 G), this group's block blk
          auto put = [&](int mrow0, int gstride, int blk, const uint32_t(&w)[4]) {
            *(uint4 *)(B + (size_t)((mrow0 + bg * gstride) / 8 + blk) * SBO + o) = make_uint4(w[0], w[1], w[2], w[3]);
          };
          if (bhalf == 0) {
            uint32_t rh[4], rl[4], ihh[4], il[4], nih[4], nil[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              rh[e] = bf2(cr[2 * e + 1], cr[2 * e]);
              ihh[e] = bf2(ci[2 * e + 1], ci[2 * e]);
              rl[e] = bf2(sa_sub(cr[2 * e + 1], __uint_as_float(rh[e] & 0xFFFF0000u)),
                          sa_sub(cr[2 * e], __uint_as_float(rh[e] << 16)));
              il[e] = bf2(sa_sub(ci[2 * e + 1], __uint_as_float(ihh[e] & 0xFFFF0000u)),
                          sa_sub(ci[2 * e], __uint_as_float(ihh[e] << 16)));
              nih[e] = ihh[e] ^ 0x80008000u;  // exact negation of both bf16 halves
              nil[e] = il[e] ^ 0x80008000u;
            }
            put(0, 32, 0, rh);          // B1: cr_hi
            put(0, 32, 1, ihh);         //     ci_hi
            put(0, 32, 2, rl);          //     cr_lo
            put(0, 32, 3, il);          //     ci_lo
            put(32 * G, 32, 0, nih);    // B2: -ci_hi
            put(32 * G, 32, 1, rh);     //     cr_hi
            put(32 * G, 32, 2, nil);    //     -ci_lo
            put(32 * G, 32, 3, rl);     //     cr_lo
          } else {
            uint32_t sr[4], si[4], nsi[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              sr[e] = bf2(sa_sgn(cr[2 * e + 1]), sa_sgn(cr[2 * e]));
              si[e] = bf2(sa_sgn(ci[2 * e + 1]), sa_sgn(ci[2 * e]));
              nsi[e] = si[e] ^ 0x80008000u;
            }
            put(64 * G, 16, 0, sr);     // B3: sgn cr
            put(64 * G, 16, 1, si);     //     sgn ci
            put(80 * G, 16, 0, nsi);    // B4: -sgn ci
            put(80 * G, 16, 1, sr);     //     sgn cr
          }
        }
        if (ch + 1 < nch) load_c(cv, ref, cbase + (int64_t)(ch + 1) * KCH, ref_len, csign);  // next chunk's values
        sa_fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05.mma
        __syncwarp();
        if (lane == 0) sa_mbar_arrive_local(&full[b]);
      }
      // epilogue of this pass (warps 0-3): the last chunk's commit tracks all prior MMAs
      if (warp < 4) {
        const uint32_t last = cc - 1;
        sa_mbar_wait(&bar[last & 1], (last >> 1) & 1);
        fence_after();
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
        const int l1 = MR == 128 ? warp * 32 + lane : warp * 16 + (lane & 15);
        const bool live = MR == 128 || lane < 16;  // MR = 64: lanes 16-31 hold no rows
#pragma unroll 1
        for (int gs = 0; gs < G; ++gs) {
          uint32_t d1[16], d2[16], d3[16];
          SA_LD16(d1, ta + 32 * gs);
          SA_LD16(d2, ta + 32 * gs + 16);
          SA_LD16(d3, ta + 32 * G + 16 * gs);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float re[8], im[8];
#pragma unroll
          for (int l0 = 0; l0 < 8; ++l0) {
            re[l0] = (__uint_as_float(d1[l0]) + __uint_as_float(d2[l0])) + __uint_as_float(d3[l0]);
            im[l0] = (__uint_as_float(d1[8 + l0]) + __uint_as_float(d2[8 + l0])) + __uint_as_float(d3[8 + l0]);
          }
          const int64_t lagb = lpass + (int64_t)gs * LGRP + 8 * l1;  // absolute lag of re[0]
          if constexpr (!BLK) {
#pragma unroll
            for (int l0 = 0; l0 < 8; ++l0) {
              const int64_t lag = lagb + l0 - l0g;  // row of z
              if (live && lag >= 0 && lag < l_count) *dst.row(z, lag, m, q) = make_float2(re[l0], im[l0]);
            }
          } else {
            // lanes (2i, 2i+1) hold the 16 lags of tile k: swap halves so that every
            // store instruction writes one whole 32-B sector of the tile's 128-B line
            const int64_t k = (lagb - lalign) >> 4;
            const bool odd = l1 & 1;
            float4 c[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) c[i] = make_float4(re[2 * i], im[2 * i], re[2 * i + 1], im[2 * i + 1]);
            float4 snd[2] = {odd ? c[0] : c[1], odd ? c[2] : c[3]}, rcv[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              rcv[i].x = __shfl_xor_sync(0xffffffffu, snd[i].x, 1);
              rcv[i].y = __shfl_xor_sync(0xffffffffu, snd[i].y, 1);
              rcv[i].z = __shfl_xor_sync(0xffffffffu, snd[i].z, 1);
              rcv[i].w = __shfl_xor_sync(0xffffffffu, snd[i].w, 1);
            }
            const int64_t t0 = lalign + 16 * k;  // tile intersects the call's rows?
            if (live && t0 + 16 > l0g && t0 < l0g + l_count) {
              float4 *ln = reinterpret_cast<float4 *>(dst.line(z, k, m, q));
              if (!odd) {
                ln[0] = c[0];
                ln[2] = c[2];
                ln[4] = rcv[0];
                ln[6] = rcv[1];
              } else {
                ln[1] = rcv[0];
                ln[3] = rcv[1];
                ln[5] = c[1];
                ln[7] = c[3];
              }
            }
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) sa_mbar_arrive_local(dempty);
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

}  // namespace

bool sa_lag_tc_supported(int dtype, int64_t tb, int64_t m, const void *surv) {
  return dtype == SA_C64 && tb >= 128 && tb % 128 == 0 && tb <= 4096 && m <= 0x7fffffff &&
         ((uintptr_t)surv & 15) == 0;
}

int sa_launch_lag_tc(const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count, int64_t m,
                     int64_t tb, int conj, void *z, int blocked, cudaStream_t s) {
  return sa_launch_lag_tc_blocks(surv, ref, ref_len, l0, l_count, m, 0, m, tb, conj, z, nullptr, 0, 0, blocked, s);
}

template <int G, bool BLK, int MR>
int launch_g(const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, int64_t q0,
             int64_t q_count, int64_t tb, int conj, void *z, const LagDst &d, cudaStream_t s) {
  const size_t bytes = smem_bytes((int)tb, MR);
  static int smem_set[64] = {};  // largest smem size set per device
  int dev = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64 || smem_set[dev] < (int)bytes) {
    SA_CUDA_TRY(cudaFuncSetAttribute(k_lag_tc<G, BLK, MR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    if (dev < 64) smem_set[dev] = (int)bytes;
  }
  k_lag_tc<G, BLK, MR><<<(unsigned)q_count, THREADS, bytes, s>>>((const float2 *)surv, (const float2 *)ref, ref_len,
                                                                 l0, l_count, m, (int)tb, conj ? -1.f : 1.f,
                                                                 (float2 *)z, q0, d);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

// Lag-group shape of a call: rows per group MR and groups per pass G, from the
// smem-operand cost per block (A: 6 kinds x MR x 32 B per 16 u; B: 96 G rows x
// 32 B) against the tensor floor (N/2 cycles per M = 64/128, K = 16 MMA).
struct LagShape {
  int mr, g;
};
LagShape lag_shape(int64_t l0, int64_t l_count, int64_t tb) {
#ifdef SA_LAG_MR
  const int only = SA_LAG_MR;
#else
  const int only = 0;
#endif
  LagShape best{128, 1};
  double best_cost = 1e300;
  for (int mr : {64, 128}) {
    if (only && mr != only) continue;
    const int64_t ngrp = ((l0 & 15) + l_count + 8 * mr - 1) / (8 * mr);
    const int g = ngrp >= 3 ? 4 : (int)ngrp;
    const int64_t npass = (ngrp + g - 1) / g;
    const double smem_cyc = (6.0 * mr * 32 + 96.0 * g * 32) / 128.0, tc_cyc = 64.0 * g;
    const double cost = (double)npass * (double)(tb + 8 * mr) / 16.0 * (smem_cyc > tc_cyc ? smem_cyc : tc_cyc);
    if (cost < best_cost) best_cost = cost, best = {mr, g};
  }
  return best;
}

int sa_launch_lag_tc_blocks(const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count, int64_t m,
                            int64_t q0, int64_t q_count, int64_t tb, int conj, void *z, void *const *dst_rows,
                            int64_t rows_base, int64_t rows_extra, int blocked, cudaStream_t s) {
  if (l_count == 0 || q_count == 0) return SA_OK;
  if (sa_lag_i8_enabled()) {
    const int rc = sa_launch_lag_i8_blocks(surv, ref, ref_len, l0, l_count, m, q0, q_count, tb, conj, z, dst_rows,
                                           rows_base, rows_extra, blocked, s);
    if (rc != SA_ERR_UNSUPPORTED) return rc;
  }
  const LagShape sh = lag_shape(l0, l_count, tb);
  const LagDst d{(float2 *const *)dst_rows, rows_base, rows_extra};
#define SA_LAG_LAUNCH(G, MR)                                                                                     \
  return blocked ? launch_g<G, true, MR>(surv, ref, ref_len, l0, l_count, m, q0, q_count, tb, conj, z, d, s)    \
                 : launch_g<G, false, MR>(surv, ref, ref_len, l0, l_count, m, q0, q_count, tb, conj, z, d, s)
  if (sh.mr == 64) {
    if (sh.g == 4) SA_LAG_LAUNCH(4, 64);
    if (sh.g == 2) SA_LAG_LAUNCH(2, 64);
    SA_LAG_LAUNCH(1, 64);
  }
  if (sh.g == 4) SA_LAG_LAUNCH(4, 128);
  if (sh.g == 2) SA_LAG_LAUNCH(2, 128);
  SA_LAG_LAUNCH(1, 128);
#undef SA_LAG_LAUNCH
}
