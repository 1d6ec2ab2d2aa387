// sa_ndft_i8.cu -- the fast-mode NDFT (transforms.py:223-251, regrouped as in
// sa_ndft.cu) on the tcgen05 tensor cores in EXACT INTEGER arithmetic: an
// Ozaki-style split of both non-sign operands into int8 digits, int8 x int8 ->
// int32 MMAs (kind::i8), floating point only in the epilogue.  complex128 (ND = 2
// digit pairs, the fp64 bound) and complex64 (ND = 1, the fp32 bound).
//
// The regrouped sum is one real GEMM per batch (sa_ndft_tc.cu):
//   D[v, o] = Σ_K S[v,K] Wv[o,K] + X[v,K] sgn(Wv)[o,K],   S = sgn(x),  o = 2k+(re|im), K = 2n+(re|im)
// One factor of every product is a sign in {-1, 0, +1} -- exact in int8.  The
// other factor is split into 2 ND signed digits in mixed radix (127, 127, 128, 127):
//   Wv ~ d0/127 + d1/127^2 [+ d2/(127^2 128) + d3/(127^3 128)]    (|Wv| <= 1, |d0| <= 127, |d1..3| <= 64)
//   x' = x_v / 2^e_v   (per-vector exponent: max|x_v| < 2^e_v), digits alike
// (round-to-nearest digits; the residual after digit 2 ND is <= 2^-15 / 2^-29).
// Two digits 127 apart share one int32 accumulator by pairing the sign operand
// with 127 x sign (still int8):
//   accW_j = Σ (127 S) dW_2j + S dW_2j+1        accX_j = Σ dx_2j (127 sW) + dx_2j+1 sW
// all exact (|acc| < 2^26 at n <= 2048), and the epilogue forms
//   D = Σ_j accW_j c_j + 2^e_v Σ_j accX_j c_j,   c_0 = 1/127^2, c_1 = c_0/(128 127)
// (fp64 for complex128, fp32 for complex64).
// Error model: per output ~ sqrt(2n) 2^-(14 ND + 1) (1 + 2^e) against ||y||_1 ~ n sqrt(2n):
//   ND = 2: the fp64 bound 1e-9 with a wide margin;
//   ND = 1: the fp32 bound 1e-4 with a wide margin
// (tests/test_gpu_ndft_i8.py).  Smaller n runs the FFMA2 / DFMA fast kernels.
//
// Pipeline: the x digit prep (one pass over x: gain, per-vector exponent, the
// 2 + 2 ND int8 planes S, 127 S, digits) -- for complex64 with n <= 1024 done by
// prep warps INSIDE k_ndft_i8 (rows released per 128-vector block through a
// ready counter the producer acquires before its bulk copies), otherwise by
// k_i8_prep / k_i8_prep_w first -- then k_ndft_i8<ND>
// (persistent CTA pairs, cluster 2, tcgen05.mma.cta_group::2.kind::i8, M = 256
// vectors, N = 512 / (2 ND) outputs, K = 32; the 2 ND accumulators fill TMEM's 512
// columns).  Both operand sets are stored in HBM as "smem images": for each
// 128-vector block (or N/2-output block) and 64-K slot the planes' tiles are
// contiguous and already SWIZZLE_64B-permuted, so one bulk copy per side fills a
// slot -- 128-B requests instead of the 64-B rows a 2-D TMA box would issue (the
// request rate bounded the first version).  Three slots per CTA.  Warp 0
// produces, warp 2 + EPI relays each CTA's slot completion to the leader, warp 1
// issues the MMAs (leader CTA), EPI epilogue warps (two per TMEM lane quarter,
// half the columns each) drain TMEM into rows of y.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <math_constants.h>
#include <mutex>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

constexpr int BM = 128;   // vectors per CTA (TMEM lanes); M = 256 per pair
constexpr int KSL = 64;   // int8 K elements per slot (64-B rows, SWIZZLE_64B)
constexpr int XT = BM * KSL;  // one x-plane tile per CTA: 8 KB
constexpr int TMEM_COLS = 512;

#ifndef SA_I8_NB_C64
#define SA_I8_NB_C64 1  // TMEM accumulator sets for complex64 (2 halves N: measured slower, L2-fed)
#endif
#ifndef SA_I8_NB_C128
#define SA_I8_NB_C128 1
#endif
#ifndef SA_I8_EPI_C64
#define SA_I8_EPI_C64 8  // epilogue warps (a multiple of 4: EPI / 4 per TMEM lane quarter)
#endif
#ifndef SA_I8_EPI_C128
#define SA_I8_EPI_C128 8
#endif
#ifndef SA_I8_T16_C128
#define SA_I8_T16_C128 1  // complex128 epilogue reads TMEM as 16x256b: 4 lanes per row, 64-B row segments per store
#endif
#ifndef SA_I8_PREP_WARP
#define SA_I8_PREP_WARP 1  // complex64 digit prep: one warp per row (0: one CTA per row)
#endif
#ifndef SA_I8_NPREP
#define SA_I8_NPREP 4  // complex64, n <= 1024: warps (pairs) per CTA that make the x planes inside the kernel (0: separate prep)
#endif
#ifndef SA_I8_PREP_LA
#define SA_I8_PREP_LA 2  // fused prep: rounds of tiles the prep may run ahead (0: unthrottled)
#endif
#ifndef SA_I8_STAGE_C64
#define SA_I8_STAGE_C64 1  // complex64 rows leave through a per-warp smem staging tile
#endif

template <int ND> struct Cfg {
  static constexpr int NPL = 2 + 2 * ND;          // planes per side: S, 127 S, 2 ND digits
  static constexpr int NACC = 2 * ND;             // accumulators: ND W-side, ND x-side
  static constexpr int NB = ND == 1 ? SA_I8_NB_C64 : SA_I8_NB_C128;  // accumulator sets in TMEM
  static constexpr int BN = TMEM_COLS / (NACC * NB);  // outputs per tile: 128 (c64, two sets; c128, one)
  static constexpr int WT = (BN / 2) * KSL;       // one W-plane tile per CTA (half the outputs)
  static constexpr int SLOT = NPL * (XT + WT);    // 48 KB (c64) / 72 KB (c128)
  static constexpr int NSLOT = (224 * 1024) / SLOT > 4 ? 4 : (224 * 1024) / SLOT;
  static constexpr int EPI = ND == 1 ? SA_I8_EPI_C64 : SA_I8_EPI_C128;  // epilogue warps
  static constexpr int RELAY_WARP = 2 + EPI;
  static constexpr int NPREP = ND == 1 ? SA_I8_NPREP : 0;  // digit-prep warps inside the kernel (complex64)
  static constexpr int THREADS = (3 + EPI + NPREP) * 32;  // producer, MMA, epilogue, relay, prep
  // complex64: per epilogue warp a 32 x 32 fp32 staging tile (rows leave as whole 128-B lines)
  static constexpr bool STAGE = ND == 1 && SA_I8_STAGE_C64;
  static constexpr int STG = STAGE ? EPI * 4096 : 0;
  static constexpr int SMEM = NSLOT * SLOT + 1024 + 256 + STG;
  // kind::i8: D = s32 (2), A = B = s8 (1), K-major, N = BN, M = 256
  static constexpr uint32_t IDESC =
      (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
};

SA_HD uint64_t sdesc(uint32_t saddr) {  // K-major SWIZZLE_64B: 64-B rows, 8-row atoms 512 B apart
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
// byte offset of (row r, K byte b) inside a SWIZZLE_64B tile of 64-B rows
SA_HD uint32_t sw64(int r, int b) { return (uint32_t)(r * 64 + ((((b >> 4) ^ (r >> 1)) & 3) << 4) + (b & 15)); }
SA_HD void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sa_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(sa_smem_u32(bar)), "l"(pol)
      : "memory");
}
SA_HD void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SA_HD void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SA_HD void commit2(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          sa_smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
SA_HD void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
#ifdef SA_I8_PROBE_NOMMA
  return;
#endif
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
SA_HD void arrive_cl(uint32_t cl_addr) { asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory"); }
SA_HD uint64_t policy(bool keep) {
  uint64_t p;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
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

#define SA_LD16(v, taddr)                                                                                  \
  asm volatile(                                                                                            \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"    \
      " [%16];"                                                                                            \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),           \
        "=r"(v[15])                                                                                        \
      : "r"(taddr))

// 16 TMEM lanes x 16 columns: thread t gets lane t/4 (regs 0,1,4,5) and t/4 + 8
// (regs 2,3,6,7), columns 2 (t%4) + {0, 1} (regs 0-3) and 8 + 2 (t%4) + {0, 1} (regs 4-7)
#define SA_LD16x256(v, taddr)                                                                              \
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                    \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),       \
                 "=r"(v[7])                                                                                \
               : "r"(taddr))

// The 2 ND signed digits (radix 127, 127, 128, 127) of |v| <= 1.
template <int ND> SA_HD void digits(double v, int (&d)[2 * ND]) {
  double y = v * 127.0;
#pragma unroll
  for (int i = 0; i < 2 * ND; ++i) {
    const double r = rint(y);
    d[i] = (int)r;
    y = (y - r) * ((i & 1) ? 128.0 : 127.0);
  }
}
// exact int64 -> double for |v| < 2^51: v added to the significand of 1.5 2^52
// (an integer add and one DADD instead of the slow 64-bit I2F)
SA_HD double i51_to_f64(long long v) {
  return __dsub_rn(__longlong_as_double(v + 0x4338000000000000LL), 6755399441055744.0);
}
SA_HD int sgn_i(double v) { return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0); }

// Four bytes (the low byte of each word) packed into one word.
SA_HD uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}
// rint(y) for |y| <= 2^21 and its two's-complement low byte, by the 1.5 2^p
// shifter: the sum's significand holds the rounded integer in its low bits.
SA_HD float rint_b(float y, uint32_t &byte) {
  const float t = __fadd_rn(y, 12582912.0f);
  byte = __float_as_uint(t);
  return __fsub_rn(t, 12582912.0f);
}
SA_HD double rint_b(double y, uint32_t &byte) {
  const double t = __dadd_rn(y, 6755399441055744.0);
  byte = (uint32_t)__double2loint(t);
  return __dsub_rn(t, 6755399441055744.0);
}

// x (batch x n complex, gain applied in the input precision as the fast kernels
// do) -> the planes as smem images: block (v / 128, K slot) holds the NPL 8 KB
// tiles of rows v % 128, SWIZZLE_64B-permuted; e[v] = per-vector exponent
// (max|x_v| < 2^e; INT_MAX for a row holding NaN / Inf: the epilogue writes NaN).
// One row per CTA iteration, read once: thread t holds elements [8 t + 2048 i,
// +8), i < IT, in registers; each plane gets one 8-byte store per thread.  The
// digits are taken in the input precision (complex64: fp32; the last digit's
// residual rounding only moves a tie).
template <int ND, typename T, int IT>
__global__ void __launch_bounds__(256) k_i8_prep(const T *__restrict__ x, int8_t *__restrict__ planes,
                                                 int *__restrict__ ex, int64_t batch, int n, T gain, int use_gain) {
  constexpr int NPL = Cfg<ND>::NPL;
  __shared__ T red[8];
  const int nk = 2 * n;
  const int kslots = nk / KSL;
  // the next row's loads are issued before this row's digit work (two rows in flight per CTA)
  auto load = [&](int64_t v, T (&t)[IT][8]) {
    const T *row = x + v * nk;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int k = threadIdx.x * 8 + 2048 * i;
      if (v < batch && k < nk) {
        if constexpr (sizeof(T) == 4) {
          const float4 u0 = __ldcs((const float4 *)&row[k]), u1 = __ldcs((const float4 *)&row[k + 4]);
          t[i][0] = u0.x, t[i][1] = u0.y, t[i][2] = u0.z, t[i][3] = u0.w;
          t[i][4] = u1.x, t[i][5] = u1.y, t[i][6] = u1.z, t[i][7] = u1.w;
        } else {
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const double2 u = __ldcs((const double2 *)&row[k + j]);
            t[i][j] = u.x, t[i][j + 1] = u.y;
          }
        }
      }
    }
  };
  T t[IT][8], tn[IT][8];
  load(blockIdx.x, t);
  for (int64_t v = blockIdx.x; v < batch; v += gridDim.x) {
    T mx = T(0);
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int k = threadIdx.x * 8 + 2048 * i;
      if (k < nk) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (use_gain) t[i][j] = sa_mul(gain, t[i][j]);
          const T a = fabs(t[i][j]);
          mx = a == a ? fmax(mx, a) : T(INFINITY);  // a NaN anywhere makes the row non-finite
        }
      }
    }
    load(v + gridDim.x, tn);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    __syncthreads();
    int e = 0;
    if (mx > T(0)) frexp((double)mx, &e);  // mx = f 2^e, f in [0.5, 1): max < 2^e
    if (!(mx <= T(sizeof(T) == 4 ? 3.4028234663852886e38 : 1.7976931348623157e308))) e = INT_MAX;
    if (threadIdx.x == 0) ex[v] = e;
    if (e == INT_MAX) e = 0;  // (digits of this row are never used)
    // 127 x 2^-e: an exact power-of-two product where the scale is normal, then 127
    const bool fast = sizeof(T) == 4 ? (e > -100 && e < 100) : (e > -900 && e < 900);
    const T sc = (T)ldexp(1.0, -e);
    int8_t *blk = planes + (size_t)(v / BM) * kslots * (NPL * XT);
    const int r = (int)(v % BM);
    // (uniform per row: one branch, not a per-element select)
    auto emit = [&](auto scaled) {
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        const int k = threadIdx.x * 8 + 2048 * i;
        if (k < nk) {
          uint32_t b[NPL][8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const T xv = t[i][j];
            const uint32_t sg = (uint32_t)((xv > T(0)) - (xv < T(0)));
            b[0][j] = sg;
            b[1][j] = sg * 127u;
            T yv = scaled(xv);
#pragma unroll
            for (int d = 0; d < 2 * ND; ++d) {
              const T rr = rint_b(yv, b[2 + d][j]);
              if (d + 1 < 2 * ND) yv = sa_mul(sa_sub(yv, rr), T((d & 1) ? 128.0 : 127.0));
            }
          }
          int8_t *tile = blk + (size_t)(k / KSL) * (NPL * XT) + sw64(r, k % KSL);  // 8 bytes, one swizzle chunk
#pragma unroll
          for (int p = 0; p < NPL; ++p)
            *(uint2 *)(tile + p * XT) = make_uint2(pack4(b[p][0], b[p][1], b[p][2], b[p][3]),
                                                   pack4(b[p][4], b[p][5], b[p][6], b[p][7]));
        }
      }
    };
    if (fast) emit([&](T xv) { return sa_mul(sa_mul(xv, sc), T(127)); });
    else emit([&](T xv) { return (T)sa_mul(ldexp((double)xv, -e), 127.0); });
#pragma unroll
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) t[i][j] = tn[i][j];
  }
}

// complex64, n <= 1024: one WARP per row (no block barriers), NV float4 per lane
// held in registers (k = 4 lane + 128 i: every load instruction is 512 contiguous
// bytes), warp-shuffle maximum, one 4-byte store per plane per float4 (a warp
// writes two whole 64-B tile rows).  Digits exactly as k_i8_prep.
template <int ND, int NV>
SA_HD void prep_row_w(const float *__restrict__ x, int8_t *__restrict__ planes, int *__restrict__ ex, int64_t v,
                      int n, float gain, int use_gain, int lane) {
  constexpr int NPL = Cfg<ND>::NPL;
  const int nk = 2 * n;
  const int kslots = nk / KSL;
  const float *row = x + v * nk;
  float4 t[NV];
  float mx = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int k = 4 * lane + 128 * i;
    t[i] = k < nk ? __ldcs((const float4 *)&row[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (use_gain) t[i] = make_float4(sa_mul(gain, t[i].x), sa_mul(gain, t[i].y), sa_mul(gain, t[i].z), sa_mul(gain, t[i].w));
    const float a[4] = {fabsf(t[i].x), fabsf(t[i].y), fabsf(t[i].z), fabsf(t[i].w)};
#pragma unroll
    for (int j = 0; j < 4; ++j) mx = a[j] == a[j] ? fmaxf(mx, a[j]) : INFINITY;  // a NaN makes the row non-finite
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.f) frexp((double)mx, &e);  // mx = f 2^e, f in [0.5, 1): max < 2^e
  if (!(mx <= 3.4028234663852886e38f)) e = INT_MAX;
  if (lane == 0) ex[v] = e;
  if (e == INT_MAX) e = 0;  // (digits of this row are never used)
  const bool fast = e > -100 && e < 100;
  const float sc = (float)ldexp(1.0, -e);
  int8_t *blk = planes + (size_t)(v / BM) * kslots * (NPL * XT);
  const int r = (int)(v % BM);
  auto emit = [&](auto scaled) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int k = 4 * lane + 128 * i;
      if (k < nk) {
        const float xs[4] = {t[i].x, t[i].y, t[i].z, t[i].w};
        uint32_t b[NPL][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float xv = xs[j];
          const uint32_t sg = (uint32_t)((xv > 0.f) - (xv < 0.f));
          b[0][j] = sg;
          b[1][j] = sg * 127u;
          float yv = scaled(xv);
#pragma unroll
          for (int d = 0; d < 2 * ND; ++d) {
            const float rr = rint_b(yv, b[2 + d][j]);
            if (d + 1 < 2 * ND) yv = sa_mul(sa_sub(yv, rr), (d & 1) ? 128.0f : 127.0f);
          }
        }
        int8_t *tile = blk + (size_t)(k / KSL) * (NPL * XT) + sw64(r, k % KSL);  // 4 bytes, inside one chunk
#pragma unroll
        for (int p = 0; p < NPL; ++p) *(uint32_t *)(tile + p * XT) = pack4(b[p][0], b[p][1], b[p][2], b[p][3]);
      }
    }
  };
  if (fast) emit([&](float xv) { return sa_mul(sa_mul(xv, sc), 127.0f); });
  else emit([&](float xv) { return (float)sa_mul(ldexp((double)xv, -e), 127.0); });
}

// complex64, n <= 1024: one WARP per row (no block barriers), NV float4 per lane
// held in registers (k = 4 lane + 128 i: every load instruction is 512 contiguous
// bytes), warp-shuffle maximum, one 4-byte store per plane per float4 (a warp
// writes two whole 64-B tile rows).  Digits exactly as k_i8_prep.
template <int ND, int NV>
__global__ void __launch_bounds__(256) k_i8_prep_w(const float *__restrict__ x, int8_t *__restrict__ planes,
                                                   int *__restrict__ ex, int64_t batch, int n, float gain,
                                                   int use_gain) {
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = w0; v < batch; v += nw) prep_row_w<ND, NV>(x, planes, ex, v, n, gain, use_gain, threadIdx.x & 31);
}

// W planes (sW, 127 sW, digits) of Wv = [[Wr, -Wi], [Wi, Wr]], W = raw[(k m) mod n]
// (the twiddle set's table: fp32 RN cast for complex64, the fp64 reference table
// transforms.py:108-146 for complex128), as smem images: block (o / (N/2), K slot).
template <int ND, typename C2T>
__global__ void k_i8_wbuild(const C2T *__restrict__ raw, int n, int8_t *__restrict__ q) {
  using C = Cfg<ND>;
  const int64_t nn = 2LL * n, total = nn * nn;
  const int kslots = (int)(nn / KSL);
  constexpr int HB = C::BN / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / nn, kk = i % nn;
    const int64_t k = o >> 1, m = kk >> 1;
    const int co = (int)(o & 1), ci = (int)(kk & 1);
    const C2T tw = raw[(k * m) % n];
    const double val = co == ci ? (double)tw.x : (co == 0 ? -(double)tw.y : (double)tw.y);
    int d[2 * ND];
    digits<ND>(val, d);
    const int sg = sgn_i(val);
    int8_t *tile = q + ((o / HB) * kslots + kk / KSL) * (C::NPL * C::WT) + sw64((int)(o % HB), (int)(kk % KSL));
    tile[0] = (int8_t)sg;
    tile[C::WT] = (int8_t)(127 * sg);
#pragma unroll
    for (int p = 0; p < 2 * ND; ++p) tile[(2 + p) * C::WT] = (int8_t)d[p];
  }
}

template <int ND, typename T>
__global__ void __launch_bounds__(Cfg<ND>::THREADS, 1)
    k_ndft_i8(const int8_t *__restrict__ xblk, const int8_t *__restrict__ wblk, const int *__restrict__ ex,
              T *__restrict__ y, int64_t batch, int n, const T *__restrict__ x, unsigned *__restrict__ ready,
              T gain, int use_gain) {
  using C = Cfg<ND>;
  constexpr int NPL = C::NPL, BN = C::BN, WT = C::WT, SLOT = C::SLOT, NSLOT = C::NSLOT, NB = C::NB;
  constexpr int EPI = C::EPI, RELAY_WARP = C::RELAY_WARP;
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + NSLOT * SLOT);  // leader: both CTAs' slot s complete
  uint64_t *empty = full + NSLOT;
  uint64_t *lfull = empty + NSLOT;                     // this CTA's bytes of slot s landed
  uint64_t *tfull = lfull + NSLOT;                     // accumulator set b holds a finished tile
  uint64_t *tempty = tfull + NB;                       // the epilogue drained set b
  uint32_t *tmem_holder = (uint32_t *)(tempty + NB);
  int64_t *okt = (int64_t *)(smem + NSLOT * SLOT + 128);  // last tile whose x block the producer verified

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int64_t cl = blockIdx.x / 2, ncl = gridDim.x / 2;
  const int nk = 2 * n;
  const int ot_count = nk / BN;
  const int64_t vt_count = (batch + 2 * BM - 1) / (2 * BM);
  const int64_t ntiles = vt_count * ot_count;
  const int kslots = nk / KSL;
  auto lead = [&](uint64_t *bar) { return sa_mapa(sa_smem_u32(bar), 0); };

  if (threadIdx.x == 0) {
    *okt = -1;
    for (int s = 0; s < NSLOT; ++s) {
      sa_mbar_init(&full[s], 2);  // the relays of both CTAs
      sa_mbar_init(&empty[s], 1);
      sa_mbar_init(&lfull[s], 1);
    }
    for (int b = 0; b < NB; ++b) {
      sa_mbar_init(&tfull[b], 1);
      sa_mbar_init(&tempty[b], EPI * 2);
    }
    sa_fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa_smem_u32(tmem_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_before();
  cluster_sync_all();
  fence_after();
  const uint32_t tmem = *tmem_holder;
  const int64_t my_tiles = cl < ntiles ? (ntiles - 1 - cl) / ncl + 1 : 0;
  const int64_t total = my_tiles * kslots;

  if (warp == 0) {
    // ---- producer: one bulk copy per side per slot (this CTA's 128 vectors / N/2 outputs) ----
    if (lane == 0) {
      const uint64_t wpol = policy(true), xpol = policy(false);
      for (int64_t it = 0; it < total; ++it) {
        const int64_t lt = it / kslots;
        const int kc = (int)(it - lt * kslots);
        const int64_t t = cl + lt * ncl;
        const int64_t vb = (t / ot_count) * 2 + rank;  // 128-vector block
        const int64_t ob = (t % ot_count) * 2 + rank;  // N/2-output block
        const int s = (int)(it % NSLOT);
#ifdef SA_I8_PROBE_NOWAIT
        if (false) {
#else
        if (C::NPREP > 0 && ready && kc == 0) {
#endif
          // fused prep: all rows of this 128-vector block have their planes (release-add per
          // row by the prep warps of every CTA); then the async-proxy reads may see them
          const int64_t need = std::min<int64_t>(BM, batch - vb * BM);
          if (need > 0) {
            unsigned got;
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(ready + vb) : "memory");
            } while ((int64_t)got < need);
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        }
        if (kc == 0)  // this tile's block has its planes and exponents: the epilogue may read ex
          asm volatile("st.release.cta.shared::cta.b64 [%0], %1;" ::"r"(sa_smem_u32(okt)), "l"(lt) : "memory");
        sa_mbar_wait(&empty[s], ((it / NSLOT) & 1) ^ 1);
        unsigned char *b = smem + s * SLOT;
        sa_mbar_expect_tx(&lfull[s], SLOT);
        bulk_g2s(b, xblk + (vb * kslots + kc) * (NPL * XT), NPL * XT, &lfull[s], xpol);
        bulk_g2s(b + NPL * XT, wblk + (ob * kslots + kc) * (NPL * WT), NPL * WT, &lfull[s], wpol);
      }
    }
  } else if (warp == RELAY_WARP) {
    // ---- relay: this CTA's slot landed -> arrive on the leader's full barrier ----
    if (lane == 0)
      for (int64_t it = 0; it < total; ++it) {
        const int s = (int)(it % NSLOT);
        sa_mbar_wait(&lfull[s], (it / NSLOT) & 1);
        arrive_cl(lead(&full[s]));
      }
  } else if (warp == 1) {
    // ---- MMA issuer (leader CTA): 4 ND MMAs per K step of 32 into the 2 ND accumulators ----
    if (lane == 0 && rank == 0) {
      uint32_t it = 0, lt = 0;
      for (int64_t t = cl; t < ntiles; t += ncl, ++lt) {
        const uint32_t ab = lt % NB, acc0 = tmem + ab * (2 * ND * BN);  // this tile's accumulator set
        sa_mbar_wait(&tempty[ab], ((lt / NB) & 1) ^ 1);
        fence_after();
        for (int kc = 0; kc < kslots; ++kc, ++it) {
          const int s = it % NSLOT;
          sa_mbar_wait(&full[s], (it / NSLOT) & 1);
          fence_after();
          const uint32_t base = sa_smem_u32(smem + s * SLOT);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t off = ks * 32;
            auto X = [&](int p) { return sdesc(base + p * XT + off); };
            auto W = [&](int p) { return sdesc(base + NPL * XT + p * WT + off); };
            const uint32_t first = (kc | ks) != 0;
#pragma unroll
            for (int j = 0; j < ND; ++j) {
              mma2(acc0 + j * BN, X(1), W(2 + 2 * j), C::IDESC, first);          // accW_j += 127 S dW_2j
              mma2(acc0 + j * BN, X(0), W(3 + 2 * j), C::IDESC, 1);              //         + S dW_2j+1
              mma2(acc0 + (ND + j) * BN, X(2 + 2 * j), W(1), C::IDESC, first);   // accX_j += dx_2j 127 sW
              mma2(acc0 + (ND + j) * BN, X(3 + 2 * j), W(0), C::IDESC, 1);       //         + dx_2j+1 sW
            }
          }
          commit2(&empty[s]);
        }
        commit2(&tfull[ab]);
      }
    }
  } else if (warp > RELAY_WARP) {
    // ---- prep warps (complex64, fused): rows taken in increasing order from one ticket
    // counter (ready[nready]) by whichever prep warps run -- no producer ever waits on a
    // row owned by a CTA that is not resident -- each row released to the producers of
    // the CTAs that read it ----
    if constexpr (C::NPREP > 0) {
      if (ready) {
        unsigned *ticket = ready + (vt_count * 2);
        for (;;) {
          unsigned vt = 0;
          if (lane == 0) vt = atomicAdd(ticket, 1u);
          const int64_t v = __shfl_sync(0xffffffffu, vt, 0);
          if (v >= batch) break;
#if SA_I8_PREP_LA > 0
          // stay at most SA_I8_PREP_LA rounds of tiles ahead of this CTA's producer (every
          // CTA advances alike), so planes are read back while still in L2
          const int64_t tfirst = (v / (2 * BM)) * ot_count;
          for (;;) {
            int64_t ok;
            asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(ok) : "r"(sa_smem_u32(okt)) : "memory");
            if (tfirst <= cl + (ok < 0 ? 0 : ok) * ncl + SA_I8_PREP_LA * ncl) break;
            __nanosleep(256);
          }
#endif
          prep_row_w<ND, 16>((const float *)x, const_cast<int8_t *>(xblk), const_cast<int *>(ex), v, n, (float)gain,
                             use_gain, lane);
#ifndef SA_I8_PROBE_NOFENCE
          asm volatile("fence.proxy.async.global;" ::: "memory");  // plane stores -> the TMA readers
#endif
          __syncwarp();
          if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ready + v / BM) : "memory");
        }
      }
    }
  } else {
    // ---- epilogue (warps 2 .. 1 + EPI): TMEM lane quarter q -> vector row v, a column share ----
    // y = c (W + 2^e X) with W, X the digit-pair sums: one conversion each and one
    // FMA against the per-row scale c 2^e (rows whose scale leaves the normal range
    // of the output type take the ldexp form).
    const int q = warp & 3;
    const int cs = (warp - 2) / 4;  // this warp's column share
    constexpr int CW = BN / (EPI / 4);
    constexpr double CD = ND == 2 ? 1.0 / (127.0 * 127.0 * 128.0 * 127.0) : 1.0 / (127.0 * 127.0);
    uint32_t lt = 0;
    for (int64_t t = cl; t < ntiles; t += ncl, ++lt) {
      const int64_t v = (t / ot_count) * (2 * BM) + rank * BM + q * 32 + lane;
      const int o0 = (int)(t % ot_count) * BN;
      const uint32_t ab = lt % NB;
      {  // the producer verified this tile's block (fused prep: ex written), then the load
        int64_t ok;
        do {
          asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(ok) : "r"(sa_smem_u32(okt)) : "memory");
        } while (ok < (int64_t)lt);
      }
      const int e = v < batch ? __ldcg(&ex[v]) : 0;  // (its latency overlaps the accumulator wait)
      sa_mbar_wait(&tfull[ab], (lt / NB) & 1);
      fence_after();
      const bool fast = ND == 2 ? (e > -960 && e < 1030) : (e > -100 && e < 100);
      const double sxd = fast ? ldexp(CD, e) : 0.0;
      const float sxf = (float)sxd;
      const uint32_t ta = tmem + ab * (2 * ND * BN) + ((uint32_t)(q * 32) << 16);
#ifdef SA_I8_PROBE_NOEPI
      if (v >= 0) {
      } else
#endif
      if constexpr (C::STAGE) {
        // complex64: 32 columns at a time through the warp's staging tile (16-B
        // chunks XOR-swizzled by row): each lane writes its row, then every store
        // instruction writes four whole 128-B lines of y.
        float *stg = (float *)(smem + NSLOT * SLOT + 256) + (warp - 2) * 1024;
        const int64_t vw = v - lane;  // this warp's first row
#pragma unroll 1
        for (int c = cs * CW; c < (cs + 1) * CW; c += 32) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t acc[2][16];
            SA_LD16(acc[0], ta + c + 16 * h);
            SA_LD16(acc[1], ta + BN + c + 16 * h);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float d[16];
            if (fast) {
#pragma unroll
              for (int j = 0; j < 16; ++j) d[j] = fmaf((float)(int)acc[1][j], sxf, sa_mul((float)(int)acc[0][j], (float)CD));
            } else {  // (rows of extreme scale, or non-finite: NaN)
#pragma unroll
              for (int j = 0; j < 16; ++j)
                d[j] = e == INT_MAX ? CUDART_NAN_F
                                    : (float)sa_add(ldexp(sa_mul((double)(int)acc[1][j], CD), e),
                                                    sa_mul((double)(int)acc[0][j], CD));
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
              *(float4 *)(stg + lane * 32 + (((4 * h + k) ^ (lane & 7)) << 2)) =
                  make_float4(d[4 * k], d[4 * k + 1], d[4 * k + 2], d[4 * k + 3]);
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = 4 * i + (lane >> 3), ch = lane & 7;
            const float4 val = *(const float4 *)(stg + r * 32 + ((ch ^ (r & 7)) << 2));
#ifdef SA_I8_PROBE_NOSTORE
            if (batch < 0)
#endif
            if (vw + r < batch) __stcs((float4 *)&y[(vw + r) * nk + o0 + c + 4 * ch], val);
          }
          __syncwarp();
        }
      } else if constexpr (ND == 2 && SA_I8_T16_C128) {
        // complex128, 16x256b: thread t holds rows rr(i) = t/4 + 8 (i & 1) + 16 (i >> 1) of the
        // warp's 32 and columns 2 (t%4) + {0, 1} and 8 + 2 (t%4) + {0, 1} of each 16-column
        // chunk; four threads store 64 contiguous bytes of a row
        const int tj = lane & 3;
        int er[4];
        double sr[4];
        bool allfast = true;
        const int64_t vw = v - lane;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t vi = vw + (lane >> 2) + 8 * (i & 1) + 16 * (i >> 1);
          er[i] = vi < batch ? ex[vi] : 0;
          const bool f = er[i] > -960 && er[i] < 1030;
          sr[i] = f ? ldexp(CD, er[i]) : 0.0;
          allfast = allfast && f;
        }
#pragma unroll 1
        for (int c = cs * CW; c < (cs + 1) * CW; c += 16) {
          uint32_t acc[4][2][8];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int h = 0; h < 2; ++h) SA_LD16x256(acc[a][h], ta + ((uint32_t)(16 * h) << 16) + a * BN + c);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t vi = vw + (lane >> 2) + 8 * (i & 1) + 16 * (i >> 1);
            const int h = i >> 1, rb = 2 * (i & 1);
            double d[4];  // columns 2 tj, 2 tj + 1, 8 + 2 tj, 9 + 2 tj
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int rg = rb + (u & 1) + 4 * (u >> 1);
              const double w = i51_to_f64((long long)(int)acc[0][h][rg] * (128 * 127) + (int)acc[1][h][rg]);
              const double xs = i51_to_f64((long long)(int)acc[2][h][rg] * (128 * 127) + (int)acc[3][h][rg]);
              if (allfast) d[u] = fma(xs, sr[i], sa_mul(w, CD));
              else d[u] = er[i] == INT_MAX ? CUDART_NAN
                          : (er[i] > -960 && er[i] < 1030) ? fma(xs, sr[i], sa_mul(w, CD))
                                                           : sa_add(ldexp(sa_mul(xs, CD), er[i]), sa_mul(w, CD));
            }
            if (vi < batch) {
              double *row = y + vi * nk + o0 + c + 2 * tj;
              __stcs((double2 *)row, make_double2(d[0], d[1]));
              __stcs((double2 *)(row + 8), make_double2(d[2], d[3]));
            }
          }
        }
      } else {
        // each lane stores its row, 16 B at a time
        T *dst = y + v * nk + o0;
#pragma unroll 1
        for (int c = cs * CW; c < (cs + 1) * CW; c += 16) {
          uint32_t acc[2 * ND][16];
#pragma unroll
          for (int a = 0; a < 2 * ND; ++a) SA_LD16(acc[a], ta + a * BN + c);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (v < batch) {
            T d[16];
            // W, X: the digit-pair sums (complex128: combined in int64, exact: |.| < 2^39)
            auto wx = [&](int j, double &w, double &xs) {
              if constexpr (ND == 2) {
                w = i51_to_f64((long long)(int)acc[0][j] * (128 * 127) + (int)acc[1][j]);
                xs = i51_to_f64((long long)(int)acc[2][j] * (128 * 127) + (int)acc[3][j]);
              } else {
                w = (double)(int)acc[0][j];
                xs = (double)(int)acc[1][j];
              }
            };
            if (fast) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if constexpr (ND == 2) {
                  double w, xs;
                  wx(j, w, xs);
                  d[j] = fma(xs, sxd, sa_mul(w, CD));
                } else {
                  d[j] = fmaf((float)(int)acc[1][j], sxf, sa_mul((float)(int)acc[0][j], (float)CD));
                }
              }
            } else {  // (rows of extreme scale, or non-finite: NaN)
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                double w, xs;
                wx(j, w, xs);
                d[j] = e == INT_MAX ? (T)CUDART_NAN : (T)sa_add(ldexp(sa_mul(xs, CD), e), sa_mul(w, CD));
              }
            }
#ifdef SA_I8_PROBE_NOSTORE
            if (batch < 0)
#endif
            if constexpr (sizeof(T) == 8) {
#pragma unroll
              for (int j = 0; j < 16; j += 2) __stcs((double2 *)&dst[c + j], make_double2(d[j], d[j + 1]));
            } else {
#pragma unroll
              for (int j = 0; j < 16; j += 4) __stcs((float4 *)&dst[c + j], make_float4(d[j], d[j + 1], d[j + 2], d[j + 3]));
            }
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) arrive_cl(lead(&tempty[ab]));
    }
  }

  fence_before();
  cluster_sync_all();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

std::mutex g_i8_mutex;

template <int ND> int64_t wbytes(int64_t n) { return (int64_t)Cfg<ND>::NPL * (2 * n) * (2 * n); }

template <int ND, typename T, typename C2T>
int launch_i8(const void *x, void *y, int64_t batch, int64_t n, SaTwiddles *tw, double gain, cudaStream_t s) {
  using C = Cfg<ND>;
  {
    // W planes built once per twiddle set, stream-ordered (event for later streams)
    std::lock_guard<std::mutex> g(g_i8_mutex);
    if (!tw->i8w) {
      void *w = nullptr;
      cudaEvent_t ev = nullptr;
      SA_CUDA_TRY(cudaMalloc(&w, wbytes<ND>(n)));
      k_i8_wbuild<ND, C2T><<<1184, 256, 0, s>>>((const C2T *)tw->raw, (int)n, (int8_t *)w);
      SA_LAUNCH_CHECK();
      SA_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      SA_CUDA_TRY(cudaEventRecord(ev, s));
      tw->i8w = w;
      tw->i8w_ready = ev;
    }
  }
  if (tw->i8w_ready) SA_CUDA_TRY(cudaStreamWaitEvent(s, (cudaEvent_t)tw->i8w_ready, 0));
  // x planes (whole 256-vector tiles: rows past the batch are never stored) + exponents
  const int64_t rows = (batch + 2 * BM - 1) / (2 * BM) * (2 * BM);
  const size_t pbytes = (size_t)C::NPL * rows * 2 * n;
  // complex64, n <= 1024: the digit prep runs inside the tensor-core kernel (prep warps,
  // one ready counter per 128-vector block); otherwise a separate prep launch
  const bool fused = C::NPREP > 0 && n <= 1024;
  const int64_t nready = rows / BM;
  int8_t *planes = nullptr;
  {
    const int rc_ = sa_scratch_alloc((void **)&planes, pbytes + (size_t)batch * sizeof(int) + 256 +
                                                           (size_t)(nready + 1) * sizeof(unsigned) + 256, s);
    if (rc_) return rc_;
  }
  int *ex = (int *)(((uintptr_t)(planes + pbytes) + 255) & ~(uintptr_t)255);
  unsigned *ready = (unsigned *)(((uintptr_t)(ex + batch) + 255) & ~(uintptr_t)255);
  int dev = 0, sms = 148;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  SA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (fused) {
    SA_CUDA_TRY(cudaMemsetAsync(ready, 0, (size_t)(nready + 1) * sizeof(unsigned), s));  // + the row ticket
    goto prepped;
  }
  if constexpr (ND == 1 && SA_I8_PREP_WARP) {
    // complex64, n <= 1024: one warp per row, a wave of resident CTAs
    if (n <= 1024) {
      auto prepw = n <= 512 ? k_i8_prep_w<1, 8> : k_i8_prep_w<1, 16>;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prepw, 256, 0) != cudaSuccess || per_sm < 1)
        per_sm = 2;
      const int64_t need = (batch + 7) / 8, pmax = (int64_t)per_sm * sms;
      prepw<<<(unsigned)(need < pmax ? need : pmax), 256, 0, s>>>((const float *)x, planes, ex, batch, (int)n,
                                                                  (float)gain, (int)(gain != 1.0));
      SA_LAUNCH_CHECK();
      goto prepped;
    }
  }
  {
    // one row per CTA iteration, one wave of resident CTAs
    auto prep = n <= 1024 ? k_i8_prep<ND, T, 1> : k_i8_prep<ND, T, 2>;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prep, 256, 0) != cudaSuccess || per_sm < 1) per_sm = 2;
    const int64_t pmax = (int64_t)per_sm * sms;
    prep<<<(unsigned)(batch < pmax ? batch : pmax), 256, 0, s>>>((const T *)x, planes, ex, batch, (int)n, (T)gain,
                                                                 (int)(gain != 1.0));
    SA_LAUNCH_CHECK();
  }
prepped:
  static bool smem_set[64] = {};
  if (dev >= 64 || !smem_set[dev]) {
    SA_CUDA_TRY(cudaFuncSetAttribute(k_ndft_i8<ND, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    if (dev < 64) smem_set[dev] = true;
  }
  const int64_t ntiles = (rows / (2 * BM)) * ((2 * n) / C::BN);
  const int64_t units = ntiles < sms / 2 ? ntiles : sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * 2));
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_ndft_i8<ND, T>, (const int8_t *)planes, (const int8_t *)tw->i8w,
                                 (const int *)ex, (T *)y, batch, (int)n, (const T *)x, fused ? ready : nullptr,
                                 (T)gain, (int)(gain != 1.0)));
  SA_LAUNCH_CHECK();
  SA_CUDA_TRY(cudaFreeAsync(planes, s));
  return SA_OK;
}

}  // namespace

// complex128: n % 64 == 0, 128 <= n <= 2048 (below 128 the fp64 margin shrinks: DFMA);
// complex64: n % 128 == 0 (whole 256-output tiles), 128 <= n <= 2048.
bool sa_ndft_i8_supported(int dtype, int64_t n) {
  if (n < 128 || n > 2048) return false;
  return dtype == SA_C128 ? n % 64 == 0 : n % 128 == 0;
}

int sa_launch_ndft_i8(const void *x, void *y, int64_t batch, int64_t n, const SaTwiddles *tw_c, double gain,
                      cudaStream_t s) {
  if (!sa_ndft_i8_supported(tw_c->dtype, n)) return SA_ERR_UNSUPPORTED;
  if (((uintptr_t)x | (uintptr_t)y) & 15) return SA_ERR_UNSUPPORTED;
  if (batch == 0) return SA_OK;
  SaTwiddles *tw = const_cast<SaTwiddles *>(tw_c);
  if (tw->dtype == SA_C128) return launch_i8<2, double, double2>(x, y, batch, n, tw, gain, s);
  return launch_i8<1, float, float2>(x, y, batch, n, tw, gain, s);
}
