// sa_lag_i8.cu -- the map's fast-mode lag stage (ambiguity.py:146-187 composed
// with the block sums, as sa_lag_tc.cu) on the tcgen05 tensor cores in EXACT
// INTEGER arithmetic, complex64: int8 digits x signs, int32 accumulation.
//
//   z_l[q] = Σ_{t<T} s[qT+t] ⊙ c[qT+t-l],   c = conj(ref) (ref outside [0, ref_len) = 0)
//   Re = Σ sgn(sr) cr + sr sgn(cr) − sgn(si) ci − si sgn(ci)
//   Im = Σ sgn(si) cr + si sgn(cr) + sgn(sr) ci + sr sgn(ci)
// (the sign-split identity of the fast ⊙, sa_ambiguity.cu).  Every term has a
// sign in {−1, 0, 1} as one factor (exact in int8); the other factor is split
// into two signed int8 digits (radix 127, 254) of x / 2^e:
//   x ≈ 2^e (254 d0 + d1) / (127 · 254),  |d0|, |d1| <= 127,  residual <= 2^e / 64516
// with e per integration block for s (its T samples) and ONE e for the whole
// reference c (so a lag's digits never depend on which lags a call covers: any
// row range or Doppler-block shard of a map is bit-identical to the full call,
// and integer sums do not depend on the summation order).
//
// Formulation ("c-Hankel").  Lag l = lb + 16 j + i (j < MR rows, i < 16 shifts),
// u = t − i in [−16, T + 16):
//   Z[j, i] = Σ_u A[j, u] B[i, u],   A[j, u] = c[qT − lb − 16 j + u],  B[i, u] = s[qT + u + i]
// A is a Hankel matrix in (j, u): stored once per lag group as a linear int8
// array per plane, rows reversed (r = MR − 1 − j) so that row r + 1 starts 16 B
// later -- exactly the K-major no-swizzle core-matrix row pitch, so the UMMA
// descriptor (LBO 16 B, SBO 128 B) reads it in place.  B (16 shifts of the
// block's s planes) is materialised per K chunk from linear s planes.  The K
// range is T + 32 whatever the lag count (no zero region).
//
// Planes.  A (c): d0 cr, d1 cr, d0 ci, d1 ci, sgn cr, sgn ci.
//          B (s): sgn sr, sgn si, d0 sr, d0 si, d1 sr, d1 si.
// Per K step (32 u) and lag group, six MMAs (M = MR, K = 32):
//   W_p  (32 cols) += A[p] x B[sgn sr; sgn si]                   p = d0cr, d1cr, d0ci, d1ci   (N = 32)
//   X_p  (64 cols) += A[p] x B[d0 sr; d0 si; d1 sr; d1 si]       p = sgn cr, sgn ci           (N = 64)
// 256 TMEM columns per group.  Epilogue (per shift i, exact int32):
//   IWre = 254 (W0r[sr] − W0i[si]) + (W1r[sr] − W1i[si]),  IWim = 254 (W0r[si] + W0i[sr]) + (W1r[si] + W1i[sr])
//   IXre = 254 (Xr[d0sr] − Xi[d0si]) + (Xr[d1sr] − Xi[d1si]), IXim = 254 (Xr[d0si] + Xi[d0sr]) + (Xr[d1si] + Xi[d1sr])
//   Re = IWre 2^ec / 32258 + IXre 2^es / 32258 (fp64, rounded once to fp32), Im alike.
// Each TMEM lane holds the 16 consecutive lags of one blocked-z tile (sa_lag_tc.cu
// layout): the thread stores one whole 128-B line.
//
// Launches per call: k_lag_absmax (|ref| partials) -> k_lag_cprep (the six
// reference digit planes over the range the call's blocks read, in HBM) ->
// k_lag_i8: one CTA per integration block q, two per SM; warp roles: 0-3
// epilogue (drain TMEM, store the blocked z tiles), 4-7 B builders (16 shifts of
// the block's s planes per 128-u chunk, 4-deep ring), 8 MMA issuer (one elected
// lane per K step's six MMAs), 9 producer (bulk copies of each lag-group pass's
// A window, double-buffered).  A non-finite value in the block (s) makes its
// column NaN; a non-finite reference value makes the whole map NaN (the exponent
// is global) -- the bf16 kernel (sa_lag_tc.cu) keeps NaN local.
#include <cuda.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <math_constants.h>

#include "sa_internal.h"
#include "sa_regs.cuh"


namespace {

#ifdef SA_LAG_TS  // probe build: per-CTA phase timestamps (globaltimer, ns), tools/probes/lag_ts.py
__device__ unsigned long long g_lag_ts[4096 * 8];
SA_HD unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TS(i)                                                                \
  do {                                                                       \
    if (blockIdx.x < 4096 && (threadIdx.x & 31) == 0) g_lag_ts[blockIdx.x * 8 + (i)] = gtime(); \
  } while (0)
#else
#define TS(i) \
  do {        \
  } while (0)
#endif

constexpr int NPL = 6;                   // planes per side
constexpr int KC = 4;                    // K32 steps per B chunk (128 u)
constexpr int CORE = 128;                // one core matrix: 8 rows x 16 B
constexpr int B_SBO = 2 * KC * CORE;     // next 8 B rows
constexpr int B_BYTES = NPL * 2 * B_SBO; // 6 planes x 16 shifts x 128 u = 12 KB
constexpr int BUILDERS = 256;
constexpr int THREADS = BUILDERS + 32;   // warp 8 issues the MMAs
constexpr int NPART_MAX = 2048;          // |ref| max partials (k_lag_absmax CTAs)
constexpr double DSC = 1.0 / (127.0 * 254.0);

struct Geo {
  int ks, psl, pcl;
  int off_pc, off_b, off_bar, bytes;
};
__host__ __device__ inline Geo geo(int tb, int mr, int g) {
  Geo o;
  o.ks = tb / 32 + 1;                           // u in [-16, T + 16)
  o.psl = (32 * o.ks + 32 + 127) & ~127;        // s planes: x = u + 16 + i
  o.pcl = (32 * o.ks + 16 * mr + 127) & ~127;   // c planes: x = u + 16 + 16 r
  o.off_pc = NPL * o.psl;
  o.off_b = (o.off_pc + g * NPL * o.pcl + 1023) & ~1023;
  o.off_bar = o.off_b + 2 * B_BYTES;
  o.bytes = o.off_bar + 256 + 1024;             // barriers, reductions, alignment slack
  return o;
}

// kind::i8: D = s32, A = B = s8, K-major, N, M
constexpr uint32_t idesc(int n, int mr) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(mr >> 4) << 24);
}
SA_HD uint64_t sdesc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46);
}
SA_HD void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
SA_HD void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   sa_smem_u32(bar))
               : "memory");
}
SA_HD bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}\n" : "=r"(p));
  return p != 0;
}
SA_HD void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SA_HD void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define SA_LD16(v, taddr)                                                                                  \
  asm volatile(                                                                                            \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"    \
      " [%16];"                                                                                            \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),           \
        "=r"(v[15])                                                                                        \
      : "r"(taddr))
SA_HD void tm_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// sign and the two digits of x at scale 127 / 2^e.  |e| < 100 (every practical
// input): fp32 with the 1.5 2^23 shifter (d0 = rint(x sc) of the rounded product, the
// residual x sc - d0 by one fma, d1 = rint(254 residual)); otherwise fp64 (x sc exact).
// The path depends only on e, so a sample's digits are the same in every call.
struct Dig {
  float sf;
  double sd;
  bool fast;
  SA_HD explicit Dig(int e) : sf(0.f), sd(ldexp(127.0, -e)), fast(e > -100 && e < 100) {
    if (fast) sf = (float)sd;  // 127 x 2^-e, exact in fp32
  }
  SA_HD uint32_t operator()(float x, uint32_t &d0, uint32_t &d1) const {
    if (fast) {
      const float t0 = __fadd_rn(__fmul_rn(x, sf), 12582912.0f);
      const float r0 = __fsub_rn(t0, 12582912.0f);
      const float t1 = __fmaf_rn(__fmaf_rn(x, sf, -r0), 254.0f, 12582912.0f);
      d0 = __float_as_uint(t0) & 0xffu;
      d1 = __float_as_uint(t1) & 0xffu;
    } else {
      const double y = (double)x * sd;
      const double r0 = rint(y);
      d0 = (uint32_t)(int)r0 & 0xffu;
      d1 = (uint32_t)(int)rint((y - r0) * 254.0) & 0xffu;
    }
    return (uint32_t)((x > 0.f) - (x < 0.f)) & 0xffu;
  }
};
SA_HD int exponent_of(float mx) {  // mx = f 2^e, f in [0.5, 1): max < 2^e
  int e = 0;
  if (mx > 0.f && mx <= FLT_MAX) frexpf(mx, &e);
  return e;
}
SA_HD float amax(float2 v) {  // max |component|; +inf for a non-finite value
  const float a = fabsf(v.x), b = fabsf(v.y);
  return (a <= FLT_MAX && b <= FLT_MAX) ? fmaxf(a, b) : INFINITY;
}

// Where the 16 lags of a tile go: blocked z (one 128-B line) or row-major z, local
// or the owning rank's z block over peer memory (sa_lag_tc.cu's LagDst).
struct LagDst {
  float2 *const *ptr;
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

// |ref| maxima: one partial per CTA (grid-stride, 16-B loads); k_lag_cprep and the
// lag kernel reduce the partials.
__global__ void __launch_bounds__(256) k_lag_absmax(const float2 *__restrict__ ref, int64_t ref_len,
                                                    float *__restrict__ part) {
  sa_pdl_trigger();  // the prep launch may become resident while this one drains
  __shared__ float red[8];
  float mx = 0.f;
  const int64_t n4 = (uintptr_t)ref & 15 ? 0 : ref_len / 4;  // 16-B aligned: float4 pairs
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = __ldg((const float4 *)&ref[4 * i]), b = __ldg((const float4 *)&ref[4 * i + 2]);
    mx = fmaxf(mx, fmaxf(fmaxf(amax(make_float2(a.x, a.y)), amax(make_float2(a.z, a.w))),
                         fmaxf(amax(make_float2(b.x, b.y)), amax(make_float2(b.z, b.w)))));
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ref_len;
       i += (int64_t)gridDim.x * blockDim.x)
    mx = fmaxf(mx, amax(__ldg(&ref[i])));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
    part[blockIdx.x] = mx;
  }
}

// s planes of every block of the call (one CTA per block): the block's exponent
// (|s| maximum; INT_MAX marks a non-finite block) and its six digit planes
// [sgn sr, sgn si, d0 sr, d0 si, d1 sr, d1 si] over x in [0, psl), t = x - 16, laid
// out contiguously per block so the lag kernel fetches them with one bulk copy.
// Block 0 also stores the reference maximum (from the k_lag_absmax partials).
// Runs as the trailing blocks of the k_lag_cprep launch.
__device__ __forceinline__ void sprep_block(int64_t qi, const float2 *__restrict__ surv, int64_t q0, int tb, int psl,
                                            unsigned char *__restrict__ splanes, int *__restrict__ es_out,
                                            const float *__restrict__ part, int npart, float *__restrict__ mc_out) {
  __shared__ float red[8];
  const float2 *sb = surv + (q0 + qi) * tb;
  float ms = 0.f;
  for (int t = threadIdx.x; t < tb; t += blockDim.x) ms = fmaxf(ms, amax(__ldg(&sb[t])));
#pragma unroll
  for (int o = 16; o; o >>= 1) ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ms;
  __syncthreads();
  for (int w = 0; w < 8; ++w) ms = fmaxf(ms, red[w]);
  const int es = !(ms <= FLT_MAX) ? INT_MAX : exponent_of(ms);
  if (threadIdx.x == 0) es_out[qi] = es;
  if (qi == 0) {  // the reference maximum, reduced once for every lag CTA
    __syncthreads();
    float mc = 0.f;
    for (int i = threadIdx.x; i < npart; i += blockDim.x) mc = fmaxf(mc, __ldcg(&part[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mc;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w) mc = fmaxf(mc, red[w]);
      *mc_out = mc;
    }
  }
  const Dig dig(es == INT_MAX ? 0 : es);
  unsigned char *ps = splanes + qi * (int64_t)(NPL * psl);
  for (int x4 = threadIdx.x; x4 < psl / 4; x4 += blockDim.x) {
    const int t = 4 * x4 - 16;
    float2 v[4] = {};
    if (t >= 0 && t < tb) {  // tb % 4 == 0: a group of 4 is all in or all out
      const float4 a = __ldg((const float4 *)&sb[t]), b = __ldg((const float4 *)&sb[t + 2]);
      v[0] = make_float2(a.x, a.y), v[1] = make_float2(a.z, a.w), v[2] = make_float2(b.x, b.y), v[3] = make_float2(b.z, b.w);
    }
    uint32_t w[NPL] = {};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t d0r, d1r, d0i, d1i;
      const uint32_t sr = dig(v[e].x, d0r, d1r), si = dig(v[e].y, d0i, d1i);
      w[0] |= sr << (8 * e), w[1] |= si << (8 * e);
      w[2] |= d0r << (8 * e), w[3] |= d0i << (8 * e);
      w[4] |= d1r << (8 * e), w[5] |= d1i << (8 * e);
    }
#pragma unroll
    for (int p = 0; p < NPL; ++p) ((uint32_t *)(ps + p * psl))[x4] = w[p];
  }
}

// c planes of the whole reference (one exponent ec for all of it): plane p holds
// byte x = c[x - guard] (zero outside [0, ref_len)), p = d0 cr, d1 cr, d0 ci, d1 ci,
// sgn cr, sgn ci; the lag kernel bulk-copies its Hankel windows out of them.
// (Two ordinary launches, not one cooperative one: a grid barrier would need every
// CTA resident, which a concurrent kernel -- e.g. an NCCL collective of the
// streaming multi-GPU map -- can prevent.)
__global__ void __launch_bounds__(256) k_lag_cprep(const float2 *__restrict__ ref, int64_t ref_len, float csign,
                                                   const float *__restrict__ part, int npart, int64_t guard,
                                                   int64_t cpl, unsigned char *__restrict__ planes, unsigned ncb,
                                                   const float2 *__restrict__ surv, int64_t q0, int tb, int psl,
                                                   unsigned char *__restrict__ splanes, int *__restrict__ es_out,
                                                   float *__restrict__ mc_out) {
  sa_pdl_trigger();
  sa_pdl_wait();  // the |ref| partials of k_lag_absmax
  if (blockIdx.x >= ncb) {  // trailing blocks: one per surveillance block
    sprep_block(blockIdx.x - ncb, surv, q0, tb, psl, splanes, es_out, part, npart, mc_out);
    return;
  }
  __shared__ float red[8];
  float mc = 0.f;
  for (int i = threadIdx.x; i < npart; i += blockDim.x) mc = fmaxf(mc, __ldcg(&part[i]));
#pragma unroll
  for (int o = 16; o; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mc;
  __syncthreads();
  for (int w = 0; w < 8; ++w) mc = fmaxf(mc, red[w]);
  const Dig dig(exponent_of(mc));
  for (int64_t x16 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x16 < cpl / 16;
       x16 += (int64_t)ncb * blockDim.x) {
    const int64_t k0 = 16 * x16 - guard;
    uint32_t w[NPL][4] = {};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      float2 v[4];
      const int64_t k = k0 + 4 * h;
      if (k >= 0 && k + 4 <= ref_len) {
        const float4 a = __ldg((const float4 *)&ref[k]), b = __ldg((const float4 *)&ref[k + 2]);
        v[0] = make_float2(a.x, a.y), v[1] = make_float2(a.z, a.w), v[2] = make_float2(b.x, b.y), v[3] = make_float2(b.z, b.w);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (k + e >= 0 && k + e < ref_len) ? __ldg(&ref[k + e]) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t d0r, d1r, d0i, d1i;
        const uint32_t sr = dig(v[e].x, d0r, d1r), si = dig(csign * v[e].y, d0i, d1i);
        w[0][h] |= d0r << (8 * e), w[1][h] |= d1r << (8 * e);
        w[2][h] |= d0i << (8 * e), w[3][h] |= d1i << (8 * e);
        w[4][h] |= sr << (8 * e), w[5][h] |= si << (8 * e);
      }
    }
#pragma unroll
    for (int p = 0; p < NPL; ++p)
      *(uint4 *)(planes + p * cpl + 16 * x16) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
  }
}

#ifndef SA_LAGI8_NB
#define SA_LAGI8_NB 4  // B chunk ring depth
#endif
#ifndef SA_LAGI8_NACC
#define SA_LAGI8_NACC 1  // accumulator sets in TMEM (2: the epilogue of pass p overlaps pass p + 1; 512 columns)
#endif
constexpr int NB = SA_LAGI8_NB;
constexpr int NACC = SA_LAGI8_NACC;

#define SA_LD8(v, taddr)                                                                                \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                  \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),    \
                 "=r"(v[7])                                                                             \
               : "r"(taddr))
SA_HD void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sa_smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(sa_smem_u32(bar))
               : "memory");
}

// Warp roles: 0-3 epilogue (TMEM lanes 0-127), 4-7 B builders, 8 MMA issuer, 9
// producer (bulk copies of the A windows, double-buffered per lag-group pass).
constexpr int NWARPS = 10;
constexpr int WB0 = 4, WMMA = 8, WPROD = 9;

template <int MR, bool BLK>
__global__ void __launch_bounds__(NWARPS * 32, 2)
    k_lag_i8(const unsigned char *__restrict__ splanes, const int *__restrict__ es_in, const float *__restrict__ mc_in,
             int64_t l0g, int64_t l_count, int64_t m, int tb, const unsigned char *__restrict__ cplanes, int64_t guard,
             int64_t cpl, float2 *__restrict__ z, int64_t q0, LagDst dst) {
  sa_pdl_trigger();  // the Doppler launch may become resident while the last wave drains
  sa_pdl_wait();     // the planes, exponents and scales of k_lag_cprep
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const Geo gm = geo(tb, MR, 2);
  const int bbytes = B_BYTES;
  unsigned char *Ps = smem;               // NPL x psl: s planes, x = t + 16
  unsigned char *Pc = smem + gm.off_pc;   // 2 x NPL x pcl: A windows (double-buffered)
  unsigned char *Bb = smem + gm.off_b;    // NB x B_BYTES
  uint64_t *bfull = (uint64_t *)(Bb + NB * bbytes);
  uint64_t *bempty = bfull + NB;
  uint64_t *afull = bempty + NB;
  uint64_t *aempty = afull + 2;
  uint64_t *tfull = aempty + 2;
  uint64_t *tempty = tfull + NACC;
  uint64_t *psfull = tempty + NACC;                    // the block's s planes landed
  uint32_t *tmem_holder = (uint32_t *)(psfull + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t q = q0 + blockIdx.x;
  constexpr int LGRP = 16 * MR;  // lags per group (one pass)
  constexpr int TMEM_COLS = 256 * NACC;
  if (tid == 0) TS(0);

  if (tid == 0) {
    for (int i = 0; i < NB; ++i) sa_mbar_init(&bfull[i], 4), sa_mbar_init(&bempty[i], 1);
    for (int i = 0; i < 2; ++i) sa_mbar_init(&afull[i], 1), sa_mbar_init(&aempty[i], 1);
    for (int i = 0; i < NACC; ++i) sa_mbar_init(&tfull[i], 1), sa_mbar_init(&tempty[i], 4);
    sa_mbar_init(psfull, 1);
    sa_fence_mbar_init();
  }
  __syncthreads();
  // exponents from the prep launch (sprep_block): this block's (INT_MAX: non-finite) and the reference maximum
  const int es_raw = es_in[blockIdx.x];
  const float mc = *mc_in;
  const bool bad = es_raw == INT_MAX || !(mc <= FLT_MAX);
  const int es = es_raw == INT_MAX ? 0 : es_raw, ec = exponent_of(mc);

  const int64_t lalign = l0g - (l0g & 15);
  const int npass = (int)((l0g - lalign + l_count + LGRP - 1) / LGRP);
  const int nch = (gm.ks + KC - 1) / KC;
  auto cstart = [&](int pi) { return q * tb - (lalign + (int64_t)pi * LGRP) - 16 * MR; };  // c index of x = 0

  // ---- producer: the A windows (six plane segments) of each pass, two buffers; the
  // first two passes are issued here, the rest (waiting for a buffer) after the role split ----
  auto produce = [&](int pi) {
    const int a = pi & 1;
    if (pi >= 2) sa_mbar_wait(&aempty[a], ((pi >> 1) - 1) & 1);
    sa_mbar_expect_tx(&afull[a], (uint32_t)(NPL * gm.pcl));
    const unsigned char *src = cplanes + guard + cstart(pi);
#pragma unroll 1
    for (int p = 0; p < NPL; ++p)
      bulk_g2s(Pc + (a * NPL + p) * gm.pcl, src + (int64_t)p * cpl, (uint32_t)gm.pcl, &afull[a]);
  };
  if (warp == WPROD && lane == 0) {
    sa_mbar_expect_tx(psfull, (uint32_t)(NPL * gm.psl));  // the block's s planes (sprep_block), one bulk copy
    bulk_g2s(Ps, splanes + (int64_t)blockIdx.x * (NPL * gm.psl), (uint32_t)(NPL * gm.psl), psfull);
    for (int pi = 0; pi < min(2, npass); ++pi) produce(pi);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa_smem_u32(tmem_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_holder;
  if (tid == 0) TS(1);

  if (warp == WPROD) {
    if (lane == 0)
      for (int pi = 2; pi < npass; ++pi) produce(pi);
  } else if (warp == WMMA) {
    // ---- MMA issuer: the whole warp runs the (uniform) loop, so descriptors live in
    // uniform registers; one elected lane issues each K step's six MMAs ----
    constexpr uint32_t IDW = idesc(32, MR), IDX = idesc(64, MR);
    const uint32_t pcbase = sa_smem_u32(Pc), bbase = sa_smem_u32(Bb);
    const uint64_t ap = (uint64_t)(gm.pcl >> 4);  // descriptor step of one plane
    uint32_t cc = 0;
    for (int pi = 0; pi < npass; ++pi) {
      const int a = pi & 1, ab = pi % NACC;
      sa_mbar_wait(&afull[a], (pi >> 1) & 1);
      if (pi == 0 && lane == 0) TS(2);
      if (pi >= NACC) sa_mbar_wait(&tempty[ab], ((pi / NACC) - 1) & 1);
      fence_after();
      const uint32_t tm = tmem + 256 * ab;
      const uint32_t pa0 = pcbase + a * NPL * gm.pcl;
      for (int ch = 0; ch < nch; ++ch, ++cc) {
        const int b = cc % NB;
        sa_mbar_wait(&bfull[b], (cc / NB) & 1);
        if (cc == 0 && lane == 0) TS(3);
        fence_after();
        const int kn = min(KC, gm.ks - ch * KC);
        for (int kk = 0; kk < kn; ++kk) {
          const int kstep = ch * KC + kk;
          const uint32_t bo = bbase + b * B_BYTES + kk * 2 * CORE;
          const uint64_t bw = sdesc_ns(bo, CORE, B_SBO), bx = sdesc_ns(bo + 4 * B_SBO, CORE, B_SBO);
          const uint64_t a0 = sdesc_ns(pa0 + 32 * kstep, 16, 128);
          asm volatile(
              "{\n .reg .pred e, p;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %12, 0;\n"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %6, %10, %13, p;\n"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%1], %7, %10, %13, p;\n"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%2], %8, %10, %13, p;\n"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%3], %9, %10, %13, p;\n"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%4], %14, %11, %15, p;\n"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%5], %16, %11, %15, p;\n}\n" ::"r"(tm),
              "r"(tm + 32), "r"(tm + 64), "r"(tm + 96), "r"(tm + 128), "r"(tm + 192), "l"(a0), "l"(a0 + ap),
              "l"(a0 + 2 * ap), "l"(a0 + 3 * ap), "l"(bw), "l"(bx), "r"((uint32_t)(kstep != 0)), "r"(IDW),
              "l"(a0 + 4 * ap), "r"(IDX), "l"(a0 + 5 * ap)
              : "memory");
        }
        if (elect_one()) commit(&bempty[b]);
        __syncwarp();
      }
      if (elect_one()) {
        commit(&aempty[a]);
        commit(&tfull[ab]);
      }
      if (lane == 0) TS(4);
      __syncwarp();
    }
  } else if (warp >= WB0 && warp < WB0 + 4) {
    // ---- builders: B chunk = 16 shifts of the six s planes, 16-B pieces ----
    const int bt = tid - WB0 * 32;
    sa_mbar_wait(psfull, 0);  // the block's s planes landed
    uint32_t cc = 0;
    for (int pi = 0; pi < npass; ++pi) {
      for (int ch = 0; ch < nch; ++ch, ++cc) {
        const int b = cc % NB;
        if (cc >= NB) sa_mbar_wait(&bempty[b], ((cc / NB) - 1) & 1);  // MMAs that read this slot are done
        unsigned char *B = Bb + b * bbytes;
#pragma unroll
        for (int it = 0; it < NPL * 16 * 2 * KC / 128; ++it) {
          const int e = it * 128 + bt;
          const int i = e & 15, kc2 = (e >> 4) & (2 * KC - 1), p = e >> 4 >> 3;  // shift, K core, plane
          if (ch * KC + (kc2 >> 1) < gm.ks) {
            const int x0 = 32 * ch * KC + 16 * kc2 + i;  // plane byte of B[i][u0]
            const uint32_t *P32 = (const uint32_t *)(Ps + p * gm.psl) + (x0 >> 2);
            const uint32_t sh = (uint32_t)(x0 & 3) * 8;
            const uint32_t a0 = P32[0], a1 = P32[1], a2 = P32[2], a3 = P32[3], a4 = P32[4];
            const uint4 o = make_uint4(__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh),
                                       __funnelshift_r(a2, a3, sh), __funnelshift_r(a3, a4, sh));
            *(uint4 *)(B + ((p * 2 + (i >> 3)) * (2 * KC) + kc2) * CORE + (i & 7) * 16) = o;
          }
        }
        sa_fence_proxy_async();
        __syncwarp();
        if (lane == 0) sa_mbar_arrive_local(&bfull[b]);
      }
    }
  } else if (warp < 4) {
    // ---- epilogue: drain each pass's accumulators; lane = row r, lags of one blocked tile ----
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
    const int r = MR == 128 ? warp * 32 + lane : warp * 16 + (lane & 15);
    const bool live = MR == 128 || lane < 16;  // M = 64: lanes 16-31 hold no rows
    const double cw = ldexp(DSC, ec), cx = ldexp(DSC, es);
    for (int pi = 0; pi < npass; ++pi) {
      const int ab = pi % NACC;
      sa_mbar_wait(&tfull[ab], (pi / NACC) & 1);
      if (warp == 0 && lane == 0) TS(5);
      fence_after();
      const uint32_t gc = ta + 256 * ab;
      const int64_t lag0 = lalign + (int64_t)pi * LGRP + 16 * (MR - 1 - r);  // lags lag0 + [0, 16) of block q
      const bool tile_in = BLK ? (lag0 + 16 > l0g && lag0 < l0g + l_count) : true;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {  // shifts 8h .. 8h + 7
        const uint32_t g8 = gc + 8 * h;
        uint32_t u[8], v[8];
        int iw[8], ix[8];
        float re[8], im[8];
        SA_LD8(u, g8 + 0);   SA_LD8(v, g8 + 32);  tm_wait();  // W0r[sr], W1r[sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] = 254 * (int)u[k] + (int)v[k];
        SA_LD8(u, g8 + 80);  SA_LD8(v, g8 + 112); tm_wait();  // W0i[si], W1i[si]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] -= 254 * (int)u[k] + (int)v[k];
        SA_LD8(u, g8 + 128); SA_LD8(v, g8 + 160); tm_wait();  // Xr[d0sr], Xr[d1sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) ix[k] = 254 * (int)u[k] + (int)v[k];
        SA_LD8(u, g8 + 208); SA_LD8(v, g8 + 240); tm_wait();  // Xi[d0si], Xi[d1si]
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          ix[k] -= 254 * (int)u[k] + (int)v[k];
          re[k] = bad ? CUDART_NAN_F : (float)((double)iw[k] * cw + (double)ix[k] * cx);
        }
        SA_LD8(u, g8 + 16);  SA_LD8(v, g8 + 48);  tm_wait();  // W0r[si], W1r[si]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] = 254 * (int)u[k] + (int)v[k];
        SA_LD8(u, g8 + 64);  SA_LD8(v, g8 + 96);  tm_wait();  // W0i[sr], W1i[sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] += 254 * (int)u[k] + (int)v[k];
        SA_LD8(u, g8 + 144); SA_LD8(v, g8 + 176); tm_wait();  // Xr[d0si], Xr[d1si]
#pragma unroll
        for (int k = 0; k < 8; ++k) ix[k] = 254 * (int)u[k] + (int)v[k];
        SA_LD8(u, g8 + 192); SA_LD8(v, g8 + 224); tm_wait();  // Xi[d0sr], Xi[d1sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          ix[k] += 254 * (int)u[k] + (int)v[k];
          im[k] = bad ? CUDART_NAN_F : (float)((double)iw[k] * cw + (double)ix[k] * cx);
        }
        // (no divergent exit from the loop: tcgen05.ld is .sync.aligned)
        if (live && tile_in) {
          if constexpr (BLK) {
            float4 *ln = reinterpret_cast<float4 *>(dst.line(z, (lag0 - lalign) >> 4, m, q)) + 4 * h;
#pragma unroll
            for (int k = 0; k < 4; ++k) ln[k] = make_float4(re[2 * k], im[2 * k], re[2 * k + 1], im[2 * k + 1]);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int64_t row = lag0 + 8 * h + k - l0g;
              if (row >= 0 && row < l_count) *dst.row(z, row, m, q) = make_float2(re[k], im[k]);
            }
          }
        }
        __syncwarp();
      }
      fence_before();
      __syncwarp();
      if (lane == 0) sa_mbar_arrive_local(&tempty[ab]);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) TS(6);
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

template <int MR, bool BLK>
int launch_i8(const unsigned char *splanes, const int *es, const float *mc, int64_t l0, int64_t l_count, int64_t m,
              int64_t q0, int64_t q_count, int64_t tb, void *z, const LagDst &d, const unsigned char *cplanes,
              int64_t guard, int64_t cpl, cudaStream_t s) {
  const Geo gm = geo((int)tb, MR, 2);
  const int bytes = gm.off_b + NB * B_BYTES + 512 + 1024;
  static int smem_set[64] = {};  // largest smem size set per device
  int dev = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64 || smem_set[dev] < bytes) {
    SA_CUDA_TRY(cudaFuncSetAttribute(k_lag_i8<MR, BLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    if (dev < 64) smem_set[dev] = bytes;
  }
  SA_CUDA_TRY(sa_launch_pdl(k_lag_i8<MR, BLK>, dim3((unsigned)q_count), dim3(NWARPS * 32), (size_t)bytes, s,
                            (const unsigned char *)splanes, (const int *)es, (const float *)mc, l0, l_count, m, (int)tb,
                            (const unsigned char *)cplanes, guard, cpl, (float2 *)z, q0, d));
  SA_LAUNCH_CHECK();
  return SA_OK;
}

}  // namespace

static int g_lag_kind = -1;  // sa_lag_kernel: SA_LAGK_I8 / SA_LAGK_BF16
static int lag_kind_now() {
  if (g_lag_kind < 0) {
    const char *e = getenv("SA_LAG_KIND");
    g_lag_kind = (e && e[0] == 'b') ? SA_LAGK_BF16 : SA_LAGK_I8;
  }
  return g_lag_kind;
}
bool sa_lag_i8_enabled() { return lag_kind_now() == SA_LAGK_I8; }
#ifdef SA_LAG_TS
extern "C" int sa_lag_ts_read(unsigned long long *host, int n) {
  return cudaMemcpyFromSymbol(host, g_lag_ts, (size_t)n * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}
#endif
extern "C" int sa_lag_kernel(int kind) {
  const int prev = lag_kind_now();
  if (kind == SA_LAGK_I8 || kind == SA_LAGK_BF16) g_lag_kind = kind;
  return prev;
}

// Lag-group shape: MR = 128 (2048 lags per group, 24 KB of A per K step) or 64
// (1024 lags, 12 KB); per K step and group the smem operand reads (A + 8 KB of B)
// bound the MMAs (N/2 = 128 tensor cycles per group): cost = groups x bytes.
int sa_launch_lag_i8_blocks(const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count, int64_t m,
                            int64_t q0, int64_t q_count, int64_t tb, int conj, void *z, void *const *dst_rows,
                            int64_t rows_base, int64_t rows_extra, int blocked, cudaStream_t s) {
  if (l_count == 0 || q_count == 0) return SA_OK;
  if (((uintptr_t)ref & 15) != 0 || tb > 4096) return SA_ERR_UNSUPPORTED;
  const int64_t span = (l0 & 15) + l_count;
  const int64_t g128 = (span + 2047) / 2048, g64 = (span + 1023) / 1024;
  const int mr = g64 * 20 < g128 * 32 ? 64 : 128;
  const LagDst d{(float2 *const *)dst_rows, rows_base, rows_extra};
  // c planes over the windows this call's blocks read: c index = x - guard, x in [0, cpl)
  // (a block-sharded rank digitises only its own blocks' range; the exponent is
  // still that of the whole reference)
  const Geo gm = geo((int)tb, mr, 2);
  const int64_t lgrp = 16 * mr, npass = (span + lgrp - 1) / lgrp;
  const int64_t clo = q0 * tb - (l0 - (l0 & 15)) - npass * lgrp - 16 * mr - 128;  // a multiple of 16
  const int64_t chi = (q0 + q_count) * tb + gm.pcl + 128;
  const int64_t guard = -clo;
  const int64_t cpl = (chi - clo + 127) / 128 * 128;
  unsigned char *ws = nullptr;
  {
    const int rc_ = sa_scratch_alloc((void **)&ws, NPART_MAX * sizeof(float) + 16 + 4 * q_count + 15 + NPL * cpl +
                                                     q_count * NPL * gm.psl, s);
    if (rc_ != SA_OK) return rc_;
  }
  float *cpart = (float *)ws;
  float *mc = cpart + NPART_MAX;
  int *es = (int *)(mc + 4);
  unsigned char *cplanes = ws + (NPART_MAX * sizeof(float) + 16 + 4 * q_count + 15) / 16 * 16;
  unsigned char *splanes = cplanes + NPL * cpl;  // cpl and psl are multiples of 16
  int sms = 148, dev = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int npart = (int)std::max<int64_t>(1, std::min<int64_t>(4 * sms, (ref_len / 4 + 255) / 256));
  k_lag_absmax<<<npart, 256, 0, s>>>((const float2 *)ref, ref_len, cpart);
  SA_LAUNCH_CHECK();
  const int64_t nb = std::min<int64_t>((cpl / 16 + 255) / 256, 8 * sms);
  SA_CUDA_TRY(sa_launch_pdl(k_lag_cprep, dim3((unsigned)(nb + q_count)), dim3(256), (size_t)0, s, (const float2 *)ref,
                            ref_len, conj ? -1.f : 1.f, (const float *)cpart, npart, guard, cpl, cplanes, (unsigned)nb,
                            (const float2 *)surv, q0, (int)tb, gm.psl, splanes, es, mc));
  SA_LAUNCH_CHECK();
  int rc;
  if (mr == 64)
    rc = blocked ? launch_i8<64, true>(splanes, es, mc, l0, l_count, m, q0, q_count, tb, z, d, cplanes, guard, cpl, s)
                 : launch_i8<64, false>(splanes, es, mc, l0, l_count, m, q0, q_count, tb, z, d, cplanes, guard, cpl, s);
  else
    rc = blocked ? launch_i8<128, true>(splanes, es, mc, l0, l_count, m, q0, q_count, tb, z, d, cplanes, guard, cpl, s)
                 : launch_i8<128, false>(splanes, es, mc, l0, l_count, m, q0, q_count, tb, z, d, cplanes, guard, cpl, s);
  SA_CUDA_TRY(cudaFreeAsync(ws, s));
  return rc;
}
