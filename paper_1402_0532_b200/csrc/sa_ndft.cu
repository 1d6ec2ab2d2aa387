// sa_ndft.cu -- batched N-point nonlinear DFT (transforms.py:223-251).
//
// X[k] = sum_m W^(km mod N) ⊙ x[m].
//
// EXACT mode: every ⊙ rounded as operator.py:124-131 and accumulated column by
// column from +0 in index order (transforms.py:244-246): value-identical to the
// reference.
//
// FAST mode (the batched hot path): with the identity a⊗b = sgn(b)a + sgn(a)b,
//   Re X[k] = Σ_m  sgn(xr)Wr + sgn(Wr)xr − sgn(xi)Wi − sgn(Wi)xi
//   Im X[k] = Σ_m  sgn(xr)Wi + sgn(Wi)xr + sgn(xi)Wr + sgn(Wr)xi
// i.e. 8 FP32/FP64 FMAs per ⊙ into two accumulators (SURVEY §7 hard part 6).
// Only the rounding of the sum changes (fp64: ~1e-16 relative).
//
// FAST kernel layout (CUDA cores; the north star excludes tensor cores):
//   CTA = 8 warps.  All warps share one tile of BV = 32*TB vectors; warp w owns
//   TK consecutive bins.  Lane l owns vectors l + 32*i (i < TB).  The twiddle
//   table {Wr, Wi, sWr, sWi} lives in smem and is read as a warp-wide
//   broadcast (every lane needs the same W^(km)); vector data {xr, xi, sxr, sxi}
//   is staged per chunk of NC samples into smem [m][v] (XOR-swizzled, so both
//   the transposing stores and the inner-loop loads are conflict-free) with a
//   register prefetch of the next chunk overlapping the FMA loop.
#include <algorithm>
#include <type_traits>

#include "sa_common.cuh"
#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

template <typename T> using C2 = typename SaVec<T>::c2;
template <typename T> using C4 = typename SaVec<T>::c4;

constexpr int NDFT_THREADS = 256;
constexpr int NDFT_WARPS = NDFT_THREADS / 32;
constexpr int NC = 16;  // samples per staged chunk

template <typename T> struct NdftCfg;
template <> struct NdftCfg<float> {
  static constexpr int TB = 4;  // vectors per lane
  static constexpr int TK = 8;  // bins per thread
};
#ifndef SA_D_TB  // fp64 tile (vectors per lane, bins per thread, min CTAs/SM); -D for sweeps
#define SA_D_TB 4
#define SA_D_TK 4
#define SA_D_MINB 1
#endif
template <> struct NdftCfg<double> {
  static constexpr int TB = SA_D_TB;
  static constexpr int TK = SA_D_TK;
};

SA_HD int swz(int mm, int vv) { return vv ^ ((mm >> 1) & 7); }

// EX: exact mode on the same tiles -- every ⊙ rounded as the reference does
// (each real ⊗ = one fma of exact sign products, rr/ri = one add each) and the
// accumulator advanced sequentially over m from +0: value-identical to
// transforms.py:223-251 (12 FP ops per ⊙ instead of 8).
// TB / TK: vectors per lane / bins per thread (NdftCfg; fp64 also a 1 x 4 tile for
// batches too small to fill the GPU with the 4 x 4 one).
template <typename T, bool POW2, bool TW_SMEM, bool EX, int TB = NdftCfg<T>::TB, int TK = NdftCfg<T>::TK>
__global__ void __launch_bounds__(NDFT_THREADS, sizeof(T) == 8 ? (TB == 1 ? 2 : SA_D_MINB) : 1)
    k_ndft_fast(const C2<T> *__restrict__ x, C2<T> *__restrict__ y, int64_t batch, int n,
                const C4<T> *__restrict__ quad, T gain, bool use_gain) {
  constexpr int BV = 32 * TB;               // vectors per CTA
  constexpr int BK = NDFT_WARPS * TK;       // bins per CTA
  constexpr int CHUNK = BV * NC;            // complex samples per chunk
  constexpr int PER_T = CHUNK / 2 / NDFT_THREADS;  // 2-sample loads per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C4<T> *xs = reinterpret_cast<C4<T> *>(smem_raw);  // [2][NC][BV]
  C4<T> *tws = xs + 2 * NC * BV;                    // [n] (TW_SMEM)

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v0 = (int64_t)blockIdx.y * BV;
  const int kbase = blockIdx.x * BK + warp * TK;

  if (TW_SMEM)
    for (int i = threadIdx.x; i < n; i += NDFT_THREADS) tws[i] = quad[i];

  // staging map: thread handles sample pairs (mm, mm+1) of vector vv; 8 lanes
  // cover one vector's NC=16 samples (128 B for c64, coalesced).
  auto ld_chunk = [&](int m0, C2<T> (&r)[PER_T][2]) {
#pragma unroll
    for (int q = 0; q < PER_T; ++q) {
      int e = threadIdx.x + q * NDFT_THREADS;
      int vv = e >> 3, mm = (e & 7) * 2;
      int64_t v = v0 + vv;
      int m = m0 + mm;
      C2<T> a = {T(0), T(0)}, b = {T(0), T(0)};
      if (v < batch) {
        const C2<T> *row = x + v * n;
        if (m < n) a = sa_ldg(row + m);
        if (m + 1 < n) b = sa_ldg(row + m + 1);
      }
      r[q][0] = a;
      r[q][1] = b;
    }
  };
  auto st_chunk = [&](int buf, C2<T> (&r)[PER_T][2]) {
    C4<T> *dst = xs + buf * NC * BV;
#pragma unroll
    for (int q = 0; q < PER_T; ++q) {
      int e = threadIdx.x + q * NDFT_THREADS;
      int vv = e >> 3, mm = (e & 7) * 2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        C2<T> a = r[q][h];
        if (use_gain) {
          a.x = sa_mul(gain, a.x);
          a.y = sa_mul(gain, a.y);
        }
        dst[(mm + h) * BV + swz(mm + h, vv)] = {a.x, a.y, sa_sgn(a.x), sa_sgn(a.y)};
      }
    }
  };

  T accr[TK][TB], acci[TK][TB];
#pragma unroll
  for (int kk = 0; kk < TK; ++kk)
#pragma unroll
    for (int i = 0; i < TB; ++i) accr[kk][i] = acci[kk][i] = T(0);

  int idx[TK];  // (k*m) mod n for the current m
  int kst[TK];  // k mod n (bins past n are computed but never stored)
#pragma unroll
  for (int kk = 0; kk < TK; ++kk) {
    idx[kk] = 0;
    kst[kk] = (kbase + kk) % n;
  }

  const int nchunks = (n + NC - 1) / NC;
  C2<T> pre[PER_T][2];
  ld_chunk(0, pre);
  st_chunk(0, pre);
  __syncthreads();

  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    if (c + 1 < nchunks) ld_chunk((c + 1) * NC, pre);
    const C4<T> *cur = xs + buf * NC * BV;
    const int mlim = min(NC, n - c * NC);
#pragma unroll 4
    for (int mm = 0; mm < mlim; ++mm) {
      C4<T> d[TB];
#pragma unroll
      for (int i = 0; i < TB; ++i) d[i] = cur[mm * BV + swz(mm, lane + 32 * i)];
      C4<T> w[TK];
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        w[kk] = TW_SMEM ? tws[idx[kk]] : sa_ldg(&quad[idx[kk]]);
        int nx = idx[kk] + kst[kk];
        if (POW2) {
          nx &= n - 1;
        } else {
          nx = nx >= n ? nx - n : nx;
        }
        idx[kk] = nx;
      }
      // d = {xr, xi, sgn xr, sgn xi} ; w = {Wr, Wi, sgn Wr, sgn Wi}.
      if constexpr (EX) {  // rr = Wr⊗xr - Wi⊗xi ; ri = Wi⊗xr + xi⊗Wr (operator.py:128-131)
#pragma unroll
        for (int i = 0; i < TB; ++i)
#pragma unroll
          for (int kk = 0; kk < TK; ++kk) {
            const T p1 = sa_fma(w[kk].z, d[i].x, sa_mul(d[i].z, w[kk].x));
            const T p2 = sa_fma(w[kk].w, d[i].y, sa_mul(d[i].w, w[kk].y));
            const T p3 = sa_fma(w[kk].w, d[i].x, sa_mul(d[i].z, w[kk].y));
            const T p4 = sa_fma(w[kk].z, d[i].y, sa_mul(d[i].w, w[kk].x));
            accr[kk][i] = sa_add(accr[kk][i], sa_sub(p1, p2));
            acci[kk][i] = sa_add(acci[kk][i], sa_add(p3, p4));
          }
        continue;
      }
      // Consecutive FMAs share the data operand (register-reuse cache, see the
      // f32x2 kernel); per accumulator the terms add in the same order as before.
#pragma unroll
      for (int i = 0; i < TB; ++i) {
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = sa_fma(d[i].z, w[kk].x, accr[kk][i]);
          acci[kk][i] = sa_fma(d[i].z, w[kk].y, acci[kk][i]);
        }
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = sa_fma(d[i].x, w[kk].z, accr[kk][i]);
          acci[kk][i] = sa_fma(d[i].x, w[kk].w, acci[kk][i]);
        }
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = sa_fma(d[i].w, -w[kk].y, accr[kk][i]);
          acci[kk][i] = sa_fma(d[i].w, w[kk].x, acci[kk][i]);
        }
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = sa_fma(d[i].y, -w[kk].w, accr[kk][i]);
          acci[kk][i] = sa_fma(d[i].y, w[kk].z, acci[kk][i]);
        }
      }
    }
    if (c + 1 < nchunks) st_chunk(buf ^ 1, pre);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < TB; ++i) {
    int64_t v = v0 + lane + 32 * i;
    if (v >= batch) continue;
    C2<T> *row = y + v * n;
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      int k = kbase + kk;
      if (k < n) row[k] = {accr[kk][i], acci[kk][i]};
    }
  }
}


// fp32 FAST kernel with packed FFMA2: two vectors per 64-bit accumulator pair.
// Per sample m and bin k a lane issues 8 FFMA2 for its 2 vector pairs (= 16
// ⊙-accumulate lane-ops of the scalar kernel's 32 FFMA), halving issue slots so
// the FMA pipe, not instruction issue/dispatch, is the limit.  smem chunk layout
// per (m, pair p): D0 = {xr_a, xr_b, xi_a, xi_b}, D1 = {sxr_a, sxr_b, sxi_a, sxi_b}.
// sample-loop unroll of the fp32 tile loop: fast 1 / 2 / 4 / 8 = 21.46 / 21.51 /
// 22.04 / 21.53 ms, exact 26.99 / 27.71 / 27.37 / 26.91 ms (C2)
#ifndef SA_F2_UNROLL_FAST
#define SA_F2_UNROLL_FAST 1
#define SA_F2_UNROLL_EXACT 8
#endif
constexpr int F2_UNR_FAST = SA_F2_UNROLL_FAST, F2_UNR_EXACT = SA_F2_UNROLL_EXACT;
#ifndef SA_F2_CPA  // stage chunks by cp.async into a raw smem ring (-D SA_F2_CPA=0 for A/B)
#define SA_F2_CPA 1
#endif
template <int TP_, int TK_, int NC_> struct F2Cfg {
  static constexpr int TP = TP_;  // vector pairs per lane
  static constexpr int TK = TK_;  // bins per thread
  static constexpr int NCH = NC_; // samples per staged chunk
  static constexpr int BP = 32 * TP;            // pairs per CTA
  static constexpr int BV = 2 * BP;             // vectors per CTA
  static constexpr int BK = NDFT_WARPS * TK;    // bins per CTA
  static constexpr size_t STAGE_BYTES =
      2 * 2 * NCH * BP * sizeof(float4) + (SA_F2_CPA ? 2 * BV * NCH * sizeof(float2) : 0);
};
// Two tiles.  Large n (>= 256): 128 vectors x 128 bins per CTA, 16 bins per
// thread, 16-sample chunks, 1 CTA/SM (250 registers): C2 fast 20.0 ms, exact
// 26.5 ms.  Small n: 128 x 64, 8 bins per thread, 8-sample chunks, 2 CTAs/SM
// (128 registers; 21.5 / 26.9 ms at C2), so n = 64 wastes no bins.  Sweep of
// (pairs/lane, bins/thread, chunk, CTAs/SM) at C2: (2,16,16,1) 20.0,
// (2,16,8,1) 20.4, (2,16,32,1) 20.5, (4,8,8,1) 21.0, (2,8,8,2) 21.5,
// (2,12,8,1) 22.5, (4,8,16,1) 24.4 ms.
#ifndef SA_F2_TP  // large-n tile shape (vector pairs per lane, bins per thread, chunk, CTAs/SM); -D for sweeps
#define SA_F2_TP 2
#define SA_F2_TK 16
#define SA_F2_NC 16
#define SA_F2_MINB 1
#endif
using F2Big = F2Cfg<SA_F2_TP, SA_F2_TK, SA_F2_NC>;
using F2Small = F2Cfg<2, 8, 8>;
constexpr int F2BIG_MINB = SA_F2_MINB, F2SMALL_MINB = 2;
constexpr int F2_BIG_MIN_N = 256;
#ifndef SA_F2_CHAIN  // chained twiddle offsets in exact mode (-D SA_F2_CHAIN=0 for A/B)
#define SA_F2_CHAIN 1
#endif
template <class F2, int MINB, bool POW2, bool TW_SMEM, bool EX>
__global__ void __launch_bounds__(NDFT_THREADS, MINB)
    k_ndft_fast_f32x2(const float2 *__restrict__ x, float2 *__restrict__ y, int64_t batch, int n,
                      const float4 *__restrict__ quad, float gain, bool use_gain) {
  using A = Ar<float>;
  using V = A::V;
  constexpr int TP = F2::TP, TK = F2::TK, NCH = F2::NCH, BP = F2::BP, BV = F2::BV, BK = F2::BK;
  constexpr int PER_T = BP * NCH / NDFT_THREADS;  // (pair, m) loads per thread per chunk
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4 *d0 = reinterpret_cast<float4 *>(smem_raw);  // [2][NCH][BP] {xr_a, xr_b, xi_a, xi_b}
  float4 *d1 = d0 + 2 * NCH * BP;                      // [2][NCH][BP] signs
  float2 *raw = reinterpret_cast<float2 *>(d1 + 2 * NCH * BP);  // [2][NCH][BV] (SA_F2_CPA)
  float4 *tws = SA_F2_CPA ? reinterpret_cast<float4 *>(raw + 2 * BV * NCH) : d1 + 2 * NCH * BP;  // [n]
  const unsigned char *twb = reinterpret_cast<const unsigned char *>(tws);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v0 = (int64_t)blockIdx.y * BV;
  const int kbase = blockIdx.x * BK + warp * TK;
  if (TW_SMEM)
    for (int i = threadIdx.x; i < n; i += NDFT_THREADS) tws[i] = quad[i];

  auto ld_chunk = [&](int m0, float2 (&r)[PER_T][2]) {
#pragma unroll
    for (int q = 0; q < PER_T; ++q) {
      int e = threadIdx.x + q * NDFT_THREADS;
      int p = e % BP, mm = e / BP;
      int m = m0 + mm;
      float2 a = {0.f, 0.f}, b = {0.f, 0.f};
      int64_t va = v0 + 2 * p;
      if (m < n) {
        if (va < batch) a = __ldg(x + va * n + m);
        if (va + 1 < batch) b = __ldg(x + (va + 1) * n + m);
      }
      r[q][0] = a;
      r[q][1] = b;
    }
  };
  auto st_chunk = [&](int buf, float2 (&r)[PER_T][2]) {
#pragma unroll
    for (int q = 0; q < PER_T; ++q) {
      int e = threadIdx.x + q * NDFT_THREADS;
      int p = e % BP, mm = e / BP;
      float2 a = r[q][0], b = r[q][1];
      if (use_gain) {
        a = {sa_mul(gain, a.x), sa_mul(gain, a.y)};
        b = {sa_mul(gain, b.x), sa_mul(gain, b.y)};
      }
      d0[(buf * NCH + mm) * BP + p] = {a.x, b.x, a.y, b.y};
      d1[(buf * NCH + mm) * BP + p] = {sa_sgn(a.x), sa_sgn(b.x), sa_sgn(a.y), sa_sgn(b.y)};
    }
  };

  V accr[TK][TP], acci[TK][TP];
#pragma unroll
  for (int kk = 0; kk < TK; ++kk)
#pragma unroll
    for (int i = 0; i < TP; ++i) accr[kk][i] = acci[kk][i] = 0ull;
  const int nb = n * (int)sizeof(float4);
  // Twiddle byte offsets (k*m mod n) * 16.  Fast mode keeps one per bin, each
  // stepped by k*16 per sample, so the twiddle loads' addresses are ready a
  // sample ahead (21.8 ms at C2).  Exact mode keeps two -- off0 for k = kbase
  // and m16 = (m mod n)*16 -- and forms bin kbase+kk by a chain of kk adds: the
  // per-bin table spilled its 12-op-per-⊙ loop (37.0 -> 27.7 ms at C2), while
  // the chain costs fast mode 2 ms.
  constexpr bool CHAIN = EX && SA_F2_CHAIN;
  constexpr int UNR = EX ? F2_UNR_EXACT : F2_UNR_FAST;
  int off[TK], kst[TK];
#pragma unroll
  for (int kk = 0; kk < TK; ++kk) {
    off[kk] = 0;
    kst[kk] = CHAIN ? 0 : ((kbase + kk) % n) * (int)sizeof(float4);
  }
  int off0 = 0, m16 = 0;
  const int kst0 = (kbase % n) * (int)sizeof(float4);
  const int nchunks = (n + NCH - 1) / NCH;
  // Fast mode stages by cp.async (21.8 -> 21.5 ms at C2); exact mode keeps the
  // register prefetch (27.7 vs 27.9 ms).
  constexpr bool CPA = SA_F2_CPA && !EX;
  float2 pre[PER_T][2];
  // cp.async ring: each thread copies, then converts, its own (pair, sample
  // pair) entries, so only the chunk barrier orders the smem traffic.  Chunk j
  // lands in raw[j & 1] two chunks ahead of use; no prefetch registers.
  constexpr int PER_C = BP * NCH / 2 / NDFT_THREADS;  // (pair, sample pair) items per thread
  static_assert(NCH % 2 == 0 && BP * NCH / 2 % NDFT_THREADS == 0, "cp.async staging tiles");
  auto issue = [&](int j) {
    if (j < nchunks) {
      const int m0 = j * NCH, rb = j & 1;
#pragma unroll
      for (int q = 0; q < PER_C; ++q) {
        const int e = threadIdx.x + q * NDFT_THREADS, p = e % BP, sp = e / BP;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t gv = v0 + 2 * p + h;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int m = m0 + 2 * sp + t;
            const bool ok = gv < batch && m < n;
            sa_cp_async8(&raw[(rb * NCH + 2 * sp + t) * BV + 2 * p + h], ok ? x + gv * n + m : x, ok ? 8 : 0);
          }
        }
      }
    }
    sa_cp_async_commit();
  };
  auto convert = [&](int j) {
    const int rb = j & 1;
#pragma unroll
    for (int q = 0; q < PER_C; ++q) {
      const int e = threadIdx.x + q * NDFT_THREADS, p = e % BP, sp = e / BP;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int mm = 2 * sp + t;
        const float4 ab = reinterpret_cast<const float4 *>(raw)[((rb * NCH + mm) * BV + 2 * p) / 2];
        float2 a = {ab.x, ab.y}, b = {ab.z, ab.w};
        if (use_gain) {
          a = {sa_mul(gain, a.x), sa_mul(gain, a.y)};
          b = {sa_mul(gain, b.x), sa_mul(gain, b.y)};
        }
        d0[(rb * NCH + mm) * BP + p] = {a.x, b.x, a.y, b.y};
        d1[(rb * NCH + mm) * BP + p] = {sa_sgn(a.x), sa_sgn(b.x), sa_sgn(a.y), sa_sgn(b.y)};
      }
    }
  };
  if constexpr (CPA) {
    issue(0);
    issue(1);
    sa_cp_async_wait<1>();
    convert(0);
  } else {
    ld_chunk(0, pre);
    st_chunk(0, pre);
  }
  __syncthreads();
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    if constexpr (CPA) issue(c + 2);  // into raw[c & 1], converted by this thread last iteration
    else if (c + 1 < nchunks) ld_chunk((c + 1) * NCH, pre);
    const float4 *c0 = d0 + buf * NCH * BP;
    const float4 *c1 = d1 + buf * NCH * BP;
    const int mlim = min(NCH, n - c * NCH);
#pragma unroll UNR
    for (int mm = 0; mm < mlim; ++mm) {
      V xr[TP], xi[TP], sr[TP], si[TP];
#pragma unroll
      for (int i = 0; i < TP; ++i) {
        float4 a = c0[mm * BP + lane + 32 * i];
        float4 b = c1[mm * BP + lane + 32 * i];
        xr[i] = A::pack(a.x, a.y);
        xi[i] = A::pack(a.z, a.w);
        sr[i] = A::pack(b.x, b.y);
        si[i] = A::pack(b.z, b.w);
      }
      float4 w[TK];
      if constexpr (CHAIN) {
        int o = off0;
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          w[kk] = TW_SMEM ? *reinterpret_cast<const float4 *>(twb + o)
                          : __ldg(reinterpret_cast<const float4 *>(
                                reinterpret_cast<const unsigned char *>(quad) + o));
          o += m16;
          if (POW2) o &= nb - 1;
          else o = o >= nb ? o - nb : o;
        }
        int nx = off0 + kst0, nm = m16 + (int)sizeof(float4);
        if (POW2) {
          nx &= nb - 1;
          nm &= nb - 1;
        } else {
          nx = nx >= nb ? nx - nb : nx;
          nm = nm >= nb ? nm - nb : nm;
        }
        off0 = nx;
        m16 = nm;
      } else {
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        w[kk] = TW_SMEM ? *reinterpret_cast<const float4 *>(twb + off[kk])
                        : __ldg(reinterpret_cast<const float4 *>(
                              reinterpret_cast<const unsigned char *>(quad) + off[kk]));
        int nx = off[kk] + kst[kk];
        if (POW2) nx &= nb - 1;
        else nx = nx >= nb ? nx - nb : nx;
        off[kk] = nx;
      }
      }
      // Operand order for the register-reuse cache: consecutive FFMA2 share the
      // data pair (slot a) and differ in twiddle scalar and accumulator, so each
      // reads one 64-bit and one 32-bit register -- within the 2-cycle pipe slot.
      // Per accumulator the terms still add in the order
      //   Re: sxr*Wr, xr*sWr, -sxi*Wi, -xi*sWi ;  Im: sxr*Wi, xr*sWi, sxi*Wr, xi*sWr.
      if constexpr (EX) {  // exact ⊙ per vector pair (see k_ndft_fast): 12 packed ops
#pragma unroll
        for (int i = 0; i < TP; ++i)
#pragma unroll
          for (int kk = 0; kk < TK; ++kk) {
            const V Wr = A::pack(w[kk].x, w[kk].x), Wi = A::pack(w[kk].y, w[kk].y);
            const V sWr = A::pack(w[kk].z, w[kk].z), sWi = A::pack(w[kk].w, w[kk].w);
            const V p1 = A::fma(sWr, xr[i], A::mul(sr[i], Wr));  // Wr⊗xr
            const V p2 = A::fma(sWi, xi[i], A::mul(si[i], Wi));  // Wi⊗xi
            const V p3 = A::fma(sWi, xr[i], A::mul(sr[i], Wi));  // Wi⊗xr
            const V p4 = A::fma(sWr, xi[i], A::mul(si[i], Wr));  // xi⊗Wr
            accr[kk][i] = A::add(accr[kk][i], A::sub(p1, p2));
            acci[kk][i] = A::add(acci[kk][i], A::add(p3, p4));
          }
        continue;
      }
#pragma unroll
      for (int i = 0; i < TP; ++i) {
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = A::fma(sr[i], A::pack(w[kk].x, w[kk].x), accr[kk][i]);
          acci[kk][i] = A::fma(sr[i], A::pack(w[kk].y, w[kk].y), acci[kk][i]);
        }
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = A::fma(xr[i], A::pack(w[kk].z, w[kk].z), accr[kk][i]);
          acci[kk][i] = A::fma(xr[i], A::pack(w[kk].w, w[kk].w), acci[kk][i]);
        }
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = A::fma(si[i], A::pack(-w[kk].y, -w[kk].y), accr[kk][i]);
          acci[kk][i] = A::fma(si[i], A::pack(w[kk].x, w[kk].x), acci[kk][i]);
        }
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          accr[kk][i] = A::fma(xi[i], A::pack(-w[kk].w, -w[kk].w), accr[kk][i]);
          acci[kk][i] = A::fma(xi[i], A::pack(w[kk].z, w[kk].z), acci[kk][i]);
        }
      }
    }
    if (c + 1 < nchunks) {
      if constexpr (CPA) {
        sa_cp_async_wait<1>();  // chunk c+1 landed (c+2 may still be in flight)
        convert(c + 1);
      } else {
        st_chunk(buf ^ 1, pre);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TP; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int64_t v = v0 + 2 * (lane + 32 * i) + h;
      if (v >= batch) continue;
      float2 *row = y + v * n;
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        int k = kbase + kk;
        float r0, r1, i0, i1;
        A::unpack(accr[kk][i], r0, r1);
        A::unpack(acci[kk][i], i0, i1);
        if (k < n) row[k] = h ? make_float2(r1, i1) : make_float2(r0, i0);
      }
    }
  }
}

// Exact sequential NDFT: one thread per (vector, bin); x[m] is a warp broadcast.
template <typename T>
__global__ void __launch_bounds__(256) k_ndft_exact(const C2<T> *__restrict__ x,
                                                    C2<T> *__restrict__ y, int n,
                                                    const C2<T> *__restrict__ raw, T gain,
                                                    bool use_gain) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t v = blockIdx.y;
  const C2<T> *row = x + v * n;
  T accr = T(0), acci = T(0);
  int idx = 0;
  const int kk = k < n ? k : 0;
  for (int m = 0; m < n; ++m) {
    C2<T> xv = sa_ldg(row + m);
    if (use_gain) {
      xv.x = sa_mul(gain, xv.x);
      xv.y = sa_mul(gain, xv.y);
    }
    C2<T> w = sa_ldg(raw + idx);
    T rr, ri;
    sa_mfc_literal<T>(w.x, w.y, xv.x, xv.y, rr, ri);  // operand order (W, x): transforms.py:243
    accr = sa_add(accr, rr);
    acci = sa_add(acci, ri);
    idx += kk;
    if (idx >= n) idx -= n;
  }
  if (k < n) y[v * n + k] = {accr, acci};
}

template <class F2, int MINB>
int launch_f32x2(const float2 *x, float2 *y, int64_t batch, int n, const SaTwiddles *tw, bool exact, float g,
                 bool use_gain, cudaStream_t s) {
  const bool pow2 = (n & (n - 1)) == 0;
  const bool tw_smem = (size_t)n * sizeof(float4) <= 64 * 1024;
  const size_t bytes = F2::STAGE_BYTES + sizeof(float4) * (tw_smem ? n : 0);
  const float4 *quad = (const float4 *)tw->quad;
  const int64_t vblocks = (batch + F2::BV - 1) / F2::BV;
  const unsigned kblocks = (unsigned)((n + F2::BK - 1) / F2::BK);
  for (int64_t vb = 0; vb < vblocks; vb += 65535) {
    const int64_t nvb = std::min<int64_t>(65535, vblocks - vb);
    const dim3 grid(kblocks, (unsigned)nvb);
    const float2 *xs = x + vb * F2::BV * n;
    float2 *ys = y + vb * F2::BV * n;
    const int64_t bleft = batch - vb * F2::BV;
#define SA_NDFT_GO(P2, TS)                                                                              \
  do {                                                                                                  \
    auto kern = exact ? k_ndft_fast_f32x2<F2, MINB, P2, TS, true> : k_ndft_fast_f32x2<F2, MINB, P2, TS, false>; \
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));   \
    kern<<<grid, NDFT_THREADS, bytes, s>>>(xs, ys, bleft, n, quad, g, use_gain);                       \
  } while (0)
    if (pow2 && tw_smem) SA_NDFT_GO(true, true);
    else if (pow2) SA_NDFT_GO(true, false);
    else if (tw_smem) SA_NDFT_GO(false, true);
    else SA_NDFT_GO(false, false);
#undef SA_NDFT_GO
  }
  SA_LAUNCH_CHECK();
  return SA_OK;
}

template <typename T>
int launch(const void *xv, void *yv, int64_t batch, int64_t n64, const SaTwiddles *tw, int mode,
           double gain, cudaStream_t s) {
  const C2<T> *x = (const C2<T> *)xv;
  C2<T> *y = (C2<T> *)yv;
  const bool use_gain = gain != 1.0;
  const T g = (T)gain;
  if (batch == 0) return SA_OK;
  if (n64 > (1 << 24)) {
    sa_set_error("sa_ndft: n=%lld too large", (long long)n64);
    return SA_ERR_UNSUPPORTED;
  }
  const int n = (int)n64;
  // fp32: packed FFMA2 kernel (F2Big / F2Small tile); fp64: scalar DFMA kernel (NdftCfg tile)
  constexpr bool F32X2 = sizeof(T) == 4;
  static_assert(F2Big::BV == F2Small::BV, "both fp32 tiles take 128 vectors");
  constexpr int BV = F32X2 ? F2Big::BV : 32 * NdftCfg<T>::TB;
  // exact mode: the tiled kernels (EX) once a batch fills a tile, else one
  // thread per (vector, bin)
  const bool exact = mode == SA_NDFT_EXACT;
  if (exact && batch < BV) {
    if (batch > 65535) {
      // grid.y limit: split into slices
      for (int64_t b = 0; b < batch; b += 65535) {
        int64_t nb = std::min<int64_t>(65535, batch - b);
        dim3 grid((n + 255) / 256, (unsigned)nb);
        k_ndft_exact<T><<<grid, 256, 0, s>>>(x + b * n, y + b * n, n, (const C2<T> *)tw->raw, g,
                                             use_gain);
      }
    } else {
      dim3 grid((n + 255) / 256, (unsigned)batch);
      k_ndft_exact<T><<<grid, 256, 0, s>>>(x, y, n, (const C2<T> *)tw->raw, g, use_gain);
    }
    SA_LAUNCH_CHECK();
    return SA_OK;
  }
  if constexpr (F32X2) {
    if (n >= F2_BIG_MIN_N)
      return launch_f32x2<F2Big, F2BIG_MINB>((const float2 *)x, (float2 *)y, batch, n, tw, exact, (float)g,
                                             use_gain, s);
    return launch_f32x2<F2Small, F2SMALL_MINB>((const float2 *)x, (float2 *)y, batch, n, tw, exact, (float)g,
                                               use_gain, s);
  }
  const bool pow2 = (n & (n - 1)) == 0;
  const bool tw_smem = (size_t)n * sizeof(C4<T>) <= 64 * 1024;
  const C4<T> *quad = (const C4<T> *)tw->quad;
  auto go = [&](auto tb_, auto tk_) -> int {
    constexpr int TBv = decltype(tb_)::value, TKv = decltype(tk_)::value;
    constexpr int BVv = 32 * TBv, BK = NDFT_WARPS * TKv;
    size_t bytes = sizeof(C4<T>) * 2 * NC * BVv + sizeof(C4<T>) * (tw_smem ? n : 0);
    int64_t vblocks = (batch + BVv - 1) / BVv;
    unsigned kblocks = (unsigned)((n + BK - 1) / BK);
    for (int64_t vb = 0; vb < vblocks; vb += 65535) {
      int64_t nvb = std::min<int64_t>(65535, vblocks - vb);
      dim3 grid(kblocks, (unsigned)nvb);
      const C2<T> *xs = x + vb * BVv * n;
      C2<T> *ys = y + vb * BVv * n;
      int64_t bleft = batch - vb * BVv;
#define SA_NDFT_GO(P2, TS)                                                                              \
  do {                                                                                                  \
    auto kern = exact ? k_ndft_fast<T, P2, TS, true, TBv, TKv> : k_ndft_fast<T, P2, TS, false, TBv, TKv>; \
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));   \
    kern<<<grid, NDFT_THREADS, bytes, s>>>(xs, ys, bleft, n, quad, g, use_gain);                       \
  } while (0)
      if (pow2 && tw_smem) SA_NDFT_GO(true, true);
      else if (pow2) SA_NDFT_GO(true, false);
      else if (tw_smem) SA_NDFT_GO(false, true);
      else SA_NDFT_GO(false, false);
#undef SA_NDFT_GO
    }
    SA_LAUNCH_CHECK();
    return SA_OK;
  };
  // fp64: the 4 x 4 tile when it fills two waves of 148 SMs, else 1 x 4 (C1: 66 -> 258 CTAs)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr int BK4 = NDFT_WARPS * NdftCfg<T>::TK;
  const int64_t ctas = ((batch + BV - 1) / BV) * ((n + BK4 - 1) / BK4);
  if (ctas < 2 * (int64_t)sms) return go(std::integral_constant<int, 1>{}, std::integral_constant<int, 4>{});
  return go(std::integral_constant<int, NdftCfg<T>::TB>{}, std::integral_constant<int, NdftCfg<T>::TK>{});
}

}  // namespace

int sa_launch_ndft(int dtype, const void *x, void *y, int64_t batch, int64_t n,
                   const SaTwiddles *tw, int mode, double gain, cudaStream_t s) {
  if (dtype == SA_C64) return launch<float>(x, y, batch, n, tw, mode, gain, s);
  return launch<double>(x, y, batch, n, tw, mode, gain, s);
}
