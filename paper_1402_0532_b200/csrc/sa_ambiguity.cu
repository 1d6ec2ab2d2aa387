// sa_ambiguity.cu -- ⊙ lag products and their block integration for the
// range-Doppler map (ambiguity.py:116-187; SURVEY §8(d) map composition).
//
//   y_l[i] = surv[i] ⊙ conj(ref[i-l])   (ref[<0] = 0, ambiguity.py:129-131,151)
//   z_l[q] = Σ_{t<T} y_l[qT + t]         (T = ns/m; T == 1 is ambiguity_eq12a)
//
// The Doppler transform of gain*z_l is sa_nlfft / sa_ndft (sa_abi.cu).
//
// FAST lag kernel (T % 8 == 0): ALU-bound correlation tiling (SURVEY §7 hard
// part 5).  One CTA = one integration block q x 64 lags (8 warps x 8 lags).
// The block's T surveillance samples and the T+63 reference samples it can see
// are staged once in smem as {re, im, sgn re, sgn im} (conjugation folded in).
// Each lane walks sub-blocks of 8 samples and holds 8 samples x 8 lags in
// registers: 8 + 15 smem loads feed 64 ⊙ = 512 FMAs (regrouped identity
// a⊗b = sgn(b)a + sgn(a)b, 8 FMA per ⊙).  Samples with i < l read zeros, which
// contribute exactly 0, so the causal edge needs no branch.  Per-lag partial
// sums are reduced across the warp with shuffles.
#include <algorithm>

#include "sa_common.cuh"
#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

template <typename T> using C2 = typename SaVec<T>::c2;
template <typename T> using C4 = typename SaVec<T>::c4;

constexpr int LAG_WARPS = 8;
constexpr int LAGS_PER_WARP = 8;
constexpr int LAGS_PER_CTA = LAG_WARPS * LAGS_PER_WARP;  // 64

__host__ __device__ __forceinline__ int pad8(int s) { return s + (s >> 3); }  // one 16B/32B pad per 8 entries

// EXACT = false: lag_product_mf (ambiguity.py:146-155); EXACT = true:
// lag_product_exact (ambiguity.py:134-143), surv * np.conj(shifted) with
// numpy's complex multiply (np.conj of the zero prefix gives imag -0).
template <typename T, bool EXACT>
__global__ void __launch_bounds__(256) k_lag_product(const C2<T> *__restrict__ surv,
                                                     const C2<T> *__restrict__ ref, int64_t n,
                                                     int64_t lag, bool conj,
                                                     C2<T> *__restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    C2<T> a = surv[i];
    T cr = T(0), ci = T(0);
    if (i >= lag) {
      C2<T> r = ref[i - lag];
      cr = r.x;
      ci = conj ? -r.y : r.y;
    } else if (EXACT && conj) {
      ci = -T(0);
    }
    C2<T> o;
    if (EXACT) {
      sa_npmul<T>(a.x, a.y, cr, ci, o.x, o.y);
    } else {
      T rr, ri;
      sa_mfc_literal<T>(a.x, a.y, cr, ci, rr, ri);  // operand order (surv, ref): :152
      sa_np_complex<T>(rr, ri, o.x, o.y);          // rr + 1j*ri (:155)
    }
    out[i] = o;
  }
}

// Exact / generic: one thread per (lag, q); every product rounded, sequential
// sum over t from +0 (identical to the oracle's composition; T == 1 -> the
// reference rows).  EXACT selects the exact-multiply lag product (eq11/eq12c).
template <typename T, bool EXACT>
__global__ void __launch_bounds__(256) k_lag_integrate_exact(
    const C2<T> *__restrict__ surv, const C2<T> *__restrict__ ref, int64_t ref_len, int64_t l0,
    int64_t l_count, int64_t m, int64_t tb, bool conj, C2<T> *__restrict__ z) {
  int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= l_count * m) return;
  int64_t l = l0 + id / m, q = id % m;
  T sr = T(0), si = T(0);
  for (int64_t t = 0; t < tb; ++t) {
    int64_t i = q * tb + t;
    C2<T> a = surv[i];
    T cr = T(0), ci = T(0);
    int64_t j = i - l;
    if (j >= 0 && j < ref_len) {
      C2<T> r = ref[j];
      cr = r.x;
      ci = conj ? -r.y : r.y;
    } else if (conj) {
      ci = -T(0);
    }
    T rr, ri;
    if (EXACT) sa_npmul<T>(a.x, a.y, cr, ci, rr, ri);
    else sa_mfc_literal<T>(a.x, a.y, cr, ci, rr, ri);
    sr = sa_add(sr, rr);
    si = sa_add(si, ri);
  }
  z[id] = {sr, si};
}

// Exact / sequential mode on smem tiles: one CTA = block q x LAGS_EXACT lags,
// one thread per lag walking the block's T samples in order from +0 -- the
// oracle's composition, value-identical -- with the surveillance block
// (broadcast reads) and the reference window staged once with signs.
constexpr int LAGS_EXACT = 256;

template <typename T, bool EXACT>
__global__ void __launch_bounds__(LAGS_EXACT) k_lag_integrate_seq(
    const C2<T> *__restrict__ surv, const C2<T> *__restrict__ ref, int64_t ref_len, int64_t l0,
    int64_t l_count, int64_t m, int tb, bool conj, C2<T> *__restrict__ z) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int win = tb + LAGS_EXACT - 1;
  C4<T> *ss = reinterpret_cast<C4<T> *>(smem_raw);  // {sr, si, sgn sr, sgn si}
  C4<T> *rs = ss + tb;                               // {cr, ci, sgn cr, sgn ci}, conj folded in
  const int64_t q = blockIdx.x;
  const int64_t lt = l0 + (int64_t)blockIdx.y * LAGS_EXACT;
  const int64_t i0 = q * tb;
  const int64_t ws = i0 - lt - (LAGS_EXACT - 1);
  for (int t = threadIdx.x; t < tb; t += blockDim.x) {
    const C2<T> a = surv[i0 + t];
    ss[t] = {a.x, a.y, sa_sgn(a.x), sa_sgn(a.y)};
  }
  for (int u = threadIdx.x; u < win; u += blockDim.x) {
    const int64_t j = ws + u;
    T cr = T(0), ci = conj ? -T(0) : T(0);
    if (j >= 0 && j < ref_len) {
      const C2<T> r = ref[j];
      cr = r.x;
      ci = conj ? -r.y : r.y;
    }
    rs[u] = {cr, ci, sa_sgn(cr), sa_sgn(ci)};
  }
  __syncthreads();
  const int l = threadIdx.x;
  if (lt + l - l0 >= l_count) return;
  const C4<T> *cw = rs + (LAGS_EXACT - 1) - l;  // sample t pairs with window slot t + 255 - l
  T sr = T(0), si = T(0);
  for (int t = 0; t < tb; ++t) {
    const C4<T> a = ss[t], c = cw[t];
    T rr, ri;
    if (EXACT) {
      sa_npmul<T>(a.x, a.y, c.x, c.y, rr, ri);
    } else {  // surv ⊙ c, operand order (surv, ref): ambiguity.py:152; identity form, one rounding each
      rr = sa_sub(sa_fma(c.z, a.x, sa_mul(a.z, c.x)), sa_fma(c.w, a.y, sa_mul(a.w, c.y)));
      ri = sa_add(sa_fma(c.z, a.y, sa_mul(a.w, c.x)), sa_fma(a.z, c.y, sa_mul(c.w, a.x)));
    }
    sr = sa_add(sr, rr);
    si = sa_add(si, ri);
  }
  z[(lt + l - l0) * m + q] = {sr, si};
}

template <typename T, bool EXACT, int NT>
__global__ void __launch_bounds__(256) k_lag_integrate_fast(
    const C2<T> *__restrict__ surv, const C2<T> *__restrict__ ref, int64_t ref_len, int64_t l0,
    int64_t l_count, int64_t m, int tb, bool conj, C2<T> *__restrict__ z) {
  constexpr int LPT = NT * LAGS_PER_CTA;  // lags staged per CTA (NT lag tiles, as k_lag_integrate_f32x2)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int win = tb + LPT - 1;
  C4<T> *ss = reinterpret_cast<C4<T> *>(smem_raw);  // surveillance block, padded
  C4<T> *rs = ss + pad8(tb) + 1;                     // reference window, padded

  const int64_t q = blockIdx.x;
  const int64_t lt0 = l0 + (int64_t)blockIdx.y * LPT;  // first lag of the CTA
  const int64_t i0 = q * tb;
  const int64_t ws = i0 - lt0 - (LPT - 1);  // global ref index of window slot 0

  // Prologue: PF loads in flight per thread (all issued before the first use).
  constexpr int PF = 8;
  for (int s0 = threadIdx.x; s0 < tb; s0 += PF * blockDim.x) {
    C2<T> a[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u)
      if (s0 + u * (int)blockDim.x < tb) a[u] = sa_ldg(&surv[i0 + s0 + u * blockDim.x]);
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int s = s0 + u * blockDim.x;
      if (s < tb) ss[pad8(s)] = {a[u].x, a[u].y, sa_sgn(a[u].x), sa_sgn(a[u].y)};
    }
  }
  for (int s0 = threadIdx.x; s0 < win; s0 += PF * blockDim.x) {
    C2<T> r[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int64_t j = ws + s0 + u * blockDim.x;
      r[u] = {T(0), T(0)};
      if (s0 + u * (int)blockDim.x < win && j >= 0 && j < ref_len) r[u] = sa_ldg(&ref[j]);
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int s = s0 + u * blockDim.x;
      const T cr = r[u].x, ci = conj ? -r[u].y : r[u].y;
      if (s < win) rs[pad8(s)] = {cr, ci, sa_sgn(cr), sa_sgn(ci)};
    }
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int k = 0; k < NT; ++k) {  // lag tile k: window offset (NT-1-k)*64, a multiple of 8 (pad8-safe)
  const int64_t lw = lt0 + k * LAGS_PER_CTA + warp * LAGS_PER_WARP;  // first lag of this warp
  if (lw - l0 >= l_count) break;  // whole warp past the last row (warp-uniform; no barrier follows)

  T accr[LAGS_PER_WARP], acci[LAGS_PER_WARP];
#pragma unroll
  for (int j = 0; j < LAGS_PER_WARP; ++j) accr[j] = acci[j] = T(0);

  const int nsb = tb >> 3;
  for (int sb = lane; sb < nsb; sb += 32) {
    const int t0 = sb * 8;
    C4<T> a[8], c[15];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ss[pad8(t0 + i)];
    // window index of (sample t0+i, lag lw+j) = t0 + 63 - 8*warp - j + i
    const int base = (NT - 1 - k) * LAGS_PER_CTA + t0 + (LAGS_PER_CTA - 1) - LAGS_PER_WARP * warp -
                     (LAGS_PER_WARP - 1);
#pragma unroll
    for (int u = 0; u < 15; ++u) c[u] = rs[pad8(base + u)];
    // Consecutive FMAs share the surveillance operand (register-reuse cache)
    // and walk the 8 lags; per lag the terms add in the order
    //   Re: scr*sr, ssr*cr, -sci*si, -ssi*ci ;  Im: scr*si, ssi*cr, ssr*ci, sci*sr.
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const C4<T> &s = a[i];  // {sr, si, sgn sr, sgn si}; reference c[i-j+7] = {cr, ci, sgn cr, sgn ci}
      if constexpr (EXACT) {  // s * c: Re += sr*cr - si*ci ; Im += sr*ci + si*cr (4 FMA)
#pragma unroll
        for (int j = 0; j < LAGS_PER_WARP; ++j) {
          accr[j] = sa_fma(s.x, c[i - j + 7].x, accr[j]);
          acci[j] = sa_fma(s.x, c[i - j + 7].y, acci[j]);
        }
#pragma unroll
        for (int j = 0; j < LAGS_PER_WARP; ++j) {
          accr[j] = sa_fma(-s.y, c[i - j + 7].y, accr[j]);
          acci[j] = sa_fma(s.y, c[i - j + 7].x, acci[j]);
        }
        continue;
      }
#pragma unroll
      for (int j = 0; j < LAGS_PER_WARP; ++j) {
        accr[j] = sa_fma(s.x, c[i - j + 7].z, accr[j]);
        acci[j] = sa_fma(s.y, c[i - j + 7].z, acci[j]);
      }
#pragma unroll
      for (int j = 0; j < LAGS_PER_WARP; ++j) {
        accr[j] = sa_fma(s.z, c[i - j + 7].x, accr[j]);
        acci[j] = sa_fma(s.w, c[i - j + 7].x, acci[j]);
      }
#pragma unroll
      for (int j = 0; j < LAGS_PER_WARP; ++j) {
        accr[j] = sa_fma(s.y, -c[i - j + 7].w, accr[j]);
        acci[j] = sa_fma(s.z, c[i - j + 7].y, acci[j]);
      }
#pragma unroll
      for (int j = 0; j < LAGS_PER_WARP; ++j) {
        accr[j] = sa_fma(s.w, -c[i - j + 7].y, accr[j]);
        acci[j] = sa_fma(s.x, c[i - j + 7].w, acci[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < LAGS_PER_WARP; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      accr[j] = sa_add(accr[j], __shfl_xor_sync(0xffffffffu, accr[j], o));
      acci[j] = sa_add(acci[j], __shfl_xor_sync(0xffffffffu, acci[j], o));
    }
  }
  if (lane < LAGS_PER_WARP) {
    T vr = accr[0], vi = acci[0];
#pragma unroll
    for (int j = 1; j < LAGS_PER_WARP; ++j)
      if (lane == j) {
        vr = accr[j];
        vi = acci[j];
      }
    int64_t row = lw + lane - l0;
    if (row < l_count) z[row * m + q] = {vr, vi};
  }
  }
}

// complex64, T % 16 == 0: entry e of S holds samples e and e + T/2, entry u of
// C window slots u and u + T/2, each as {x, x'}, {y, y'} (S0/C0) and the signs
// {sx, sx'}, {sy, sy'} (S1/C1), in pad8-strided float4 arrays.
#ifndef SA_LAG2_LPW  // packed kernel: lags per warp, min CTAs per SM (-D for sweeps)
#define SA_LAG2_LPW 8
#define SA_LAG2_MINB 2
#endif
#ifndef SA_LAG2_RS  // reduce-scatter epilogue (16 values per lane; -D for A/B)
#define SA_LAG2_RS (SA_LAG2_LPW == 8)
#endif
constexpr int L2_LPW = SA_LAG2_LPW;
constexpr int L2_LPC = LAG_WARPS * L2_LPW;  // lags per CTA
constexpr int L2_WIN = 8 + L2_LPW - 1;      // window pairs per 8-sample sub-block
// Each CTA stages one block + window for NT consecutive lag tiles (template
// NT, chosen per launch): the staging prologue's global loads, index math and
// sign computation (IMAD/FSET/LOP3 contending with the FFMA2 stream; ~50% of
// the warp-stall samples at NT = 1) are paid once per NT * L2_LPC lags.
// C4 lag stage: NT 1 / 2 / 4 / 8 / 16 = 0.388 / 0.369 / 0.357 / 0.353 / 0.402 ms.

// Packed pair layout views of one CTA's dynamic shared memory.
struct Lag2Smem {
  float4 *S0, *S1, *C0, *C1;
  __device__ Lag2Smem(unsigned char *base, int h, int hw) {
    S0 = reinterpret_cast<float4 *>(base);
    S1 = S0 + pad8(h) + 1;
    C0 = S1 + pad8(h) + 1;
    C1 = C0 + pad8(hw) + 1;
  }
  __host__ __device__ static size_t bytes(int h, int hw) {
    return 2 * sizeof(float4) * ((size_t)pad8(h) + 1 + pad8(hw) + 1);
  }
};

// One (block q, L2_LPC lags) tile from the staged pair layout: lag ⊙ products
// summed over the block, then the warp reduction and the store of z rows.
template <bool EXACT>
__device__ __forceinline__ void lag2_tile(const Lag2Smem &sm, int h, int64_t lt, int64_t l0, int64_t l_count,
                                          int64_t m, int64_t q, int coff, float2 *__restrict__ z) {
  using A = Ar<float>;
  using V = A::V;
  const float4 *S0 = sm.S0, *S1 = sm.S1, *C0 = sm.C0, *C1 = sm.C1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t lw = lt + warp * L2_LPW;
  if (lw - l0 >= l_count) return;  // warp-uniform; no barrier follows

  V accr[L2_LPW], acci[L2_LPW];
#pragma unroll
  for (int j = 0; j < L2_LPW; ++j) accr[j] = acci[j] = 0ull;

  const int nsb = h >> 3;
  for (int sb = lane; sb < nsb; sb += 32) {
    const int t0 = sb * 8;
    const int base = coff + t0 + (L2_LPC - 1) - L2_LPW * warp - (L2_LPW - 1);
    V cx[L2_WIN], cy[L2_WIN], cz[L2_WIN], cw[L2_WIN];  // window pairs {re}, {im}, {sgn re}, {sgn im}
#pragma unroll
    for (int u = 0; u < L2_WIN; ++u) {
      const float4 c0 = C0[pad8(base + u)];
      cx[u] = A::pack(c0.x, c0.y);
      cy[u] = A::pack(c0.z, c0.w);
      if (!EXACT) {
        const float4 c1 = C1[pad8(base + u)];
        cz[u] = A::pack(c1.x, c1.y);
        cw[u] = A::pack(c1.z, c1.w);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 s0 = S0[pad8(t0 + i)];
      const V sx = A::pack(s0.x, s0.y), sy = A::pack(s0.z, s0.w);
      if constexpr (EXACT) {  // s * c: Re += sx*cx - sy*cy ; Im += sx*cy + sy*cx (4 FFMA2 per lag)
#pragma unroll
        for (int j = 0; j < L2_LPW; ++j) accr[j] = A::fma(sx, cx[i - j + L2_LPW - 1], accr[j]);
#pragma unroll
        for (int j = 0; j < L2_LPW; ++j) acci[j] = A::fma(sx, cy[i - j + L2_LPW - 1], acci[j]);
#pragma unroll
        for (int j = 0; j < L2_LPW; ++j) accr[j] = A::fma(A::neg(sy), cy[i - j + L2_LPW - 1], accr[j]);
#pragma unroll
        for (int j = 0; j < L2_LPW; ++j) acci[j] = A::fma(sy, cx[i - j + L2_LPW - 1], acci[j]);
        continue;
      }
      const float4 s1 = S1[pad8(t0 + i)];
      const V sz = A::pack(s1.x, s1.y), sw = A::pack(s1.z, s1.w);
      // consecutive FFMA2 share the surveillance pair; per lag the terms add as
      //   Re: sx*cz, sz*cx, -sy*cw, -sw*cy ;  Im: sy*cz, sw*cx, sz*cy, sx*cw
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) accr[j] = A::fma(sx, cz[i - j + L2_LPW - 1], accr[j]);
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) acci[j] = A::fma(sy, cz[i - j + L2_LPW - 1], acci[j]);
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) accr[j] = A::fma(sz, cx[i - j + L2_LPW - 1], accr[j]);
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) acci[j] = A::fma(sw, cx[i - j + L2_LPW - 1], acci[j]);
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) accr[j] = A::fma(A::neg(sy), cw[i - j + L2_LPW - 1], accr[j]);
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) acci[j] = A::fma(sz, cy[i - j + L2_LPW - 1], acci[j]);
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) accr[j] = A::fma(A::neg(sw), cy[i - j + L2_LPW - 1], accr[j]);
#pragma unroll
      for (int j = 0; j < L2_LPW; ++j) acci[j] = A::fma(sx, cw[i - j + L2_LPW - 1], acci[j]);
    }
  }
#if SA_LAG2_RS
  // Reduce-scatter over the warp: 2*L2_LPW partial sums per lane, halved at
  // each xor level (8+4+2+1 shuffles for 16 values, + 1 for the last pair)
  // instead of a full butterfly per value (80).  Lane bits 4..1 select the
  // value; lanes l and l^1 end with the same sum.
  static_assert(L2_LPW == 8, "reduce-scatter epilogue assumes 16 values per lane");
  float v[16];
#pragma unroll
  for (int j = 0; j < L2_LPW; ++j) {
    float a, b;
    A::unpack(accr[j], a, b);
    v[2 * j] = sa_add(a, b);
    A::unpack(acci[j], a, b);
    v[2 * j + 1] = sa_add(a, b);
  }
#pragma unroll
  for (int half = 8; half >= 1; half >>= 1) {
    const bool up = lane & (half << 1);  // keep the upper half of the current values
#pragma unroll
    for (int k = 0; k < half; ++k) {
      const float keep = up ? v[k + half] : v[k], send = up ? v[k] : v[k + half];
      v[k] = sa_add(keep, __shfl_xor_sync(0xffffffffu, send, half << 1));
    }
  }
  v[0] = sa_add(v[0], __shfl_xor_sync(0xffffffffu, v[0], 1));
  if (!(lane & 1)) {
    const int idx = lane >> 1;  // value 2j + c: lag j, component c
    const int64_t row = lw + (idx >> 1) - l0;
    if (row < l_count) reinterpret_cast<float *>(z + row * m + q)[idx & 1] = v[0];
  }
#else
  float vr[L2_LPW], vi[L2_LPW];
#pragma unroll
  for (int j = 0; j < L2_LPW; ++j) {
    float a, b;
    A::unpack(accr[j], a, b);
    vr[j] = sa_add(a, b);
    A::unpack(acci[j], a, b);
    vi[j] = sa_add(a, b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      vr[j] = sa_add(vr[j], __shfl_xor_sync(0xffffffffu, vr[j], o));
      vi[j] = sa_add(vi[j], __shfl_xor_sync(0xffffffffu, vi[j], o));
    }
  }
  if (lane < L2_LPW) {
    float r = vr[0], i = vi[0];
#pragma unroll
    for (int j = 1; j < L2_LPW; ++j)
      if (lane == j) {
        r = vr[j];
        i = vi[j];
      }
    const int64_t row = lw + lane - l0;
    if (row < l_count) z[row * m + q] = {r, i};
  }
#endif
}

template <bool EXACT, int L2_NT>
__global__ void __launch_bounds__(256, SA_LAG2_MINB) k_lag_integrate_f32x2(
    const float2 *__restrict__ surv, const float2 *__restrict__ ref, int64_t ref_len, int64_t l0,
    int64_t l_count, int64_t m, int tb, bool conj, float2 *__restrict__ z) {
  constexpr int L2_LPT = L2_NT * L2_LPC;  // lags staged per CTA
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int h = tb >> 1;
  const int hw = h + L2_LPT - 1;  // window pair entries for the CTA's L2_NT lag tiles
  const Lag2Smem sm(smem_raw, h, hw);
  float4 *S0 = sm.S0, *S1 = sm.S1, *C0 = sm.C0, *C1 = sm.C1;

  const int64_t q = blockIdx.x;
  const int64_t lt = l0 + (int64_t)blockIdx.y * L2_LPT;
  const int64_t i0 = q * tb;
  const int64_t ws = i0 - lt - (L2_LPT - 1);

  constexpr int PF = 4;
  for (int e0 = threadIdx.x; e0 < h; e0 += PF * blockDim.x) {
    float2 a[PF], b[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < h) {
        a[u] = __ldg(&surv[i0 + e]);
        b[u] = __ldg(&surv[i0 + e + h]);
      }
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < h) {
        S0[pad8(e)] = {a[u].x, b[u].x, a[u].y, b[u].y};
        S1[pad8(e)] = {sa_sgn(a[u].x), sa_sgn(b[u].x), sa_sgn(a[u].y), sa_sgn(b[u].y)};
      }
    }
  }
  for (int e0 = threadIdx.x; e0 < hw; e0 += PF * blockDim.x) {
    float2 a[PF], b[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int e = e0 + u * blockDim.x;
      const int64_t j = ws + e, k = j + h;
      a[u] = b[u] = {0.f, 0.f};
      if (e < hw && j >= 0 && j < ref_len) a[u] = __ldg(&ref[j]);
      if (e < hw && k >= 0 && k < ref_len) b[u] = __ldg(&ref[k]);
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int e = e0 + u * blockDim.x;
      const float ai = conj ? -a[u].y : a[u].y, bi = conj ? -b[u].y : b[u].y;
      if (e < hw) {
        C0[pad8(e)] = {a[u].x, b[u].x, ai, bi};
        C1[pad8(e)] = {sa_sgn(a[u].x), sa_sgn(b[u].x), sa_sgn(ai), sa_sgn(bi)};
      }
    }
  }
  __syncthreads();
  // the staged block and window serve L2_NT consecutive lag tiles (tile k's
  // window starts (L2_NT-1-k)*L2_LPC entries in, a multiple of 8: pad8-safe)
#pragma unroll 1
  for (int k = 0; k < L2_NT; ++k)
    lag2_tile<EXACT>(sm, h, lt + k * L2_LPC, l0, l_count, m, q, (L2_NT - 1 - k) * L2_LPC, z);
}

template <typename T, int NT>
int launch_lag_fast(bool exact_lag, const C2<T> *surv, const C2<T> *ref, int64_t ref_len, int64_t l0,
                    int64_t l_count, int64_t m, int64_t tb, int conj, C2<T> *z, size_t bytes, cudaStream_t s) {
  constexpr int LPT = NT * LAGS_PER_CTA;
  const int64_t ltiles = (l_count + LPT - 1) / LPT;
  auto kern = exact_lag ? k_lag_integrate_fast<T, true, NT> : k_lag_integrate_fast<T, false, NT>;
  SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  for (int64_t t0 = 0; t0 < ltiles; t0 += 65535) {
    const int64_t nt = std::min<int64_t>(65535, ltiles - t0);
    kern<<<dim3((unsigned)m, (unsigned)nt), 256, bytes, s>>>(surv, ref, ref_len, l0 + t0 * LPT,
                                                             l_count - t0 * LPT, m, (int)tb, conj != 0,
                                                             z + t0 * LPT * m);
  }
  SA_LAUNCH_CHECK();
  return SA_OK;
}

template <int NT>
int launch_lag2(bool exact_lag, const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count,
                int64_t m, int64_t tb, int conj, void *z, cudaStream_t s) {
  constexpr int LPT = NT * L2_LPC;
  const int h = (int)tb / 2, hw = h + LPT - 1;
  const int64_t ltiles = (l_count + LPT - 1) / LPT;
  const size_t bytes = Lag2Smem::bytes(h, hw);
  auto k2 = exact_lag ? k_lag_integrate_f32x2<true, NT> : k_lag_integrate_f32x2<false, NT>;
  SA_CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  for (int64_t t0 = 0; t0 < ltiles; t0 += 65535) {
    const int64_t nt = std::min<int64_t>(65535, ltiles - t0);
    k2<<<dim3((unsigned)m, (unsigned)nt), 256, bytes, s>>>(
        (const float2 *)surv, (const float2 *)ref, ref_len, l0 + t0 * LPT, l_count - t0 * LPT, m, (int)tb,
        conj != 0, (float2 *)z + t0 * LPT * m);
  }
  SA_LAUNCH_CHECK();
  return SA_OK;
}

template <typename T>
int launch_integrate(int lag_kind, const void *survv, const void *refv, int64_t ns, int64_t ref_len,
                     int64_t l0, int64_t l_count, int64_t m, int conj, int mode, void *zv, cudaStream_t s) {
  const C2<T> *surv = (const C2<T> *)survv;
  const C2<T> *ref = (const C2<T> *)refv;
  C2<T> *z = (C2<T> *)zv;
  const int64_t tb = ns / m;
  if (l_count == 0 || m == 0) return SA_OK;
  const bool exact_lag = lag_kind == SA_LAG_EXACT;
  int dev = 0, sms = 148, smem_max = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  SA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SA_CUDA_TRY(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t smax = (size_t)smem_max;
  const bool tiles_ok = mode == SA_NDFT_FAST && tb % 8 == 0 && tb <= 0x3fffffff && m <= 0x7fffffff;
#ifndef SA_NO_LAG_TC
  // fast mode, complex64, T % 128 == 0: Hankel GEMM on the tcgen05 tensor cores (sa_lag_tc.cu)
  if (mode == SA_NDFT_FAST && !exact_lag && sa_lag_tc_supported(sizeof(T) == 4 ? SA_C64 : SA_C128, tb, m, survv))
    return sa_launch_lag_tc(survv, refv, ref_len, l0, l_count, m, tb, conj, zv, 0, s);
#endif

  // fast mode, complex64, T % 16 == 0: packed pair kernel.  NT is the largest of
  // 8/4/2/1 that leaves >= 3 waves of 2 CTAs per SM and fits shared memory.
  if (tiles_ok && sizeof(T) == 4 && tb % 16 == 0) {
    const int h = (int)tb / 2;
    int nt = 8;
    while (nt > 1 && ((l_count + L2_LPC * nt - 1) / (L2_LPC * nt) * m < 3 * 2 * (int64_t)sms ||
                      Lag2Smem::bytes(h, h + nt * L2_LPC - 1) > smax))
      nt >>= 1;
    if (Lag2Smem::bytes(h, h + nt * L2_LPC - 1) <= smax) switch (nt) {
        case 8: return launch_lag2<8>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, s);
        case 4: return launch_lag2<4>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, s);
        case 2: return launch_lag2<2>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, s);
        default: return launch_lag2<1>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, s);
      }
  }
  // fast mode, T % 8 == 0: scalar lag tiles, NT as above (1 CTA per SM when
  // the complex128 block + window take > 113 KB)
  auto fast_bytes = [&](int nt) {
    return sizeof(C4<T>) * ((size_t)pad8((int)tb) + 1 + pad8((int)(tb + nt * LAGS_PER_CTA - 1)) + 1);
  };
  if (tiles_ok && fast_bytes(1) <= smax) {
    int nt = 8;
    while (nt > 1) {
      const size_t b = fast_bytes(nt);
      const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(2, (int64_t)(228 * 1024) / (int64_t)(b + 1024)));
      if (b <= smax && (l_count + LAGS_PER_CTA * nt - 1) / (LAGS_PER_CTA * nt) * m >= 3 * per_sm * sms) break;
      nt >>= 1;
    }
    switch (nt) {
      case 8: return launch_lag_fast<T, 8>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, fast_bytes(8), s);
      case 4: return launch_lag_fast<T, 4>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, fast_bytes(4), s);
      case 2: return launch_lag_fast<T, 2>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, fast_bytes(2), s);
      default: return launch_lag_fast<T, 1>(exact_lag, surv, ref, ref_len, l0, l_count, m, tb, conj, z, fast_bytes(1), s);
    }
  }
  // sequential order (exact mode, or fast mode when no tile shape fits): smem
  // tiles when the block + window fit, else one thread per (lag, block)
  const size_t seq_bytes = sizeof(C4<T>) * (size_t)(2 * tb + LAGS_EXACT - 1);
  if (tb >= 8 && tb <= 0x3fffffff && seq_bytes <= smax && m <= 0x7fffffff) {
    auto kern = exact_lag ? k_lag_integrate_seq<T, true> : k_lag_integrate_seq<T, false>;
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)seq_bytes));
    const int64_t lt = (l_count + LAGS_EXACT - 1) / LAGS_EXACT;
    for (int64_t t0 = 0; t0 < lt; t0 += 65535) {
      const int64_t nt = std::min<int64_t>(65535, lt - t0);
      kern<<<dim3((unsigned)m, (unsigned)nt), LAGS_EXACT, seq_bytes, s>>>(
          surv, ref, ref_len, l0 + t0 * LAGS_EXACT, l_count - t0 * LAGS_EXACT, m, (int)tb, conj != 0,
          z + t0 * LAGS_EXACT * m);
    }
    SA_LAUNCH_CHECK();
    return SA_OK;
  }
  const int64_t tot = l_count * m;
  auto kern = exact_lag ? k_lag_integrate_exact<T, true> : k_lag_integrate_exact<T, false>;
  kern<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(surv, ref, ref_len, l0, l_count, m, tb, conj != 0, z);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

}  // namespace

int64_t sa_ambiguity_ws_bytes(int dtype, int64_t l_count, int64_t m) {
  // + 30 rows: the blocked z layout pads the call's rows to whole 16-lag tiles (sa_lag_tc.cu)
  return (l_count + 30) * m * (dtype == SA_C64 ? (int64_t)sizeof(float2) : (int64_t)sizeof(double2));
}

template <typename T>
void launch_lag_product(int lag_kind, const void *surv, const void *ref, int64_t n, int64_t lag, int conj,
                        void *out, cudaStream_t s) {
  const int g = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  auto kern = lag_kind == SA_LAG_EXACT ? k_lag_product<T, true> : k_lag_product<T, false>;
  kern<<<g, 256, 0, s>>>((const C2<T> *)surv, (const C2<T> *)ref, n, lag, conj != 0, (C2<T> *)out);
}

int sa_launch_lag_product(int dtype, int lag_kind, const void *surv, const void *ref, int64_t n,
                          int64_t ref_len, int64_t lag, int conj, void *out, cudaStream_t s) {
  (void)ref_len;
  if (n == 0) return SA_OK;
  if (dtype == SA_C64) launch_lag_product<float>(lag_kind, surv, ref, n, lag, conj, out, s);
  else launch_lag_product<double>(lag_kind, surv, ref, n, lag, conj, out, s);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

int sa_launch_lag_integrate(int dtype, int lag_kind, const void *surv, const void *ref, int64_t ns,
                            int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, int conj,
                            int mode, void *z, cudaStream_t s) {
  if (dtype == SA_C64)
    return launch_integrate<float>(lag_kind, surv, ref, ns, ref_len, l0, l_count, m, conj, mode, z, s);
  return launch_integrate<double>(lag_kind, surv, ref, ns, ref_len, l0, l_count, m, conj, mode, z, s);
}
