// sa_common.cuh -- shared device arithmetic for the sign-additive (⊙) kernels.
//
// Exactness rules (SURVEY §7 "hard part 1"):
//   * compiled with -fmad=false: the only FMAs are the explicit fma() calls below;
//   * no fast-math, FTZ off (np.sign(5e-324) == 1);
//   * every real ⊗ rounds exactly once, every combining add rounds once, in the
//     reference order (operator.py:124-131);
//   * twiddles are the host reference table (transforms.py:122-133), never sincos.
//
// Real ⊗ identity used by the fast forms:  a⊗b = sgn(b)·a + sgn(a)·b.  With
// sgn(.) ∈ {-1, 0, +1} both products are exact, so fma(sgn(a), b, sgn(b)·a) is the
// correctly rounded sign(ab)(|a|+|b|) -- value-identical to the reference (signed
// zeros may differ).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#define SA_HD __device__ __forceinline__

template <typename T> struct SaVec;
template <> struct SaVec<float> {
  using c2 = float2;
  using c4 = float4;
};
template <> struct SaVec<double> {
  using c2 = double2;
  using c4 = double4;
};

// ---------------------------------------------------------------------------
// Sign helpers
// ---------------------------------------------------------------------------
// np.sign value semantics (operator.py:121): +1 / -1 / +0 for ±0.
SA_HD float sa_sgn_np(float v) { return v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f); }
SA_HD double sa_sgn_np(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// Two-instruction sign: FSET(|v| > 0) -> 1.0f/0.0f, then OR in v's sign bit.
// Value-identical to np.sign (returns -0 for -0, which only ever multiplies).
SA_HD float sa_sgn(float v) {
  float t;
  asm("set.gt.f32.f32 %0, %1, 0f00000000;" : "=f"(t) : "f"(fabsf(v)));
  return __int_as_float(__float_as_int(t) | (__float_as_int(v) & 0x80000000));
}
SA_HD double sa_sgn(double v) {
  int hi = __double2hiint(v);
  unsigned m = (fabs(v) > 0.0) ? 0x3FF00000u : 0u;
  return __hiloint2double((int)(m | ((unsigned)hi & 0x80000000u)), 0);
}

// ---------------------------------------------------------------------------
// Exact (literal) forms -- operator.py:118-131, evaluated as numpy does
// ---------------------------------------------------------------------------
SA_HD float sa_add(float a, float b) { return __fadd_rn(a, b); }
SA_HD double sa_add(double a, double b) { return __dadd_rn(a, b); }
SA_HD float sa_sub(float a, float b) { return __fsub_rn(a, b); }
SA_HD double sa_sub(double a, double b) { return __dsub_rn(a, b); }
SA_HD float sa_mul(float a, float b) { return __fmul_rn(a, b); }
SA_HD double sa_mul(double a, double b) { return __dmul_rn(a, b); }
SA_HD float sa_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
SA_HD double sa_fma(double a, double b, double c) { return __fma_rn(a, b, c); }

// sign(a)*sign(b)*(|a|+|b|) exactly as operator.py:124-125 (incl. signed zeros)
template <typename T> SA_HD T sa_mfr_literal(T a, T b) {
  return sa_mul(sa_mul(sa_sgn_np(a), sa_sgn_np(b)), sa_add(fabs(a), fabs(b)));
}

// operator.py:128-131: rr = ar⊗br − ai⊗bi ; ri = ai⊗br + bi⊗ar
template <typename T> SA_HD void sa_mfc_literal(T ar, T ai, T br, T bi, T &rr, T &ri) {
  rr = sa_sub(sa_mfr_literal(ar, br), sa_mfr_literal(ai, bi));
  ri = sa_add(sa_mfr_literal(ai, br), sa_mfr_literal(bi, ar));
}

// numpy assembles results as `rr + 1j * ri` (operator.py:173, ambiguity.py:155):
// imag = +0 + ri (so -0 becomes +0), real = rr + (0*ri - 0).  Emulated so the
// elementwise drop-ins are byte-identical, signed zeros included.
template <typename T> SA_HD void sa_np_complex(T rr, T ri, T &re, T &im) {
  re = sa_add(rr, sa_sub(sa_mul(T(0), ri), T(0)));
  im = sa_add(ri, T(0));
}

// numpy's complex absolute value on the reference host (SIMD loop, verified
// bit-exact in tests/golden/make_golden.py): L = max(|re|,|im|), S = min,
// r = S/L (0 when L == 0), |v| = sqrt(fma(r, r, 1)) * L.
template <typename T> SA_HD T np_cabs(T re, T im) {
  re = fabs(re);
  im = fabs(im);
  const T inf = T(INFINITY);
  if (re == inf || im == inf) return inf;
  if (re != re || im != im) return T(NAN);
  const T L = re > im ? re : im, S = re > im ? im : re;
  const T r = (L == T(0)) ? T(0) : S / L;
  return sqrt(fma(r, r, T(1))) * L;
}

// numpy complex multiply a*b as the reference host's SIMD loop computes it
// (verified bit-exact, oracle/signadd_oracle.c or_npmul):
//   re = fma(ar, br, -(ai*bi)),  im = fma(ar, bi, ai*br)
// Used by the exact-multiply variants: fft_exact (transforms.py:212) and
// lag_product_exact (ambiguity.py:134-143).
template <typename T> SA_HD void sa_npmul(T ar, T ai, T br, T bi, T &rr, T &ri) {
  const T p = sa_mul(ai, bi), q = sa_mul(ai, br);
  rr = sa_fma(ar, br, -p);
  ri = sa_fma(ar, bi, q);
}

// Same value, identity form with precomputed signs (sa = sgn(a) etc.)
template <typename T> SA_HD T sa_mfr_id(T a, T sa, T b, T sb) { return sa_fma(sa, b, sa_mul(sb, a)); }

template <typename T>
SA_HD void sa_mfc_id(T ar, T ai, T sar, T sai, T br, T bi, T sbr, T sbi, T &rr, T &ri) {
  rr = sa_sub(sa_mfr_id(ar, sar, br, sbr), sa_mfr_id(ai, sai, bi, sbi));
  ri = sa_add(sa_mfr_id(ai, sai, br, sbr), sa_mfr_id(bi, sbi, ar, sar));
}

// ---------------------------------------------------------------------------
// Twiddle-split form for the NL-FFT: w = (wr, wi) given as A=|wr|, B=|wi|,
// s=sgn(wr), t=sgn(wi).  Computes w ⊗ b, value-identical to operator.py:128-131:
//   wr⊗br = s·(sgn(br)·A + br)   wi⊗bi = t·(sgn(bi)·B + bi)
//   wi⊗br = t·(sgn(br)·B + br)   bi⊗wr = s·(sgn(bi)·A + bi)
//   rr = s·P1 − t·P2 ;  ri = t·P3 + s·P4      (products by s,t are exact)
// 8 FP instructions + 2 signs.
// ---------------------------------------------------------------------------
template <typename T>
SA_HD void sa_tw_mul(T A, T B, T s, T t, T br, T bi, T &rr, T &ri) {
  T sbr = sa_sgn(br), sbi = sa_sgn(bi);
  T p1 = sa_fma(sbr, A, br);
  T p2 = sa_fma(sbi, B, bi);
  T p3 = sa_fma(sbr, B, br);
  T p4 = sa_fma(sbi, A, bi);
  rr = sa_fma(s, p1, -sa_mul(t, p2));
  ri = sa_fma(s, p4, sa_mul(t, p3));
}

// 1 ⊗ b (the unity twiddle of the DIT bottom stage, transforms.py:279-280):
// (sgn(br)(1+|br|) − 0⊗bi, 0⊗br + sgn(bi)(|bi|+1))
template <typename T> SA_HD void sa_one_mul(T br, T bi, T &rr, T &ri) {
  rr = sa_fma(sa_sgn(br), T(1), br);
  ri = sa_fma(sa_sgn(bi), T(1), bi);
}

SA_HD int sa_brev(int v, int bits) { return bits ? (int)(__brev((unsigned)v) >> (32 - bits)) : 0; }

SA_HD int sa_ilog2(int64_t n) { return 63 - __clzll(n); }

inline int sa_ilog2_host(int64_t n) {
  int b = 0;
  while ((int64_t(1) << (b + 1)) <= n) ++b;
  return b;
}

// read-only loads (double4 has no __ldg overload)
SA_HD float2 sa_ldg(const float2 *p) { return __ldg(p); }
SA_HD double2 sa_ldg(const double2 *p) { return __ldg(p); }
SA_HD float4 sa_ldg(const float4 *p) { return __ldg(p); }
SA_HD double4 sa_ldg(const double4 *p) {
  double2 a = __ldg(reinterpret_cast<const double2 *>(p));
  double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
  return {a.x, a.y, b.x, b.y};
}
