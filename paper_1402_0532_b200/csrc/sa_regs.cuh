// sa_regs.cuh -- register-level complex ⊙ arithmetic for the NL-FFT butterflies,
// and TMA / mbarrier helpers.
//
// fp32 values live as packed {re, im} pairs in 64-bit registers and use the
// sm_100 packed instructions (fma/mul/add.rn.f32x2 -> FFMA2/FMUL2/FADD2).  ptxas
// folds the scalar broadcasts {w,w}, the pair swap {hi,lo} and the partial
// negation {t,-t} into operand modifiers, so a full DIT butterfly
//   t = w ⊙ b ; a' = a + t ; b' = a − t
// is 6 packed FP instructions + 2 two-instruction signs.  Every lane result is
// rounded exactly as sa_tw_mul (sa_common.cuh) -- value-identical to the
// reference (operator.py:124-131, transforms.py:282-295).
#pragma once
#include <cuda.h>

#include "sa_common.cuh"

typedef unsigned long long sa_u64;

template <typename T> struct Ar;

template <> struct Ar<float> {
  using V = sa_u64;
  using C2 = float2;
  using C4 = float4;
  static SA_HD V pack(float lo, float hi) {
    V r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
  }
  static SA_HD void unpack(V v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  }
  static SA_HD V from(C2 c) { return pack(c.x, c.y); }
  static SA_HD C2 to(V v) {
    C2 c;
    unpack(v, c.x, c.y);
    return c;
  }
  static SA_HD V add(V a, V b) {
    V d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
  }
  static SA_HD V sub(V a, V b) {
    V d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
  }
  static SA_HD V mul(V a, V b) {
    V d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
  }
  static SA_HD V fma(V a, V b, V c) {
    V d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
  }
  static SA_HD V sgn(V b) {
    float lo, hi;
    unpack(b, lo, hi);
    return pack(sa_sgn(lo), sa_sgn(hi));
  }
  static SA_HD V scale(V a, float g) { return mul(pack(g, g), a); }
  static SA_HD V swap(V v) {
    float lo, hi;
    unpack(v, lo, hi);
    return pack(hi, lo);
  }
  static SA_HD V neg(V v) {  // folds into the consuming FFMA2/FADD2 operand (-R.F32x2)
    float lo, hi;
    unpack(v, lo, hi);
    return pack(-lo, -hi);
  }
  static SA_HD V neg_hi(V v) {
    float lo, hi;
    unpack(v, lo, hi);
    return pack(lo, -hi);
  }
  // w ⊙ b with w = {|wr|, |wi|, sgn wr, sgn wi}.  Written so that every pair
  // shuffle is an operand modifier (LO_HI swap, scalar broadcast, negated
  // broadcast, high-half negation): 4 packed instructions, no MOVs.
  static SA_HD V twmul(const C4 &w, V b) {
    V sb = sgn(b);
    V q1 = fma(sb, pack(w.x, w.x), b);                   // {P1, P4}
    V q2 = fma(swap(sb), pack(w.y, w.y), swap(b));       // {P2, P3}
    V tq = mul(pack(-w.w, -w.w), q2);                    // {−tP2, −tP3}
    return fma(pack(w.z, w.z), q1, neg_hi(tq));          // {sP1 − tP2, sP4 + tP3}
  }
  // w ⊙ b for a twiddle with wr != 0 and wi < 0 (every stage j except 0 and
  // h/2): sgn wi = −1 and sgn wr = ±1 come from the raw value, no FMUL2.
  //   rr = σP1 + P2 ; ri = σP4 − P3
  static SA_HD V twmul_fast(const C2 &w, V b) {
    V sb = sgn(b);
    const float A = fabsf(w.x), B = fabsf(w.y);
    const float s = __int_as_float((__float_as_int(w.x) & 0x80000000) | 0x3f800000);
    V q1 = fma(sb, pack(A, A), b);              // {P1, P4}
    V q2 = fma(swap(sb), pack(B, B), swap(b));  // {P2, P3}
    return fma(pack(s, s), q1, neg_hi(q2));     // {σP1 + P2, σP4 − P3}
  }
  static SA_HD V one_mul(V b) { return add(sgn(b), b); }  // 1 ⊙ b
  static SA_HD V mj_mul(V b) {                            // (−j) ⊙ b = {u.hi, −u.lo}
    return neg_hi(swap(add(sgn(b), b)));
  }
};

template <> struct Ar<double> {
  using V = double2;
  using C2 = double2;
  using C4 = double4;
  static SA_HD V from(C2 c) { return c; }
  static SA_HD C2 to(V v) { return v; }
  static SA_HD V add(V a, V b) { return {sa_add(a.x, b.x), sa_add(a.y, b.y)}; }
  static SA_HD V sub(V a, V b) { return {sa_sub(a.x, b.x), sa_sub(a.y, b.y)}; }
  static SA_HD V scale(V a, double g) { return {sa_mul(g, a.x), sa_mul(g, a.y)}; }
  static SA_HD V twmul(const C4 &w, V b) {
    V r;
    sa_tw_mul<double>(w.x, w.y, w.z, w.w, b.x, b.y, r.x, r.y);
    return r;
  }
  static SA_HD V twmul_fast(const C2 &w, V b) {  // wr != 0, wi < 0
    const double sbr = sa_sgn(b.x), sbi = sa_sgn(b.y);
    const double A = fabs(w.x), B = fabs(w.y), s = w.x < 0.0 ? -1.0 : 1.0;
    const double p1 = sa_fma(sbr, A, b.x), p4 = sa_fma(sbi, A, b.y);
    const double p2 = sa_fma(sbi, B, b.y), p3 = sa_fma(sbr, B, b.x);
    return {sa_fma(s, p1, p2), sa_fma(s, p4, -p3)};
  }
  static SA_HD V one_mul(V b) { return {sa_fma(sa_sgn(b.x), 1.0, b.x), sa_fma(sa_sgn(b.y), 1.0, b.y)}; }
  static SA_HD V mj_mul(V b) {
    V u = one_mul(b);
    return {u.y, -u.x};
  }
};

// DIT butterflies on registers
template <typename T> SA_HD void r_dit(typename Ar<T>::V &a, typename Ar<T>::V &b,
                                       const typename Ar<T>::C4 &w) {
  auto t = Ar<T>::twmul(w, b);
  b = Ar<T>::sub(a, t);
  a = Ar<T>::add(a, t);
}
template <typename T> SA_HD void r_dit_fast(typename Ar<T>::V &a, typename Ar<T>::V &b,
                                            const typename Ar<T>::C2 &w) {
  auto t = Ar<T>::twmul_fast(w, b);
  b = Ar<T>::sub(a, t);
  a = Ar<T>::add(a, t);
}
template <typename T> SA_HD void r_dif_fast(typename Ar<T>::V &a, typename Ar<T>::V &b,
                                            const typename Ar<T>::C2 &w) {
  auto d = Ar<T>::sub(a, b);
  a = Ar<T>::add(a, b);
  b = Ar<T>::twmul_fast(w, d);
}
template <typename T> SA_HD void r_dit_one(typename Ar<T>::V &a, typename Ar<T>::V &b) {
  auto t = Ar<T>::one_mul(b);
  b = Ar<T>::sub(a, t);
  a = Ar<T>::add(a, t);
}
template <typename T> SA_HD void r_dit_mj(typename Ar<T>::V &a, typename Ar<T>::V &b) {
  auto t = Ar<T>::mj_mul(b);
  b = Ar<T>::sub(a, t);
  a = Ar<T>::add(a, t);
}
// bottom stage: full 2-point NDFT (transforms.py:270-280)
template <typename T> SA_HD void r_two_point(typename Ar<T>::V &a, typename Ar<T>::V &b) {
  auto u = Ar<T>::one_mul(a);
  auto t = Ar<T>::one_mul(b);
  a = Ar<T>::add(u, t);
  b = Ar<T>::sub(u, t);
}
// DIF butterfly: a' = a + b ; b' = w ⊙ (a − b)
template <typename T> SA_HD void r_dif(typename Ar<T>::V &a, typename Ar<T>::V &b,
                                       const typename Ar<T>::C4 &w) {
  auto d = Ar<T>::sub(a, b);
  a = Ar<T>::add(a, b);
  b = Ar<T>::twmul(w, d);
}
template <typename T> SA_HD void r_dif_one(typename Ar<T>::V &a, typename Ar<T>::V &b) {
  auto d = Ar<T>::sub(a, b);
  a = Ar<T>::add(a, b);
  b = Ar<T>::one_mul(d);
}
template <typename T> SA_HD void r_dif_mj(typename Ar<T>::V &a, typename Ar<T>::V &b) {
  auto d = Ar<T>::sub(a, b);
  a = Ar<T>::add(a, b);
  b = Ar<T>::mj_mul(d);
}

// ---------------------------------------------------------------------------
// shared-memory addresses, mbarriers, TMA
// ---------------------------------------------------------------------------
SA_HD uint32_t sa_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

SA_HD void sa_mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa_smem_u32(bar)), "r"(count));
}
SA_HD void sa_mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
SA_HD void sa_mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SA_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SA_WAIT_%=;\n}\n" ::"r"(sa_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
SA_HD void sa_fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SA_HD void sa_fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 2-D TMA tile load global -> this CTA's smem, completion on an mbarrier
SA_HD void sa_tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(sa_smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(sa_smem_u32(bar))
      : "memory");
}

// split cluster barrier: arrive early, wait late.  release only where DSMEM
// writes must be published; relaxed where only execution order matters (a CTA's
// own smem reads completed -- their values were consumed -- before it arrives).
SA_HD void sa_cluster_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
SA_HD void sa_cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
SA_HD void sa_cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// DSMEM producer -> consumer hand-off without fences: st.async writes into a
// cluster peer's smem and credits the bytes to the peer's mbarrier
// (complete_tx); the peer waits on its own mbarrier with cluster-scope acquire.
SA_HD uint32_t sa_mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
SA_HD void sa_st_async(uint32_t addr, float2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "r"(mbar)
               : "memory");
}
SA_HD void sa_st_async(uint32_t addr, double2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "d"(v.x), "d"(v.y), "r"(mbar)
               : "memory");
}
SA_HD void sa_mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SA_WAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SA_WAITC_%=;\n}\n" ::"r"(sa_smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// remote arrive on a peer CTA's mbarrier (address from sa_mapa).  Relaxed:
// used only to say "my reads of the storage you write into are complete".
SA_HD void sa_mbar_arrive_local(uint64_t *bar) {  // release.cta: prior smem writes visible to waiters
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa_smem_u32(bar)) : "memory");
}
SA_HD void sa_mbar_arrive_remote_release(uint32_t cluster_addr) {  // publishes prior global writes
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
SA_HD void sa_mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

// cp.async (LDGSTS): global -> shared without a register round trip.
// src_bytes < 8 zero-fills the rest of the 8-byte destination.
SA_HD void sa_cp_async8(void *smem, const void *gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa_smem_u32(smem)), "l"(gmem),
               "r"(src_bytes)
               : "memory");
}
SA_HD void sa_cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> SA_HD void sa_cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
