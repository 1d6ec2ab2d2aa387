// sa_ndft_i8.cu -- complex128 fast-mode NDFT (transforms.py:223-251, regrouped as
// in sa_ndft.cu) on the tcgen05 tensor cores in EXACT INTEGER arithmetic: an
// Ozaki-style split of both non-sign operands into int8 digits, int8 x int8 ->
// int32 MMAs (kind::i8), fp64 only in the epilogue.
//
// The regrouped sum is one real GEMM per batch (sa_ndft_tc.cu):
//   D[v, o] = Σ_K S[v,K] Wv[o,K] + X[v,K] sgn(Wv)[o,K],   S = sgn(x),  o = 2k+(re|im), K = 2n+(re|im)
// One factor of every product is a sign in {-1, 0, +1} -- exact in int8.  The
// other factor is split into four signed digits in mixed radix (64, 127, 128, 127):
//   Wv ~ d0/64 + d1/(64 127) + d2/(64 127 128) + d3/(64 127 128 127)    (|Wv| <= 1, |d| <= 64)
//   x' = x_v / 2^e_v   (per-vector exponent: max|x_v| < 2^e_v), digits alike
// (round-to-nearest digits; the residual after the fourth digit is <= 2^-28).
// Two digits 127 apart share one int32 accumulator by pairing the sign operand
// with 127 x sign (still int8):
//   accWH = Σ (127 S) dW0 + S dW1        accWL = Σ (127 S) dW2 + S dW3
//   accXH = Σ dx0 (127 sW) + dx1 sW      accXL = Σ dx2 (127 sW) + dx3 sW
// all exact (|acc| < 2^25 at n <= 2048), and the epilogue forms, in fp64,
//   D = accWH c1 + accWL c2 + 2^e_v (accXH c1 + accXL c2),  c1 = 1/(64 127), c2 = c1/(128 127).
// Error model: per output ~ sqrt(2n) 2^-28 (1 + 2^e) against ||y||_1 ~ n sqrt(2n):
// the fp64 bound 1e-9 holds from n = 128 up; measured max|Δ|/‖y‖₁ ~1e-11 on C2
// (tests/test_gpu_ndft_i8.py).  Smaller n runs the DFMA fast kernel.
//
// Pipeline: k_i8_prep (one pass over x: gain, per-vector exponent, the six int8
// planes S, 127 S, dx0..dx3) -> k_ndft_i8 (persistent CTA pairs, cluster 2,
// tcgen05.mma.cta_group::2.kind::i8, M = 256 vectors, N = 128 outputs, K = 32;
// the four accumulators fill TMEM's 512 columns).  Both operand sets are stored
// in HBM as "smem images": for each 128-vector block (or 64-output block) and
// 64-K slot the six planes' tiles are contiguous and already SWIZZLE_64B-permuted,
// so one bulk copy per side (48 KB of x planes, 24 KB of W planes: sW, 127 sW,
// dW0..dW3, built once per twiddle set) fills a slot -- 128-B requests instead of
// the 64-B rows a 2-D TMA box would issue (the request rate bounded the first
// version: 2.48 ms with the MMAs skipped or not).  Three 72 KB slots per CTA.
// Warp 0 produces, warp 2 + EPI relays each CTA's slot completion to the leader,
// warp 1 issues the MMAs (leader CTA), warps 2 .. 1 + EPI drain TMEM into
// complex128 rows of y (EPI = 8: two warps per TMEM lane quarter, half the columns each).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <map>
#include <math_constants.h>
#include <mutex>
#include <tuple>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

constexpr int BM = 128;               // vectors per CTA (TMEM lanes); M = 256 per pair
constexpr int BN = 128;               // outputs per tile (each accumulator: 128 TMEM columns)
constexpr int KSL = 64;               // int8 K elements per slot (64-B rows, SWIZZLE_64B)
constexpr int NPL = 6;                // planes per operand side: S, 127 S, four digits
constexpr int XT = BM * KSL;          // one x-plane tile per CTA: 8 KB
constexpr int WT = (BN / 2) * KSL;    // one W-plane tile per CTA (half the outputs): 4 KB
constexpr int SLOT = NPL * XT + NPL * WT;  // 72 KB
constexpr int NSLOT = 3;
constexpr int SMEM = NSLOT * SLOT + 1024 + 256;
#ifndef SA_I8_EPI_WARPS
#define SA_I8_EPI_WARPS 8
#endif
constexpr int EPI = SA_I8_EPI_WARPS;  // epilogue warps: EPI / 4 per TMEM lane quarter, each a column share
constexpr int RELAY_WARP = 2 + EPI;
#ifndef SA_I8_NP
#define SA_I8_NP 1  // CTA pairs per cluster sharing (TMA-multicast) the x planes of one vector tile
#endif
constexpr int NP = SA_I8_NP;
#ifndef SA_I8_SCALE
#define SA_I8_SCALE 0  // 1: the 127 x sign tiles are made in smem from the sign tiles (5 planes per side in HBM)
#endif
constexpr int NMEM = SA_I8_SCALE ? 5 : 6;  // planes per side in HBM (smem images), order S, [127 S,] digits
constexpr int NSCALE = SA_I8_SCALE ? 2 : 0;  // scaler warps (they also relay); else one relay warp
constexpr int THREADS = (2 + EPI + (NSCALE ? NSCALE : 1)) * 32;  // producer, MMA, epilogue, scaler/relay
constexpr int TMEM_COLS = 512;
// kind::i8: D = s32 (2), A = B = s8 (1), K-major, N = 128, M = 256
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);

SA_HD uint64_t sdesc(uint32_t saddr) {  // K-major SWIZZLE_64B: 64-B rows, 8-row atoms 512 B apart
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
// byte offset of (row r, K byte b) inside a SWIZZLE_64B tile of 64-B rows
SA_HD uint32_t sw64(int r, int b) { return (uint32_t)(r * 64 + ((((b >> 4) ^ (r >> 1)) & 3) << 4) + (b & 15)); }
SA_HD void bulk_g2s_mc(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint16_t mask, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4, %5;" ::"r"(sa_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(sa_smem_u32(bar)), "h"(mask), "l"(pol)
      : "memory");
}
SA_HD void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sa_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(sa_smem_u32(bar)), "l"(pol)
      : "memory");
}
SA_HD void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SA_HD void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SA_HD void commit2(uint64_t *bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          sa_smem_u32(bar)),
      "h"(mask)
      : "memory");
}
SA_HD void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
#ifdef SA_I8_PROBE_NOMMA
  return;
#endif
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc)
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

// The four signed digits (radix 64, 127, 128, 127; each |d| <= 64) of |v| <= 1.
SA_HD void digits(double v, int &d0, int &d1, int &d2, int &d3) {
  double y = v * 64.0;
  double r = rint(y);
  d0 = (int)r;
  y = (y - r) * 127.0;
  r = rint(y);
  d1 = (int)r;
  y = (y - r) * 128.0;
  r = rint(y);
  d2 = (int)r;
  y = (y - r) * 127.0;
  d3 = (int)rint(y);
}
SA_HD int sgn_i(double v) { return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0); }

// x (batch x n complex128, gain applied) -> the six planes (S, 127 S, dx0..dx3; K =
// 2m + re/im) as smem images: block (v / 128, K slot kc) holds the six 8 KB
// tiles of rows v % 128, SWIZZLE_64B-permuted; e[v] = per-vector exponent (max|x_v| < 2^e).
template <int IT>
__global__ void __launch_bounds__(256) k_i8_prep(const double *__restrict__ x, int8_t *__restrict__ planes,
                                                 int *__restrict__ ex, int64_t batch, int n, double gain,
                                                 int use_gain) {
  // one row per CTA iteration; thread t holds doubles [8 t + 2048 i, +8), i < IT, in
  // registers (2n <= 2048 IT), so the row is read once and every plane store is 8 bytes
  __shared__ double red[8];
  const int nk = 2 * n;
  const int kslots = nk / KSL;
  for (int64_t v = blockIdx.x; v < batch; v += gridDim.x) {
    const double *row = x + v * nk;
    double t[IT][8];
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int k = threadIdx.x * 8 + 2048 * i;
      if (k < nk) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          double2 u = __ldcs((const double2 *)&row[k + j]);
          t[i][j] = use_gain ? sa_mul(gain, u.x) : u.x;
          t[i][j + 1] = use_gain ? sa_mul(gain, u.y) : u.y;
          // max |x|; a NaN / Inf anywhere makes mx = +Inf (fmax would drop a NaN)
          const double a0 = fabs(t[i][j]), a1 = fabs(t[i][j + 1]);
          mx = (a0 == a0 && a1 == a1) ? fmax(mx, fmax(a0, a1)) : INFINITY;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    __syncthreads();
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): max < 2^e
    if (!(mx <= 1.7976931348623157e308)) e = INT_MAX;  // non-finite row: the epilogue writes NaN
    if (threadIdx.x == 0) ex[v] = e;
    if (e == INT_MAX) e = 0;  // (digits of this row are never used)
    int8_t *blk = planes + (size_t)(v / BM) * kslots * (NMEM * XT);
    const int r = (int)(v % BM);
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int k = threadIdx.x * 8 + 2048 * i;
      if (k < nk) {
        uint64_t w[6] = {};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          int d0, d1, d2, d3;
          digits(ldexp(t[i][j], -e), d0, d1, d2, d3);
          const int sh = 8 * j, sg = sgn_i(t[i][j]);
          w[0] |= (uint64_t)(uint8_t)sg << sh;
          w[1] |= (uint64_t)(uint8_t)(127 * sg) << sh;
          w[2] |= (uint64_t)(uint8_t)d0 << sh;
          w[3] |= (uint64_t)(uint8_t)d1 << sh;
          w[4] |= (uint64_t)(uint8_t)d2 << sh;
          w[5] |= (uint64_t)(uint8_t)d3 << sh;
        }
        int8_t *tile = blk + (size_t)(k / KSL) * (NMEM * XT) + sw64(r, k % KSL);  // 8 bytes, one swizzle chunk
#pragma unroll
        for (int p = 0; p < NMEM; ++p) *(uint64_t *)(tile + p * XT) = w[p + (NMEM == 5 && p > 0)];
      }
    }
  }
}

// The same as k_i8_prep with one warp per row (no block barriers, ~8 doubles live
// per lane): pass 1 takes the row max, pass 2 re-reads the row (L1) and writes
// the digit planes, 8 bytes per plane per lane.
__global__ void __launch_bounds__(256) k_i8_prep_w(const double *__restrict__ x, int8_t *__restrict__ planes,
                                                   int *__restrict__ ex, int64_t batch, int n, double gain,
                                                   int use_gain) {
  const int nk = 2 * n;
  const int kslots = nk / KSL;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  auto ld8 = [&](const double *row, int k, double (&t)[8]) {
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      double2 u = *(const double2 *)&row[k + j];
      t[j] = use_gain ? sa_mul(gain, u.x) : u.x;
      t[j + 1] = use_gain ? sa_mul(gain, u.y) : u.y;
    }
  };
  for (int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < batch; v += nw) {
    const double *row = x + v * nk;
    double mx = 0.0;
    for (int k = lane * 8; k < nk; k += 256) {
      double t[8];
      ld8(row, k, t);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double a = fabs(t[j]);
        mx = a == a ? fmax(mx, a) : INFINITY;  // a NaN anywhere makes the row non-finite
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    if (!(mx <= 1.7976931348623157e308)) e = INT_MAX;  // non-finite row: the epilogue writes NaN
    if (lane == 0) ex[v] = e;
    if (e == INT_MAX) e = 0;
    int8_t *blk = planes + (size_t)(v / BM) * kslots * (NMEM * XT);
    const int r = (int)(v % BM);
    for (int k = lane * 8; k < nk; k += 256) {
      double t[8];
      ld8(row, k, t);
      uint64_t w[6] = {};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int d0, d1, d2, d3;
        digits(ldexp(t[j], -e), d0, d1, d2, d3);
        const int sh = 8 * j, sg = sgn_i(t[j]);
        w[0] |= (uint64_t)(uint8_t)sg << sh;
        w[1] |= (uint64_t)(uint8_t)(127 * sg) << sh;
        w[2] |= (uint64_t)(uint8_t)d0 << sh;
        w[3] |= (uint64_t)(uint8_t)d1 << sh;
        w[4] |= (uint64_t)(uint8_t)d2 << sh;
        w[5] |= (uint64_t)(uint8_t)d3 << sh;
      }
      int8_t *tile = blk + (size_t)(k / KSL) * (NMEM * XT) + sw64(r, k % KSL);
#pragma unroll
      for (int p = 0; p < NMEM; ++p) *(uint64_t *)(tile + p * XT) = w[p + (NMEM == 5 && p > 0)];
    }
  }
}

// W planes Q[p][o][K] (p = sW, dW0..dW3) of Wv = [[Wr, -Wi], [Wi, Wr]],
// W = raw[(k m) mod n] (the fp64 reference table, transforms.py:108-146).
__global__ void k_i8_wbuild(const double2 *__restrict__ raw, int n, int8_t *__restrict__ q) {
  // smem images: block (o / 64, K slot kc) holds the six 4 KB tiles of rows o % 64
  const int64_t nn = 2LL * n, total = nn * nn;
  const int kslots = (int)(nn / KSL);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / nn, kk = i % nn;
    const int64_t k = o >> 1, m = kk >> 1;
    const int co = (int)(o & 1), ci = (int)(kk & 1);
    const double2 tw = raw[(k * m) % n];
    const double val = co == ci ? tw.x : (co == 0 ? -tw.y : tw.y);
    int d0, d1, d2, d3;
    digits(val, d0, d1, d2, d3);
    const int sg = sgn_i(val);
    const int8_t v[NPL] = {(int8_t)sg, (int8_t)(127 * sg), (int8_t)d0, (int8_t)d1, (int8_t)d2, (int8_t)d3};
    int8_t *tile = q + ((o / (BN / 2)) * kslots + kk / KSL) * (NMEM * WT) + sw64((int)(o % (BN / 2)), (int)(kk % KSL));
#pragma unroll
    for (int p = 0; p < NMEM; ++p) tile[p * WT] = v[p + (NMEM == 5 && p > 0)];
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    k_ndft_i8(const int8_t *__restrict__ xblk, const int8_t *__restrict__ wblk, const int *__restrict__ ex,
              double *__restrict__ y, int64_t batch, int n) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + NSLOT * SLOT);  // leader: both CTAs' slot s complete
  uint64_t *empty = full + NSLOT;
  uint64_t *lfull = empty + NSLOT;                       // this CTA's TMA bytes of slot s landed
  uint64_t *tfull = lfull + NSLOT;
  uint64_t *tempty = tfull + 1;
  uint32_t *tmem_holder = (uint32_t *)(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster = NP CTA pairs on the same vector tile, pair pr on output tile NP otp + pr
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1, pr = crank >> 1;
  const int64_t cl = blockIdx.x / (2 * NP), ncl = gridDim.x / (2 * NP);
  const int nk = 2 * n;
  const int ot_count = nk / BN;
  const int64_t vt_count = (batch + 2 * BM - 1) / (2 * BM);
  const int64_t ntiles = vt_count * (ot_count / NP);  // cluster tiles
  const int kslots = nk / KSL;
  const uint16_t pair_mask = (uint16_t)(3u << (2 * pr)), all_mask = (uint16_t)((1u << (2 * NP)) - 1);
  auto lead = [&](uint64_t *bar) { return sa_mapa(sa_smem_u32(bar), crank & ~1u); };
  auto vt_of = [&](int64_t t) { return t / (ot_count / NP); };
  auto ot_of = [&](int64_t t) { return (int)(t % (ot_count / NP)) * NP + (int)pr; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      sa_mbar_init(&full[s], 2 * (NSCALE ? NSCALE : 1));  // the relay / scaler warps of both CTAs
      sa_mbar_init(&empty[s], NP);  // every pair's MMAs on slot s are done (x tiles are shared)
      sa_mbar_init(&lfull[s], 1);
    }
    sa_mbar_init(tfull, 1);
    sa_mbar_init(tempty, EPI * 2);
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
    // ---- producer: one bulk copy per side per slot (this CTA's 128 vectors / 64 outputs) ----
    if (lane == 0) {
      const uint64_t wpol = policy(true), xpol = policy(false);
      for (int64_t it = 0; it < total; ++it) {
        const int64_t lt = it / kslots;
        const int kc = (int)(it - lt * kslots);
        const int64_t t = cl + lt * ncl;
        const int64_t vb = vt_of(t) * 2 + rank;                   // 128-vector block
        const int64_t ob = (int64_t)ot_of(t) * 2 + rank;          // 64-output block
        const int s = (int)(it % NSLOT);
        sa_mbar_wait(&empty[s], ((it / NSLOT) & 1) ^ 1);          // every pair is done with slot s
        unsigned char *b = smem + s * SLOT;
        sa_mbar_expect_tx(&lfull[s], NMEM * (XT + WT));
        const int8_t *xs = xblk + (vb * kslots + kc) * (NMEM * XT);
        const int8_t *ws_ = wblk + (ob * kslots + kc) * (NMEM * WT);
        if (NMEM == 6) {
          if (NP == 1) bulk_g2s(b, xs, NPL * XT, &lfull[s], xpol);
          else if (pr == 0)  // the x tile of rows `rank` goes to the same CTA of every pair
            bulk_g2s_mc(b, xs, NPL * XT, &lfull[s], (uint16_t)(0x5u << rank), xpol);
          bulk_g2s(b + NPL * XT, ws_, NPL * WT, &lfull[s], wpol);
        } else {  // S -> tile 0, digits -> tiles 2..5 (tile 1 = 127 S is made by the scalers)
          bulk_g2s(b, xs, XT, &lfull[s], xpol);
          bulk_g2s(b + 2 * XT, xs + XT, 4 * XT, &lfull[s], xpol);
          bulk_g2s(b + NPL * XT, ws_, WT, &lfull[s], wpol);
          bulk_g2s(b + NPL * XT + 2 * WT, ws_ + WT, 4 * WT, &lfull[s], wpol);
        }
      }
    }
  } else if (warp >= RELAY_WARP) {
    // ---- relay (+ scalers): this CTA's slot landed [127 S / 127 sW tiles made from
    // the sign tiles: bytes {-1,0,1} -> (x & 1) * 127, negated where negative] ->
    // arrive on the leader's full barrier ----
    const int st = threadIdx.x - RELAY_WARP * 32, nst = (NSCALE ? NSCALE : 1) * 32;
    for (int64_t it = 0; it < total; ++it) {
      const int s = (int)(it % NSLOT);
      sa_mbar_wait(&lfull[s], (it / NSLOT) & 1);
      if (NSCALE) {
        unsigned char *b = smem + s * SLOT;
        auto scale_tile = [&](const unsigned char *src, unsigned char *dst, int bytes) {
          for (int o = st * 16; o < bytes; o += nst * 16) {
            uint4 v = *(const uint4 *)(src + o);
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t t = (w[i] & 0x01010101u) * 0x7Fu;
              const uint32_t ng = (w[i] >> 7) & 0x01010101u;
              w[i] = (t ^ (ng * 0xFFu)) + ng;
            }
            *(uint4 *)(dst + o) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        };
        scale_tile(b, b + XT, XT);
        scale_tile(b + NPL * XT, b + NPL * XT + WT, WT);
        sa_fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05.mma
      }
      __syncwarp();
      if (lane == 0) arrive_cl(lead(&full[s]));
    }
  } else if (warp == 1) {
    // ---- MMA issuer (leader CTA): 8 MMAs per K step of 32 into the four accumulators ----
    if (lane == 0 && rank == 0) {
      uint32_t it = 0, lt = 0;
      for (int64_t t = cl; t < ntiles; t += ncl, ++lt) {
        sa_mbar_wait(tempty, (lt & 1) ^ 1);
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
            mma2(tmem + 0, X(1), W(2), first);    // accWH += 127 S dW0
            mma2(tmem + 0, X(0), W(3), 1);        //        + S dW1
            mma2(tmem + 128, X(1), W(4), first);  // accWL += 127 S dW2
            mma2(tmem + 128, X(0), W(5), 1);      //        + S dW3
            mma2(tmem + 256, X(2), W(1), first);  // accXH += dx0 127 sW
            mma2(tmem + 256, X(3), W(0), 1);      //        + dx1 sW
            mma2(tmem + 384, X(4), W(1), first);  // accXL += dx2 127 sW
            mma2(tmem + 384, X(5), W(0), 1);      //        + dx3 sW
          }
          commit2(&empty[s], all_mask);
        }
        commit2(tfull, pair_mask);
      }
    }
  } else {
    // ---- epilogue (warps 2 .. 2 + EPI - 1): TMEM lane quarter q -> vector row v, a share of the 128 outputs ----
    const int q = warp & 3;
    const int cs = (warp - 2) / 4;  // this warp's column share
    constexpr int CW = BN / (EPI / 4);
    uint32_t lt = 0;
    for (int64_t t = cl; t < ntiles; t += ncl, ++lt) {
      const int64_t v = vt_of(t) * (2 * BM) + rank * BM + q * 32 + lane;
      const int o0 = ot_of(t) * BN;
      const int e = v < batch ? ex[v] : 0;
      sa_mbar_wait(tfull, lt & 1);
      fence_after();
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16);
      double *dst = y + v * nk + o0;
#ifdef SA_I8_PROBE_NOEPI
      if (v < 0)
#endif
#pragma unroll 1
      for (int c = cs * CW; c < (cs + 1) * CW; c += 16) {
        uint32_t wh[16], wl[16], xh[16], xl[16];
        SA_LD16(wh, ta + c);
        SA_LD16(wl, ta + 128 + c);
        SA_LD16(xh, ta + 256 + c);
        SA_LD16(xl, ta + 384 + c);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v < batch) {
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            double d[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              // pair digits in int64 (exact), then one conversion and one scaling each
              constexpr double C2 = 1.0 / (64.0 * 127.0 * 128.0 * 127.0);
              const long long W = (long long)(int)wh[j + h] * (128 * 127) + (int)wl[j + h];
              const long long X = (long long)(int)xh[j + h] * (128 * 127) + (int)xl[j + h];
              d[h] = e == INT_MAX ? CUDART_NAN : sa_add(ldexp(sa_mul((double)X, C2), e), sa_mul((double)W, C2));
            }
            __stcs((double2 *)&dst[c + j], make_double2(d[0], d[1]));
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) arrive_cl(lead(tempty));
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

}  // namespace

bool sa_ndft_i8_supported(int dtype, int64_t n) {
  return dtype == SA_C128 && n >= 128 && n <= 2048 && n % (64 * NP) == 0;  // 2n <= 2 x 2048 (k_i8_prep); whole cluster tiles
}

int64_t sa_ndft_i8_wbytes(int64_t n) { return (int64_t)NMEM * (2 * n) * (2 * n); }

int sa_launch_ndft_i8(const void *x, void *y, int64_t batch, int64_t n, const SaTwiddles *tw_c, double gain,
                      cudaStream_t s) {
  if (!sa_ndft_i8_supported(tw_c->dtype, n)) return SA_ERR_UNSUPPORTED;
  if (((uintptr_t)x | (uintptr_t)y) & 15) return SA_ERR_UNSUPPORTED;
  if (batch == 0) return SA_OK;
  SaTwiddles *tw = const_cast<SaTwiddles *>(tw_c);
  {
    // W planes built once per twiddle set, stream-ordered (event for later streams)
    std::lock_guard<std::mutex> g(g_i8_mutex);
    if (!tw->i8w) {
      void *w = nullptr;
      cudaEvent_t ev = nullptr;
      SA_CUDA_TRY(cudaMalloc(&w, sa_ndft_i8_wbytes(n)));
      k_i8_wbuild<<<1184, 256, 0, s>>>((const double2 *)tw->raw, (int)n, (int8_t *)w);
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
  const size_t pbytes = (size_t)NMEM * rows * 2 * n;
  int8_t *planes = nullptr;
  {
    const int rc_ = sa_scratch_alloc((void **)&planes, pbytes + (size_t)batch * sizeof(int) + 256, s);
    if (rc_) return rc_;
  }
  int *ex = (int *)(((uintptr_t)(planes + pbytes) + 255) & ~(uintptr_t)255);
  int dev = 0, sms = 148;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  SA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int pgrid = (int)(batch < 8LL * sms ? batch : 8LL * sms);
  auto prep = n <= 1024 ? k_i8_prep<1> : k_i8_prep<2>;
  prep<<<pgrid, 256, 0, s>>>((const double *)x, planes, ex, batch, (int)n, gain, (int)(gain != 1.0));
  SA_LAUNCH_CHECK();
  static bool smem_set[64] = {};
  if (dev >= 64 || !smem_set[dev]) {
    SA_CUDA_TRY(cudaFuncSetAttribute(k_ndft_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    if (dev < 64) smem_set[dev] = true;
  }
  const int64_t ntiles = (rows / (2 * BM)) * ((2 * n) / BN / NP);  // cluster tiles
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * NP;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(2 * NP * (sms / (2 * NP))));
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, k_ndft_i8, &cfg) != cudaSuccess || max_clusters < 1)
    max_clusters = sms / (2 * NP);
  const int64_t units = ntiles < max_clusters ? ntiles : max_clusters;
  cfg.gridDim = dim3((unsigned)(units * 2 * NP));
  SA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_ndft_i8, (const int8_t *)planes, (const int8_t *)tw->i8w, (const int *)ex,
                                 (double *)y, batch, (int)n));
  SA_LAUNCH_CHECK();
  SA_CUDA_TRY(cudaFreeAsync(planes, s));
  return SA_OK;
}
