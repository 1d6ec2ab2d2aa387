// MEASURED ALTERNATIVE, NOT BUILT: the diagonal lag kernel (one
// reference window for blocks w and w + 1, both blocks' shifts stacked along N,
// 512 TMEM columns, 1 CTA per SM).  Bit-identical rows; C5 map 0.499 vs 0.446 ms.
// To try it: paste into csrc/sa_lag_i8.cu (inside the anonymous namespace, after
// k_lag_i8) and dispatch launch_i8d when npass == 2 and 16 MR == T.

// Diagonal variant (two lag groups of exactly T lags each, i.e. npass == 2 and
// 16 MR == T -- the C5 shape): A(q, lb) = A(q + 1, lb + T), so CTA w reads ONE
// c window and computes block w's lags [lalign, lalign + T) and block w + 1's lags
// [lalign + T, lalign + 2T): both blocks' s shifts are stacked along N (four
// N = 64 and two N = 128 MMAs per K step, all 512 TMEM columns), which cuts the
// smem operand bytes per MAC by 1.6x (A is 24 KB of the 32 KB per K step and unit).
template <int MR, bool BLK>
__global__ void __launch_bounds__(NWARPS * 32, 1)
    k_lag_i8d(const float2 *__restrict__ surv, int64_t l0g, int64_t l_count, int64_t m, int tb,
              const float *__restrict__ cpart, int npart, const unsigned char *__restrict__ cplanes, int64_t guard,
              int64_t cpl, float2 *__restrict__ z, int64_t q0, int64_t q_count, LagDst dst) {
  constexpr int U = 2;
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const Geo gm = geo(tb, MR, 1);
  unsigned char *Ps = smem;                                    // U x NPL x psl
  unsigned char *Pc = smem + U * NPL * gm.psl;                 // NPL x pcl: the A window
  unsigned char *Bb = smem + ((U * NPL * gm.psl + NPL * gm.pcl + 1023) & ~1023);  // NB x U B chunks
  constexpr int BU = U * B_BYTES;
  uint64_t *bfull = (uint64_t *)(Bb + NB * BU);
  uint64_t *bempty = bfull + NB;
  uint64_t *afull = bempty + NB;
  uint64_t *tfull = afull + 1;
  uint32_t *tmem_holder = (uint32_t *)(tfull + 1);
  float *red = (float *)(tmem_holder + 2);  // (U + 1) x NWARPS partial maxima

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t w = q0 + (int64_t)blockIdx.x - (U - 1);  // blocks w (pass 0) and w + 1 (pass 1)
  constexpr int LGRP = 16 * MR;
  bool valid[U];
#pragma unroll
  for (int u = 0; u < U; ++u) valid[u] = w + u >= q0 && w + u < q0 + q_count;

  {
    float ms[U] = {}, mc = 0.f;
    for (int i = tid; i < npart; i += NWARPS * 32) mc = fmaxf(mc, cpart[i]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (valid[u])
        for (int t = tid; t < tb; t += NWARPS * 32) ms[u] = fmaxf(ms[u], amax(__ldg(&surv[(w + u) * tb + t])));
#pragma unroll
    for (int o = 16; o; o >>= 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) ms[u] = fmaxf(ms[u], __shfl_xor_sync(0xffffffffu, ms[u], o));
      mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) red[u * NWARPS + warp] = ms[u];
      red[U * NWARPS + warp] = mc;
    }
  }
  if (tid == 0) {
    for (int i = 0; i < NB; ++i) sa_mbar_init(&bfull[i], 4), sa_mbar_init(&bempty[i], 1);
    sa_mbar_init(afull, 1);
    sa_mbar_init(tfull, 1);
    sa_fence_mbar_init();
  }
  __syncthreads();
  float ms[U] = {}, mc = 0.f;
#pragma unroll
  for (int i = 0; i < NWARPS; ++i) {
#pragma unroll
    for (int u = 0; u < U; ++u) ms[u] = fmaxf(ms[u], red[u * NWARPS + i]);
    mc = fmaxf(mc, red[U * NWARPS + i]);
  }
  const int ec = exponent_of(mc);
  const int64_t lalign = l0g - (l0g & 15);
  const int nch = (gm.ks + KC - 1) / KC;

  if (warp == WPROD && lane == 0) {  // the one A window: c index w T - lalign - 16 MR + x
    sa_mbar_expect_tx(afull, (uint32_t)(NPL * gm.pcl));
    const unsigned char *src = cplanes + guard + (w * tb - lalign - 16 * MR);
#pragma unroll 1
    for (int p = 0; p < NPL; ++p) bulk_g2s(Pc + p * gm.pcl, src + (int64_t)p * cpl, (uint32_t)gm.pcl, afull);
  }
  if (warp != WPROD) {  // s planes of both blocks (zero for a block outside the call)
#pragma unroll 1
    for (int u = 0; u < U; ++u) {
      const Dig dig(exponent_of(ms[u]));
      const float2 *sb = surv + (w + u) * tb;
      unsigned char *ps = Ps + u * NPL * gm.psl;
      for (int x4 = tid; x4 < gm.psl / 4; x4 += (NWARPS - 1) * 32) {
        const int t = 4 * x4 - 16;
        float2 v[4] = {};
        if (valid[u] && t >= 0 && t < tb) {
          const float4 a = __ldg((const float4 *)&sb[t]), b = __ldg((const float4 *)&sb[t + 2]);
          v[0] = make_float2(a.x, a.y), v[1] = make_float2(a.z, a.w), v[2] = make_float2(b.x, b.y), v[3] = make_float2(b.z, b.w);
        }
        uint32_t wd[NPL] = {};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t d0r, d1r, d0i, d1i;
          const uint32_t sr = dig(v[e].x, d0r, d1r), si = dig(v[e].y, d0i, d1i);
          wd[0] |= sr << (8 * e), wd[1] |= si << (8 * e);
          wd[2] |= d0r << (8 * e), wd[3] |= d0i << (8 * e);
          wd[4] |= d1r << (8 * e), wd[5] |= d1i << (8 * e);
        }
#pragma unroll
        for (int p = 0; p < NPL; ++p) ((uint32_t *)(ps + p * gm.psl))[x4] = wd[p];
      }
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa_smem_u32(tmem_holder)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == WMMA) {
    // B chunk rows: [sgn sr, sgn si] of block w then w + 1 (W window, 64 rows), then
    // [d0 sr, d0 si, d1 sr, d1 si] of w then w + 1 (X window, 128 rows)
    constexpr uint32_t IDW = idesc(32 * U, MR), IDX = idesc(64 * U, MR);
    const uint32_t pa0 = sa_smem_u32(Pc), bbase = sa_smem_u32(Bb);
    const uint64_t ap = (uint64_t)(gm.pcl >> 4);
    sa_mbar_wait(afull, 0);
    fence_after();
    for (int ch = 0; ch < nch; ++ch) {
      const int b = ch % NB;
      sa_mbar_wait(&bfull[b], (ch / NB) & 1);
      fence_after();
      const int kn = min(KC, gm.ks - ch * KC);
      for (int kk = 0; kk < kn; ++kk) {
        const int kstep = ch * KC + kk;
        const uint32_t bo = bbase + b * BU + kk * 2 * CORE;
        const uint64_t bw = sdesc_ns(bo, CORE, B_SBO), bx = sdesc_ns(bo + 4 * U * B_SBO, CORE, B_SBO);
        const uint64_t a0 = sdesc_ns(pa0 + 32 * kstep, 16, 128);
        asm volatile(
            "{\n .reg .pred e, p;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %12, 0;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %6, %10, %13, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%1], %7, %10, %13, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%2], %8, %10, %13, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%3], %9, %10, %13, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%4], %14, %11, %15, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%5], %16, %11, %15, p;\n}\n" ::"r"(tmem),
            "r"(tmem + 32 * U), "r"(tmem + 64 * U), "r"(tmem + 96 * U), "r"(tmem + 128 * U), "r"(tmem + 192 * U),
            "l"(a0), "l"(a0 + ap), "l"(a0 + 2 * ap), "l"(a0 + 3 * ap), "l"(bw), "l"(bx),
            "r"((uint32_t)(kstep != 0)), "r"(IDW), "l"(a0 + 4 * ap), "r"(IDX), "l"(a0 + 5 * ap)
            : "memory");
      }
      if (elect_one()) commit(&bempty[b]);
      __syncwarp();
    }
    if (elect_one()) commit(tfull);
    __syncwarp();
  } else if (warp >= WB0 && warp < WB0 + 4) {
    const int bt = tid - WB0 * 32;
    for (int ch = 0; ch < nch; ++ch) {
      const int b = ch % NB;
      if (ch >= NB) sa_mbar_wait(&bempty[b], ((ch / NB) - 1) & 1);
      unsigned char *B = Bb + b * BU;
#pragma unroll
      for (int it = 0; it < U * NPL * 16 * 2 * KC / 128; ++it) {
        const int e = it * 128 + bt;
        const int i = e & 15, kc2 = (e >> 4) & (2 * KC - 1), pu = e >> 4 >> 3;  // shift, K core, (unit, plane)
        const int u = pu / NPL, p = pu % NPL;
        if (ch * KC + (kc2 >> 1) < gm.ks) {
          const int x0 = 32 * ch * KC + 16 * kc2 + i;
          const uint32_t *P32 = (const uint32_t *)(Ps + (u * NPL + p) * gm.psl) + (x0 >> 2);
          const uint32_t sh = (uint32_t)(x0 & 3) * 8;
          const uint32_t a0 = P32[0], a1 = P32[1], a2 = P32[2], a3 = P32[3], a4 = P32[4];
          const uint4 o = make_uint4(__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh),
                                     __funnelshift_r(a2, a3, sh), __funnelshift_r(a3, a4, sh));
          // row block: W planes (p < 2) at 4 u + 2 p, X planes at 4 U + 8 u + 2 (p - 2)
          const int rb = (p < 2 ? 4 * u + 2 * p : 4 * U + 8 * u + 2 * (p - 2)) + (i >> 3);
          *(uint4 *)(B + (rb * (2 * KC) + kc2) * CORE + (i & 7) * 16) = o;
        }
      }
      sa_fence_proxy_async();
      __syncwarp();
      if (lane == 0) sa_mbar_arrive_local(&bfull[b]);
    }
  } else if (warp < 4) {
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
    const int r = MR == 128 ? warp * 32 + lane : warp * 16 + (lane & 15);
    const bool live = MR == 128 || lane < 16;
    const double cw = ldexp(DSC, ec);
    sa_mbar_wait(tfull, 0);
    fence_after();
#pragma unroll 1
    for (int u = 0; u < U; ++u) {
      const int es = exponent_of(ms[u]);
      const bool bad = !(ms[u] <= FLT_MAX) || !(mc <= FLT_MAX);
      const double cx = ldexp(DSC, es);
      const int64_t q = w + u;
      const int64_t lag0 = lalign + (int64_t)u * LGRP + 16 * (MR - 1 - r);
      const bool tile_in = valid[u] && (BLK ? (lag0 + 16 > l0g && lag0 < l0g + l_count) : true);
      const uint32_t gw = ta + 32 * u, gx = ta + 256 + 64 * u;  // W_p at 64 p, X_p at 256 + 128 p'
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t a[8], c[8];
        int iw[8], ix[8];
        float re[8], im[8];
        const uint32_t w8 = gw + 8 * h, x8 = gx + 8 * h;
        SA_LD8(a, w8 + 0);   SA_LD8(c, w8 + 64);  tm_wait();   // W0r[sr], W1r[sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] = 254 * (int)a[k] + (int)c[k];
        SA_LD8(a, w8 + 144); SA_LD8(c, w8 + 208); tm_wait();   // W0i[si], W1i[si]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] -= 254 * (int)a[k] + (int)c[k];
        SA_LD8(a, x8 + 0);   SA_LD8(c, x8 + 32);  tm_wait();   // Xr[d0sr], Xr[d1sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) ix[k] = 254 * (int)a[k] + (int)c[k];
        SA_LD8(a, x8 + 144); SA_LD8(c, x8 + 176); tm_wait();   // Xi[d0si], Xi[d1si]
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          ix[k] -= 254 * (int)a[k] + (int)c[k];
          re[k] = bad ? CUDART_NAN_F : (float)((double)iw[k] * cw + (double)ix[k] * cx);
        }
        SA_LD8(a, w8 + 16);  SA_LD8(c, w8 + 80);  tm_wait();   // W0r[si], W1r[si]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] = 254 * (int)a[k] + (int)c[k];
        SA_LD8(a, w8 + 128); SA_LD8(c, w8 + 192); tm_wait();   // W0i[sr], W1i[sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) iw[k] += 254 * (int)a[k] + (int)c[k];
        SA_LD8(a, x8 + 16);  SA_LD8(c, x8 + 48);  tm_wait();   // Xr[d0si], Xr[d1si]
#pragma unroll
        for (int k = 0; k < 8; ++k) ix[k] = 254 * (int)a[k] + (int)c[k];
        SA_LD8(a, x8 + 128); SA_LD8(c, x8 + 160); tm_wait();   // Xi[d0sr], Xi[d1sr]
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          ix[k] += 254 * (int)a[k] + (int)c[k];
          im[k] = bad ? CUDART_NAN_F : (float)((double)iw[k] * cw + (double)ix[k] * cx);
        }
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
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int MR, bool BLK>
int launch_i8d(const void *surv, int64_t l0, int64_t l_count, int64_t m, int64_t q0, int64_t q_count, int64_t tb,
               void *z, const LagDst &d, const float *cpart, int npart, const unsigned char *cplanes, int64_t guard,
               int64_t cpl, cudaStream_t s) {
  const Geo gm = geo((int)tb, MR, 1);
  const int bytes = ((2 * NPL * gm.psl + NPL * gm.pcl + 1023) & ~1023) + NB * 2 * B_BYTES + 512 + 1024;
  static int smem_set[64] = {};
  int dev = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64 || smem_set[dev] < bytes) {
    SA_CUDA_TRY(cudaFuncSetAttribute(k_lag_i8d<MR, BLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    if (dev < 64) smem_set[dev] = bytes;
  }
  k_lag_i8d<MR, BLK><<<(unsigned)(q_count + 1), NWARPS * 32, bytes, s>>>(
      (const float2 *)surv, l0, l_count, m, (int)tb, cpart, npart, cplanes, guard, cpl, (float2 *)z, q0, q_count, d);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

