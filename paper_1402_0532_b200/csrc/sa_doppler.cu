// sa_doppler.cu -- the map's Doppler stage: DIT NL-FFT of gain*z_l for a range of
// delay rows, with M = 2^6 .. 2^11 (C4: 512, C5: 2048), straight from the lag
// kernel's blocked z layout (sa_lag_tc.cu).
//
//   row_l = nfft(gain * z_l)            (ambiguity.py:174-178; transforms.py:254-298)
//
// z layout "blocked": rows in tiles of 16 consecutive absolute lags (tile k
// holds rows 16k .. 16k+15 counted from the call's 16-aligned lag base), and
// inside a tile element q of the 16 rows is one 128-B line:
//   zb[(k * M + q) * 16 + j]  =  z[16k + j][q]
// so the lag kernel's epilogue writes whole sectors and this kernel reads whole
// lines.  A row-major z (stride M) is accepted as well (tile = 0).
//
// One CTA = R consecutive rows (R = 16, or 8 / 4 where 16 rows do not fit in
// shared memory).  Rows are staged in smem in bit-reversed order (the
// reference's y = x[bitrev], transforms.py:268) with one pad element per 16 and
// an odd row stride (bank-conflict free), then the log2 M stages run as
// register radix-16 rounds (the last round radix 2^(log M mod 4)): each thread
// loads the 16 (or 2^r) nodes of one butterfly group, runs its stages with the
// stage-table twiddles (sa_regs.cuh: value-identical to the reference), and
// stores them back.  Stage 1 is the full 2-point NDFT (transforms.py:270-280).
// The output rows are written coalesced, natural order, to out[(row) * M + i].
#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

constexpr int THREADS = 512;

template <typename T, int LOGM> struct Dop {
  static constexpr int M = 1 << LOGM;
  static constexpr int R = sizeof(T) == 4 ? (LOGM <= 10 ? 16 : 8) : (LOGM <= 10 ? 8 : 4);
  static constexpr int STRIDE = M + M / 16 + 1;  // padded, odd: rows land in distinct banks
  using C2 = typename Ar<T>::C2;
  using C4 = typename Ar<T>::C4;
  static constexpr size_t SM_DATA = sizeof(C2) * (size_t)R * STRIDE;
  static constexpr size_t SMEM = SM_DATA + sizeof(C4) * (size_t)(M - 1);
};

SA_HD int pad16(int p) { return p + (p >> 4); }

// One round: stages t0 .. t0 + NST - 1 on every butterfly group of the R rows.
template <typename T, int LOGM, int NST>
SA_HD void round_dit(typename Ar<T>::C2 *sm, const typename Ar<T>::C4 *tws, int t0) {
  using D = Dop<T, LOGM>;
  using A = Ar<T>;
  using V = typename A::V;
  constexpr int GS = 1 << NST;             // nodes per group
  constexpr int GPR = D::M / GS;           // groups per row
  const int lo = 1 << (t0 - 1);            // node stride of the group
  for (int gid = threadIdx.x; gid < D::R * GPR; gid += THREADS) {
    const int row = gid / GPR, g = gid % GPR;
    const int base = (g & (lo - 1)) + ((g >> (t0 - 1)) << (t0 - 1 + NST));
    typename A::C2 *rs = sm + row * D::STRIDE;
    V v[GS];
#pragma unroll
    for (int k = 0; k < GS; ++k) v[k] = A::from(rs[pad16(base + k * lo)]);
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      const int t = t0 + s, h = 1 << (t - 1);
      if (t == 1) {
#pragma unroll
        for (int k = 0; k < GS; k += 2) r_two_point<T>(v[k], v[k + 1]);
      } else {
#pragma unroll
        for (int k = 0; k < GS; ++k)
          if (!(k & (1 << s))) {
            const int j = (base & (lo - 1)) + (k & ((1 << s) - 1)) * lo;  // p_k mod h
            r_dit<T>(v[k], v[k + (1 << s)], tws[(h - 1) + j]);
          }
      }
    }
#pragma unroll
    for (int k = 0; k < GS; ++k) rs[pad16(base + k * lo)] = A::to(v[k]);
  }
  __syncthreads();
}

template <typename T, int LOGM>
__global__ void __launch_bounds__(THREADS, 1)
    k_doppler(const typename Ar<T>::C2 *__restrict__ z, typename Ar<T>::C2 *__restrict__ out, int row_off,
              int64_t l_count, int blocked, const typename Ar<T>::C4 *__restrict__ stage, T gain, int use_gain) {
  using D = Dop<T, LOGM>;
  using C2 = typename D::C2;
  using C4 = typename D::C4;
  constexpr int M = D::M, R = D::R;
  sa_pdl_wait();  // launched with programmatic serialization: the lag kernel's z is complete from here on
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C2 *sm = reinterpret_cast<C2 *>(smem_raw);
  C4 *tws = reinterpret_cast<C4 *>(smem_raw + D::SM_DATA);
  // twiddles and rows: every thread issues a batch of independent loads before its
  // shared-memory stores (a load-store-load chain would pay the L2 latency per element)
  constexpr int TB = (M - 1 + THREADS - 1) / THREADS;
  {
    C4 t[TB];
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const int e = threadIdx.x + j * THREADS;
      if (e < M - 1) t[j] = stage[e];
    }
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const int e = threadIdx.x + j * THREADS;
      if (e < M - 1) tws[e] = t[j];
    }
  }
  // rows of this CTA: absolute (16-aligned) rows a0 .. a0 + R - 1; valid rows are
  // row_off .. row_off + l_count - 1 (output row = a - row_off)
  const int64_t a0 = (int64_t)blockIdx.x * R;
  constexpr int LB = (M * R / THREADS) < 8 ? (M * R / THREADS) : 8;  // loads in flight per thread
  static_assert((M * R) % (LB * THREADS) == 0, "row staging: whole batches");
  for (int e0 = threadIdx.x; e0 < M * R; e0 += LB * THREADS) {
    C2 v[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int e = e0 + b * THREADS;
      const int j = e % R, pos = e / R;  // R consecutive threads: one q, R rows
      const int q = (int)(__brev((unsigned)pos) >> (32 - LOGM));
      const int64_t a = a0 + j;
      v[b] = {T(0), T(0)};
      if (a >= row_off && a < row_off + l_count)
        v[b] = blocked ? z[((a >> 4) * M + q) * 16 + (a & 15)] : z[(a - row_off) * M + q];
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int e = e0 + b * THREADS;
      const int j = e % R, pos = e / R;
      C2 x = v[b];
      if (use_gain) x = {sa_mul(gain, x.x), sa_mul(gain, x.y)};
      sm[j * D::STRIDE + pad16(pos)] = x;
    }
  }
  __syncthreads();
  constexpr int FULL = LOGM / 4, REM = LOGM % 4;
#pragma unroll
  for (int r = 0; r < FULL; ++r) round_dit<T, LOGM, 4>(sm, tws, 1 + 4 * r);
  if constexpr (REM > 0) round_dit<T, LOGM, REM>(sm, tws, 1 + 4 * FULL);
  for (int e = threadIdx.x; e < M * R; e += THREADS) {
    const int j = e / M, i = e % M;
    const int64_t a = a0 + j;
    if (a >= row_off && a < row_off + l_count) __stcs(&out[(a - row_off) * M + i], sm[j * D::STRIDE + pad16(i)]);
  }
}

template <typename T, int LOGM>
int launch_dop(const void *z, void *out, int row_off, int64_t l_count, int blocked, const SaTwiddles *tw,
               double gain, cudaStream_t s) {
  using D = Dop<T, LOGM>;
  static int smem_set[64] = {};
  int dev = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64 || !smem_set[dev]) {
    SA_CUDA_TRY(cudaFuncSetAttribute(k_doppler<T, LOGM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D::SMEM));
    if (dev < 64) smem_set[dev] = 1;
  }
  const int64_t rows = row_off + l_count;
  const int64_t grid = (rows + D::R - 1) / D::R;
  SA_CUDA_TRY(sa_launch_pdl(k_doppler<T, LOGM>, dim3((unsigned)grid), dim3(THREADS), (size_t)D::SMEM, s,
                            (const typename D::C2 *)z, (typename D::C2 *)out, (int)row_off, (int64_t)l_count,
                            (int)blocked, (const typename D::C4 *)tw->stage, (T)gain, (int)(gain != 1.0)));
  SA_LAUNCH_CHECK();
  return SA_OK;
}

template <typename T>
int launch_dop_t(const void *z, void *out, int row_off, int64_t l_count, int64_t m, int blocked,
                 const SaTwiddles *tw, double gain, cudaStream_t s) {
  switch (m) {
    case 64: return launch_dop<T, 6>(z, out, row_off, l_count, blocked, tw, gain, s);
    case 128: return launch_dop<T, 7>(z, out, row_off, l_count, blocked, tw, gain, s);
    case 256: return launch_dop<T, 8>(z, out, row_off, l_count, blocked, tw, gain, s);
    case 512: return launch_dop<T, 9>(z, out, row_off, l_count, blocked, tw, gain, s);
    case 1024: return launch_dop<T, 10>(z, out, row_off, l_count, blocked, tw, gain, s);
    case 2048: return launch_dop<T, 11>(z, out, row_off, l_count, blocked, tw, gain, s);
    default: return SA_ERR_UNSUPPORTED;
  }
}

}  // namespace

bool sa_doppler_supported(int64_t m) { return m >= 64 && m <= 2048 && (m & (m - 1)) == 0; }

// DIT NL-FFT of gain * z rows (blocked: zb tiles of 16 rows counted from the
// 16-aligned base, valid rows row_off .. row_off + l_count - 1; row-major:
// z[(row) * m + q], row_off must be 0) into out (l_count x m, row-major).
int sa_launch_doppler_nlfft(int dtype, const void *z, void *out, int row_off, int64_t l_count, int64_t m,
                            int blocked, const SaTwiddles *tw, double gain, cudaStream_t s) {
  if (l_count == 0) return SA_OK;
  if (!sa_doppler_supported(m) || !tw->stage) return SA_ERR_UNSUPPORTED;
  if (dtype == SA_C64) return launch_dop_t<float>(z, out, row_off, l_count, m, blocked, tw, gain, s);
  return launch_dop_t<double>(z, out, row_off, l_count, m, blocked, tw, gain, s);
}
