// sa_nlfft.cu -- nonlinear radix-2 FFT (⊙ replaces every twiddle product).
//
// DIT is value-identical to nfft (transforms.py:254-298): bottom stage is the
// full 2-point NDFT (1⊗a, 1⊗b; y0=u+t, y1=u−t, :270-280); stages m=4..N apply
// w_j = entries[j*N/m] to the odd branch, top = a + w⊗b and bot = a + (−w)⊗b,
// evaluated as a − (w⊗b) which is exactly equal (test_operator.py:225-229).
// DIF follows the DESIGN.md convention (no reference; "parity unpinned").
// The same kernels run fft_exact (transforms.py:200-220, variant SA_FFT_EXACT):
// every stage an exact butterfly with numpy's complex multiply of the raw twiddle.
//
// Node layout is free (SURVEY §7 hard part 4): the reference's bit-reversed
// array is never materialised in HBM; bit reversal is folded into smem
// addressing.  Sizes that fit on chip run in ONE pass (one HBM read + write).
// Larger sizes use N = N1*N2 and two passes over tiles of TC sub-transforms:
//   DIT pass A  ("rows"): global stages 1..log N2 on the stride-N1 subsequences
//               x[c + N1*i] (they are the reference's bit-reversed blocks), result
//               written as row rev_N1(c) of the N1 x N2 node matrix;
//   DIT pass B  ("cols"): stages log N2 + 1 .. log N along the rows index R of
//               each column q, twiddle j = (R mod 2^(t-1))*N2 + q.
// DIF runs the mirror image (cols first, then rows + bit-reversed store).
#include <algorithm>
#include <cstdlib>

#include "sa_common.cuh"
#include "sa_internal.h"

namespace {

template <typename T> using C2 = typename SaVec<T>::c2;
template <typename T> using C4 = typename SaVec<T>::c4;

template <typename T> SA_HD C2<T> scale(C2<T> v, T g, bool use) {
  if (use) {
    v.x = sa_mul(g, v.x);
    v.y = sa_mul(g, v.y);
  }
  return v;
}

// DIT butterfly: t = w ⊗ b ; a <- a + t ; b <- a − t
template <typename T> SA_HD void bfly_dit(C2<T> &a, C2<T> &b, const C4<T> &w) {
  T tr, ti;
  sa_tw_mul<T>(w.x, w.y, w.z, w.w, b.x, b.y, tr, ti);
  C2<T> top = {sa_add(a.x, tr), sa_add(a.y, ti)};
  C2<T> bot = {sa_sub(a.x, tr), sa_sub(a.y, ti)};
  a = top;
  b = bot;
}

// DIT bottom / DIF final stage: full 2-point NDFT with the unity entries
template <typename T> SA_HD void bfly_two_point(C2<T> &a, C2<T> &b) {
  T ur, ui, tr, ti;
  sa_one_mul<T>(a.x, a.y, ur, ui);
  sa_one_mul<T>(b.x, b.y, tr, ti);
  a = {sa_add(ur, tr), sa_add(ui, ti)};
  b = {sa_sub(ur, tr), sa_sub(ui, ti)};
}

// Exact DIT butterfly of fft_exact (transforms.py:210-214): t = w * b with
// numpy's complex multiply, a <- a + t, b <- a − t.  Raw twiddle (wr, wi).
template <typename T> SA_HD void bfly_exact(C2<T> &a, C2<T> &b, const C2<T> &w) {
  T tr, ti;
  sa_npmul<T>(w.x, w.y, b.x, b.y, tr, ti);
  C2<T> top = {sa_add(a.x, tr), sa_add(a.y, ti)};
  C2<T> bot = {sa_sub(a.x, tr), sa_sub(a.y, ti)};
  a = top;
  b = bot;
}

// DIF butterfly: a <- a + b ; b <- w ⊗ (a − b)
template <typename T> SA_HD void bfly_dif(C2<T> &a, C2<T> &b, const C4<T> &w) {
  T dr = sa_sub(a.x, b.x), di = sa_sub(a.y, b.y);
  a = {sa_add(a.x, b.x), sa_add(a.y, b.y)};
  T tr, ti;
  sa_tw_mul<T>(w.x, w.y, w.z, w.w, dr, di, tr, ti);
  b = {tr, ti};
}

// One stage over a smem tile sm[pos*TC + col] holding TC transforms of length L.
// Pairs (p, p+h), h = 2^(t-1), p with bit t-1 clear.  The twiddle functor maps
// (h, p, col) -> stage-table entry.
template <typename T, int KIND, class TwF>
__device__ void tile_stage(C2<T> *sm, int TC, int L, int t, const TwF &twf) {
  const int h = 1 << (t - 1);
  const int nb = TC * (L >> 1);
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    int col = b % TC;
    int k = b / TC;
    int p = ((k >> (t - 1)) << t) | (k & (h - 1));
    C2<T> x = sm[p * TC + col];
    C2<T> y = sm[(p + h) * TC + col];
    if constexpr (KIND == 0) {
      bfly_two_point<T>(x, y);
    } else if constexpr (KIND == 1) {
      bfly_dit<T>(x, y, twf(h, p, col));
    } else if constexpr (KIND == 2) {
      bfly_dif<T>(x, y, twf(h, p, col));
    } else {
      bfly_exact<T>(x, y, twf(h, p, col));
    }
    sm[p * TC + col] = x;
    sm[(p + h) * TC + col] = y;
  }
  __syncthreads();
}

// Twiddle for a stage whose block index lives entirely in the tile position:
// stage-table offset h-1, j = p & (h-1).
template <typename T> struct TwLocal {
  const C4<T> *stage;
  SA_HD C4<T> operator()(int h, int p, int) const { return sa_ldg(&stage[(h - 1) + (p & (h - 1))]); }
};

// Twiddle for the "cols" pass: global stage s = log2(N2) + t, h_global = h*N2,
// j = (R & (h-1))*N2 + q where R = tile position, q = q0 + col.
template <typename T> struct TwCols {
  const C4<T> *stage;
  int n2, q0;
  SA_HD C4<T> operator()(int h, int R, int col) const {
    int64_t hg = (int64_t)h * n2;
    return sa_ldg(&stage[(hg - 1) + (int64_t)(R & (h - 1)) * n2 + q0 + col]);
  }
};

// Raw-twiddle functors for the exact FFT (stage-packed raw table, same indexing)
template <typename T> struct TwLocalRaw {
  const C2<T> *stage2;
  SA_HD C2<T> operator()(int h, int p, int) const { return sa_ldg(&stage2[(h - 1) + (p & (h - 1))]); }
};
template <typename T> struct TwColsRaw {
  const C2<T> *stage2;
  int n2, q0;
  SA_HD C2<T> operator()(int h, int R, int col) const {
    int64_t hg = (int64_t)h * n2;
    return sa_ldg(&stage2[(hg - 1) + (int64_t)(R & (h - 1)) * n2 + q0 + col]);
  }
};

// V: 0 = DIT nfft, 1 = DIF, 2 = exact radix-2 DIT FFT (fft_exact).
// ---------------------------------------------------------------------------
// Single pass: SPB whole transforms per CTA, all log2 N stages on chip.
// ---------------------------------------------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(256) k_nlfft_single(const C2<T> *__restrict__ x, C2<T> *y,
                                                      int64_t batch, int logn, int spb,
                                                      const C4<T> *__restrict__ stage,
                                                      const C2<T> *__restrict__ stage2, T gain,
                                                      bool use_gain) {
  constexpr bool DIF = V == 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C2<T> *sm = reinterpret_cast<C2<T> *>(smem_raw);
  const int n = 1 << logn;
  const int64_t b0 = (int64_t)blockIdx.x * spb;
  const int nsig = (int)(batch - b0 < spb ? batch - b0 : spb);
  const int tot = nsig * n;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    int sig = e >> logn, i = e & (n - 1);
    C2<T> v = scale<T>(x[(b0 + sig) * n + i], gain, use_gain);
    int pos = DIF ? i : sa_brev(i, logn);  // DIT: y0[pos] = x[rev(pos)] (transforms.py:268)
    sm[pos * spb + sig] = v;
  }
  // unused columns of a partial last tile: zeros (never stored)
  for (int e = tot + threadIdx.x; e < spb * n; e += blockDim.x) {
    int sig = e >> logn, i = e & (n - 1);
    sm[i * spb + sig] = {T(0), T(0)};
  }
  __syncthreads();
  TwLocal<T> twf{stage};
  if constexpr (V == 2) {
    TwLocalRaw<T> twr{stage2};
    for (int t = 1; t <= logn; ++t) tile_stage<T, 3>(sm, spb, n, t, twr);
  } else if constexpr (!DIF) {
    tile_stage<T, 0>(sm, spb, n, 1, twf);
    for (int t = 2; t <= logn; ++t) tile_stage<T, 1>(sm, spb, n, t, twf);
  } else {
    for (int t = logn; t >= 2; --t) tile_stage<T, 2>(sm, spb, n, t, twf);
    tile_stage<T, 0>(sm, spb, n, 1, twf);
  }
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    int sig = e >> logn, i = e & (n - 1);
    int pos = DIF ? sa_brev(i, logn) : i;  // DIF output is bit-reversed in place
    y[(b0 + sig) * n + i] = sm[pos * spb + sig];
  }
}

// ---------------------------------------------------------------------------
// Two-pass, "rows" kernel: TC sub-transforms of length N2 per CTA.
//   DIT (pass A): sub-transform c reads x[i*N1 + c] (natural i), stages 1..log N2
//                 (stage 1 = 2-point NDFT), writes node row rev_N1(c): buf[R*N2 + q].
//   DIF (pass 2): sub-transform for row R = rev_N1(c) reads buf[R*N2 + q], DIF
//                 stages log N2..2 + final 2-point, writes out[rev_N2(q)*N1 + c].
// ---------------------------------------------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(256) k_nlfft_rows(const C2<T> *__restrict__ in, C2<T> *out,
                                                    int logn1, int logn2, int tc,
                                                    const C4<T> *__restrict__ stage,
                                                    const C2<T> *__restrict__ stage2, T gain,
                                                    bool use_gain) {
  constexpr bool DIF = V == 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C2<T> *sm = reinterpret_cast<C2<T> *>(smem_raw);
  const int n1 = 1 << logn1, n2 = 1 << logn2;
  const int64_t n = (int64_t)n1 * n2;
  const int tiles = n1 / tc;
  const int64_t sig = blockIdx.x / tiles;
  const int c0 = (blockIdx.x % tiles) * tc;
  const C2<T> *src = in + sig * n;
  C2<T> *dst = out + sig * n;
  const int tot = tc * n2;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    int cc = e % tc, i = e / tc;
    if (!DIF) {
      C2<T> v = scale<T>(src[(int64_t)i * n1 + c0 + cc], gain, use_gain);
      sm[sa_brev(i, logn2) * tc + cc] = v;
    } else {
      int R = sa_brev(c0 + cc, logn1);
      sm[i * tc + cc] = src[(int64_t)R * n2 + i];
    }
  }
  __syncthreads();
  TwLocal<T> twf{stage};
  if (!DIF) {
    if constexpr (V == 2) {
      TwLocalRaw<T> twr{stage2};
      for (int t = 1; t <= logn2; ++t) tile_stage<T, 3>(sm, tc, n2, t, twr);
    } else {
      tile_stage<T, 0>(sm, tc, n2, 1, twf);
      for (int t = 2; t <= logn2; ++t) tile_stage<T, 1>(sm, tc, n2, t, twf);
    }
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      int q = e % n2, cc = e / n2;  // each sub-transform row contiguous in HBM
      int R = sa_brev(c0 + cc, logn1);
      dst[(int64_t)R * n2 + q] = sm[q * tc + cc];
    }
  } else {
    for (int t = logn2; t >= 2; --t) tile_stage<T, 2>(sm, tc, n2, t, twf);
    tile_stage<T, 0>(sm, tc, n2, 1, twf);
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      int cc = e % tc, u = e / tc;  // output row u = rev_N2(q)
      dst[(int64_t)u * n1 + c0 + cc] = sm[sa_brev(u, logn2) * tc + cc];
    }
  }
}

// ---------------------------------------------------------------------------
// Two-pass, "cols" kernel: TC columns q of the N1 x N2 node matrix per CTA,
// transform along R.  DIT pass B (stages log N2+1..log N) or DIF pass 1
// (stages log N..log N2+1).  In place is safe (tile read fully before write).
// ---------------------------------------------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(256) k_nlfft_cols(const C2<T> *in, C2<T> *out, int logn1,
                                                    int logn2, int tc,
                                                    const C4<T> *__restrict__ stage,
                                                    const C2<T> *__restrict__ stage2, T gain,
                                                    bool use_gain) {
  constexpr bool DIF = V == 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C2<T> *sm = reinterpret_cast<C2<T> *>(smem_raw);
  const int n1 = 1 << logn1, n2 = 1 << logn2;
  const int64_t n = (int64_t)n1 * n2;
  const int tiles = n2 / tc;
  const int64_t sig = blockIdx.x / tiles;
  const int q0 = (blockIdx.x % tiles) * tc;
  const C2<T> *src = in + sig * n;
  C2<T> *dst = out + sig * n;
  const int tot = tc * n1;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    int cc = e % tc, R = e / tc;
    sm[R * tc + cc] = scale<T>(src[(int64_t)R * n2 + q0 + cc], gain, use_gain);
  }
  __syncthreads();
  TwCols<T> twf{stage, n2, q0};
  if constexpr (V == 2) {
    TwColsRaw<T> twr{stage2, n2, q0};
    for (int t = 1; t <= logn1; ++t) tile_stage<T, 3>(sm, tc, n1, t, twr);
  } else if constexpr (!DIF) {
    for (int t = 1; t <= logn1; ++t) tile_stage<T, 1>(sm, tc, n1, t, twf);
  } else {
    for (int t = logn1; t >= 1; --t) tile_stage<T, 2>(sm, tc, n1, t, twf);
  }
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    int cc = e % tc, R = e / tc;
    dst[(int64_t)R * n2 + q0 + cc] = sm[R * tc + cc];
  }
}

template <typename K> int set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) {
    SA_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)bytes));
  }
  return SA_OK;
}

template <typename T>
int launch(int variant, const void *xv, void *yv, int64_t batch, int64_t n, const SaTwiddles *tw,
           double gain, cudaStream_t s) {
  const C2<T> *x = (const C2<T> *)xv;
  C2<T> *y = (C2<T> *)yv;
  const C4<T> *stage = (const C4<T> *)tw->stage;
  const C2<T> *stage2 = (const C2<T> *)tw->stage2;
  const bool use_gain = gain != 1.0;
  const T g = (T)gain;
  const int logn = sa_ilog2_host(n);
  const int single_max_log = sizeof(T) == 4 ? 13 : 12;  // 64 KiB of nodes per CTA
  if (batch == 0) return SA_OK;
  if (logn <= single_max_log) {
    int spb = (int)std::max<int64_t>(1, 4096 >> logn);
    spb = (int)std::min<int64_t>(spb, batch);
    size_t bytes = sizeof(C2<T>) * (size_t)spb * n;
    int64_t blocks = (batch + spb - 1) / spb;
    auto kern = variant == SA_DIT ? k_nlfft_single<T, 0>
                : variant == SA_DIF ? k_nlfft_single<T, 1> : k_nlfft_single<T, 2>;
    if (set_smem(kern, bytes)) return SA_ERR_CUDA;
    kern<<<(unsigned)blocks, 256, bytes, s>>>(x, y, batch, logn, spb, stage, stage2, g, use_gain);
    SA_LAUNCH_CHECK();
    return SA_OK;
  }
  if (variant != SA_FFT_EXACT) {
    // N = 2^16: persistent work-queue kernel (out of place) or the cluster kernel
    // default: cluster kernel (measured faster); SA_NLFFT_IMPL=2p selects the
    // persistent work-queue kernel (out of place, DIT) for comparison.
    static int impl = -1;
    if (impl < 0) {
      const char *e = getenv("SA_NLFFT_IMPL");
      impl = (e && e[0] == '2') ? 0 : 1;
    }
    const int d = sizeof(T) == 4 ? SA_C64 : SA_C128;
    int rc = SA_ERR_UNSUPPORTED;
    if (impl == 0) rc = sa_launch_nlfft2p(d, variant, xv, yv, batch, n, tw, gain, s);
    if (rc == SA_ERR_UNSUPPORTED) rc = sa_launch_nlfft64k(d, variant, xv, yv, batch, n, tw, gain, s);
    if (rc != SA_ERR_UNSUPPORTED) return rc;
  }
  if (x == y) {
    sa_set_error("sa_nlfft: n=%lld needs two passes; in-place (x == y) is not supported",
                 (long long)n);
    return SA_ERR_ARG;
  }
  const int logn1 = logn / 2, logn2 = logn - logn1;
  if (logn2 > 12) {
    sa_set_error("sa_nlfft: n=2^%d exceeds the supported 2^24", logn);
    return SA_ERR_UNSUPPORTED;
  }
  const int maxl = 1 << logn2;
  const int tc = std::max(1, std::min(16, 4096 / maxl));
  const int n1 = 1 << logn1, n2 = 1 << logn2;
  size_t bytes_rows = sizeof(C2<T>) * (size_t)tc * n2;
  size_t bytes_cols = sizeof(C2<T>) * (size_t)tc * n1;
  int64_t grid_rows = batch * (n1 / tc);
  int64_t grid_cols = batch * (n2 / tc);
  if (variant != SA_DIF) {
    auto rows = variant == SA_DIT ? k_nlfft_rows<T, 0> : k_nlfft_rows<T, 2>;
    auto cols = variant == SA_DIT ? k_nlfft_cols<T, 0> : k_nlfft_cols<T, 2>;
    if (set_smem(rows, bytes_rows)) return SA_ERR_CUDA;
    if (set_smem(cols, bytes_cols)) return SA_ERR_CUDA;
    rows<<<(unsigned)grid_rows, 256, bytes_rows, s>>>(x, y, logn1, logn2, tc, stage, stage2, g, use_gain);
    cols<<<(unsigned)grid_cols, 256, bytes_cols, s>>>(y, y, logn1, logn2, tc, stage, stage2, g, false);
  } else {
    if (set_smem(k_nlfft_rows<T, 1>, bytes_rows)) return SA_ERR_CUDA;
    if (set_smem(k_nlfft_cols<T, 1>, bytes_cols)) return SA_ERR_CUDA;
    // pass 2 scatters rows to bit-reversed output columns, so it cannot run in
    // place: pass 1 writes a stream-ordered scratch, pass 2 reads it.
    C2<T> *scratch = nullptr;
    {
      const int rc_ = sa_scratch_alloc((void **)&scratch, sizeof(C2<T>) * (size_t)(batch * n), s);
      if (rc_) return rc_;
    }
    k_nlfft_cols<T, 1><<<(unsigned)grid_cols, 256, bytes_cols, s>>>(x, scratch, logn1, logn2, tc, stage,
                                                                    stage2, g, use_gain);
    k_nlfft_rows<T, 1><<<(unsigned)grid_rows, 256, bytes_rows, s>>>(scratch, y, logn1, logn2, tc, stage,
                                                                    stage2, g, false);
    SA_CUDA_TRY(cudaFreeAsync(scratch, s));
  }
  SA_LAUNCH_CHECK();
  return SA_OK;
}

}  // namespace

int sa_launch_nlfft(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
                    const SaTwiddles *tw, double gain, cudaStream_t s) {
  if (dtype == SA_C64) return launch<float>(variant, x, y, batch, n, tw, gain, s);
  return launch<double>(variant, x, y, batch, n, tw, gain, s);
}
