// sa_internal.h -- internal launchers shared by the kernel translation units and
// the C ABI (sa_abi.cu).  Not part of the public interface (see include/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/signadd_b200.h"

// Device-resident twiddle set for one (device, n, dtype).  Built from the HOST
// reference table (transforms.py:122-133) -- never from device sincos.
struct SaTwiddles {
  int dtype;
  int64_t n;
  int device;
  void *raw;    // n complex entries (c64: round-to-nearest cast of the fp64 table)
  void *quad;   // n x {wr, wi, sgn wr, sgn wi}                      (NDFT)
  void *stage;  // (n-1) x {|wr|, |wi|, sgn wr, sgn wi}, stage-packed:
                //   stage s (1..log2 n) at offset 2^(s-1)-1, entry j = table[j*n/2^s]
  void *stage2; // (n-1) x {wr, wi}, same stage-packed order (8/16-byte entries)
  void *tcw;    // tensor-core NDFT operands [W0; W1; sgn Wv] (bf16, 3 x 2n x 2n), built on first use
  void *tcw_ready;  // cudaEvent_t recorded after the tcw build (streams wait on it)
  void *i8w;        // complex128 tensor-core NDFT: six int8 planes of Wv (sa_ndft_i8.cu), built on first use
  void *i8w_ready;
};

void sa_set_error(const char *fmt, ...);
// stream-ordered scratch from a per-device pool that keeps its memory (free with cudaFreeAsync)
int sa_scratch_alloc(void **p, size_t bytes, cudaStream_t s);

#define SA_CUDA_TRY(expr)                                                       \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      sa_set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),       \
                   __FILE__, __LINE__);                                         \
      return SA_ERR_CUDA;                                                       \
    }                                                                           \
  } while (0)

#define SA_LAUNCH_CHECK()                                                       \
  do {                                                                          \
    cudaError_t _e = cudaGetLastError();                                        \
    if (_e != cudaSuccess) {                                                    \
      sa_set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e),  \
                   __FILE__, __LINE__);                                         \
      return SA_ERR_CUDA;                                                       \
    }                                                                           \
  } while (0)

// sa_twiddles.cu
int sa_twiddles_build(SaTwiddles *tw, const double *host_table, cudaStream_t s);

// sa_mf.cu
int sa_launch_mf_complex(int dtype, const void *a, const void *b, void *out, int64_t count,
                         cudaStream_t s);
int sa_launch_check_finite(int dtype, const void *x, int64_t count, int *d_flag, cudaStream_t s);
int sa_launch_fma_peak(int dtype, int64_t iters, void *d_sink, int blocks, cudaStream_t s);

// sa_ndft.cu
int sa_launch_ndft(int dtype, const void *x, void *y, int64_t batch, int64_t n,
                   const SaTwiddles *tw, int mode, double gain, cudaStream_t s);

// sa_ndft_tc.cu (tensor-core fast mode; SA_ERR_UNSUPPORTED -> use the FFMA2 kernels)
bool sa_ndft_tc_supported(int dtype, int64_t n);
int sa_launch_ndft_tc(const void *x, void *y, int64_t batch, int64_t n, const SaTwiddles *tw, double gain,
                      cudaStream_t s);
// sa_ndft_i8.cu (complex128 fast mode on tcgen05 kind::i8, exact integer digits)
bool sa_ndft_i8_supported(int dtype, int64_t n);
int sa_launch_ndft_i8(const void *x, void *y, int64_t batch, int64_t n, const SaTwiddles *tw, double gain,
                      cudaStream_t s);

// sa_lag_tc.cu (tensor-core fast-mode lag integration, complex64)
bool sa_lag_tc_supported(int dtype, int64_t tb, int64_t m, const void *surv);
int sa_launch_lag_tc(const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count, int64_t m,
                     int64_t tb, int conj, void *z, int blocked, cudaStream_t s);
int sa_launch_lag_tc_blocks(const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count, int64_t m,
                            int64_t q0, int64_t q_count, int64_t tb, int conj, void *z, void *const *dst_rows,
                            int64_t rows_base, int64_t rows_extra, int blocked, cudaStream_t s);
// sa_lag_i8.cu (the same lag stage on tcgen05 kind::i8, exact integer digits; the default,
// SA_LAG_KIND=bf16 selects sa_lag_tc.cu; SA_ERR_UNSUPPORTED -> the bf16 kernel)
bool sa_lag_i8_enabled();
int sa_launch_lag_i8_blocks(const void *surv, const void *ref, int64_t ref_len, int64_t l0, int64_t l_count, int64_t m,
                            int64_t q0, int64_t q_count, int64_t tb, int conj, void *z, void *const *dst_rows,
                            int64_t rows_base, int64_t rows_extra, int blocked, cudaStream_t s);
// blocked z: tiles of 16 lags from the 16-aligned base (sa_lag_tc.cu), rows padded to whole tiles
inline int64_t sa_zblk_rows(int64_t l0, int64_t l_count) { return (((l0 & 15) + l_count + 15) / 16) * 16; }

// sa_doppler.cu (the map's Doppler NL-FFT straight from (blocked) z, M = 64 .. 2048)
bool sa_doppler_supported(int64_t m);
int sa_launch_doppler_nlfft(int dtype, const void *z, void *out, int row_off, int64_t l_count, int64_t m,
                            int blocked, const SaTwiddles *tw, double gain, cudaStream_t s);

// sa_nlfft.cu
int sa_launch_nlfft(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
                    const SaTwiddles *tw, double gain, cudaStream_t s);

// sa_nlfft64k.cu (fused single-pass N = 2^16; SA_ERR_UNSUPPORTED -> use the generic path)
int sa_launch_nlfft64k(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
                       const SaTwiddles *tw, double gain, cudaStream_t s);

// sa_nlfft2p.cu (persistent work-queue two-pass N = 2^16, DIT, out of place)
int sa_launch_nlfft2p(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
                      const SaTwiddles *tw, double gain, cudaStream_t s);

// sa_ambiguity.cu
int64_t sa_ambiguity_ws_bytes(int dtype, int64_t l_count, int64_t m);
int64_t sa_peaks_ws_bytes(int64_t rows, int64_t cols, int k);
int sa_launch_map_peaks(int dtype, const void *map, int64_t rows, int64_t cols, int k, long long *idx, double *mag,
                        int *count, void *ws, cudaStream_t s);
int sa_launch_map_floor(int dtype, const void *map, int64_t rows, int64_t cols, const int *centers, int ncent,
                        int g0, int g1, unsigned long long *out, cudaStream_t s);
int sa_launch_stereo_fm(int dtype, const double *u, int64_t n, double f_s, double ca, double cb, double cc,
                        double ck, void *out, cudaStream_t s);
int sa_launch_echoes(const void *ref, int64_t d, int ne, const int64_t *delays, const double *amps, const double *w,
                     double inv_fs, void *out, cudaStream_t s);
int64_t sa_power_ws_bytes(int64_t d);
int sa_launch_power(const void *x, int64_t d, double *ws, double *sum, cudaStream_t s);
int sa_launch_noise_gain(int dtype, const void *x, int64_t d, int kind, const double *z, const double *u, double scale,
                         double eps, double s1, double s2, double gain, void *out, cudaStream_t s);
int sa_launch_lag_product(int dtype, int lag_kind, const void *surv, const void *ref, int64_t n, int64_t ref_len,
                          int64_t lag, int conj, void *out, cudaStream_t s);
int sa_launch_lag_integrate(int dtype, int lag_kind, const void *surv, const void *ref, int64_t ns,
                            int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, int conj,
                            int mode, void *z, cudaStream_t s);

// Launch with programmatic stream serialization (PDL): the kernel's CTAs may become
// resident while the previous kernel in the stream drains, if that kernel executed
// griddepcontrol.launch_dependents; the launched kernel must execute
// griddepcontrol.wait before touching anything its predecessor wrote (sa_pdl_wait()).
// Off by default (SA_MAP_PDL=1 in the environment enables it): one full GPU test run with it
// showed a stale scale read in the lag kernel (test_lag_i8_nonfinite, not reproducible alone) --
// L1 / read-only-cache lines of a recycled scratch address are not known to be invalidated for a
// programmatically launched grid, and the kernels of the chain read their predecessors' outputs
// with cached loads (with ld.global.cg loads four full runs passed, at ~1% cost on the C5 map:
// DESIGN 5.3e).  Experimental: not safe as built.  The griddepcontrol instructions are no-ops
// for normal launches.
#ifdef __CUDACC__
#include <cstdlib>
#include <utility>
inline bool sa_pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SA_MAP_PDL");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}
template <typename... KArgs, typename... Args>
inline cudaError_t sa_launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                 Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = sa_pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
__device__ __forceinline__ void sa_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void sa_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif
