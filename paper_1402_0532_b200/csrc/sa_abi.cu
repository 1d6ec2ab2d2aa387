// sa_abi.cu -- the extern "C" boundary (include/signadd_b200.h).
//
// Argument validation mirrors the reference contracts so the Python shim can
// map status codes to the reference exception classes:
//   SA_ERR_CONTRACT <-> ContractError (transforms.py:166-169; ambiguity.py:121-128)
//   SA_ERR_DOMAIN   <-> DomainError   (operator.py:112-115; transforms.py:161-162)
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "sa_common.cuh"
#include <cstring>

#include "sa_internal.h"

static thread_local char g_err[512] = "";

void sa_set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

#define SA_REQUIRE(cond, code, ...) \
  do {                              \
    if (!(cond)) {                  \
      sa_set_error(__VA_ARGS__);    \
      return code;                  \
    }                               \
  } while (0)

static bool dtype_ok(int d) { return d == SA_C64 || d == SA_C128; }
static bool pow2(int64_t n) { return n >= 2 && (n & (n - 1)) == 0; }

static int check_tw(const void *tw, int dtype, int64_t n, bool need_stage) {
  const SaTwiddles *t = (const SaTwiddles *)tw;
  SA_REQUIRE(t != nullptr, SA_ERR_ARG, "twiddle handle is null");
  SA_REQUIRE(t->dtype == dtype, SA_ERR_ARG, "twiddle dtype %d != %d", t->dtype, dtype);
  SA_REQUIRE(t->n == n, SA_ERR_ARG, "twiddle set is for n=%lld, call needs n=%lld",
             (long long)t->n, (long long)n);
  SA_REQUIRE(!need_stage || t->stage != nullptr, SA_ERR_ARG, "twiddle set has no stage table");
  int dev = -1;
  cudaGetDevice(&dev);
  SA_REQUIRE(dev == t->device, SA_ERR_ARG, "twiddle set lives on device %d, current is %d",
             t->device, dev);
  return SA_OK;
}

extern "C" {

int sa_version(void) { return SA_ABI_VERSION; }

const char *sa_last_error(void) { return g_err; }

int sa_twiddle_create(int device, int dtype, int64_t n, const double *host_table, void *stream,
                      void **handle) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(n >= 1, SA_ERR_CONTRACT, "TwiddleTable: size must be >= 1");
  SA_REQUIRE(host_table && handle, SA_ERR_ARG, "null pointer");
  int prev = 0;
  SA_CUDA_TRY(cudaGetDevice(&prev));
  SA_CUDA_TRY(cudaSetDevice(device));
  SaTwiddles *tw = new SaTwiddles{dtype, n, device, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int rc = sa_twiddles_build(tw, host_table, (cudaStream_t)stream);
  cudaSetDevice(prev);
  if (rc != SA_OK) {
    cudaFree(tw->raw);
    cudaFree(tw->quad);
    cudaFree(tw->stage);
    cudaFree(tw->stage2);
    cudaFree(tw->tcw);
    delete tw;
    return rc;
  }
  *handle = tw;
  return SA_OK;
}

int sa_twiddle_destroy(void *handle) {
  SaTwiddles *tw = (SaTwiddles *)handle;
  if (!tw) return SA_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(tw->device);
  cudaFree(tw->raw);
  cudaFree(tw->quad);
  cudaFree(tw->stage);
  cudaFree(tw->stage2);
  cudaFree(tw->tcw);
  if (tw->tcw_ready) cudaEventDestroy((cudaEvent_t)tw->tcw_ready);
  cudaFree(tw->i8w);
  if (tw->i8w_ready) cudaEventDestroy((cudaEvent_t)tw->i8w_ready);
  cudaSetDevice(prev);
  delete tw;
  return SA_OK;
}

int sa_mf_complex(int dtype, const void *a, const void *b, void *out, int64_t count,
                  void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(count >= 0, SA_ERR_ARG, "negative count");
  SA_REQUIRE(count == 0 || (a && b && out), SA_ERR_ARG, "null pointer");
  return sa_launch_mf_complex(dtype, a, b, out, count, (cudaStream_t)stream);
}

int sa_check_finite(int dtype, const void *x, int64_t count, int *d_flag, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(count >= 0 && d_flag, SA_ERR_ARG, "bad arguments");
  SA_REQUIRE(count == 0 || x, SA_ERR_ARG, "null pointer");
  return sa_launch_check_finite(dtype, x, count, d_flag, (cudaStream_t)stream);
}

int sa_ndft(int dtype, const void *x, void *y, int64_t batch, int64_t n, const void *tw, int mode,
            double gain, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(n >= 1, SA_ERR_CONTRACT, "transform input must be a 1-d sequence of length >= 1");
  SA_REQUIRE(batch >= 0, SA_ERR_ARG, "negative batch");
  SA_REQUIRE(mode == SA_NDFT_FAST || mode == SA_NDFT_EXACT || mode == SA_NDFT_TC || mode == SA_NDFT_TC_I8,
             SA_ERR_ARG, "bad mode %d", mode);
  SA_REQUIRE(batch == 0 || (x && y), SA_ERR_ARG, "null pointer");
  SA_REQUIRE(x != y || batch == 0, SA_ERR_ARG, "sa_ndft: x and y must not overlap");
  int rc = check_tw(tw, dtype, n, false);
  if (rc) return rc;
  if (mode == SA_NDFT_TC || mode == SA_NDFT_TC_I8) {
    rc = (dtype == SA_C64 && mode == SA_NDFT_TC)
             ? sa_launch_ndft_tc(x, y, batch, n, (const SaTwiddles *)tw, gain, (cudaStream_t)stream)
             : sa_launch_ndft_i8(x, y, batch, n, (const SaTwiddles *)tw, gain, (cudaStream_t)stream);
    if (rc != SA_ERR_UNSUPPORTED) return rc;
    mode = SA_NDFT_FAST;  // other shapes / unaligned views: the same regrouped sum on the FFMA2 kernels
  }
  return sa_launch_ndft(dtype, x, y, batch, n, (const SaTwiddles *)tw, mode, gain,
                        (cudaStream_t)stream);
}

int sa_nlfft(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
             const void *tw, double gain, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(variant == SA_DIT || variant == SA_DIF || variant == SA_FFT_EXACT, SA_ERR_ARG, "bad variant %d",
             variant);
  SA_REQUIRE(pow2(n), SA_ERR_CONTRACT, "nfft: size must be a power of two >= 2, got %lld",
             (long long)n);
  SA_REQUIRE(batch >= 0, SA_ERR_ARG, "negative batch");
  SA_REQUIRE(batch == 0 || (x && y), SA_ERR_ARG, "null pointer");
  int rc = check_tw(tw, dtype, n, true);
  if (rc) return rc;
  return sa_launch_nlfft(dtype, variant, x, y, batch, n, (const SaTwiddles *)tw, gain,
                         (cudaStream_t)stream);
}

// ambiguity.py:116-131 guards
static int lag_guards(int64_t n, int64_t surv_len, int64_t ref_len, int64_t lag) {
  SA_REQUIRE(lag >= 0, SA_ERR_CONTRACT, "lag must be non-negative, got %lld", (long long)lag);
  SA_REQUIRE(lag < ref_len, SA_ERR_CONTRACT, "lag %lld is not below the reference length %lld",
             (long long)lag, (long long)ref_len);
  SA_REQUIRE(surv_len >= n, SA_ERR_CONTRACT, "surveillance signal shorter than n=%lld",
             (long long)n);
  SA_REQUIRE(ref_len >= n - lag, SA_ERR_CONTRACT, "reference signal too short for n=%lld, lag=%lld",
             (long long)n, (long long)lag);
  return SA_OK;
}

int sa_lag_product_mf(int dtype, const void *surv, const void *ref, int64_t n, int64_t ref_len,
                      int64_t lag, int conj, void *out, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(n >= 0, SA_ERR_ARG, "negative n");
  int rc = lag_guards(n, n, ref_len, lag);
  if (rc) return rc;
  SA_REQUIRE(n == 0 || (surv && ref && out), SA_ERR_ARG, "null pointer");
  return sa_launch_lag_product(dtype, SA_LAG_MF, surv, ref, n, ref_len, lag, conj, out, (cudaStream_t)stream);
}

int sa_lag_product_exact(int dtype, const void *surv, const void *ref, int64_t n, int64_t ref_len,
                         int64_t lag, int conj, void *out, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(n >= 0, SA_ERR_ARG, "negative n");
  int rc = lag_guards(n, n, ref_len, lag);
  if (rc) return rc;
  SA_REQUIRE(n == 0 || (surv && ref && out), SA_ERR_ARG, "null pointer");
  return sa_launch_lag_product(dtype, SA_LAG_EXACT, surv, ref, n, ref_len, lag, conj, out,
                               (cudaStream_t)stream);
}

int sa_ambiguity_workspace_bytes(int dtype, int64_t l_count, int64_t m, int64_t *bytes) {
  SA_REQUIRE(dtype_ok(dtype) && bytes && l_count >= 0 && m >= 1, SA_ERR_ARG, "bad arguments");
  *bytes = sa_ambiguity_ws_bytes(dtype, l_count, m);
  return SA_OK;
}

int sa_ambiguity_map(int dtype, const void *surv, const void *ref, int64_t ns, int64_t ref_len,
                     int64_t l0, int64_t l_count, int64_t m, double gain, int conj, int doppler,
                     int mode, const void *tw, void *out, void *workspace, int64_t ws_bytes,
                     void *stream) {
  return sa_ambiguity_map_v(dtype, SA_LAG_MF, surv, ref, ns, ref_len, l0, l_count, m, gain, conj, doppler,
                            mode, tw, out, workspace, ws_bytes, stream);
}

int sa_ambiguity_map_v(int dtype, int lag_kind, const void *surv, const void *ref, int64_t ns,
                       int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, double gain, int conj,
                       int doppler, int mode, const void *tw, void *out, void *workspace,
                       int64_t ws_bytes, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(lag_kind == SA_LAG_MF || lag_kind == SA_LAG_EXACT, SA_ERR_ARG, "bad lag kind %d", lag_kind);
  SA_REQUIRE(l_count >= 1, SA_ERR_CONTRACT, "l_bins must be >= 1");
  SA_REQUIRE(m >= 1 && ns >= m && ns % m == 0, SA_ERR_CONTRACT,
             "map: ns=%lld must be a positive multiple of m=%lld", (long long)ns, (long long)m);
  SA_REQUIRE(doppler == SA_DOPPLER_NLFFT || doppler == SA_DOPPLER_NDFT || doppler == SA_DOPPLER_FFT_EXACT,
             SA_ERR_ARG, "bad doppler %d", doppler);
  SA_REQUIRE(doppler == SA_DOPPLER_NDFT || pow2(m), SA_ERR_CONTRACT,
             "nfft: size must be a power of two >= 2, got %lld", (long long)m);
  SA_REQUIRE(mode == SA_NDFT_FAST || mode == SA_NDFT_EXACT, SA_ERR_ARG, "bad mode %d", mode);
  // the largest lag must satisfy the lag_product_mf guards for n = ns
  int rc = lag_guards(ns, ns, ref_len, l0 + l_count - 1);
  if (rc) return rc;
  rc = lag_guards(ns, ns, ref_len, l0);
  if (rc) return rc;
  SA_REQUIRE(surv && ref && out, SA_ERR_ARG, "null pointer");
  int64_t need = sa_ambiguity_ws_bytes(dtype, l_count, m);
  SA_REQUIRE(workspace && ws_bytes >= need, SA_ERR_ARG, "workspace too small: %lld < %lld bytes",
             (long long)ws_bytes, (long long)need);
  rc = check_tw(tw, dtype, m, doppler != SA_DOPPLER_NDFT);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (doppler == SA_DOPPLER_NLFFT && sa_doppler_supported(m)) {
    // lag stage -> Doppler NL-FFT (sa_doppler.cu, register radix-16 rounds); on the
    // tensor-core lag path z travels in the blocked layout (whole-sector stores)
    const bool blk = mode == SA_NDFT_FAST && lag_kind == SA_LAG_MF && ns != m &&
                     sa_lag_tc_supported(dtype, ns / m, m, surv);
    rc = blk ? sa_launch_lag_tc(surv, ref, ref_len, l0, l_count, m, ns / m, conj, workspace, 1, s)
             : sa_launch_lag_integrate(dtype, lag_kind, surv, ref, ns, ref_len, l0, l_count, m, conj, mode,
                                       workspace, s);
    if (rc) return rc;
    return sa_launch_doppler_nlfft(dtype, workspace, out, blk ? (int)(l0 & 15) : 0, l_count, m, blk ? 1 : 0,
                                   (const SaTwiddles *)tw, gain, s);
  }
  rc = sa_launch_lag_integrate(dtype, lag_kind, surv, ref, ns, ref_len, l0, l_count, m, conj, mode,
                               workspace, s);
  if (rc) return rc;
  if (doppler != SA_DOPPLER_NDFT)
    return sa_launch_nlfft(dtype, doppler == SA_DOPPLER_NLFFT ? SA_DIT : SA_FFT_EXACT, workspace, out, l_count,
                           m, (const SaTwiddles *)tw, gain, s);
  if (ns != m && mode == SA_NDFT_FAST) {  // fast-mode Doppler NDFT: the tensor-core kernel where it applies
    rc = sa_launch_ndft_tc(workspace, out, l_count, m, (const SaTwiddles *)tw, gain, s);
    if (rc != SA_ERR_UNSUPPORTED) return rc;
  }
  return sa_launch_ndft(dtype, workspace, out, l_count, m, (const SaTwiddles *)tw,
                        ns == m ? SA_NDFT_EXACT : mode, gain, s);
}

int sa_ambiguity_integrate(int dtype, const void *surv, const void *ref, int64_t ns,
                           int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, int conj,
                           int mode, void *z, void *stream) {
  return sa_ambiguity_integrate_v(dtype, SA_LAG_MF, surv, ref, ns, ref_len, l0, l_count, m, conj, mode, z,
                                  stream);
}

int sa_ambiguity_integrate_v(int dtype, int lag_kind, const void *surv, const void *ref, int64_t ns,
                             int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, int conj,
                             int mode, void *z, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(lag_kind == SA_LAG_MF || lag_kind == SA_LAG_EXACT, SA_ERR_ARG, "bad lag kind %d", lag_kind);
  SA_REQUIRE(l_count >= 1, SA_ERR_CONTRACT, "l_bins must be >= 1");
  SA_REQUIRE(m >= 1 && ns >= m && ns % m == 0, SA_ERR_CONTRACT,
             "map: ns=%lld must be a positive multiple of m=%lld", (long long)ns, (long long)m);
  SA_REQUIRE(mode == SA_NDFT_FAST || mode == SA_NDFT_EXACT, SA_ERR_ARG, "bad mode %d", mode);
  int rc = lag_guards(ns, ns, ref_len, l0 + l_count - 1);
  if (rc) return rc;
  rc = lag_guards(ns, ns, ref_len, l0);
  if (rc) return rc;
  SA_REQUIRE(surv && ref && z, SA_ERR_ARG, "null pointer");
  return sa_launch_lag_integrate(dtype, lag_kind, surv, ref, ns, ref_len, l0, l_count, m, conj, mode, z,
                                 (cudaStream_t)stream);
}

int sa_ambiguity_integrate_blocks(int dtype, const void *surv, const void *ref, int64_t ns, int64_t ref_len,
                                  int64_t l0, int64_t l_count, int64_t m, int64_t q0, int64_t q_count, int conj,
                                  void *const *dst_rows, int64_t n_dst, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(l_count >= 1, SA_ERR_CONTRACT, "l_bins must be >= 1");
  SA_REQUIRE(m >= 1 && ns >= m && ns % m == 0, SA_ERR_CONTRACT,
             "map: ns=%lld must be a positive multiple of m=%lld", (long long)ns, (long long)m);
  SA_REQUIRE(q0 >= 0 && q_count >= 0 && q0 + q_count <= m, SA_ERR_ARG, "bad block range");
  SA_REQUIRE(n_dst >= 1 && n_dst <= l_count && dst_rows, SA_ERR_ARG, "bad destination rows");
  // owners' rows are whole 16-lag tiles of the blocked z layout
  SA_REQUIRE(l0 == 0 && l_count % (16 * n_dst) == 0, SA_ERR_UNSUPPORTED,
             "block-sharded lag stage needs l0 = 0 and l_count a multiple of 16 x n_dst");
  int rc = lag_guards(ns, ns, ref_len, l0 + l_count - 1);
  if (rc) return rc;
  rc = lag_guards(ns, ns, ref_len, l0);
  if (rc) return rc;
  SA_REQUIRE(surv && ref, SA_ERR_ARG, "null pointer");
  if (!sa_lag_tc_supported(dtype, ns / m, m, surv)) return SA_ERR_UNSUPPORTED;
  return sa_launch_lag_tc_blocks(surv, ref, ref_len, l0, l_count, m, q0, q_count, ns / m, conj, nullptr, dst_rows,
                                 l_count / n_dst, l_count % n_dst, 1, (cudaStream_t)stream);
}

int sa_doppler_nlfft_blocked(int dtype, const void *zb, void *out, int64_t l_count, int64_t m, const void *tw,
                             double gain, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(l_count >= 0 && sa_doppler_supported(m), SA_ERR_UNSUPPORTED,
             "blocked Doppler NL-FFT needs m = 64 .. 2048, a power of two (got %lld)", (long long)m);
  SA_REQUIRE(zb && out, SA_ERR_ARG, "null pointer");
  int rc = check_tw(tw, dtype, m, true);
  if (rc) return rc;
  return sa_launch_doppler_nlfft(dtype, zb, out, 0, l_count, m, 1, (const SaTwiddles *)tw, gain,
                                 (cudaStream_t)stream);
}

int sa_peaks_workspace_bytes(int64_t rows, int64_t cols, int k, int64_t *bytes) {
  SA_REQUIRE(bytes && rows >= 1 && cols >= 1 && k >= 1, SA_ERR_ARG, "bad arguments");
  *bytes = sa_peaks_ws_bytes(rows, cols, k);
  return SA_OK;
}

int sa_map_peaks(int dtype, const void *map, int64_t rows, int64_t cols, int k, int64_t *idx,
                 double *mag, int32_t *count, void *workspace, int64_t ws_bytes, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(k >= 1, SA_ERR_CONTRACT, "find_peaks: k must be >= 1");
  SA_REQUIRE(k <= 1024, SA_ERR_UNSUPPORTED, "find_peaks: k = %d > 1024", k);
  SA_REQUIRE(rows >= 1 && cols >= 1, SA_ERR_ARG, "empty map");
  SA_REQUIRE(map && idx && mag && count && workspace, SA_ERR_ARG, "null pointer");
  SA_REQUIRE(ws_bytes >= sa_peaks_ws_bytes(rows, cols, k), SA_ERR_ARG, "workspace too small");
  return sa_launch_map_peaks(dtype, map, rows, cols, k, (long long *)idx, mag, count, workspace,
                             (cudaStream_t)stream);
}

int sa_map_floor(int dtype, const void *map, int64_t rows, int64_t cols, const int32_t *centers,
                 int ncent, int g0, int g1, uint64_t *out, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(g0 >= 0 && g1 >= 0 && ncent >= 0, SA_ERR_ARG, "bad guard");
  SA_REQUIRE(rows >= 1 && cols >= 1, SA_ERR_ARG, "empty map");
  SA_REQUIRE(map && out && (centers || ncent == 0), SA_ERR_ARG, "null pointer");
  return sa_launch_map_floor(dtype, map, rows, cols, centers, ncent, g0, g1, (unsigned long long *)out,
                             (cudaStream_t)stream);
}

int sa_scene_stereo_fm(int dtype, const double *u, int64_t n, double f_s, double ca, double cb, double cc,
                       double ck, void *out, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(n >= 0, SA_ERR_ARG, "negative length");
  SA_REQUIRE(n == 0 || (u && out), SA_ERR_ARG, "null pointer");
  SA_REQUIRE(f_s > 0.0, SA_ERR_CONTRACT, "gen_stereo_fm: f_s must be positive");
  return sa_launch_stereo_fm(dtype, u, n, f_s, ca, cb, cc, ck, out, (cudaStream_t)stream);
}

int sa_scene_echoes(const void *ref, int64_t d, int ne, const int64_t *delays, const double *amps,
                    const double *w, double inv_fs, void *out, void *stream) {
  SA_REQUIRE(ne >= 1, SA_ERR_CONTRACT, "synth_surveillance: need at least one obstacle");
  SA_REQUIRE(ne <= 64, SA_ERR_UNSUPPORTED, "synth_surveillance: %d obstacles > 64", ne);
  SA_REQUIRE(d >= 0, SA_ERR_ARG, "negative length");
  SA_REQUIRE(delays && amps && w && (d == 0 || (ref && out)), SA_ERR_ARG, "null pointer");
  for (int k = 0; k < ne; ++k) SA_REQUIRE(delays[k] >= 0, SA_ERR_CONTRACT, "negative delay");
  return sa_launch_echoes(ref, d, ne, delays, amps, w, inv_fs, out, (cudaStream_t)stream);
}

int sa_scene_power_workspace_bytes(int64_t d, int64_t *bytes) {
  SA_REQUIRE(bytes && d >= 0, SA_ERR_ARG, "bad arguments");
  *bytes = sa_power_ws_bytes(d);
  return SA_OK;
}

int sa_scene_power(const void *x, int64_t d, double *sum, void *workspace, int64_t ws_bytes, void *stream) {
  SA_REQUIRE(d >= 1, SA_ERR_CONTRACT, "add_awgn: empty input");
  SA_REQUIRE(x && sum && workspace, SA_ERR_ARG, "null pointer");
  SA_REQUIRE(ws_bytes >= sa_power_ws_bytes(d), SA_ERR_ARG, "workspace too small");
  return sa_launch_power(x, d, (double *)workspace, sum, (cudaStream_t)stream);
}

int sa_scene_noise_gain(int dtype, const void *x, int64_t d, int kind, const double *z, const double *u,
                        double scale, double eps, double s1, double s2, double gain, void *out, void *stream) {
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(kind == SA_NOISE_NONE || kind == SA_NOISE_AWGN || kind == SA_NOISE_EPS, SA_ERR_ARG,
             "bad noise kind %d", kind);
  SA_REQUIRE(d >= 0, SA_ERR_ARG, "negative length");
  SA_REQUIRE(d == 0 || (x && out), SA_ERR_ARG, "null pointer");
  SA_REQUIRE(kind == SA_NOISE_NONE || z, SA_ERR_ARG, "null noise draws");
  SA_REQUIRE(kind != SA_NOISE_EPS || u, SA_ERR_ARG, "null mixture draws");
  return sa_launch_noise_gain(dtype, x, d, kind, z, u, scale, eps, s1, s2, gain, out, (cudaStream_t)stream);
}

int sa_enable_peer_access(int peer_device) {
  int dev = 0, n = 0, ok = 0;
  SA_CUDA_TRY(cudaGetDevice(&dev));
  SA_CUDA_TRY(cudaGetDeviceCount(&n));
  SA_REQUIRE(peer_device >= 0 && peer_device < n, SA_ERR_ARG, "bad peer device %d", peer_device);
  if (peer_device == dev) return SA_OK;
  SA_CUDA_TRY(cudaDeviceCanAccessPeer(&ok, dev, peer_device));
  SA_REQUIRE(ok, SA_ERR_UNSUPPORTED, "device %d cannot access peer %d", dev, peer_device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SA_OK;
  }
  SA_CUDA_TRY(e);
  return SA_OK;
}

int sa_ambiguity_map_multi(int ndev, const int *devs, int dtype, int lag_kind, const void *const *surv,
                           const void *const *ref, int64_t ns, int64_t ref_len, int64_t l0, int64_t l_count,
                           int64_t m, double gain, int conj, int doppler, int mode, const void *const *tw,
                           void *out, void *const *workspace, const int64_t *ws_bytes, void *const *stream) {
  SA_REQUIRE(ndev >= 1 && devs && surv && ref && tw && workspace && ws_bytes && stream && out, SA_ERR_ARG,
             "bad arguments");
  SA_REQUIRE(dtype_ok(dtype), SA_ERR_ARG, "bad dtype %d", dtype);
  SA_REQUIRE(l_count >= 1, SA_ERR_CONTRACT, "l_bins must be >= 1");
  int prev = 0;
  SA_CUDA_TRY(cudaGetDevice(&prev));
  const int64_t row_bytes = m * (dtype == SA_C64 ? 8 : 16);
  const int64_t base = l_count / ndev, extra = l_count % ndev;
  int rc = SA_OK;
  for (int g = 0; g < ndev && rc == SA_OK; ++g) {
    const int64_t count = base + (g < extra ? 1 : 0);
    const int64_t first = g * base + (g < extra ? g : extra);
    if (cudaSetDevice(devs[g]) != cudaSuccess) {
      sa_set_error("cudaSetDevice(%d) failed", devs[g]);
      rc = SA_ERR_CUDA;
      break;
    }
    if (devs[g] != devs[0]) rc = sa_enable_peer_access(devs[0]);
    if (rc == SA_OK && count > 0)
      rc = sa_ambiguity_map_v(dtype, lag_kind, surv[g], ref[g], ns, ref_len, l0 + first, count, m, gain, conj,
                              doppler, mode, tw[g], (char *)out + first * row_bytes, workspace[g], ws_bytes[g],
                              stream[g]);
  }
  cudaSetDevice(prev);
  return rc;
}

int sa_ipc_open(const void *handle64, void **dptr) {
  SA_REQUIRE(handle64 && dptr, SA_ERR_ARG, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  SA_CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SA_OK;
}

int sa_ipc_close(void *dptr) {
  SA_REQUIRE(dptr, SA_ERR_ARG, "null pointer");
  SA_CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return SA_OK;
}

int sa_fma_peak(int dtype, int64_t iters, void *d_sink, int blocks, void *stream) {
  SA_REQUIRE((dtype_ok(dtype) || dtype == 2) && d_sink && iters > 0 && blocks > 0, SA_ERR_ARG,
             "bad arguments");
  return sa_launch_fma_peak(dtype, iters, d_sink, blocks, (cudaStream_t)stream);
}

}  // extern "C"
