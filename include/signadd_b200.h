/*
 * signadd_b200.h -- C ABI of the B200 (sm_100a) sign-additive hot path.
 *
 * Drop-in boundary for the reference package signadd 0.1.0 (pure Python/numpy;
 * it has no FFI of its own -- its boundary is its Python call surface, which
 * paper_1402_0532_b200/ mirrors on top of this ABI via ctypes).  Each entry
 * point names the reference interface it replaces.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes, no C++ or torch types.
 *   - Complex data is interleaved {re, im}: dtype SA_C64 = float2 (complex64),
 *     SA_C128 = double2 (complex128), matching numpy/torch layouts.
 *   - All data pointers are DEVICE pointers on the current CUDA device, owned
 *     by the caller.  The library owns only twiddle sets (create/destroy).
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered,
 *     performs no host synchronisation and is re-entrant per stream.
 *   - Return 0 on success, a negative SA_ERR_* on failure; sa_last_error()
 *     gives a thread-local message.  No exceptions cross the ABI.
 */
#ifndef SIGNADD_B200_H
#define SIGNADD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SA_ABI_VERSION 1

enum sa_dtype { SA_C64 = 0, SA_C128 = 1 };

enum sa_status {
  SA_OK = 0,
  SA_ERR_ARG = -1,         /* null pointer / bad enum / negative size        */
  SA_ERR_CONTRACT = -2,    /* reference ContractError: size, power of two, lag */
  SA_ERR_DOMAIN = -3,      /* reference DomainError: NaN / Inf operand       */
  SA_ERR_CUDA = -4,        /* CUDA runtime error                             */
  SA_ERR_UNSUPPORTED = -5  /* valid request this build does not implement    */
};

enum sa_ndft_mode {
  SA_NDFT_FAST = 0,  /* sign-split regrouped accumulation (8 FMA per ⊙)        */
  SA_NDFT_EXACT = 1, /* per-⊙ rounding, sequential accumulation: value-identical
                        to transforms.py:223-251                               */
  SA_NDFT_TC = 2,    /* the fast-mode sum on the tcgen05 tensor cores: complex64
                        as a sign-split bf16 GEMM (n % 128 == 0, n <= 4096;
                        ≤1e-4), complex128 with exact int8 digits (n % 64 == 0,
                        128 <= n <= 2048; ≤1e-9); other shapes run SA_NDFT_FAST */
  SA_NDFT_TC_I8 = 3  /* the fast-mode sum on tcgen05 kind::i8 with exact int8
                        digits for both dtypes (complex64: one digit pair,
                        n % 128 == 0, 128 <= n <= 2048, ≤1e-4; complex128 as
                        SA_NDFT_TC); other shapes run SA_NDFT_FAST */
};

enum sa_nlfft_variant {
  SA_DIT = 0,       /* nonlinear FFT, nfft (transforms.py:254-298)                  */
  SA_DIF = 1,       /* nonlinear FFT, decimation in frequency      */
  SA_FFT_EXACT = 2  /* exact radix-2 DIT FFT, fft_exact (transforms.py:200-220):
                       numpy's complex multiply of the twiddle, bit-exact           */
};

enum sa_doppler { SA_DOPPLER_NLFFT = 0, SA_DOPPLER_NDFT = 1, SA_DOPPLER_FFT_EXACT = 2 };

enum sa_lag_kind {
  SA_LAG_MF = 0,    /* sign-additive lag product, lag_product_mf (eq12a / eq12b)   */
  SA_LAG_EXACT = 1  /* exact multiply, lag_product_exact (eq11 / eq12c)            */
};

/* ABI version (SA_ABI_VERSION). */
int sa_version(void);

/* Thread-local description of the last failure. */
const char *sa_last_error(void);

/* Build a device twiddle set from the HOST reference table.
 * Replaces: TwiddleTable / twiddle_table (transforms.py:108-146); the table
 * itself (cos/sin of (-2pi)m/n with exact quadrant entries) is computed by the
 * caller exactly as the reference does and passed in as n interleaved
 * complex128 values.  For SA_C64 the entries are rounded to nearest float. */
int sa_twiddle_create(int device, int dtype, int64_t n, const double *host_table, void *stream,
                      void **handle);
int sa_twiddle_destroy(void *handle);

/* out[i] = a[i] ⊙ b[i] (complex sign-additive product).
 * Replaces: mf_complex / _mf_complex_raw (operator.py:128-131,159-176). */
int sa_mf_complex(int dtype, const void *a, const void *b, void *out, int64_t count, void *stream);

/* Sets *d_flag (device int) to 1 if any component of x is NaN/Inf.
 * Replaces: _require_finite / _as_samples checks (operator.py:112-115,
 * transforms.py:161-162) for device-resident inputs. */
int sa_check_finite(int dtype, const void *x, int64_t count, int *d_flag, void *stream);

/* Batched N-point nonlinear DFT: y[b,k] = sum_m W^(km mod n) ⊙ (gain*x[b,m]).
 * Replaces: ndft (transforms.py:223-251), batched over `batch` contiguous rows.
 * gain == 1.0 skips the scaling (as ambiguity.py:176-177).  tw: twiddle set
 * for n.  x and y must not overlap. */
int sa_ndft(int dtype, const void *x, void *y, int64_t batch, int64_t n, const void *tw, int mode,
            double gain, void *stream);

/* Batched N-point nonlinear FFT, n a power of two >= 2.
 * SA_DIT replaces nfft (transforms.py:254-298), value-identical.
 * SA_DIF is the decimation-in-frequency convention of DESIGN.md (no reference).
 * SA_FFT_EXACT replaces fft_exact (transforms.py:200-220), bit-exact.
 * Input scaled by gain first (gain == 1.0: untouched).  x == y is allowed. */
int sa_nlfft(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
             const void *tw, double gain, void *stream);

/* One ⊙ lag-product row: out[i] = surv[i] ⊙ conj?(ref[i-lag]), ref[<0] = 0.
 * Replaces: lag_product_mf (ambiguity.py:146-155) incl. its guards
 * (ambiguity.py:121-128 -> SA_ERR_CONTRACT). */
int sa_lag_product_mf(int dtype, const void *surv, const void *ref, int64_t n, int64_t ref_len,
                      int64_t lag, int conj, void *out, void *stream);

/* One exact lag-product row: out[i] = surv[i] * conj?(ref[i-lag]) with numpy's
 * complex multiply, ref[<0] = 0.  Replaces: lag_product_exact
 * (ambiguity.py:134-143), same guards as sa_lag_product_mf. */
int sa_lag_product_exact(int dtype, const void *surv, const void *ref, int64_t n, int64_t ref_len,
                         int64_t lag, int conj, void *out, void *stream);

/* Workspace needed by sa_ambiguity_map (may be 0). */
int sa_ambiguity_workspace_bytes(int dtype, int64_t l_count, int64_t m, int64_t *bytes);

/* Range-Doppler map rows l0..l0+l_count-1 (row-major l_count x m):
 *   y_l[i] = surv[i] ⊙ conj?(ref[i-l])               (lag_product_mf, n = ns)
 *   z_l[q] = sum_{t<T} y_l[qT+t],  T = ns/m            (block integration)
 *   row_l  = NLFFT_m(gain*z_l) or NDFT_m(gain*z_l)      (_surface row, :174-178)
 * With m == ns (T == 1) this is ambiguity_eq12a (ambiguity.py:197-202) for the
 * rows requested, value-identical for the NL-FFT Doppler transform.
 * mode: SA_NDFT_FAST uses the regrouped 8-FMA lag accumulation for T > 1;
 * SA_NDFT_EXACT rounds every ⊙ (always used when T == 1).  In SA_NDFT_FAST,
 * complex64, T > 1: the lag stage runs on tcgen05 when T % 128 == 0, and an
 * NDFT Doppler stage runs as SA_NDFT_TC when m % 128 == 0 (both within the
 * fp32 tolerance; the first tensor-core call per twiddle set builds its
 * 3 x (2m)^2 bf16 operands, kept until sa_twiddle_destroy, stream-ordered).
 * tw: twiddle set for m.  Rows are independent (ambiguity.py:27-28): any row
 * range may be computed on any device (delay-bin sharding). */
int sa_ambiguity_map(int dtype, const void *surv, const void *ref, int64_t ns, int64_t ref_len,
                     int64_t l0, int64_t l_count, int64_t m, double gain, int conj, int doppler,
                     int mode, const void *tw, void *out, void *workspace, int64_t ws_bytes,
                     void *stream);

/* Stage 1 of sa_ambiguity_map alone: z (l_count x m) = block sums of the ⊙
 * lag products (no gain, no Doppler transform).  Same guards and modes. */
int sa_ambiguity_integrate(int dtype, const void *surv, const void *ref, int64_t ns,
                           int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, int conj,
                           int mode, void *z, void *stream);

/* sa_ambiguity_map for every variant of ambiguity.py:5-14: lag_kind
 * SA_LAG_MF / SA_LAG_EXACT and doppler SA_DOPPLER_NLFFT / _NDFT / _FFT_EXACT.
 * With m == ns: eq11 = (EXACT, FFT_EXACT), eq12a = (MF, NLFFT),
 * eq12b = (MF, FFT_EXACT), eq12c = (EXACT, NLFFT) (ambiguity.py:190-221), all
 * value-identical.  The exact lag product is always summed sequentially. */
int sa_ambiguity_map_v(int dtype, int lag_kind, const void *surv, const void *ref, int64_t ns,
                       int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, double gain, int conj,
                       int doppler, int mode, const void *tw, void *out, void *workspace,
                       int64_t ws_bytes, void *stream);

/* sa_ambiguity_integrate with a lag kind. */
int sa_ambiguity_integrate_v(int dtype, int lag_kind, const void *surv, const void *ref, int64_t ns,
                             int64_t ref_len, int64_t l0, int64_t l_count, int64_t m, int conj,
                             int mode, void *z, void *stream);

/* Which tensor-core kernel runs the complex64 fast-mode lag stage (T % 128 == 0):
 * SA_LAGK_I8 (default; int8 digits x signs on tcgen05 kind::i8, exact int32 sums,
 * one exponent for the whole reference) or SA_LAGK_BF16 (two-piece bf16 operands,
 * fp32 sums).  Process-wide; the environment variable SA_LAG_KIND=bf16 sets the
 * initial value.  kind < 0 only queries.  Returns the previous kind. */
enum sa_lag_kernel { SA_LAGK_I8 = 0, SA_LAGK_BF16 = 1 };
int sa_lag_kernel(int kind);

/* Block-sharded lag stage for multi-GPU maps (ambiguity.py:27-28: delay rows and
 * integration blocks are independent): fast-mode ⊙ lag integration of blocks
 * [q0, q0 + q_count) for lags [0, l_count), each lag row stored into the z
 * rows of its owner -- dst_rows is a DEVICE array of n_dst row-block bases
 * (peer / IPC pointers); owner o holds lags [o*l_count/n_dst, (o+1)*l_count/n_dst)
 * in the BLOCKED layout: tiles of 16 lags, element q of a tile's rows one 128-B
 * line, zb[(k * m + q) * 16 + j] = z[16 k + j][q] (k counted from the owner's
 * first row), so every peer store is a whole 32-B sector.  Needs l0 == 0 and
 * l_count % (16 * n_dst) == 0; tensor-core path only (complex64, T % 128 == 0);
 * anything else returns SA_ERR_UNSUPPORTED and the caller shards delay rows. */
int sa_ambiguity_integrate_blocks(int dtype, const void *surv, const void *ref, int64_t ns, int64_t ref_len,
                                  int64_t l0, int64_t l_count, int64_t m, int64_t q0, int64_t q_count, int conj,
                                  void *const *dst_rows, int64_t n_dst, void *stream);

/* The map's Doppler stage on a blocked z (sa_ambiguity_integrate_blocks'
 * layout): out (l_count x m, row-major) = nfft(gain * z row) per row, DIT,
 * value-identical to nfft (transforms.py:254-298); m = 64 .. 2048, a power of
 * two (SA_ERR_UNSUPPORTED otherwise). */
int sa_doppler_nlfft_blocked(int dtype, const void *zb, void *out, int64_t l_count, int64_t m, const void *tw,
                             double gain, void *stream);

/* Host-side writers (§8(f)-4; cli.py:74-116).  sa_format_surface_csv formats
 * a rows x cols dB map (row-major doubles, the reference's
 * AmbiguitySurface.magnitude_db) as the reference's surface CSV, byte for
 * byte: "# manifest=<manifest>\nl,p,magnitude_db\n" and one "l,p,repr(db)"
 * line per cell (cli.py:184-191 through _write_csv, floats as Python repr()),
 * in nthreads host threads (<= 0: all).  *out is malloc'ed: free it with
 * sa_free_host.  sa_format_float_repr writes repr(x) (cap >= 32); returns its
 * length. */
int sa_format_surface_csv(const double *db, int64_t rows, int64_t cols, const char *manifest, char **out,
                          int64_t *out_len, int nthreads);
int sa_format_float_repr(double x, char *out, int cap);
void sa_free_host(void *p);

/* Workspace bytes for sa_map_peaks. */
int sa_peaks_workspace_bytes(int64_t rows, int64_t cols, int k, int64_t *bytes);

/* The k strongest strict local maxima of |map| (rows x cols, device).
 * Replaces: detection.find_peaks (detection.py:85-108).  A cell qualifies when
 * strictly greater than its 8 neighbours (cells beyond the edge never block);
 * |v| is numpy's complex absolute value, max*sqrt(fma(r, r, 1)) with
 * r = min/max of |re|, |im| (bit-exact to np.abs on the reference host).
 * Peaks come strongest first, equal magnitudes in row-major order.
 * Outputs (device): idx[k] = row-major cell index (-1 past the last peak),
 * mag[k] = magnitude as double, *count = number of peaks found (<= k).
 * 1 <= k <= 1024 (SA_ERR_UNSUPPORTED above). */
int sa_map_peaks(int dtype, const void *map, int64_t rows, int64_t cols, int k, int64_t *idx,
                 double *mag, int32_t *count, void *workspace, int64_t ws_bytes, void *stream);

/* The two maxima behind detection.sidelobe_floor_db (detection.py:148-171):
 * out (device, 3 x uint64) = {bit pattern of max |map|, bit pattern of max
 * |map| outside every guard box, number of outside cells}.  Box b covers rows
 * |l - centers[2b]| <= g0 and Doppler bins at circular distance <= g1 from
 * centers[2b+1] (device int32 centers[2 * ncent]), as _guard_mask
 * (detection.py:137-145).  The dB arithmetic stays with the caller. */
int sa_map_floor(int dtype, const void *map, int64_t rows, int64_t cols, const int32_t *centers,
                 int ncent, int g0, int g1, uint64_t *out, void *stream);

/* Single-process multi-GPU map (SURVEY §8(b,e)), no NCCL: device devs[g]
 * computes the contiguous delay rows of shard g ([g*L/G .. (g+1)*L/G), uneven L
 * allowed) and its transform kernel stores them straight into `out`, an
 * (l_count x m) allocation on the root devs[0]; peer access from every device to
 * the root is enabled here.  Per shard: surv[g], ref[g] (inputs on devs[g]),
 * tw[g] (twiddle set for m on devs[g]), workspace[g] / ws_bytes[g] (for its row
 * count), stream[g] (on devs[g]).  Asynchronous per stream: the map is
 * complete when all streams are.  Other arguments as sa_ambiguity_map_v.  The
 * same device may appear more than once (shards on one GPU, separate streams). */
int sa_ambiguity_map_multi(int ndev, const int *devs, int dtype, int lag_kind, const void *const *surv,
                           const void *const *ref, int64_t ns, int64_t ref_len, int64_t l0, int64_t l_count,
                           int64_t m, double gain, int conj, int doppler, int mode, const void *const *tw,
                           void *out, void *const *workspace, const int64_t *ws_bytes, void *const *stream);

/* Multi-GPU plumbing: enable direct loads/stores from the current device to
 * `peer_device` memory (NVLink / NVSwitch).  Idempotent.  Used by the sharded
 * map, whose Doppler-transform kernels write their rows straight into the
 * root's map (an IPC mapping of it) instead of gathering afterwards. */
int sa_enable_peer_access(int peer_device);

/* Open a peer process's device allocation (64-byte cudaIpcMemHandle_t, e.g.
 * from torch's storage export) in the CURRENT device's context, with lazy
 * peer access, so this device's kernels can store into it directly; close it
 * with sa_ipc_close.  The sharded map opens the root's map this way. */
int sa_ipc_open(const void *handle64, void **dptr);
int sa_ipc_close(void *dptr);

/* --- scene synthesis (radar.py) ----------------------------
 * Device versions of the reference's signal builders for CPI-scale inputs.
 * Random draws are the caller's (the reference's numpy streams, uploaded);
 * every arithmetic step follows numpy's evaluation order, so the outputs
 * agree with the reference up to the device sin/cos (an ulp or two).  All
 * buffers are device memory; work is stream-ordered. */
enum sa_noise_kind {
  SA_NOISE_NONE = 0, /* NoiseKind.NONE                                   */
  SA_NOISE_AWGN = 1, /* add_awgn (radar.py:245-256)                      */
  SA_NOISE_EPS = 2   /* add_contaminated (radar.py:259-267)              */
};

/* gen_stereo_fm (radar.py:179-192).  u = the 2 x n draws of
 * default_rng(seed).uniform(-1, 1, (2, n)) (doubles, row-major).  The constant
 * factors are the reference's Python scalars: ca = 2*pi*2*f_p, cb = 2*pi*3*f_p,
 * cc = 2*pi*f_p (each left to right), ck = 2*pi*k_f.  out: n complex (dtype
 * SA_C128 or SA_C64, cast on store) = (cos phase, sin phase). */
int sa_scene_stereo_fm(int dtype, const double *u, int64_t n, double f_s, double ca, double cb, double cc,
                       double ck, void *out, void *stream);

/* The echo mixture of synth_surveillance (radar.py:215-243), before noise and
 * gain: out[i] = sum over echoes k, in order from +0, of
 * amp_k * ref[i - delay_k] (0 for i < delay_k) * exp(j (w_k i) / f_s).
 * ref, out: d complex128.  Host arrays: delays[ne], amps[2 ne] (re, im),
 * w[ne] = 2*pi*doppler_hz (0 for clutter: no Doppler factor, as the
 * reference's doppler_hz == 0 branch), inv_fs = 1 / f_s (numpy divides by the
 * reciprocal).  1 <= ne <= 64. */
int sa_scene_echoes(const void *ref, int64_t d, int ne, const int64_t *delays, const double *amps,
                    const double *w, double inv_fs, void *out, void *stream);

/* sum over i of |x_i|^2 (numpy's complex abs, squared) for add_awgn's signal
 * power: x = d complex128; *sum (device double).  workspace >=
 * sa_scene_power_workspace_bytes(d) bytes of device memory. */
int sa_scene_power_workspace_bytes(int64_t d, int64_t *bytes);
int sa_scene_power(const void *x, int64_t d, double *sum, void *workspace, int64_t ws_bytes, void *stream);

/* apply_noise + the surveillance gain (radar.py:243,245-275):
 * out = (x + noise) * gain with noise = z * scale (SA_NOISE_AWGN; z = the
 * 2 x d normals of default_rng(seed).standard_normal, scale =
 * sqrt(p_noise / 2) as the reference computes it), z * (u < eps ? s1 : s2)
 * (SA_NOISE_EPS; u = the 2 x d draws of .random, then z from the same
 * generator), or none.  x: d complex128; out: dtype SA_C128 or SA_C64. */
int sa_scene_noise_gain(int dtype, const void *x, int64_t d, int kind, const double *z, const double *u,
                        double scale, double eps, double s1, double s2, double gain, void *out, void *stream);

/* FMA-pipe peak microbenchmark (roofline denominator): `blocks` CTAs x 256
 * (dtype 2 = packed fp32x2 FFMA2)
 * threads each run `iters` iterations of 8 independent FMA chains; writes a
 * sink value to d_sink (8 bytes).  dtype selects FFMA or DFMA. */
int sa_fma_peak(int dtype, int64_t iters, void *d_sink, int blocks, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SIGNADD_B200_H */
