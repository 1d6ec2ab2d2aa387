/*
 * signadd_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels and the "port" CPU baseline in bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path (paper_1402_0532_b200/) never links it.
 *
 * Every routine restates the reference algorithm operation-for-operation, in
 * the reference's evaluation order, so that the fp64 build is value-identical
 * to signadd 0.1.0 (numpy 2.3.5) and the fp32 build is the same algorithm
 * evaluated in binary32:
 *
 *   sign-additive product   operator.py:118-131  (_sign_product, _mf_real_raw,
 *                                                 _mf_complex_raw)
 *   NDFT                    transforms.py:223-251 (sequential accumulation over
 *                                                 columns from +0.0, :244-246)
 *   NL-FFT (DIT)            transforms.py:254-298 (bit reverse :268, bottom
 *                                                 2-point NDFT :270-280, stages
 *                                                 m=4..N with w and -w :282-295)
 *   bit reversal            transforms.py:172-178
 *   lag product (⊙)         ambiguity.py:116-131,146-155
 *   row assembly / gain     ambiguity.py:158-187 (gain * y, :176-177)
 *
 * The DIF NL-FFT has no reference; its convention is defined
 * here and in DESIGN.md ("parity unpinned").  The block-integrated map
 * (T = Ns/M samples summed per Doppler input) is the composition defined in
 * SURVEY.md §8(d); with T == 1 it is exactly ambiguity_eq12a.
 *
 * Build: see oracle/Makefile (-O2 -ffp-contract=off: no FMA contraction, no
 * fast-math; every product below is by a sign in {-1,0,+1} and is exact).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* tiny parallel-for over [0, count) using pthreads                          */
/* ------------------------------------------------------------------------ */
typedef void (*or_body_fn)(void *ctx, int64_t lo, int64_t hi);

typedef struct {
    or_body_fn fn;
    void *ctx;
    int64_t lo, hi;
} or_task;

static void *or_task_main(void *p) {
    or_task *t = (or_task *)p;
    if (t->hi > t->lo) t->fn(t->ctx, t->lo, t->hi);
    return NULL;
}

static void or_parallel_for(int64_t count, int nthreads, or_body_fn fn, void *ctx) {
    if (nthreads <= 1 || count <= 1) {
        fn(ctx, 0, count);
        return;
    }
    if (nthreads > count) nthreads = (int)count;
    pthread_t th[256];
    or_task tasks[256];
    if (nthreads > 256) nthreads = 256;
    int64_t chunk = (count + nthreads - 1) / nthreads;
    for (int i = 0; i < nthreads; ++i) {
        tasks[i].fn = fn;
        tasks[i].ctx = ctx;
        tasks[i].lo = (int64_t)i * chunk;
        tasks[i].hi = tasks[i].lo + chunk > count ? count : tasks[i].lo + chunk;
        if (tasks[i].lo > count) tasks[i].lo = count;
        pthread_create(&th[i], NULL, or_task_main, &tasks[i]);
    }
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

static int64_t or_log2_pow2(int64_t n) {
    if (n < 2 || (n & (n - 1)) != 0) return -1;
    int64_t b = 0;
    while ((1LL << b) < n) ++b;
    return b;
}

/* transforms.py:172-178 */
static int64_t or_bitrev(int64_t i, int64_t bits) {
    int64_t r = 0;
    for (int64_t b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    return r;
}

/* ------------------------------------------------------------------------ */
/* Templated body: instantiated for double (f64) and float (f32)            */
/* ------------------------------------------------------------------------ */
#define OR_DEFINE(T, SFX, FABS, FMA)                                               \
    /* np.sign: +1 / -1 / +0 (np.sign(-0.0) == +0.0) -- operator.py:121 */         \
    static inline T or_sgn_##SFX(T v) { return v > (T)0 ? (T)1 : (v < (T)0 ? (T)-1 : (T)0); } \
    /* operator.py:124-125: sign(a)*sign(b)*(|a|+|b|), one rounding (the sum) */   \
    static inline T or_mfr_##SFX(T a, T b) {                                       \
        return or_sgn_##SFX(a) * or_sgn_##SFX(b) * (FABS(a) + FABS(b));            \
    }                                                                              \
    /* operator.py:128-131 */                                                      \
    static inline void or_mfc_##SFX(T ar, T ai, T br, T bi, T *rr, T *ri) {         \
        *rr = or_mfr_##SFX(ar, br) - or_mfr_##SFX(ai, bi);                         \
        *ri = or_mfr_##SFX(ai, br) + or_mfr_##SFX(bi, ar);                         \
    }                                                                              \
    /* numpy complex multiply a*b as the reference host computes it (SIMD loop, \
     * verified bit-exact): re = fma(ar, br, -(ai*bi)), im = fma(ar, bi, ai*br). \
     * Used by fft_exact (transforms.py:212) and lag_product_exact            \
     * (ambiguity.py:134-143). */                                               \
    static inline void or_npmul_##SFX(T ar, T ai, T br, T bi, T *rr, T *ri) {      \
        T p = ai * bi, q = ai * br;                                                \
        *rr = FMA(ar, br, -p);                                                     \
        *ri = FMA(ar, bi, q);                                                      \
    }                                                                              \
    void or_mf_complex_##SFX(int64_t count, const T *a, const T *b, T *out) {      \
        for (int64_t i = 0; i < count; ++i)                                        \
            or_mfc_##SFX(a[2 * i], a[2 * i + 1], b[2 * i], b[2 * i + 1],           \
                         &out[2 * i], &out[2 * i + 1]);                            \
    }                                                                              \
    /* transforms.py:223-251: X[k] = sum_m W^(km mod N) (x) x[m], sequential */    \
    static void or_ndft_one_##SFX(int64_t n, const T *x, const T *tw, T *y) {      \
        for (int64_t k = 0; k < n; ++k) {                                          \
            T accr = (T)0, acci = (T)0;                                            \
            for (int64_t m = 0; m < n; ++m) {                                      \
                int64_t idx = (k * m) % n;                                         \
                T rr, ri;                                                          \
                or_mfc_##SFX(tw[2 * idx], tw[2 * idx + 1], x[2 * m], x[2 * m + 1], \
                             &rr, &ri);                                            \
                accr += rr;                                                        \
                acci += ri;                                                        \
            }                                                                      \
            y[2 * k] = accr;                                                       \
            y[2 * k + 1] = acci;                                                   \
        }                                                                          \
    }                                                                              \
    /* transforms.py:254-298 */                                                    \
    static void or_nfft_dit_one_##SFX(int64_t n, const T *x, const T *tw, T *y,    \
                                      T *tmp) {                                    \
        int64_t bits = or_log2_pow2(n);                                            \
        for (int64_t i = 0; i < n; ++i) {                                          \
            int64_t r = or_bitrev(i, bits);                                        \
            tmp[2 * i] = x[2 * r];                                                 \
            tmp[2 * i + 1] = x[2 * r + 1];                                         \
        }                                                                          \
        /* bottom stage: full 2-point NDFT, unity product applied once */          \
        for (int64_t p = 0; p < n / 2; ++p) {                                      \
            T ar = tmp[4 * p], ai = tmp[4 * p + 1];                                \
            T br = tmp[4 * p + 2], bi = tmp[4 * p + 3];                            \
            T ur, ui, tr, ti;                                                      \
            or_mfc_##SFX((T)1, (T)0, ar, ai, &ur, &ui);                            \
            or_mfc_##SFX((T)1, (T)0, br, bi, &tr, &ti);                            \
            y[4 * p] = ur + tr;                                                    \
            y[4 * p + 1] = ui + ti;                                                \
            y[4 * p + 2] = ur - tr;                                                \
            y[4 * p + 3] = ui - ti;                                                \
        }                                                                          \
        for (int64_t m = 4; m <= n; m *= 2) {                                      \
            int64_t h = m / 2, stride = n / m;                                     \
            for (int64_t base = 0; base < n; base += m) {                          \
                for (int64_t j = 0; j < h; ++j) {                                  \
                    T wr = tw[2 * (j * stride)], wi = tw[2 * (j * stride) + 1];    \
                    T ar = y[2 * (base + j)], ai = y[2 * (base + j) + 1];          \
                    T br = y[2 * (base + j + h)], bi = y[2 * (base + j + h) + 1];  \
                    T t1r, t1i, t2r, t2i;                                          \
                    or_mfc_##SFX(wr, wi, br, bi, &t1r, &t1i);                      \
                    or_mfc_##SFX(-wr, -wi, br, bi, &t2r, &t2i);                    \
                    y[2 * (base + j)] = ar + t1r;                                  \
                    y[2 * (base + j) + 1] = ai + t1i;                              \
                    y[2 * (base + j + h)] = ar + t2r;                              \
                    y[2 * (base + j + h) + 1] = ai + t2i;                          \
                }                                                                  \
            }                                                                      \
        }                                                                          \
    }                                                                              \
    /* DIF NL-FFT (no reference; convention in DESIGN.md): Gentleman-Sande      \
     * stages m = N..4 with top = a + b, bot = W^(j N/m) (x) (a - b); a final    \
     * full 2-point NDFT stage (4 applications per pair, as the DIT bottom);     \
     * output reordered from bit-reversed to natural order. */                    \
    static void or_nfft_dif_one_##SFX(int64_t n, const T *x, const T *tw, T *y,    \
                                      T *tmp) {                                    \
        int64_t bits = or_log2_pow2(n);                                            \
        memcpy(tmp, x, sizeof(T) * 2 * n);                                         \
        for (int64_t m = n; m >= 4; m /= 2) {                                      \
            int64_t h = m / 2, stride = n / m;                                     \
            for (int64_t base = 0; base < n; base += m) {                          \
                for (int64_t j = 0; j < h; ++j) {                                  \
                    T wr = tw[2 * (j * stride)], wi = tw[2 * (j * stride) + 1];    \
                    T ar = tmp[2 * (base + j)], ai = tmp[2 * (base + j) + 1];      \
                    T br = tmp[2 * (base + j + h)], bi = tmp[2 * (base + j + h) + 1]; \
                    T dr = ar - br, di = ai - bi;                                  \
                    T tr, ti;                                                      \
                    or_mfc_##SFX(wr, wi, dr, di, &tr, &ti);                        \
                    tmp[2 * (base + j)] = ar + br;                                 \
                    tmp[2 * (base + j) + 1] = ai + bi;                             \
                    tmp[2 * (base + j + h)] = tr;                                  \
                    tmp[2 * (base + j + h) + 1] = ti;                              \
                }                                                                  \
            }                                                                      \
        }                                                                          \
        for (int64_t p = 0; p < n / 2; ++p) {                                      \
            T ar = tmp[4 * p], ai = tmp[4 * p + 1];                                \
            T br = tmp[4 * p + 2], bi = tmp[4 * p + 3];                            \
            T ur, ui, tr, ti;                                                      \
            or_mfc_##SFX((T)1, (T)0, ar, ai, &ur, &ui);                            \
            or_mfc_##SFX((T)1, (T)0, br, bi, &tr, &ti);                            \
            tmp[4 * p] = ur + tr;                                                  \
            tmp[4 * p + 1] = ui + ti;                                              \
            tmp[4 * p + 2] = ur - tr;                                              \
            tmp[4 * p + 3] = ui - ti;                                              \
        }                                                                          \
        for (int64_t i = 0; i < n; ++i) {                                          \
            int64_t r = or_bitrev(i, bits);                                        \
            y[2 * r] = tmp[2 * i];                                                 \
            y[2 * r + 1] = tmp[2 * i + 1];                                         \
        }                                                                          \
    }                                                                              \
    /* transforms.py:200-220 fft_exact: bit-reversed input, stages m = 2..N,   \
     * t = w_j * b (numpy complex multiply, w_j = entries[j*N/m]),             \
     * y = [a + t, a - t] per block. */                                           \
    static void or_fft_exact_one_##SFX(int64_t n, const T *x, const T *tw, T *y) { \
        int64_t bits = or_log2_pow2(n);                                            \
        for (int64_t i = 0; i < n; ++i) {                                          \
            int64_t r = or_bitrev(i, bits);                                        \
            y[2 * i] = x[2 * r];                                                   \
            y[2 * i + 1] = x[2 * r + 1];                                           \
        }                                                                          \
        for (int64_t m = 2; m <= n; m <<= 1) {                                     \
            int64_t h = m / 2;                                                     \
            for (int64_t b0 = 0; b0 < n; b0 += m)                                  \
                for (int64_t j = 0; j < h; ++j) {                                  \
                    int64_t w = j * (n / m);                                       \
                    T *a = y + 2 * (b0 + j), *b = y + 2 * (b0 + j + h);            \
                    T tr, ti;                                                      \
                    or_npmul_##SFX(tw[2 * w], tw[2 * w + 1], b[0], b[1], &tr, &ti); \
                    T ar = a[0], ai = a[1];                                        \
                    a[0] = ar + tr;                                                \
                    a[1] = ai + ti;                                                \
                    b[0] = ar - tr;                                                \
                    b[1] = ai - ti;                                                \
                }                                                                  \
        }                                                                          \
    }                                                                              \
    typedef struct {                                                               \
        int64_t n;                                                                 \
        const T *x;                                                                \
        const T *tw;                                                               \
        T *y;                                                                      \
        int kind; /* 0 ndft, 1 dit, 2 dif, 3 fft_exact */                          \
    } or_tctx_##SFX;                                                               \
    static void or_tbody_##SFX(void *p, int64_t lo, int64_t hi) {                  \
        or_tctx_##SFX *c = (or_tctx_##SFX *)p;                                     \
        T *tmp = c->kind ? (T *)malloc(sizeof(T) * 2 * c->n) : NULL;               \
        for (int64_t b = lo; b < hi; ++b) {                                        \
            const T *xb = c->x + 2 * c->n * b;                                     \
            T *yb = c->y + 2 * c->n * b;                                           \
            if (c->kind == 0) or_ndft_one_##SFX(c->n, xb, c->tw, yb);              \
            else if (c->kind == 1) or_nfft_dit_one_##SFX(c->n, xb, c->tw, yb, tmp); \
            else if (c->kind == 2) or_nfft_dif_one_##SFX(c->n, xb, c->tw, yb, tmp); \
            else or_fft_exact_one_##SFX(c->n, xb, c->tw, yb);                      \
        }                                                                          \
        free(tmp);                                                                 \
    }                                                                              \
    int or_ndft_##SFX(int64_t batch, int64_t n, const T *x, const T *tw, T *y,     \
                      int nthreads) {                                              \
        if (n < 1 || batch < 0) return -1;                                         \
        or_tctx_##SFX c = {n, x, tw, y, 0};                                        \
        or_parallel_for(batch, nthreads, or_tbody_##SFX, &c);                      \
        return 0;                                                                  \
    }                                                                              \
    int or_nfft_##SFX(int64_t batch, int64_t n, int variant, const T *x,           \
                      const T *tw, T *y, int nthreads) {                           \
        if (or_log2_pow2(n) < 0 || batch < 0) return -1;                           \
        or_tctx_##SFX c = {n, x, tw, y, variant == 1 ? 2 : 1};                     \
        or_parallel_for(batch, nthreads, or_tbody_##SFX, &c);                      \
        return 0;                                                                  \
    }                                                                              \
    int or_fft_exact_##SFX(int64_t batch, int64_t n, const T *x, const T *tw, T *y, \
                           int nthreads) {                                         \
        if (or_log2_pow2(n) < 0 || batch < 0) return -1;                           \
        or_tctx_##SFX c = {n, x, tw, y, 3};                                        \
        or_parallel_for(batch, nthreads, or_tbody_##SFX, &c);                      \
        return 0;                                                                  \
    }                                                                              \
    /* ambiguity.py:134-143 lag_product_exact: y = surv * conj(shifted), where  \
     * shifted[i] = ref[i-l] (0 for i < l) and np.conj negates the imaginary    \
     * part (0 -> -0); numpy complex multiply. */                                 \
    int or_lag_product_exact_##SFX(int64_t n, const T *surv, const T *ref,         \
                                   int64_t lag, int conj, T *out) {                \
        for (int64_t i = 0; i < n; ++i) {                                          \
            T cr = (T)0, ci = (T)0;                                                \
            if (i >= lag) {                                                        \
                cr = ref[2 * (i - lag)];                                           \
                ci = ref[2 * (i - lag) + 1];                                       \
            }                                                                      \
            if (conj) ci = -ci;                                                    \
            or_npmul_##SFX(surv[2 * i], surv[2 * i + 1], cr, ci, &out[2 * i],      \
                           &out[2 * i + 1]);                                       \
        }                                                                          \
        return 0;                                                                  \
    }                                                                              \
    /* ambiguity.py:116-131,146-155: y[i] = surv[i] (x) conj(ref[i-l]), ref      \
     * taken as zero for i < l (the conjugate is a negation of the imaginary    \
     * part, ambiguity.py:151). */                                                \
    int or_lag_product_mf_##SFX(int64_t n, const T *surv, const T *ref,            \
                                int64_t lag, int conj, T *out) {                   \
        for (int64_t i = 0; i < n; ++i) {                                          \
            T rr_ = (T)0, ri_ = (T)0;                                              \
            if (i >= lag) {                                                        \
                rr_ = ref[2 * (i - lag)];                                          \
                ri_ = conj ? -ref[2 * (i - lag) + 1] : ref[2 * (i - lag) + 1];     \
            } else {                                                               \
                ri_ = conj ? -(T)0 : (T)0;                                         \
            }                                                                      \
            or_mfc_##SFX(surv[2 * i], surv[2 * i + 1], rr_, ri_, &out[2 * i],      \
                         &out[2 * i + 1]);                                         \
        }                                                                          \
        return 0;                                                                  \
    }                                                                              \
    typedef struct {                                                               \
        int64_t ns, m, l0;                                                         \
        const T *surv, *ref, *tw;                                                  \
        double gain;                                                               \
        int conj, doppler, lag_kind;                                               \
        T *out;                                                                    \
    } or_actx_##SFX;                                                               \
    static void or_abody_##SFX(void *p, int64_t lo, int64_t hi) {                  \
        or_actx_##SFX *c = (or_actx_##SFX *)p;                                     \
        T *y = (T *)malloc(sizeof(T) * 2 * c->ns);                                 \
        T *z = (T *)malloc(sizeof(T) * 2 * c->m);                                  \
        T *tmp = (T *)malloc(sizeof(T) * 2 * c->m);                                \
        int64_t tb = c->ns / c->m;                                                 \
        for (int64_t r = lo; r < hi; ++r) {                                        \
            if (c->lag_kind == 0)                                                  \
                or_lag_product_mf_##SFX(c->ns, c->surv, c->ref, c->l0 + r, c->conj, y); \
            else                                                                   \
                or_lag_product_exact_##SFX(c->ns, c->surv, c->ref, c->l0 + r, c->conj, y); \
            for (int64_t q = 0; q < c->m; ++q) {                                   \
                T sr = (T)0, si = (T)0;                                            \
                for (int64_t t = 0; t < tb; ++t) {                                 \
                    sr += y[2 * (q * tb + t)];                                     \
                    si += y[2 * (q * tb + t) + 1];                                 \
                }                                                                  \
                if (c->gain != 1.0) {                                              \
                    sr = (T)c->gain * sr;                                          \
                    si = (T)c->gain * si;                                          \
                }                                                                  \
                z[2 * q] = sr;                                                     \
                z[2 * q + 1] = si;                                                 \
            }                                                                      \
            T *row = c->out + 2 * c->m * r;                                        \
            if (c->doppler == 0) or_nfft_dit_one_##SFX(c->m, z, c->tw, row, tmp);  \
            else if (c->doppler == 1) or_ndft_one_##SFX(c->m, z, c->tw, row);      \
            else or_fft_exact_one_##SFX(c->m, z, c->tw, row);                      \
        }                                                                          \
        free(y);                                                                   \
        free(z);                                                                   \
        free(tmp);                                                                 \
    }                                                                              \
    /* Map rows l = l0 .. l0+l_count-1: lag product over ns samples, sums of     \
     * T = ns/m consecutive products (sequential, from +0), times gain, then     \
     * the M-point NL-FFT (doppler 0) or NDFT (doppler 1).  T == 1 is exactly    \
     * ambiguity_eq12a (ambiguity.py:197-202). */                                 \
    /* lag_kind 0: sign-additive lag product (eq12a/b), 1: exact multiply      \
     * (eq11/eq12c); doppler 0: nfft, 1: ndft, 2: fft_exact. */                   \
    int or_ambiguity_map_v_##SFX(int64_t ns, const T *surv, const T *ref,          \
                                 int64_t l0, int64_t l_count, int64_t m,           \
                                 double gain, int conj, int lag_kind, int doppler, \
                                 const T *tw, T *out, int nthreads) {              \
        if (m < 1 || ns % m != 0 || l0 < 0 || l_count < 0) return -1;              \
        if (doppler != 1 && or_log2_pow2(m) < 0) return -1;                        \
        or_actx_##SFX c = {ns, m, l0, surv, ref, tw, gain, conj, doppler, lag_kind, out}; \
        or_parallel_for(l_count, nthreads, or_abody_##SFX, &c);                    \
        return 0;                                                                  \
    }                                                                              \
    int or_ambiguity_map_##SFX(int64_t ns, const T *surv, const T *ref,            \
                               int64_t l0, int64_t l_count, int64_t m,             \
                               double gain, int conj, int doppler, const T *tw,    \
                               T *out, int nthreads) {                             \
        return or_ambiguity_map_v_##SFX(ns, surv, ref, l0, l_count, m, gain, conj, 0, \
                                        doppler, tw, out, nthreads);               \
    }

OR_DEFINE(double, f64, fabs, fma)
OR_DEFINE(float, f32, fabsf, fmaf)

/* ---- detection (detection.py:85-171), SURVEY §8(f)-1 ------------------------
 * Magnitude: numpy's complex absolute value, as its SIMD loop computes it on the
 * reference host (L = max, S = min of |re|, |im|; r = S/L, 0 when L == 0;
 * |v| = sqrt(fma(r, r, 1)) * L), pinned against np.abs by the golden vectors.
 * find_peaks: strict 8-neighbour maxima (detection.py:96-104; cells beyond the
 * edge never block), ordered as the stable argsort of -|v| over the row-major
 * candidates (detection.py:106): magnitude descending, then row-major index.
 * Floor inputs: max |v| and max |v| outside every guard box (_guard_mask,
 * detection.py:137-145) plus the outside-cell count. */
typedef struct {
    double mag;
    int64_t idx;
} or_cand;

static int or_cand_cmp(const void *a, const void *b) {
    const or_cand *x = (const or_cand *)a, *y = (const or_cand *)b;
    if (x->mag != y->mag) return x->mag > y->mag ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

#define OR_DETECT(T, SFX, FABS, FMA, SQRT)                                         \
    T or_cabs_np_##SFX(T re, T im) {                                               \
        re = FABS(re);                                                             \
        im = FABS(im);                                                             \
        if (isinf(re) || isinf(im)) return (T)INFINITY;                            \
        if (isnan(re) || isnan(im)) return (T)NAN;                                 \
        T L = re > im ? re : im, S = re > im ? im : re;                            \
        T r = (L == (T)0) ? (T)0 : S / L;                                          \
        return SQRT(FMA(r, r, (T)1)) * L;                                          \
    }                                                                              \
    void or_abs_np_##SFX(int64_t n, const T *z, T *out) {                          \
        for (int64_t i = 0; i < n; ++i) out[i] = or_cabs_np_##SFX(z[2 * i], z[2 * i + 1]); \
    }                                                                              \
    /* returns the number of peaks written (<= k), -1 on bad arguments */         \
    int64_t or_find_peaks_##SFX(int64_t rows, int64_t cols, const T *v, int64_t k, \
                                int64_t *out_idx, double *out_mag) {               \
        if (rows < 1 || cols < 1 || k < 1) return -1;                              \
        T *mag = (T *)malloc(sizeof(T) * rows * cols);                             \
        or_cand *c = (or_cand *)malloc(sizeof(or_cand) * rows * cols);             \
        int64_t nc = 0;                                                            \
        for (int64_t i = 0; i < rows * cols; ++i)                                  \
            mag[i] = or_cabs_np_##SFX(v[2 * i], v[2 * i + 1]);                     \
        for (int64_t l = 0; l < rows; ++l)                                         \
            for (int64_t p = 0; p < cols; ++p) {                                   \
                T m = mag[l * cols + p];                                           \
                int strict = 1;                                                    \
                for (int dl = -1; dl <= 1; ++dl)                                   \
                    for (int dp = -1; dp <= 1; ++dp) {                             \
                        if (!dl && !dp) continue;                                  \
                        int64_t ll = l + dl, pp = p + dp;                          \
                        if (ll < 0 || ll >= rows || pp < 0 || pp >= cols) continue; \
                        if (!(m > mag[ll * cols + pp])) strict = 0;                \
                    }                                                              \
                if (strict) {                                                      \
                    c[nc].mag = (double)m;                                         \
                    c[nc].idx = l * cols + p;                                      \
                    ++nc;                                                          \
                }                                                                  \
            }                                                                      \
        qsort(c, (size_t)nc, sizeof(or_cand), or_cand_cmp);                        \
        int64_t n = nc < k ? nc : k;                                               \
        for (int64_t i = 0; i < n; ++i) {                                          \
            out_idx[i] = c[i].idx;                                                 \
            out_mag[i] = c[i].mag;                                                 \
        }                                                                          \
        free(mag);                                                                 \
        free(c);                                                                   \
        return n;                                                                  \
    }                                                                              \
    void or_map_floor_##SFX(int64_t rows, int64_t cols, const T *v,                \
                            const int32_t *centers, int ncent, int g0, int g1,     \
                            double *out3) {                                        \
        double all = 0.0, outside = 0.0, n_out = 0.0;                              \
        for (int64_t l = 0; l < rows; ++l)                                         \
            for (int64_t p = 0; p < cols; ++p) {                                   \
                double m = (double)or_cabs_np_##SFX(v[2 * (l * cols + p)],         \
                                                    v[2 * (l * cols + p) + 1]);    \
                int in = 0;                                                        \
                for (int b = 0; b < ncent && !in; ++b) {                           \
                    int64_t dl = l - centers[2 * b];                               \
                    int64_t d = (p - centers[2 * b + 1]) % cols;                   \
                    if (d < 0) d += cols;                                          \
                    int64_t dp = d < cols - d ? d : cols - d;                      \
                    in = dl <= g0 && dl >= -g0 && dp <= g1;                        \
                }                                                                  \
                if (m > all) all = m;                                              \
                if (!in) {                                                         \
                    if (m > outside) outside = m;                                  \
                    n_out += 1.0;                                                  \
                }                                                                  \
            }                                                                      \
        out3[0] = all;                                                             \
        out3[1] = outside;                                                         \
        out3[2] = n_out;                                                           \
    }

OR_DETECT(double, f64, fabs, fma, sqrt)
OR_DETECT(float, f32, fabsf, fmaf, sqrtf)

int or_version(void) { return 1; }
