/* abi_host.c -- the C ABI driven from plain C (no Python, no torch), as a C, Go
 * (cgo) or Java (JNI) host of the reference's path would drive it.  Test
 * infrastructure: tests/test_c_host.py compiles it against
 * paper_1402_0532_b200/libsignadd_b200.so and oracle/liboracle.so and runs it on
 * the GPU.
 *
 * It builds the reference twiddle table on the host (cos/sin of -2*pi*m/n, the
 * entries with 4m = 0 mod n set exactly to 1, -j, -1, j: transforms.py:122-133),
 * runs mf_complex, the exact NDFT and the DIT NL-FFT (complex128) through
 * cudaMalloc'd buffers, and compares every value with the C oracle.  Prints
 * "c-host ok" and exits 0 on success. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "signadd_b200.h"

/* oracle (oracle/signadd_oracle.c) */
void or_mf_complex_f64(int64_t count, const double *a, const double *b, double *out);
int or_ndft_f64(int64_t batch, int64_t n, const double *x, const double *tw, double *y, int nthreads);
int or_nfft_f64(int64_t batch, int64_t n, int variant, const double *x, const double *tw, double *y,
                int nthreads);

#define CK(call)                                                                      \
  do {                                                                                \
    int rc_ = (call);                                                                 \
    if (rc_) {                                                                        \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, rc_,       \
              sa_last_error());                                                       \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

static void table(int64_t n, double *t) { /* interleaved complex128 */
  for (int64_t m = 0; m < n; ++m) {
    if ((4 * m) % n == 0) {
      static const double q[4][2] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};
      int k = (int)((4 * m) / n);
      t[2 * m] = q[k][0];
      t[2 * m + 1] = q[k][1];
    } else {
      double a = (-2.0 * M_PI) * (double)m / (double)n;
      t[2 * m] = cos(a);
      t[2 * m + 1] = sin(a);
    }
  }
}

static uint64_t s = 14020532;
static double rnd(void) { /* xorshift, uniform in [-1, 1) */
  s ^= s << 13;
  s ^= s >> 7;
  s ^= s << 17;
  return (double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0;
}

static int same(const double *a, const double *b, int64_t n, const char *what) {
  for (int64_t i = 0; i < n; ++i)
    if (!(a[i] == b[i])) {
      fprintf(stderr, "%s: mismatch at %lld: %.17g vs %.17g\n", what, (long long)i, a[i], b[i]);
      return 0;
    }
  return 1;
}

int main(void) {
  const int64_t batch = 8, n_ndft = 64, n_fft = 1024, cnt = 4096;
  const int64_t nmax = batch * n_fft;
  double *hx = malloc(sizeof(double) * 2 * nmax), *hy = malloc(sizeof(double) * 2 * nmax);
  double *hr = malloc(sizeof(double) * 2 * nmax), *tw = malloc(sizeof(double) * 2 * n_fft);
  double *hb = malloc(sizeof(double) * 2 * cnt);
  void *dx, *dy, *db;
  if (sa_version() != SA_ABI_VERSION) return 1;
  if (cudaMalloc(&dx, sizeof(double) * 2 * nmax) || cudaMalloc(&dy, sizeof(double) * 2 * nmax) ||
      cudaMalloc(&db, sizeof(double) * 2 * cnt))
    return 1;
  int ok = 1;

  /* mf_complex (operator.py:159-176), with zeros and a subnormal */
  for (int64_t i = 0; i < 2 * cnt; ++i) {
    hx[i] = rnd() * 100.0;
    hb[i] = rnd();
  }
  hx[0] = 0.0;
  hb[3] = 4e-320;
  cudaMemcpy(dx, hx, sizeof(double) * 2 * cnt, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, sizeof(double) * 2 * cnt, cudaMemcpyHostToDevice);
  CK(sa_mf_complex(SA_C128, dx, db, dy, cnt, NULL));
  cudaMemcpy(hy, dy, sizeof(double) * 2 * cnt, cudaMemcpyDeviceToHost);
  or_mf_complex_f64(cnt, hx, hb, hr);
  ok &= same(hy, hr, 2 * cnt, "mf_complex");

  /* exact NDFT (transforms.py:223-251), batched */
  void *h64 = NULL;
  table(n_ndft, tw);
  CK(sa_twiddle_create(0, SA_C128, n_ndft, tw, NULL, &h64));
  for (int64_t i = 0; i < 2 * batch * n_ndft; ++i) hx[i] = rnd();
  cudaMemcpy(dx, hx, sizeof(double) * 2 * batch * n_ndft, cudaMemcpyHostToDevice);
  CK(sa_ndft(SA_C128, dx, dy, batch, n_ndft, h64, SA_NDFT_EXACT, 1.0, NULL));
  cudaMemcpy(hy, dy, sizeof(double) * 2 * batch * n_ndft, cudaMemcpyDeviceToHost);
  or_ndft_f64(batch, n_ndft, hx, tw, hr, 1);
  ok &= same(hy, hr, 2 * batch * n_ndft, "ndft");

  /* DIT NL-FFT (transforms.py:254-298), batched, in place */
  void *h1k = NULL;
  table(n_fft, tw);
  CK(sa_twiddle_create(0, SA_C128, n_fft, tw, NULL, &h1k));
  for (int64_t i = 0; i < 2 * nmax; ++i) hx[i] = rnd();
  cudaMemcpy(dx, hx, sizeof(double) * 2 * nmax, cudaMemcpyHostToDevice);
  CK(sa_nlfft(SA_C128, SA_DIT, dx, dx, batch, n_fft, h1k, 1.0, NULL));
  cudaMemcpy(hy, dx, sizeof(double) * 2 * nmax, cudaMemcpyDeviceToHost);
  or_nfft_f64(batch, n_fft, 0, hx, tw, hr, 1);
  ok &= same(hy, hr, 2 * nmax, "nlfft");

  /* contract errors come back as status codes, not crashes */
  ok &= sa_nlfft(SA_C128, SA_DIT, dx, dy, 1, 12, h1k, 1.0, NULL) == SA_ERR_CONTRACT;

  CK(sa_twiddle_destroy(h64));
  CK(sa_twiddle_destroy(h1k));
  cudaFree(dx);
  cudaFree(dy);
  cudaFree(db);
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  puts(ok ? "c-host ok" : "c-host FAILED");
  return ok ? 0 : 1;
}
