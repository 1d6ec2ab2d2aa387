// sa_scene.cu -- scene synthesis on the device: the
// reference's radar.py builds the stereo-FM illuminator and the surveillance
// echo mixture with numpy; these kernels compute the same expressions for
// CPI-scale inputs (2^20 - 2^22 samples) straight into HBM.
//
// Reproducibility: every random draw stays numpy's -- the host draws the
// reference's exact streams (default_rng(seed).uniform / standard_normal /
// random) and uploads them -- and every arithmetic step is the one numpy
// performs, in the same order (checked against the reference in
// tests/golden/make_golden.py):
//   gen_stereo_fm (radar.py:179-192): t = i / f_s; the cosine arguments are
//     the Python constants ((2*pi)*2)*f_p etc. times t; m adds left to right;
//     phase = ((2*pi)*k_f) * m; out = (cos phase, sin phase).
//   synth_surveillance (radar.py:215-243): the Doppler phase of
//     2j*pi*f*i/fs is ((2*pi*f)*i) * (1/fs) (numpy divides a complex array by
//     a real scalar through its reciprocal); exp(+-0 + j phase) = (cos, sin);
//     amplitude*shifted*exp are numpy complex products (sa_npmul), summed per
//     obstacle in order from +0.
//   add_awgn / add_contaminated (radar.py:245-267): x + z0 + 1j*z1 with z the
//     host-drawn normals times the scale (or the per-component sigma).
//   * surv_gain: each part times the gain.
// The device sin/cos differ from the host libm by an ulp or two, and the
// AWGN power is a device reduction (numpy sums pairwise), so the outputs
// agree with the reference to ~1e-15 relative -- not bitwise.
#include <algorithm>

#include "sa_common.cuh"
#include "sa_internal.h"

namespace {

template <typename T> using C2 = typename SaVec<T>::c2;

struct SceneEcho {
  long long delay;
  double ar, ai;  // complex amplitude
  double w;       // 2*pi*f (Python: (2j*pi*f).imag); 0 = clutter (no Doppler term)
};
constexpr int MAX_ECHOES = 64;
struct SceneEchoes {
  SceneEcho e[MAX_ECHOES];
};

template <typename TO>
__global__ void k_stereo_fm(const double *__restrict__ u, int64_t n, double f_s, double ca, double cb,
                            double cc, double ck, C2<TO> *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x1 = u[i], x2 = u[n + i];
    const double t = (double)i / f_s;
    double m = sa_mul(0.9, sa_add(x1, x2));
    m = sa_add(m, sa_mul(sa_mul(0.5, sa_sub(x1, x2)), cos(sa_mul(ca, t))));
    m = sa_add(m, sa_mul(0.25, cos(sa_mul(cb, t))));
    m = sa_add(m, sa_mul(0.1, cos(sa_mul(cc, t))));
    double s, c;
    sincos(sa_mul(ck, m), &s, &c);
    out[i] = {(TO)c, (TO)s};
  }
}

__global__ void k_echoes(const double2 *__restrict__ ref, int64_t d, int ne, const __grid_constant__ SceneEchoes ech,
                         double inv_fs, double2 *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    double accr = 0.0, acci = 0.0;
    for (int k = 0; k < ne; ++k) {
      const SceneEcho &e = ech.e[k];
      double sr = 0.0, si = 0.0;
      if (i >= e.delay) {
        const double2 r = ref[i - e.delay];
        sr = r.x;
        si = r.y;
      }
      double pr, pi;
      sa_npmul<double>(e.ar, e.ai, sr, si, pr, pi);  // amplitude * shifted
      if (e.w != 0.0) {
        double s, c;
        sincos(sa_mul(sa_mul(e.w, (double)i), inv_fs), &s, &c);
        double qr, qi;
        sa_npmul<double>(pr, pi, c, s, qr, qi);  // (...) * exp(j phase)
        pr = qr;
        pi = qi;
      }
      accr = sa_add(accr, pr);
      acci = sa_add(acci, pi);
    }
    out[i] = {accr, acci};
  }
}

// sum of |x|^2 (numpy abs, squared): per-block partials, then one block
__global__ void k_power_partial(const double2 *__restrict__ x, int64_t d, double *__restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = np_cabs<double>(x[i].x, x[i].y);
    acc = sa_add(acc, sa_mul(a, a));
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = sa_add(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_power_final(const double *__restrict__ part, int np, double *__restrict__ sum) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc = sa_add(acc, part[i]);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = sa_add(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *sum = sh[0];
}

template <typename TO>
__global__ void k_noise_gain(const double2 *__restrict__ x, int64_t d, int kind, const double *__restrict__ z,
                             const double *__restrict__ u, double scale, double eps, double s1, double s2,
                             double gain, C2<TO> *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    double re = x[i].x, im = x[i].y;
    if (kind == SA_NOISE_AWGN) {
      re = sa_add(re, sa_mul(z[i], scale));
      im = sa_add(im, sa_mul(z[d + i], scale));
    } else if (kind == SA_NOISE_EPS) {
      re = sa_add(re, sa_mul(z[i], u[i] < eps ? s1 : s2));
      im = sa_add(im, sa_mul(z[d + i], u[d + i] < eps ? s1 : s2));
    }
    out[i] = {(TO)sa_mul(re, gain), (TO)sa_mul(im, gain)};
  }
}

unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

int sa_launch_stereo_fm(int dtype, const double *u, int64_t n, double f_s, double ca, double cb, double cc,
                        double ck, void *out, cudaStream_t s) {
  if (n == 0) return SA_OK;
  if (dtype == SA_C128)
    k_stereo_fm<double><<<grid_for(n), 256, 0, s>>>(u, n, f_s, ca, cb, cc, ck, (double2 *)out);
  else
    k_stereo_fm<float><<<grid_for(n), 256, 0, s>>>(u, n, f_s, ca, cb, cc, ck, (float2 *)out);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

int sa_launch_echoes(const void *ref, int64_t d, int ne, const int64_t *delays, const double *amps, const double *w,
                     double inv_fs, void *out, cudaStream_t s) {
  if (d == 0) return SA_OK;
  SceneEchoes e{};
  for (int k = 0; k < ne; ++k) e.e[k] = {(long long)delays[k], amps[2 * k], amps[2 * k + 1], w[k]};
  k_echoes<<<grid_for(d), 256, 0, s>>>((const double2 *)ref, d, ne, e, inv_fs, (double2 *)out);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

int64_t sa_power_ws_bytes(int64_t d) { return (int64_t)sizeof(double) * (int64_t)grid_for(d); }

int sa_launch_power(const void *x, int64_t d, double *ws, double *sum, cudaStream_t s) {
  const unsigned g = grid_for(d);
  k_power_partial<<<g, 256, 0, s>>>((const double2 *)x, d, ws);
  k_power_final<<<1, 256, 0, s>>>(ws, (int)g, sum);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

int sa_launch_noise_gain(int dtype, const void *x, int64_t d, int kind, const double *z, const double *u, double scale,
                         double eps, double s1, double s2, double gain, void *out, cudaStream_t s) {
  if (d == 0) return SA_OK;
  if (dtype == SA_C128)
    k_noise_gain<double><<<grid_for(d), 256, 0, s>>>((const double2 *)x, d, kind, z, u, scale, eps, s1, s2, gain,
                                                     (double2 *)out);
  else
    k_noise_gain<float><<<grid_for(d), 256, 0, s>>>((const double2 *)x, d, kind, z, u, scale, eps, s1, s2, gain,
                                                    (float2 *)out);
  SA_LAUNCH_CHECK();
  return SA_OK;
}
