/*
 * ocean_oracle.c — TEST INFRASTRUCTURE ONLY (see ocean_oracle.h).
 *
 * fp64 restatement of the reference algorithm; each function cites the
 * reference file:line (relative to /root/reference/proj) it restates. The
 * operation order follows the reference so that, built with
 * -ffp-contract=off against the same libm, results are bit-identical to the
 * reference build in oracle/_ref (checked in tests/test_oracle_vs_ref.py).
 */
#include "ocean_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define KPI 3.14159265358979323846
#define KGRAVITY 9.80665

/* ======================================================================== */
/* rng.hpp:14-57 — Philox4x32-10 with the 128-bit key XOR-folded to 2 words. */
void orc_philox(uint64_t key_lo, uint64_t key_hi, uint64_t ctr_lo, uint64_t ctr_hi,
                uint32_t out[4]) {
  uint32_t k0 = (uint32_t)key_lo ^ (uint32_t)key_hi;
  uint32_t k1 = (uint32_t)(key_lo >> 32) ^ (uint32_t)(key_hi >> 32);
  uint32_t c[4] = {(uint32_t)ctr_lo, (uint32_t)(ctr_lo >> 32), (uint32_t)ctr_hi,
                   (uint32_t)(ctr_hi >> 32)};
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  memcpy(out, c, sizeof(c));
}

/* rng.hpp:60-76 — uniform in (0,1], Box-Muller, /sqrt(2). */
void orc_gaussian_complex(uint64_t seed, uint32_t stream, uint32_t i, uint32_t j, double out[2]) {
  uint32_t b[4];
  orc_philox(seed, 0x6F63656E00000000ull | stream, ((uint64_t)i << 32) | j, 0, b);
  double u1 = ((double)b[0] + 1.0) * (1.0 / 4294967296.0);
  double u2 = ((double)b[1] + 1.0) * (1.0 / 4294967296.0);
  double r = sqrt(-2.0 * log(u1));
  double g1 = r * cos(2.0 * KPI * u2);
  double g2 = r * sin(2.0 * KPI * u2);
  out[0] = g1 / sqrt(2.0);
  out[1] = g2 / sqrt(2.0);
}

/* ======================================================================== */
/* spectra.cpp:10-32 */
double orc_alpha(const ocn_spectrum_params* p) {
  return 0.076 * pow(p->wind_speed * p->wind_speed / (p->fetch * p->gravity), 0.22);
}
double orc_peak_omega(const ocn_spectrum_params* p) {
  if (p->has_peak_omega_override) return p->peak_omega_override;
  return 22.0 * p->gravity * p->gravity / (p->wind_speed * p->fetch);
}
double orc_standard_peak_omega(const ocn_spectrum_params* p) {
  return 22.0 * cbrt(p->gravity * p->gravity / (p->wind_speed * p->fetch));
}
int orc_spectrum_validate(const ocn_spectrum_params* p) {
  if (!(p->wind_speed > 0.0)) return OCN_ERR_CONFIG;
  if (!(p->fetch > 0.0)) return OCN_ERR_CONFIG;
  if (p->swell < 0.0 || p->swell > 1.0) return OCN_ERR_CONFIG;
  if (p->direction_mix < 0.0 || p->direction_mix > 1.0) return OCN_ERR_CONFIG;
  if (!(p->gravity > 0.0)) return OCN_ERR_CONFIG;
  if (p->has_peak_omega_override && !(p->peak_omega_override > 0.0)) return OCN_ERR_CONFIG;
  return OCN_OK;
}

/* spectra.cpp:34 */
double orc_dispersion(double k, double g) { return sqrt(g * k); }

/* spectra.cpp:36-47 */
int orc_jonswap(double omega, const ocn_spectrum_params* p, double* out) {
  if (!(omega > 0.0)) return OCN_ERR_DOMAIN;
  double g = p->gravity;
  double wp = orc_peak_omega(p);
  double sigma = omega <= wp ? 0.07 : 0.09;
  double d = (omega - wp) / (sigma * wp);
  double r = exp(-0.5 * d * d);
  double ratio = wp / omega;
  double ratio4 = ratio * ratio * ratio * ratio;
  *out = orc_alpha(p) * g * g / pow(omega, 5.0) * exp(-1.25 * ratio4) * pow(3.3, r);
  return OCN_OK;
}

/* spectra.cpp:49-54 */
double orc_beta_s(double r) {
  if (r < 0.95) return 2.61 * pow(r, 1.3);
  if (r < 1.6) return 2.28 * pow(r, -1.3);
  double eps = 0.8393 * exp(-0.567 * log(r * r)) - 0.4;
  return pow(10.0, eps);
}

/* spectra.cpp:56-59 */
double orc_directional_kernel(double beta, double theta) {
  double sech = 1.0 / cosh(beta * theta);
  return 0.5 * beta * sech * sech / tanh(beta * KPI);
}

/* spectra.cpp:61-63 */
double orc_donelan_banner(double omega, double theta, double omega_p) {
  return orc_directional_kernel(orc_beta_s(omega / omega_p), theta);
}

/* spectra.cpp:65-72 */
double orc_swell_spread(double omega, double theta, double omega_p, double xi) {
  double r = omega / omega_p;
  double s = 16.0 * tanh(1.0 / r) * xi * xi;
  if (s == 0.0) return 1.0;
  double c = fabs(cos(0.5 * theta));
  if (c == 0.0) return 0.0;
  return pow(c, 2.0 * s);
}

/* spectra.cpp:74-82 */
double orc_q_dbxi_approx(double r) {
  if (r < 0.94) return 7.1467551 * r * r - 13.4662001 * r + 7.75651088;
  if (r < 5.0) return -0.69906109 * r * r + 0.77975933 * r + 0.10169164;
  if (r < 100.0) return -2.1860997 * r * r + 0.0269209 * r + 0.00016283;
  return 1.2038847 * r + 0.0008147;
}

/* spectra.cpp:84-98: composite Simpson over [-pi, pi]. */
static double quad_integrand(double theta, double beta, double s) {
  double c = fabs(cos(0.5 * theta));
  double spread = (s == 0.0) ? 1.0 : (c == 0.0 ? 0.0 : pow(c, 2.0 * s));
  return orc_directional_kernel(beta, theta) * spread;
}
double orc_q_dbxi_quadrature(double r, double xi, int panels) {
  double beta = orc_beta_s(r);
  double s = 16.0 * tanh(1.0 / r) * xi * xi;
  double h = 2.0 * KPI / panels;
  double acc = quad_integrand(-KPI, beta, s) + quad_integrand(KPI, beta, s);
  for (int i = 1; i < panels; ++i)
    acc += quad_integrand(-KPI + h * i, beta, s) * ((i & 1) ? 4.0 : 2.0);
  double integral = acc * h / 3.0;
  return 1.0 / integral;
}

/* spectra.cpp:100-109 */
double orc_directional(double omega, double theta, const ocn_spectrum_params* p) {
  double uniform = 1.0 / (2.0 * KPI);
  double delta = p->direction_mix;
  if (delta == 0.0) return uniform;
  double wp = orc_peak_omega(p);
  double d = orc_q_dbxi_approx(omega / wp) * orc_donelan_banner(omega, theta, wp) *
             orc_swell_spread(omega, theta, wp, p->swell);
  if (d < 0.0) d = 0.0;
  return (1.0 - delta) * uniform + delta * d;
}

/* spectra.cpp:119-130 */
double orc_h0_variance(double kx, double kz, double k, double omega, double L,
                       const ocn_spectrum_params* p) {
  if (k <= 0.0) return 0.0;
  double dk = 2.0 * KPI / L;
  double theta = atan2(kz, kx) - p->wind_direction;
  double s = 0.0;
  orc_jonswap(omega, p, &s);
  double d = orc_directional(omega, theta, p);
  double domega_dk = p->gravity / (2.0 * omega);
  return s * d * domega_dk * dk * dk / k;
}

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
static int neg_index(int s, int n) { return s == 0 ? 0 : n - s; } /* fft.hpp:20 */

/* spectra.cpp:132-179 */
int orc_generate_h0(int n, double length, double band_min, double band_max,
                    const ocn_spectrum_params* p, uint32_t cascade, double* h0, double* h0cn,
                    uint8_t* in_band, double* waves) {
  if (!is_pow2(n) || n < 2) return OCN_ERR_CONFIG;
  if (!(length > 0.0)) return OCN_ERR_CONFIG;
  if (!(band_min >= 0.0) || !(band_max > band_min)) return OCN_ERR_CONFIG;
  int st = orc_spectrum_validate(p);
  if (st) return st;
  size_t nn = (size_t)n * n;
  memset(h0, 0, 2 * nn * sizeof(double));
  double dk = 2.0 * KPI / length;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      size_t q = (size_t)i * n + j;
      double kx = dk * (i - n / 2);
      double kz = dk * (j - n / 2);
      double k = hypot(kx, kz);
      double omega = orc_dispersion(k, p->gravity);
      if (waves) {
        waves[4 * q + 0] = kx;
        waves[4 * q + 1] = kz;
        waves[4 * q + 2] = k;
        waves[4 * q + 3] = omega;
      }
      int banded = k > 0.0 && k >= band_min && k < band_max;
      if (in_band) in_band[q] = (uint8_t)banded;
      if (!banded) continue;
      double xi[2];
      orc_gaussian_complex(p->rng_seed, cascade, (uint32_t)i, (uint32_t)j, xi);
      double amp = sqrt(orc_h0_variance(kx, kz, k, omega, length, p));
      h0[2 * q + 0] = xi[0] * amp;
      h0[2 * q + 1] = xi[1] * amp;
    }
  }
  if (h0cn) {
    for (int i = 0; i < n; ++i) {
      int ni = neg_index(i, n);
      for (int j = 0; j < n; ++j) {
        int nj = neg_index(j, n);
        size_t q = (size_t)i * n + j, m = (size_t)ni * n + nj;
        h0cn[2 * q + 0] = h0[2 * m + 0];
        h0cn[2 * q + 1] = -h0[2 * m + 1];
      }
    }
  }
  return OCN_OK;
}

/* ======================================================================== */
/* fft.cpp:17-37: in-place radix-2, exponent +i, unnormalized. */
static void fft1d(double* a, int n, const double* tw) {
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double tr = a[2 * i], ti = a[2 * i + 1];
      a[2 * i] = a[2 * j];
      a[2 * i + 1] = a[2 * j + 1];
      a[2 * j] = tr;
      a[2 * j + 1] = ti;
    }
  }
  for (int len = 2; len <= n; len <<= 1) {
    int stride = n / len, half = len / 2;
    for (int i = 0; i < n; i += len) {
      for (int k = 0; k < half; ++k) {
        double wr = tw[2 * (k * stride)], wi = tw[2 * (k * stride) + 1];
        double* u = a + 2 * (i + k);
        double* v = a + 2 * (i + k + half);
        double vr = v[0] * wr - v[1] * wi;
        double vi = v[0] * wi + v[1] * wr;
        double ur = u[0], ui = u[1];
        u[0] = ur + vr;
        u[1] = ui + vi;
        v[0] = ur - vr;
        v[1] = ui - vi;
      }
    }
  }
}

/* fft.cpp:39-53 rows then columns; fft.cpp:69-77 (-1)^(i+j). */
int orc_ifft2_centered(int n, double* f) {
  if (n < 2 || !is_pow2(n)) return OCN_ERR_CONFIG;
  double* tw = (double*)malloc(sizeof(double) * (size_t)n);
  double* col = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  for (int j = 0; j < n / 2; ++j) {
    tw[2 * j] = cos(2.0 * KPI * j / n);
    tw[2 * j + 1] = sin(2.0 * KPI * j / n);
  }
  for (int i = 0; i < n; ++i) fft1d(f + 2 * (size_t)i * n, n, tw);
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < n; ++i) {
      col[2 * i] = f[2 * ((size_t)i * n + j)];
      col[2 * i + 1] = f[2 * ((size_t)i * n + j) + 1];
    }
    fft1d(col, n, tw);
    for (int i = 0; i < n; ++i) {
      f[2 * ((size_t)i * n + j)] = col[2 * i];
      f[2 * ((size_t)i * n + j) + 1] = col[2 * i + 1];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if ((i + j) & 1) {
        size_t q = (size_t)i * n + j;
        f[2 * q] = -f[2 * q];
        f[2 * q + 1] = -f[2 * q + 1];
      }
  free(tw);
  free(col);
  return OCN_OK;
}

/* fft.cpp:79-101 (check = false path): pack X + iY, transform, split. */
int orc_ifft2_pair(int n, const double* x, const double* y, double* re, double* im) {
  if (n < 2 || !is_pow2(n)) return OCN_ERR_CONFIG;
  size_t nn = (size_t)n * n;
  double* packed = (double*)malloc(2 * nn * sizeof(double));
  for (size_t q = 0; q < nn; ++q) {
    /* x + (0,1) * y : (0*yr - 1*yi, 0*yi + 1*yr) */
    packed[2 * q] = x[2 * q] + (0.0 * y[2 * q] - 1.0 * y[2 * q + 1]);
    packed[2 * q + 1] = x[2 * q + 1] + (0.0 * y[2 * q + 1] + 1.0 * y[2 * q]);
  }
  orc_ifft2_centered(n, packed);
  for (size_t q = 0; q < nn; ++q) {
    if (re) re[q] = packed[2 * q];
    if (im) im[q] = packed[2 * q + 1];
  }
  free(packed);
  return OCN_OK;
}

/* ======================================================================== */
/* complex helpers: (a+bi)(c+di) = (ac - bd) + (ad + bc)i, as std::complex. */
static inline void cmul(double ar, double ai, double br, double bi, double* outr, double* outi) {
  *outr = ar * br - ai * bi;
  *outi = ar * bi + ai * br;
}

/* surface.cpp:39-68 */
int orc_assemble_coefficients(int n, double length, double gravity, const double* h0,
                              const double* h0cn, const uint8_t* in_band, double t,
                              double chop, double* out) {
  size_t nn = (size_t)n * n;
  memset(out, 0, 8 * 2 * nn * sizeof(double));
  double dk = 2.0 * KPI / length;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      size_t q = (size_t)i * n + j;
      if (!in_band[q]) continue;
      double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
      double k = hypot(kx, kz);
      double omega = sqrt(gravity * k);
      double cr = cos(omega * t), si = sin(omega * t);
      double ar, ai, br, bi;
      cmul(h0[2 * q], h0[2 * q + 1], cr, si, &ar, &ai);
      cmul(h0cn[2 * q], h0cn[2 * q + 1], cr, -si, &br, &bi);
      double htr = ar + br, hti = ai + bi;
      double ux = kx / k, uz = kz / k;
      double dxr, dxi, dzr, dzi, tr, ti;
      /* cplx(0,1) * ux -> (0*ux, 1*ux); * ht; * choppiness */
      cmul(0.0 * ux, 1.0 * ux, htr, hti, &tr, &ti);
      dxr = tr * chop;
      dxi = ti * chop;
      cmul(0.0 * uz, 1.0 * uz, htr, hti, &tr, &ti);
      dzr = tr * chop;
      dzi = ti * chop;
      double* f[8];
      for (int m = 0; m < 8; ++m) f[m] = out + (size_t)m * 2 * nn + 2 * q;
      f[0][0] = htr;
      f[0][1] = hti;
      f[1][0] = dxr;
      f[1][1] = dxi;
      f[2][0] = dzr;
      f[2][1] = dzi;
      cmul(0.0, -kx, dxr, dxi, &f[3][0], &f[3][1]);
      cmul(0.0, -kx, dzr, dzi, &f[4][0], &f[4][1]);
      cmul(0.0, -kz, dzr, dzi, &f[5][0], &f[5][1]);
      cmul(0.0, kx, htr, hti, &f[6][0], &f[6][1]);
      cmul(0.0, kz, htr, hti, &f[7][0], &f[7][1]);
    }
  }
  return OCN_OK;
}

/* surface.cpp:70-103; pairs surface.cpp:77-80. */
int orc_generate_maps(int n, int C, const double* lengths, double gravity, const double* h0,
                      const double* h0cn, const uint8_t* in_band, double t, double chop,
                      int single_precision, double* maps) {
  static const int pairs[4][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}};
  size_t nn = (size_t)n * n;
  double* coef = (double*)malloc(8 * 2 * nn * sizeof(double));
  for (int c = 0; c < C; ++c) {
    orc_assemble_coefficients(n, lengths[c], gravity, h0 + (size_t)c * 2 * nn,
                              h0cn + (size_t)c * 2 * nn, in_band + (size_t)c * nn, t, chop, coef);
    for (int p = 0; p < 4; ++p) {
      double* re = maps + ((size_t)c * 8 + pairs[p][0]) * nn;
      double* im = maps + ((size_t)c * 8 + pairs[p][1]) * nn;
      orc_ifft2_pair(n, coef + (size_t)pairs[p][0] * 2 * nn, coef + (size_t)pairs[p][1] * 2 * nn,
                     re, im);
    }
  }
  free(coef);
  if (single_precision)
    for (size_t q = 0; q < (size_t)C * 8 * nn; ++q) maps[q] = (double)(float)maps[q];
  return OCN_OK;
}

/* ======================================================================== */
/* velocity.cpp:10 */
double orc_attenuation(double k, double y) { return y > 0.0 ? 1.0 + k * y : exp(k * y); }

/* velocity.cpp:65-71 */
int orc_log_distribution(double y, double y_min, double* out) {
  if (!(y_min < 0.0)) return OCN_ERR_DOMAIN;
  const double alpha = 0.0001;
  double beta = -y_min / (2.0 * log(alpha * y_min * y_min + 1.0));
  double v = beta * log(alpha * y * y + 1.0);
  *out = y > 0.0 ? v : -v;
  return OCN_OK;
}

/* velocity.cpp:73-82 */
int orc_exp_interp(double a, double fa, double b, double fb, double x, double* out) {
  if (a == b) return OCN_ERR_DOMAIN;
  int degenerate = fabs(fa) < 1e-12 || fabs(fb) < 1e-12 || ((fa < 0.0) != (fb < 0.0));
  if (degenerate) {
    double u = (x - a) / (b - a);
    *out = fa + (fb - fa) * u;
    return OCN_OK;
  }
  double beta = (log(fabs(fb)) - log(fabs(fa))) / (b - a);
  *out = fa * exp(beta * (x - a));
  return OCN_OK;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* velocity.cpp:84-102 */
int orc_slice_depths(const ocn_slice_config* cfg, double* depths) {
  if (!(cfg->y_min < cfg->y_max)) return OCN_ERR_CONFIG;
  if (cfg->count < 2) return OCN_ERR_CONFIG;
  if (cfg->distribution == OCN_DEPTH_LOGARITHMIC && !(cfg->y_min < 0.0)) return OCN_ERR_CONFIG;
  for (int i = 0; i < cfg->count; ++i) {
    double pre = cfg->y_min + (cfg->y_max - cfg->y_min) * i / (cfg->count - 1);
    if (cfg->distribution == OCN_DEPTH_LOGARITHMIC)
      orc_log_distribution(pre, cfg->y_min, &depths[i]);
    else
      depths[i] = pre;
  }
  qsort(depths, (size_t)cfg->count, sizeof(double), cmp_double);
  return OCN_OK;
}

/* velocity.cpp:16-20: G = h0 e^{iwt} - h0cn e^{-iwt}. */
static void time_factor(const double* h0, const double* h0cn, size_t q, double omega, double t,
                        double* gr, double* gi) {
  double cr = cos(omega * t), si = sin(omega * t);
  double ar, ai, br, bi;
  cmul(h0[2 * q], h0[2 * q + 1], cr, si, &ar, &ai);
  cmul(h0cn[2 * q], h0cn[2 * q + 1], cr, -si, &br, &bi);
  *gr = ar - br;
  *gi = ai - bi;
}

/* velocity.cpp:104-179 */
int orc_build_slices(int n, int C, const double* lengths, double gravity, const double* h0,
                     const double* h0cn, const uint8_t* in_band, double t,
                     const ocn_slice_config* cfg, double* depths, double* slices) {
  int st = orc_slice_depths(cfg, depths);
  if (st) return st;
  int D = cfg->count;
  size_t nn = (size_t)n * n;
  /* coefficients per (depth, cascade): vx, vy, vz (complex) */
  double* coef = (double*)calloc((size_t)D * C * 3 * 2 * nn, sizeof(double));
  double* zero = (double*)calloc(2 * nn, sizeof(double));
  for (int d = 0; d < D; ++d) {
    for (int c = 0; c < C; ++c) {
      const double* H0 = h0 + (size_t)c * 2 * nn;
      const double* H0C = h0cn + (size_t)c * 2 * nn;
      const uint8_t* band = in_band + (size_t)c * nn;
      double* vx = coef + (((size_t)d * C + c) * 3 + 0) * 2 * nn;
      double* vy = vx + 2 * nn;
      double* vz = vy + 2 * nn;
      double dk = 2.0 * KPI / lengths[c];
      double y = depths[d];
      for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
          size_t q = (size_t)i * n + j;
          if (!band[q]) continue;
          double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
          double k = hypot(kx, kz);
          double omega = sqrt(gravity * k);
          double gr, gi;
          time_factor(H0, H0C, q, omega, t, &gr, &gi);
          double e = orc_attenuation(k, y);
          gr *= e;
          gi *= e;
          double sx = -kx * gravity / omega;
          double sz = -kz * gravity / omega;
          vx[2 * q] = gr * sx;
          vx[2 * q + 1] = gi * sx;
          cmul(gr, gi, 0.0, omega, &vy[2 * q], &vy[2 * q + 1]);
          vz[2 * q] = gr * sz;
          vz[2 * q + 1] = gi * sz;
        }
      }
    }
  }
  for (int d = 0; d < D; ++d)
    for (int c = 0; c < C; ++c) {
      double* vx = coef + (((size_t)d * C + c) * 3 + 0) * 2 * nn;
      double* out_x = slices + (((size_t)d * C + c) * 3 + 0) * nn;
      double* out_z = slices + (((size_t)d * C + c) * 3 + 2) * nn;
      orc_ifft2_pair(n, vx, vx + 4 * nn, out_x, out_z);
    }
  for (int d0 = 0; d0 < D; d0 += 2)
    for (int c = 0; c < C; ++c) {
      double* vy0 = coef + (((size_t)d0 * C + c) * 3 + 1) * 2 * nn;
      double* out0 = slices + (((size_t)d0 * C + c) * 3 + 1) * nn;
      if (d0 + 1 < D) {
        double* vy1 = coef + (((size_t)(d0 + 1) * C + c) * 3 + 1) * 2 * nn;
        double* out1 = slices + (((size_t)(d0 + 1) * C + c) * 3 + 1) * nn;
        orc_ifft2_pair(n, vy0, vy1, out0, out1);
      } else {
        orc_ifft2_pair(n, vy0, zero, out0, NULL);
      }
    }
  free(coef);
  free(zero);
  if (cfg->single_precision)
    for (size_t q = 0; q < (size_t)D * C * 3 * nn; ++q) slices[q] = (double)(float)slices[q];
  return OCN_OK;
}

/* velocity.cpp:24-59 */
int orc_direct_velocity(int n, int C, const double* lengths, double gravity, const double* h0,
                        const double* h0cn, const uint8_t* in_band, double t, int64_t npts,
                        const double* xzy, double* out) {
  size_t nn = (size_t)n * n;
  size_t cap = (size_t)C * nn, m = 0;
  double* modes = (double*)malloc(cap * 9 * sizeof(double));
  for (int c = 0; c < C; ++c) {
    double dk = 2.0 * KPI / lengths[c];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        size_t q = (size_t)i * n + j;
        if (!in_band[(size_t)c * nn + q]) continue;
        double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
        double k = hypot(kx, kz);
        double omega = sqrt(gravity * k);
        double gr, gi;
        time_factor(h0 + (size_t)c * 2 * nn, h0cn + (size_t)c * 2 * nn, q, omega, t, &gr, &gi);
        if (gr == 0.0 && gi == 0.0) continue;
        double* md = modes + 9 * m++;
        md[0] = kx;
        md[1] = kz;
        md[2] = k;
        double sx = -kx * gravity / omega, sz = -kz * gravity / omega;
        md[3] = gr * sx;
        md[4] = gi * sx;
        cmul(gr, gi, 0.0, omega, &md[5], &md[6]);
        md[7] = gr * sz;
        md[8] = gi * sz;
      }
  }
  for (int64_t p = 0; p < npts; ++p) {
    double x = xzy[3 * p], z = xzy[3 * p + 1], y = xzy[3 * p + 2];
    double vx = 0.0, vy = 0.0, vz = 0.0;
    for (size_t q = 0; q < m; ++q) {
      const double* md = modes + 9 * q;
      double phase = md[0] * x + md[1] * z;
      double c = cos(phase), s = sin(phase);
      double e = orc_attenuation(md[2], y);
      vx += e * (md[3] * c - md[4] * s);
      vy += e * (md[5] * c - md[6] * s);
      vz += e * (md[7] * c - md[8] * s);
    }
    out[3 * p] = vx;
    out[3 * p + 1] = vy;
    out[3 * p + 2] = vz;
  }
  free(modes);
  return OCN_OK;
}

/* ======================================================================== */
/* surface.cpp:107-121 (same helper in velocity.cpp:190-201) */
static double bilinear_periodic(const double* f, int n, double length, double x, double z) {
  double u = x / length * n;
  double v = z / length * n;
  double fu = u - floor(u);
  double fv = v - floor(v);
  int i0 = (int)floor(u) % n;
  if (i0 < 0) i0 += n;
  int j0 = (int)floor(v) % n;
  if (j0 < 0) j0 += n;
  int i1 = (i0 + 1) % n, j1 = (j0 + 1) % n;
  return f[(size_t)i0 * n + j0] * (1 - fu) * (1 - fv) + f[(size_t)i1 * n + j0] * fu * (1 - fv) +
         f[(size_t)i0 * n + j1] * (1 - fu) * fv + f[(size_t)i1 * n + j1] * fu * fv;
}

static const double* map_field(const orc_surface* s, int c, int field) {
  return s->maps + ((size_t)c * 8 + field) * (size_t)s->n * s->n;
}

/* surface.cpp:125-129 */
int orc_maps_sample(const orc_surface* s, int field, int64_t npts, const double* xz, double* out) {
  for (int64_t p = 0; p < npts; ++p) {
    double acc = 0.0;
    for (int c = 0; c < s->C; ++c)
      acc += bilinear_periodic(map_field(s, c, field), s->n, s->lengths[c], xz[2 * p], xz[2 * p + 1]);
    out[p] = acc;
  }
  return OCN_OK;
}

/* surface.cpp:131-139 */
static void sample_disp(const orc_surface* s, double x, double z, double d[3]) {
  d[0] = d[1] = d[2] = 0.0;
  for (int c = 0; c < s->C; ++c) {
    d[0] += bilinear_periodic(map_field(s, c, 1), s->n, s->lengths[c], x, z);
    d[1] += bilinear_periodic(map_field(s, c, 0), s->n, s->lengths[c], x, z);
    d[2] += bilinear_periodic(map_field(s, c, 2), s->n, s->lengths[c], x, z);
  }
}
int orc_sample_displacement(const orc_surface* s, int64_t npts, const double* xz, double* out) {
  for (int64_t p = 0; p < npts; ++p) sample_disp(s, xz[2 * p], xz[2 * p + 1], out + 3 * p);
  return OCN_OK;
}

/* surface.cpp:141-151 (kHeightRetrievalIters = 4, surface.hpp:96) */
static double height_at1(const orc_surface* s, double x, double z) {
  double wx = 0.0, wz = 0.0, h = 0.0, d[3];
  for (int it = 0; it < 4; ++it) {
    sample_disp(s, x - wx, z - wz, d);
    wx = d[0];
    wz = d[2];
    h = d[1];
  }
  return h;
}
int orc_height_at(const orc_surface* s, int64_t npts, const double* xz, double* out) {
  for (int64_t p = 0; p < npts; ++p) out[p] = height_at1(s, xz[2 * p], xz[2 * p + 1]);
  return OCN_OK;
}

/* surface.cpp:153-169 */
int orc_height_at_tolerance(const orc_surface* s, int64_t npts, const double* xz, double tol,
                            int max_iters, double* out, int32_t* iterations) {
  for (int64_t p = 0; p < npts; ++p) {
    double wx = 0.0, wz = 0.0, h_prev = 0.0, d[3];
    int done = 0;
    for (int it = 1; it <= max_iters; ++it) {
      sample_disp(s, xz[2 * p] - wx, xz[2 * p + 1] - wz, d);
      wx = d[0];
      wz = d[2];
      if (fabs(d[1] - h_prev) < tol) {
        out[p] = d[1];
        if (iterations) iterations[p] = it;
        done = 1;
        break;
      }
      h_prev = d[1];
    }
    if (!done) {
      out[p] = h_prev;
      if (iterations) iterations[p] = max_iters;
    }
  }
  return OCN_OK;
}

/* velocity.cpp:203-211 */
static void sample_slice1(const orc_slices* s, int d, double x, double z, double v[3]) {
  size_t nn = (size_t)s->n * s->n;
  v[0] = v[1] = v[2] = 0.0;
  for (int c = 0; c < s->C; ++c) {
    const double* base = s->data + ((size_t)d * s->C + c) * 3 * nn;
    v[0] += bilinear_periodic(base, s->n, s->lengths[c], x, z);
    v[1] += bilinear_periodic(base + nn, s->n, s->lengths[c], x, z);
    v[2] += bilinear_periodic(base + 2 * nn, s->n, s->lengths[c], x, z);
  }
}
int orc_sample_slice(const orc_slices* s, int depth, int64_t npts, const double* xz, double* out) {
  for (int64_t p = 0; p < npts; ++p) sample_slice1(s, depth, xz[2 * p], xz[2 * p + 1], out + 3 * p);
  return OCN_OK;
}

/* std::min / std::max / std::clamp semantics (not fmin / fmax). */
static double dmin(double a, double b) { return b < a ? b : a; }
static double dmax(double a, double b) { return a < b ? b : a; }
static double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* core.hpp:190-195 */
static double wrap_angle(double a) {
  a = fmod(a + KPI, 2.0 * KPI);
  if (a <= 0.0) a += 2.0 * KPI;
  return a - KPI;
}
static double lerp1(double a, double b, double t) { return (1.0 - t) * a + t * b; }

/* velocity.cpp:213-265 */
static int velocity_at1(const orc_slices* s, double x, double z, double y, int interp,
                        double out[3]) {
  if (y < s->y_min || y > s->y_max) return OCN_ERR_DOMAIN;
  const double* dep = s->depths;
  int D = s->D;
  double va[3], vb[3];
  if (y <= dep[0]) {
    sample_slice1(s, 0, x, z, vb);
    double u = (y - s->y_min) / (dep[0] - s->y_min);
    out[0] = vb[0] * u;
    out[1] = vb[1] * u;
    out[2] = vb[2] * u;
    return OCN_OK;
  }
  if (y >= dep[D - 1]) {
    int last = D - 1;
    sample_slice1(s, last - 1, x, z, va);
    sample_slice1(s, last, x, z, vb);
    double u = (y - dep[last - 1]) / (dep[last] - dep[last - 1]);
    for (int m = 0; m < 3; ++m) out[m] = va[m] + (vb[m] - va[m]) * u;
    return OCN_OK;
  }
  int hi = 0;
  while (hi < D && !(y < dep[hi])) ++hi; /* upper_bound */
  int lo = hi - 1;
  double a = dep[lo], b = dep[hi];
  sample_slice1(s, lo, x, z, va);
  sample_slice1(s, hi, x, z, vb);
  double u_lin = (y - a) / (b - a);
  if (interp == OCN_INTERP_LINEAR) {
    for (int m = 0; m < 3; ++m) out[m] = va[m] + (vb[m] - va[m]) * u_lin;
    return OCN_OK;
  }
  double mag_a = hypot(va[0], va[2]);
  double mag_b = hypot(vb[0], vb[2]);
  double mag, vy;
  orc_exp_interp(a, mag_a, b, mag_b, y, &mag);
  orc_exp_interp(a, va[1], b, vb[1], y, &vy);
  double ang_a = atan2(va[2], va[0]);
  double ang_b = atan2(vb[2], vb[0]);
  double dphi = wrap_angle(ang_b - ang_a);
  double hx, hz;
  if (fabs(dphi) > KPI - 0.1) {
    hx = lerp1(va[0], vb[0], u_lin);
    hz = lerp1(va[2], vb[2], u_lin);
  } else {
    double u = u_lin;
    if (mag_a > 1e-12 && mag_b > 1e-12) {
      double beta = (log(mag_b) - log(mag_a)) / (b - a);
      if (fabs(beta) > 1e-12) u = expm1(beta * (y - a)) / expm1(beta * (b - a));
    }
    double phi = ang_a + dphi * u;
    hx = mag * cos(phi);
    hz = mag * sin(phi);
  }
  out[0] = hx;
  out[1] = vy;
  out[2] = hz;
  return OCN_OK;
}

int orc_velocity_at(const orc_slices* s, int64_t npts, const double* xzy, int interp, int clamp,
                    double* out) {
  for (int64_t p = 0; p < npts; ++p) {
    double y = xzy[3 * p + 2];
    if (clamp) y = dclamp(y, s->y_min, s->y_max); /* sim.cpp:40 */
    int st = velocity_at1(s, xzy[3 * p], xzy[3 * p + 1], y, interp, out + 3 * p);
    if (st) return st;
  }
  return OCN_OK;
}

/* ======================================================================== */
/* Small vector helpers restating core.hpp:38-186 arithmetic. */
typedef struct { double x, y, z; } v3;
static v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 vadd(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 vsub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vmul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static v3 vdiv(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 vcross(v3 a, v3 b) {
  return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double vnorm(v3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
static v3 vload(const double* p) { return V(p[0], p[1], p[2]); }
static void vstore(double* p, v3 a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }

/* Quat::rotate, core.hpp:164-169 */
static v3 qrotate(const double q[4], v3 v) {
  v3 u = V(q[1], q[2], q[3]);
  v3 t = vmul(vcross(u, v), 2.0);
  return vadd(vadd(v, vmul(t, q[0])), vcross(u, t));
}
/* BodyPose, hydro.hpp:24-33 */
static v3 pose_to_world(const ocn_pose* p, v3 b) {
  return vadd(vload(p->position), qrotate(p->orientation, vsub(b, vload(p->com_body))));
}
static v3 pose_point_velocity(const ocn_pose* p, v3 w) {
  return vadd(vload(p->linear_velocity), vcross(vload(p->angular_velocity), vsub(w, vload(p->position))));
}

/* ---- mesh.cpp:18-37 validate_closed: sort directed edges. ---- */
typedef struct { int a, b; } edge2;
static int cmp_edge(const void* x, const void* y) {
  const edge2* p = (const edge2*)x;
  const edge2* q = (const edge2*)y;
  if (p->a != q->a) return (p->a > q->a) - (p->a < q->a);
  return (p->b > q->b) - (p->b < q->b);
}
static int find_edge(const edge2* e, size_t m, int a, int b) {
  size_t lo = 0, hi = m;
  while (lo < hi) {
    size_t mid = (lo + hi) / 2;
    if (e[mid].a < a || (e[mid].a == a && e[mid].b < b)) lo = mid + 1;
    else hi = mid;
  }
  return lo < m && e[lo].a == a && e[lo].b == b;
}

/* mesh.cpp:48-116 */
int orc_mesh_build(int nv, const double* verts, int nt, int32_t* tris, double* normals,
                   double* areas, double* props) {
  if (nv <= 0 || nt <= 0) return OCN_ERR_MESH;
  size_t m = (size_t)nt * 3;
  edge2* e = (edge2*)malloc(m * sizeof(edge2));
  for (int t = 0; t < nt; ++t)
    for (int k = 0; k < 3; ++k) {
      int a = tris[3 * t + k], b = tris[3 * t + (k + 1) % 3];
      if (a < 0 || b < 0 || a >= nv || b >= nv || a == b) { free(e); return OCN_ERR_MESH; }
      e[3 * t + k].a = a;
      e[3 * t + k].b = b;
    }
  qsort(e, m, sizeof(edge2), cmp_edge);
  for (size_t q = 1; q < m; ++q)
    if (e[q].a == e[q - 1].a && e[q].b == e[q - 1].b) { free(e); return OCN_ERR_MESH; }
  for (size_t q = 0; q < m; ++q)
    if (!find_edge(e, m, e[q].b, e[q].a)) { free(e); return OCN_ERR_MESH; }
  free(e);
  /* signed volume mesh.cpp:39-44, re-orient when negative (mesh.cpp:52-53) */
  double sv = 0.0;
  for (int t = 0; t < nt; ++t) {
    v3 a = vload(verts + 3 * tris[3 * t]), b = vload(verts + 3 * tris[3 * t + 1]),
       c = vload(verts + 3 * tris[3 * t + 2]);
    sv += vdot(a, vcross(b, c)) / 6.0;
  }
  if (sv < 0.0)
    for (int t = 0; t < nt; ++t) {
      int32_t s = tris[3 * t + 1];
      tris[3 * t + 1] = tris[3 * t + 2];
      tris[3 * t + 2] = s;
    }
  v3 bmin = vload(verts), bmax = vload(verts);
  for (int i = 0; i < nv; ++i) {
    v3 v = vload(verts + 3 * i);
    bmin = V(dmin(bmin.x, v.x), dmin(bmin.y, v.y), dmin(bmin.z, v.z));
    bmax = V(dmax(bmax.x, v.x), dmax(bmax.y, v.y), dmax(bmax.z, v.z));
  }
  double vol = 0.0, total_area = 0.0, second[3][3] = {{0}};
  v3 first = V(0, 0, 0);
  int degenerate = 0;
  for (int t = 0; t < nt; ++t) {
    v3 a = vload(verts + 3 * tris[3 * t]), b = vload(verts + 3 * tris[3 * t + 1]),
       c = vload(verts + 3 * tris[3 * t + 2]);
    v3 nrm = vcross(vsub(b, a), vsub(c, a));
    double nlen = vnorm(nrm);
    areas[t] = 0.5 * nlen;
    if (nlen < 1e-14) {
      ++degenerate;
      vstore(normals + 3 * t, V(0, 0, 0));
    } else {
      vstore(normals + 3 * t, vdiv(nrm, nlen));
    }
    total_area += areas[t];
    double vt = vdot(a, vcross(b, c)) / 6.0;
    vol += vt;
    first = vadd(first, vmul(vadd(vadd(a, b), c), vt / 4.0));
    v3 s = vadd(vadd(a, b), c);
    const v3 pts[4] = {a, b, c, s};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 4; ++k) {
          double pi = i == 0 ? pts[k].x : (i == 1 ? pts[k].y : pts[k].z);
          double pj = j == 0 ? pts[k].x : (j == 1 ? pts[k].y : pts[k].z);
          acc += pi * pj;
        }
        second[i][j] += vt / 20.0 * acc;
      }
  }
  if (!(vol > 0.0)) return OCN_ERR_MESH;
  v3 cen = vdiv(first, vol);
  double cm[3] = {cen.x, cen.y, cen.z};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) second[i][j] -= vol * cm[i] * cm[j];
  double tr = second[0][0] + second[1][1] + second[2][2];
  props[0] = vol;
  props[1] = cen.x;
  props[2] = cen.y;
  props[3] = cen.z;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) props[4 + 3 * i + j] = (i == j ? tr : 0.0) - second[i][j];
  props[13] = bmin.x;
  props[14] = bmin.y;
  props[15] = bmin.z;
  props[16] = bmax.x;
  props[17] = bmax.y;
  props[18] = bmax.z;
  props[19] = total_area;
  props[20] = degenerate;
  return OCN_OK;
}

/* ======================================================================== */
/* interactive.cpp:10-13 */
double orc_damping_factor(double speed, double d0, double d_max, double v_max) {
  double u = speed / v_max;
  u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
  return (1.0 - u) * d0 + u * d_max;
}


/* interactive.cpp:33-52 */
int orc_zone_create(const ocn_fdm_config* cfg, double body_size, double bx, double bz, double dt,
                    orc_zone** out) {
  if (cfg->grid_size < 8) return OCN_ERR_CONFIG;
  if (cfg->margin <= 1 || 2 * cfg->margin >= cfg->grid_size) return OCN_ERR_CONFIG;
  orc_zone* z = (orc_zone*)calloc(1, sizeof(orc_zone));
  z->cfg = *cfg;
  z->n = cfg->grid_size;
  z->margin = cfg->margin;
  if (z->cfg.delta_min <= 0.0) z->cfg.delta_min = dmax(2.0 * body_size, 1e-3) / z->n;
  if (z->cfg.delta_max <= 0.0) z->cfg.delta_max = 10.0 * z->cfg.delta_min;
  if (z->cfg.delta_max < z->cfg.delta_min) { free(z); return OCN_ERR_CONFIG; }
  size_t nn = (size_t)z->n * z->n;
  z->curr = (double*)calloc(nn, sizeof(double));
  z->prev = (double*)calloc(nn, sizeof(double));
  z->pos_curr[0] = bx;
  z->pos_curr[1] = bz;
  z->damping = cfg->d0;
  z->delta = dclamp(0.999 * dt, z->cfg.delta_min, z->cfg.delta_max);
  z->c = sqrt(0.49) * z->delta / dt;
  z->origin[0] = bx - 0.5 * z->n * z->delta;
  z->origin[1] = bz - 0.5 * z->n * z->delta;
  *out = z;
  return OCN_OK;
}

void orc_zone_destroy(orc_zone* z) {
  if (!z) return;
  free(z->curr);
  free(z->prev);
  free(z);
}

/* interactive.cpp:54-65 */
int orc_zone_update_stability(orc_zone* z, double speed, double dt) {
  if (!(dt > 0.0)) return OCN_ERR_DOMAIN;
  double target = speed < 1.0 ? 0.999 * dt : speed * 0.999 * dt;
  target = dclamp(target, z->cfg.delta_min, z->cfg.delta_max);
  double lo = z->delta * (1.0 - z->cfg.delta_rate_limit);
  double hi = z->delta * (1.0 + z->cfg.delta_rate_limit);
  z->delta = dclamp(target, lo, hi);
  z->delta = dclamp(z->delta, z->cfg.delta_min, z->cfg.delta_max);
  z->c = sqrt(0.49) * z->delta / dt;
  z->damping = orc_damping_factor(speed, z->cfg.d0, z->cfg.d_max, z->cfg.v_max);
  return OCN_OK;
}

static double zread(const orc_zone* z, const double* f, int i, int j) {
  return (i < 0 || j < 0 || i >= z->n || j >= z->n) ? 0.0 : f[(size_t)i * z->n + j];
}

/* interactive.cpp:67-111 */
int orc_zone_step(orc_zone* z, double dt, double bx, double bz) {
  int n = z->n, m = z->margin;
  double mx = bx - z->pos_curr[0], mz = bz - z->pos_curr[1];
  double rx = mx / z->delta + z->carry[0];
  double rz = mz / z->delta + z->carry[1];
  int wx = (int)floor(rx), wz = (int)floor(rz);
  z->carry[0] = rx - wx;
  z->carry[1] = rz - wz;
  int max_shift = m - 1;
  size_t nn = (size_t)n * n;
  if (abs(wx) > max_shift || abs(wz) > max_shift) {
    wx = wx < -max_shift ? -max_shift : (max_shift < wx ? max_shift : wx);
    wz = wz < -max_shift ? -max_shift : (max_shift < wz ? max_shift : wz);
    memset(z->curr, 0, nn * sizeof(double));
    memset(z->prev, 0, nn * sizeof(double));
    ++z->dropped_wake;
  }
  int ox = wx + z->last_shift[0], oz = wz + z->last_shift[1];
  double a = z->c * z->c * dt * dt / (z->delta * z->delta);
  double d = z->damping;
  double* next = (double*)calloc(nn, sizeof(double));
  for (int i = m; i < n - m; ++i)
    for (int j = m; j < n - m; ++j) {
      int k = i + wx, l = j + wz;
      double lap = zread(z, z->curr, k + 1, l) + zread(z, z->curr, k - 1, l) +
                   zread(z, z->curr, k, l + 1) + zread(z, z->curr, k, l - 1) -
                   4.0 * zread(z, z->curr, k, l);
      next[(size_t)i * n + j] =
          d * (a * lap + 2.0 * zread(z, z->curr, k, l) - zread(z, z->prev, i + ox, j + oz));
    }
  free(z->prev);
  z->prev = z->curr;
  z->curr = next;
  z->origin[0] += wx * z->delta;
  z->origin[1] += wz * z->delta;
  z->last_shift[0] = wx;
  z->last_shift[1] = wz;
  z->pos_curr[0] = bx;
  z->pos_curr[1] = bz;
  return OCN_OK;
}

/* interactive.cpp:113-118 */
int orc_zone_apply_cells(orc_zone* z, int n, const int32_t* ij, const double* h) {
  int m = z->margin;
  for (int q = 0; q < n; ++q) {
    int i = ij[2 * q], j = ij[2 * q + 1];
    if (i < m || j < m || i >= z->n - m || j >= z->n - m) continue;
    z->curr[(size_t)i * z->n + j] = h[q];
  }
  return OCN_OK;
}

/* interactive.cpp:120-129 */
double orc_zone_sample(const orc_zone* z, double x, double zc) {
  int n = z->n;
  double u = (x - z->origin[0]) / z->delta;
  double v = (zc - z->origin[1]) / z->delta;
  if (u < 0.0 || v < 0.0 || u > n - 1 || v > n - 1) return 0.0;
  int i0 = (int)u < n - 2 ? (int)u : n - 2;
  int j0 = (int)v < n - 2 ? (int)v : n - 2;
  double fu = u - i0, fv = v - j0;
  const double* f = z->curr;
  return f[(size_t)i0 * n + j0] * (1 - fu) * (1 - fv) + f[(size_t)(i0 + 1) * n + j0] * fu * (1 - fv) +
         f[(size_t)i0 * n + j0 + 1] * (1 - fu) * fv + f[(size_t)(i0 + 1) * n + j0 + 1] * fu * fv;
}

/* interactive.cpp:21-31 */
int orc_mask_height(double x, double z, const ocn_mask_frame* f, double speed,
                    const ocn_mask_params* p, double* out) {
  if (!(f->half_beam > 0.0) || !(f->z_max > f->z_min)) return OCN_ERR_DOMAIN;
  double fx = fabs(x - f->center_x) / f->half_beam;
  double h_f = speed * f->mesh_height * p->intensity * f->volume_ratio;
  double b_z = f->z_max - f->z_min;
  double a = (h_f - p->back_height) / b_z;
  double b = p->back_height - a * f->z_min;
  *out = p->amplitude * (fx + a * z + b);
  return OCN_OK;
}

/* interactive.cpp:131-144 */
int orc_point_in_loops(double px, double pz, int n_loops, const int32_t* off, const double* pts) {
  int crossings = 0;
  for (int l = 0; l < n_loops; ++l) {
    int n = off[l + 1] - off[l];
    const double* L = pts + 2 * (size_t)off[l];
    for (int e = 0; e + 1 < n; ++e) {
      double ax = L[2 * e], az = L[2 * e + 1], bxx = L[2 * e + 2], bzz = L[2 * e + 3];
      if ((ax > px) == (bxx > px)) continue;
      double zi = az + (px - ax) / (bxx - ax) * (bzz - az);
      if (zi > pz) ++crossings;
    }
  }
  return (crossings & 1) != 0;
}

/* interactive.cpp:146-195 */
int orc_compute_mask(const orc_zone* z, int n_loops, const int32_t* loop_offsets,
                     const double* points, double yaw, double bx, double bz, double speed,
                     const ocn_mask_frame* frame, const ocn_mask_params* params, int capacity,
                     int32_t* ij, double* h, int* n_cells) {
  *n_cells = 0;
  if (n_loops == 0) return OCN_OK;
  double cy = cos(-yaw), sy = sin(-yaw);
  int total = loop_offsets[n_loops];
  double* loc = (double*)malloc(sizeof(double) * 2 * (size_t)(total > 0 ? total : 1));
  int32_t* off = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_loops + 1));
  int kept = 0, np = 0;
  double lox = 1e300, loz = 1e300, hix = -1e300, hiz = -1e300;
  off[0] = 0;
  for (int l = 0; l < n_loops; ++l) {
    int cnt = loop_offsets[l + 1] - loop_offsets[l];
    if (cnt < 4) continue;
    for (int q = loop_offsets[l]; q < loop_offsets[l + 1]; ++q) {
      double qx = points[3 * q] - bx, qz = points[3 * q + 2] - bz;
      double lx = cy * qx + sy * qz, lz = -sy * qx + cy * qz;
      loc[2 * np] = lx;
      loc[2 * np + 1] = lz;
      ++np;
      lox = dmin(lox, lx);
      loz = dmin(loz, lz);
      hix = dmax(hix, lx);
      hiz = dmax(hiz, lz);
    }
    off[++kept] = np;
  }
  if (kept == 0) { free(loc); free(off); return OCN_OK; }
  double rad = hypot(dmax(fabs(lox), fabs(hix)), dmax(fabs(loz), fabs(hiz)));
  int n = z->n, m = z->margin;
#define CELL_OF(w, o) ((int)floor(((w) - (o)) / z->delta))
  int i0 = CELL_OF(bx - rad, z->origin[0]);
  if (i0 < m) i0 = m;
  int i1 = CELL_OF(bx + rad, z->origin[0]) + 2;
  if (i1 > n - m) i1 = n - m;
  int j0 = CELL_OF(bz - rad, z->origin[1]);
  if (j0 < m) j0 = m;
  int j1 = CELL_OF(bz + rad, z->origin[1]) + 2;
  if (j1 > n - m) j1 = n - m;
#undef CELL_OF
  int cnt = 0, st = OCN_OK;
  for (int i = i0; i < i1 && !st; ++i)
    for (int j = j0; j < j1; ++j) {
      double wx = z->origin[0] + i * z->delta, wz = z->origin[1] + j * z->delta;
      double qx = wx - bx, qz = wz - bz;
      double lx = cy * qx + sy * qz, lz = -sy * qx + cy * qz;
      if (lx < lox || lx > hix || lz < loz || lz > hiz) continue;
      if (!orc_point_in_loops(lx, lz, kept, off, loc)) continue;
      double hv;
      st = orc_mask_height(lx, lz, frame, speed, params, &hv);
      if (st) break;
      if (cnt < capacity) {
        ij[2 * cnt] = i;
        ij[2 * cnt + 1] = j;
        h[cnt] = hv;
      }
      ++cnt;
    }
  free(loc);
  free(off);
  *n_cells = cnt;
  return st;
}

/* ======================================================================== */
/* hydro.cpp:11-23 */
static double density_at(const orc_fluid* f, double y) {
  int n = f->n_profile;
  const double* p = f->profile;
  if (n == 0) return f->water_density;
  if (y <= p[0]) return p[1];
  if (y >= p[2 * (n - 1)]) return p[2 * (n - 1) + 1];
  for (int i = 1; i < n; ++i)
    if (y <= p[2 * i]) {
      double y0 = p[2 * (i - 1)], r0 = p[2 * (i - 1) + 1], y1 = p[2 * i], r1 = p[2 * i + 1];
      return lerp1(r0, r1, (y - y0) / (y1 - y0));
    }
  return f->water_density;
}

/* Simulation::compose_height sim.cpp:44-51 : height_at + other zones. */
static double surface_height(const orc_fluid* f, double x, double z) {
  double h = f->surface ? height_at1(f->surface, x, z) : 0.0;
  for (int q = 0; q < f->n_zones; ++q) h += orc_zone_sample(f->zones[q], x, z);
  return h;
}

/* hydro.cpp:69-76 */
int orc_vertex_depths(int nv, const double* verts, const ocn_pose* pose, const orc_fluid* fluid,
                      double* wpos, double* depth) {
  for (int i = 0; i < nv; ++i) {
    v3 w = pose_to_world(pose, vload(verts + 3 * i));
    vstore(wpos + 3 * i, w);
    depth[i] = w.y - surface_height(fluid, w.x, w.z);
  }
  return OCN_OK;
}

typedef struct { int a, b; } ekey; /* EdgeKey hydro.cpp:34-38 (a = min, b = max) */
static ekey mk_key(int u, int v) { ekey k = {u < v ? u : v, u < v ? v : u}; return k; }
static int key_lt(ekey p, ekey q) { return p.a != q.a ? p.a < q.a : p.b < q.b; }
static int key_eq(ekey p, ekey q) { return p.a == q.a && p.b == q.b; }

typedef struct { ekey k; int seg; } key_seg;
static int cmp_key_seg(const void* x, const void* y) {
  const key_seg* p = (const key_seg*)x;
  const key_seg* q = (const key_seg*)y;
  if (key_lt(p->k, q->k)) return -1;
  if (key_lt(q->k, p->k)) return 1;
  return (p->seg > q->seg) - (p->seg < q->seg);
}

static void emit(orc_clip_out* out, int* count, int parent, int status, v3 a, v3 b, v3 c,
                 double da, double db, double dc, v3 n) {
  if (*count < out->capacity_states) {
    ocn_triangle_state* s = &out->states[*count];
    s->parent = parent;
    s->status = status;
    s->area = 0.5 * vnorm(vcross(vsub(b, a), vsub(c, a)));
    vstore(s->centroid, vdiv(vadd(vadd(a, b), c), 3.0));
    s->depth = (da + db + dc) / 3.0;
    vstore(s->normal, n);
  }
  ++*count;
}

/* hydro.cpp:63-215 */
int orc_classify_clip(int nv, const double* wpos, const double* depth, int nt,
                      const int32_t* tris, const double* normals, const double* areas,
                      const ocn_pose* pose, orc_clip_out* out) {
  (void)nv;
  int count = 0, nseg = 0;
  out->submerged_area = out->dry_area = 0.0;
  out->degenerate_skipped = 0;
  ekey* seg_a = (ekey*)malloc(sizeof(ekey) * (size_t)nt);
  ekey* seg_b = (ekey*)malloc(sizeof(ekey) * (size_t)nt);
  v3* pt_a = (v3*)malloc(sizeof(v3) * (size_t)nt);
  v3* pt_b = (v3*)malloc(sizeof(v3) * (size_t)nt);
  for (int ti = 0; ti < nt; ++ti) {
    if (areas[ti] <= 0.0) {
      ++out->degenerate_skipped;
      continue;
    }
    int i0 = tris[3 * ti], i1 = tris[3 * ti + 1], i2 = tris[3 * ti + 2];
    double d0 = depth[i0], d1 = depth[i1], d2 = depth[i2];
    v3 n = qrotate(pose->orientation, vload(normals + 3 * ti));
    int ab0 = d0 >= 0.0, ab1 = d1 >= 0.0, ab2 = d2 >= 0.0;
    int above = ab0 + ab1 + ab2;
    int first = count;
    if (above == 3 || above == 0) {
      emit(out, &count, ti, above == 3 ? 1 : 0, vload(wpos + 3 * i0), vload(wpos + 3 * i1),
           vload(wpos + 3 * i2), d0, d1, d2, n);
    } else {
      int a, b, c, odd_above;
      if (above == 1) {
        odd_above = 1;
        if (ab0) a = i0, b = i1, c = i2;
        else if (ab1) a = i1, b = i2, c = i0;
        else a = i2, b = i0, c = i1;
      } else {
        odd_above = 0;
        if (!ab0) a = i0, b = i1, c = i2;
        else if (!ab1) a = i1, b = i2, c = i0;
        else a = i2, b = i0, c = i1;
      }
      double da = depth[a], db = depth[b], dc = depth[c];
      double alpha_ab = da / (da - db);
      double alpha_ac = da / (da - dc);
      v3 wa = vload(wpos + 3 * a), wb = vload(wpos + 3 * b), wc = vload(wpos + 3 * c);
      v3 pab = vadd(wa, vmul(vsub(wb, wa), alpha_ab));
      v3 pac = vadd(wa, vmul(vsub(wc, wa), alpha_ac));
      int odd_status = odd_above ? 1 : 0, rest = odd_above ? 0 : 1;
      emit(out, &count, ti, odd_status, wa, pab, pac, da, 0.0, 0.0, n);
      emit(out, &count, ti, rest, pab, wb, wc, 0.0, db, dc, n);
      emit(out, &count, ti, rest, pab, wc, pac, 0.0, dc, 0.0, n);
      ekey ka = mk_key(a, b), kb = mk_key(a, c);
      if (key_lt(ka, kb) || key_lt(kb, ka)) {
        seg_a[nseg] = ka;
        seg_b[nseg] = kb;
        pt_a[nseg] = pab;
        pt_b[nseg] = pac;
        ++nseg;
      }
    }
    /* ordered gather hydro.cpp:151-163: area sums in state order */
    for (int s = first; s < count && s < out->capacity_states; ++s) {
      if (out->states[s].status == 0) out->submerged_area += out->states[s].area;
      else out->dry_area += out->states[s].area;
    }
  }
  out->n_states = count;

  /* chaining hydro.cpp:165-213. by_edge: sorted (key, seg); cross_point:
   * last writer in segment order wins (std::map operator[] overwrite). */
  key_seg* ks = (key_seg*)malloc(sizeof(key_seg) * (size_t)(2 * nseg + 1));
  for (int s = 0; s < nseg; ++s) {
    ks[2 * s].k = seg_a[s];
    ks[2 * s].seg = s;
    ks[2 * s + 1].k = seg_b[s];
    ks[2 * s + 1].seg = s;
  }
  qsort(ks, (size_t)2 * nseg, sizeof(key_seg), cmp_key_seg);
  char* used = (char*)calloc((size_t)nseg + 1, 1);
  int nl = 0, np = 0;
  if (out->capacity_loops > 0 && out->loop_offsets) out->loop_offsets[0] = 0;
#define FIND_RANGE(key, lo_, hi_)                                        \
  do {                                                                   \
    size_t L_ = 0, H_ = (size_t)2 * nseg;                                \
    while (L_ < H_) {                                                    \
      size_t M_ = (L_ + H_) / 2;                                         \
      if (key_lt(ks[M_].k, key)) L_ = M_ + 1; else H_ = M_;              \
    }                                                                    \
    lo_ = L_;                                                            \
    while (L_ < (size_t)2 * nseg && key_eq(ks[L_].k, key)) ++L_;         \
    hi_ = L_;                                                            \
  } while (0)
  /* canonical crossing point of a key: from the largest segment touching it */
#define CROSS_POINT(key, outp)                                           \
  do {                                                                   \
    size_t lo_c, hi_c;                                                   \
    FIND_RANGE(key, lo_c, hi_c);                                         \
    int sg = ks[hi_c - 1].seg; (void)lo_c;                               \
    outp = key_eq(seg_a[sg], key) ? pt_a[sg] : pt_b[sg];                 \
  } while (0)
  v3* loop = (v3*)malloc(sizeof(v3) * (size_t)(nseg + 2));
  for (int start = 0; start < nseg; ++start) {
    if (used[start]) continue;
    int lp = 0, seg = start, closed = 0;
    ekey first_entry = seg_a[start], entry = first_entry;
    for (;;) {
      used[seg] = 1;
      CROSS_POINT(entry, loop[lp]);
      ++lp;
      ekey ex = key_eq(seg_a[seg], entry) ? seg_b[seg] : seg_a[seg];
      if (key_eq(ex, first_entry)) {
        closed = 1;
        break;
      }
      size_t lo, hi;
      FIND_RANGE(ex, lo, hi);
      int next = seg;
      for (size_t q = lo; q < hi; ++q)
        if (ks[q].seg != seg && !used[ks[q].seg]) next = ks[q].seg;
      if (next == seg) {
        CROSS_POINT(ex, loop[lp]);
        ++lp;
        break;
      }
      entry = ex;
      seg = next;
    }
    if (lp >= 3) {
      if (closed) loop[lp++] = loop[0];
      for (int q = 0; q < lp; ++q) {
        if (np + q < out->capacity_points && out->points) vstore(out->points + 3 * (np + q), loop[q]);
      }
      np += lp;
      ++nl;
      if (nl < out->capacity_loops && out->loop_offsets) out->loop_offsets[nl] = np;
    }
  }
#undef CROSS_POINT
#undef FIND_RANGE
  out->n_loops = nl;
  out->n_points = np;
  free(loop);
  free(used);
  free(ks);
  free(seg_a);
  free(seg_b);
  free(pt_a);
  free(pt_b);
  return OCN_OK;
}

/* hydro.cpp:242-251 */
static v3 drag1(const ocn_triangle_state* s, v3 medium, double rho, double cd, const ocn_pose* p) {
  v3 vrel = vsub(pose_point_velocity(p, vload(s->centroid)), medium);
  double speed = vnorm(vrel);
  if (speed < 1e-12 || s->area <= 0.0) return V(0, 0, 0);
  double facing = vdot(vload(s->normal), vdiv(vrel, speed));
  if (facing <= 0.0) return V(0, 0, 0);
  double a_perp = s->area * facing;
  return vmul(vrel, -(0.5 * cd * rho * a_perp * speed));
}

/* hydro.cpp:253-306 (+ the load composition of sim.cpp:114-122) */
int orc_aggregate(int nv, const double* verts, int nt, const int32_t* tris,
                  const double* normals, const double* areas, double mesh_volume,
                  const ocn_pose* pose, const orc_fluid* fluid, const double* vertex_depth,
                  ocn_hydro_report* r, orc_clip_out* clip) {
  double* wpos = (double*)malloc(sizeof(double) * 3 * (size_t)nv);
  double* depth = (double*)malloc(sizeof(double) * (size_t)nv);
  orc_vertex_depths(nv, verts, pose, fluid, wpos, depth);
  if (vertex_depth) memcpy(depth, vertex_depth, sizeof(double) * (size_t)nv);
  orc_classify_clip(nv, wpos, depth, nt, tris, normals, areas, pose, clip);
  free(wpos);
  free(depth);
  if (clip->n_states > clip->capacity_states) return OCN_ERR_ARG;
  memset(r, 0, sizeof(*r));
  r->submerged_area = clip->submerged_area;
  r->dry_area = clip->dry_area;
  r->state_count = clip->n_states;
  r->degenerate_skipped = clip->degenerate_skipped;
  r->waterline_loops = clip->n_loops;
  r->waterline_points = clip->n_points;
  const ocn_triangle_state* S = clip->states;
  int ns = clip->n_states;
  /* submerged_volume hydro.cpp:217-223 via deterministic_sum parallel.hpp:23-39 */
  double vw = 0.0;
  for (int c0 = 0; c0 < ns; c0 += 1024) {
    double acc = 0.0;
    for (int i = c0; i < ns && i < c0 + 1024; ++i)
      acc += S[i].status == 0 ? S[i].area * S[i].depth * S[i].normal[1] : 0.0;
    vw += acc;
  }
  if (vw < 0.0) {
    vw = 0.0;
    ++r->volume_clamped;
  } else if (vw > mesh_volume) {
    vw = mesh_volume;
    ++r->volume_clamped;
  }
  r->submerged_volume = vw;
  /* center_of_immersion hydro.cpp:225-238 */
  double cw = 0.0;
  v3 moment = V(0, 0, 0);
  for (int i = 0; i < ns; ++i) {
    if (S[i].status != 0) continue;
    double w = S[i].area * S[i].depth * S[i].normal[1];
    v3 pc = V(S[i].centroid[0], S[i].centroid[1] - 0.5 * S[i].depth, S[i].centroid[2]);
    cw += w;
    moment = vadd(moment, vmul(pc, w));
  }
  v3 coi = V(0, 0, 0);
  r->has_center_of_immersion = cw > 1e-12;
  if (r->has_center_of_immersion) coi = vdiv(moment, cw);
  vstore(r->center_of_immersion, coi);
  double rho_w = fluid->water_density;
  if (fluid->n_profile > 0 && r->has_center_of_immersion) rho_w = density_at(fluid, coi.y);
  /* water / air drag: deterministic_sum over 1024-chunks */
  v3 fw = V(0, 0, 0), fa = V(0, 0, 0);
  int st = OCN_OK;
  for (int c0 = 0; c0 < ns; c0 += 1024) {
    v3 accw = V(0, 0, 0), acca = V(0, 0, 0);
    for (int i = c0; i < ns && i < c0 + 1024; ++i) {
      if (S[i].status == 0) {
        double med[3] = {0, 0, 0};
        if (fluid->slices) {
          double q[3] = {S[i].centroid[0], S[i].centroid[2], S[i].centroid[1]};
          int s2 = orc_velocity_at(fluid->slices, 1, q, OCN_INTERP_EXPONENTIAL,
                                   fluid->velocity_clamp, med);
          if (s2) st = s2;
        }
        accw = vadd(accw, drag1(&S[i], vload(med), rho_w, fluid->cd_water, pose));
      } else {
        acca = vadd(acca, drag1(&S[i], vload(fluid->wind), fluid->air_density, fluid->cd_air, pose));
      }
    }
    fw = vadd(fw, accw);
    fa = vadd(fa, acca);
  }
  if (st) return st;
  vstore(r->water_drag, fw);
  vstore(r->air_drag, fa);
  v3 fb = V(0, 0, 0), wc = vload(pose->position);
  if (r->has_center_of_immersion) {
    fb = vmul(V(0.0, -KGRAVITY, 0.0), -(vw * rho_w)); /* hydro.cpp:240, 290 */
    wc = coi;
  }
  vstore(r->buoyancy_force, fb);
  vstore(r->water_center, wc);
  double dry_area = 0.0;
  v3 dry_moment = V(0, 0, 0);
  for (int i = 0; i < ns; ++i) {
    if (S[i].status != 1) continue;
    dry_area += S[i].area;
    dry_moment = vadd(dry_moment, vmul(vload(S[i].centroid), S[i].area));
  }
  v3 ac = dry_area > 1e-12 ? vdiv(dry_moment, dry_area) : vload(pose->position);
  vstore(r->air_center, ac);
  /* rigid_body.cpp:36-39 applied as in sim.cpp:114-122 */
  v3 F = V(0, 0, 0), T = V(0, 0, 0), P = vload(pose->position);
  if (r->has_center_of_immersion) {
    F = vadd(F, fb);
    T = vadd(T, vcross(vsub(wc, P), fb));
    F = vadd(F, fw);
    T = vadd(T, vcross(vsub(wc, P), fw));
  }
  F = vadd(F, fa);
  T = vadd(T, vcross(vsub(ac, P), fa));
  vstore(r->force, F);
  vstore(r->torque, T);
  return OCN_OK;
}

/* ======================================================================== */
/* Large single grids (16384^2 cannot hold CascadeSet + generate_maps
 * in host memory). One packed surface pair of one grid, computed mode by mode:
 * h0(i, j) is a pure function of (i, j) (counter-based Philox, spectra.cpp:150-169),
 * so h0 and conj(h0(-k)) (spectra.cpp:171-177) are evaluated on the fly instead
 * of being stored; the two coefficients of the pair follow surface.cpp:45-66
 * exactly as orc_assemble_coefficients, are packed as fft.cpp:88-91, and the
 * packed field goes through the same radix-2 ifft2_centered (fft.cpp:39-77) with
 * rows / columns spread over `threads` OpenMP threads (each row / column
 * transform is unchanged, so the result does not depend on the thread count).
 * Before the transform, the packed spectrum is also summed directly at the
 * grid nodes `ab` (npts pairs a, b): out[a, b] = sum_{i,j} P(i, j)
 * e^{+2 pi i ((i - N/2) a + (j - N/2) b) / N}, the definition fft.hpp:10-17 the
 * FFT implements (an independent check of the transform at spot points). */
static void h0_mode_at(int n, double dk, double length, double bmin, double bmax,
                       const ocn_spectrum_params* p, uint32_t cascade, int i, int j,
                       int* banded_out, double out[2]) {
  double kx = dk * (i - n / 2);
  double kz = dk * (j - n / 2);
  double k = hypot(kx, kz);
  double omega = orc_dispersion(k, p->gravity);
  int banded = k > 0.0 && k >= bmin && k < bmax;
  if (banded_out) *banded_out = banded;
  out[0] = out[1] = 0.0;
  if (!banded) return;
  double xi[2];
  orc_gaussian_complex(p->rng_seed, cascade, (uint32_t)i, (uint32_t)j, xi);
  double amp = sqrt(orc_h0_variance(kx, kz, k, omega, length, p));
  out[0] = xi[0] * amp;
  out[1] = xi[1] * amp;
}

static void ifft2_centered_mt(int n, double* f, int threads) {
  double* tw = (double*)malloc(sizeof(double) * (size_t)n);
  for (int j = 0; j < n / 2; ++j) {
    tw[2 * j] = cos(2.0 * KPI * j / n);
    tw[2 * j + 1] = sin(2.0 * KPI * j / n);
  }
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
  for (int i = 0; i < n; ++i) fft1d(f + 2 * (size_t)i * n, n, tw);
  const int CB = 8; /* columns gathered together (same per-column arithmetic) */
#pragma omp parallel num_threads(threads)
  {
    double* col = (double*)malloc(sizeof(double) * 2 * (size_t)n * CB);
#pragma omp for schedule(dynamic, 1)
    for (int j0 = 0; j0 < n; j0 += CB) {
      int cb = n - j0 < CB ? n - j0 : CB;
      for (int i = 0; i < n; ++i)
        for (int c = 0; c < cb; ++c) {
          col[2 * ((size_t)c * n + i)] = f[2 * ((size_t)i * n + j0 + c)];
          col[2 * ((size_t)c * n + i) + 1] = f[2 * ((size_t)i * n + j0 + c) + 1];
        }
      for (int c = 0; c < cb; ++c) fft1d(col + 2 * (size_t)c * n, n, tw);
      for (int i = 0; i < n; ++i)
        for (int c = 0; c < cb; ++c) {
          double sgn = ((i + j0 + c) & 1) ? -1.0 : 1.0;
          f[2 * ((size_t)i * n + j0 + c)] = sgn * col[2 * ((size_t)c * n + i)];
          f[2 * ((size_t)i * n + j0 + c) + 1] = sgn * col[2 * ((size_t)c * n + i) + 1];
        }
    }
    free(col);
  }
  free(tw);
}

int orc_surface_pair_large(int n, double length, double band_min, double band_max,
                           const ocn_spectrum_params* p, uint32_t cascade, double t, double chop,
                           int pair, int threads, int npts, const int32_t* ab, double* direct,
                           double* re, double* im) {
  static const int pairs[4][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}};
  if (!is_pow2(n) || n < 2 || !(length > 0.0) || pair < 0 || pair > 3) return OCN_ERR_CONFIG;
  int st = orc_spectrum_validate(p);
  if (st) return st;
  if (threads < 1) threads = 1;
  size_t nn = (size_t)n * n;
  double* packed = (double*)malloc(2 * nn * sizeof(double));
  if (!packed) return OCN_ERR_ARG;
  const double dk = 2.0 * KPI / length;
  const double gravity = p->gravity;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
  for (int i = 0; i < n; ++i) {
    const int ni = neg_index(i, n);
    for (int j = 0; j < n; ++j) {
      size_t q = (size_t)i * n + j;
      double a[2], m[2];
      int banded;
      h0_mode_at(n, dk, length, band_min, band_max, p, cascade, i, j, &banded, a);
      double f[8][2];
      memset(f, 0, sizeof f);
      if (banded) {
        h0_mode_at(n, dk, length, band_min, band_max, p, cascade, ni, neg_index(j, n), NULL, m);
        const double h0cr = m[0], h0ci = -m[1];
        /* surface.cpp:45-66, operation order of orc_assemble_coefficients */
        double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
        double k = hypot(kx, kz);
        double omega = sqrt(gravity * k);
        double cr = cos(omega * t), si = sin(omega * t);
        double ar, ai, br, bi;
        cmul(a[0], a[1], cr, si, &ar, &ai);
        cmul(h0cr, h0ci, cr, -si, &br, &bi);
        double htr = ar + br, hti = ai + bi;
        double ux = kx / k, uz = kz / k;
        double tr, ti, dxr, dxi, dzr, dzi;
        cmul(0.0 * ux, 1.0 * ux, htr, hti, &tr, &ti);
        dxr = tr * chop;
        dxi = ti * chop;
        cmul(0.0 * uz, 1.0 * uz, htr, hti, &tr, &ti);
        dzr = tr * chop;
        dzi = ti * chop;
        f[0][0] = htr;
        f[0][1] = hti;
        f[1][0] = dxr;
        f[1][1] = dxi;
        f[2][0] = dzr;
        f[2][1] = dzi;
        cmul(0.0, -kx, dxr, dxi, &f[3][0], &f[3][1]);
        cmul(0.0, -kx, dzr, dzi, &f[4][0], &f[4][1]);
        cmul(0.0, -kz, dzr, dzi, &f[5][0], &f[5][1]);
        cmul(0.0, kx, htr, hti, &f[6][0], &f[6][1]);
        cmul(0.0, kz, htr, hti, &f[7][0], &f[7][1]);
      }
      const double* x = f[pairs[pair][0]];
      const double* y = f[pairs[pair][1]];
      packed[2 * q] = x[0] + (0.0 * y[0] - 1.0 * y[1]);
      packed[2 * q + 1] = x[1] + (0.0 * y[1] + 1.0 * y[0]);
    }
  }
  if (npts > 0 && direct) {
    double* tw = (double*)malloc(2 * sizeof(double) * (size_t)n);
    for (int q = 0; q < n; ++q) {
      tw[2 * q] = cos(2.0 * KPI * q / n);
      tw[2 * q + 1] = sin(2.0 * KPI * q / n);
    }
    for (int s = 0; s < npts; ++s) {
      const long long a = ab[2 * s], b = ab[2 * s + 1];
      double sr = 0.0, si = 0.0;
#pragma omp parallel for reduction(+ : sr, si) schedule(static) num_threads(threads)
      for (int i = 0; i < n; ++i) {
        const long long pa = (long long)(i - n / 2) * a;
        for (int j = 0; j < n; ++j) {
          long long ph = (pa + (long long)(j - n / 2) * b) % n;
          if (ph < 0) ph += n;
          const double* w = tw + 2 * ph;
          const double* v = packed + 2 * ((size_t)i * n + j);
          sr += v[0] * w[0] - v[1] * w[1];
          si += v[0] * w[1] + v[1] * w[0];
        }
      }
      direct[2 * s] = sr;
      direct[2 * s + 1] = si;
    }
    free(tw);
  }
  ifft2_centered_mt(n, packed, threads);
  for (size_t q = 0; q < nn; ++q) {
    if (re) re[q] = packed[2 * q];
    if (im) im[q] = packed[2 * q + 1];
  }
  free(packed);
  return OCN_OK;
}
