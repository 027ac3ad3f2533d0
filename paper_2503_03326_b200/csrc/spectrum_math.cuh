// spectrum_math.cuh — fp64 spectrum model shared by the K1 kernel and the
// host scalar entry points (same source, __host__ __device__).
//
// Model: JONSWAP (spectra.cpp:36-47) x Donelan-Banner/Horvath directional
// spreading with swell and delta-mix (spectra.cpp:49-109), per-mode variance
// with the grid-cell measure (spectra.cpp:119-130). Random amplitudes:
// Philox4x32-10 keyed (seed, "ocen"|cascade), counter ((i<<32)|j, 0), words
// 0 and 1, Box-Muller, /sqrt(2) (rng.hpp:14-76) — integer part bit-exact.
#pragma once

#include <math.h>
#include <stdint.h>

#include "../../include/ocean_b200.h"

#ifdef __CUDACC__
#define OCN_HD __host__ __device__ __forceinline__
#else
#define OCN_HD inline
#endif

namespace ocn {
namespace sm {

constexpr double kPiD = 3.14159265358979323846;

// ---- Philox4x32-10 with the 128-bit key XOR-folded into two round keys ----
struct Philox4 {
  uint32_t v[4];
};

OCN_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

OCN_HD Philox4 philox(uint64_t key_lo, uint64_t key_hi, uint64_t ctr_lo, uint64_t ctr_hi) {
  uint32_t k0 = (uint32_t)key_lo ^ (uint32_t)key_hi;
  uint32_t k1 = (uint32_t)(key_lo >> 32) ^ (uint32_t)(key_hi >> 32);
  uint32_t c0 = (uint32_t)ctr_lo, c1 = (uint32_t)(ctr_lo >> 32);
  uint32_t c2 = (uint32_t)ctr_hi, c3 = (uint32_t)(ctr_hi >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t m0 = 0xD2511F53u, m1 = 0xCD9E8D57u;
    uint32_t hi0 = mulhi32(m0, c0), lo0 = m0 * c0;
    uint32_t hi1 = mulhi32(m1, c2), lo1 = m1 * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0, c1 = lo1, c2 = n2, c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  Philox4 out;
  out.v[0] = c0, out.v[1] = c1, out.v[2] = c2, out.v[3] = c3;
  return out;
}

OCN_HD void gaussian_complex(uint64_t seed, uint32_t stream, uint32_t i, uint32_t j, double* re,
                             double* im) {
  Philox4 b = philox(seed, 0x6F63656E00000000ull | stream, ((uint64_t)i << 32) | j, 0);
  double u1 = ((double)b.v[0] + 1.0) * (1.0 / 4294967296.0);
  double u2 = ((double)b.v[1] + 1.0) * (1.0 / 4294967296.0);
  double r = sqrt(-2.0 * log(u1));
  double s, c;
  double a = 2.0 * kPiD * u2;
  s = sin(a);
  c = cos(a);
  *re = r * c / sqrt(2.0);
  *im = r * s / sqrt(2.0);
}

// |k| = hypot(kx, kz) exactly as the reference's libm computes it (glibc
// 2.35+ e_hypot.c, non-FMA kernel: one Newton-style correction of
// sqrt(ax^2 + ay^2)). It is NOT correctly rounded (~0.6% of the grid modes
// differ from the correctly rounded value by 1 ulp), so a "better" hypot would
// break the bit-exact |k| / band mask. Explicitly rounded ops: no contraction.
#ifdef __CUDA_ARCH__
#define OCN_ADD(a, b) __dadd_rn(a, b)
#define OCN_SUB(a, b) __dsub_rn(a, b)
#define OCN_MUL(a, b) __dmul_rn(a, b)
#define OCN_DIV(a, b) __ddiv_rn(a, b)
#define OCN_SQRT(a) __dsqrt_rn(a)
#else
#define OCN_ADD(a, b) ((a) + (b))
#define OCN_SUB(a, b) ((a) - (b))
#define OCN_MUL(a, b) ((a) * (b))
#define OCN_DIV(a, b) ((a) / (b))
#define OCN_SQRT(a) sqrt(a)
#endif
OCN_HD double hypot_kernel(double ax, double ay) {
  double h = OCN_SQRT(OCN_ADD(OCN_MUL(ax, ax), OCN_MUL(ay, ay)));
  double t1, t2;
  if (h <= 2.0 * ay) {
    const double delta = OCN_SUB(h, ay);
    t1 = OCN_MUL(ax, OCN_SUB(2.0 * delta, ax));
    t2 = OCN_MUL(OCN_SUB(delta, 2.0 * OCN_SUB(ax, ay)), delta);
  } else {
    const double delta = OCN_SUB(h, ax);
    t1 = OCN_MUL(2.0 * delta, OCN_SUB(ax, 2.0 * ay));
    t2 = OCN_ADD(OCN_MUL(OCN_SUB(4.0 * delta, ay), ay), OCN_MUL(delta, delta));
  }
  return OCN_SUB(h, OCN_DIV(OCN_ADD(t1, t2), 2.0 * h));
}

OCN_HD double hypot_ref(double x, double y) {
  x = fabs(x), y = fabs(y);
  const double ax = x < y ? y : x;
  const double ay = x < y ? x : y;
  const double kScale = 0x1p-600, kEps = 0x1p-54;
  if (ax > 0x1p+511) {
    if (ay <= ax * kEps) return ax + ay;
    return hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay / kEps) return ax + ay;
    return hypot_kernel(ax / kScale, ay / kScale) * kScale;
  }
  if (ay <= ax * kEps) return ax + ay;
  return hypot_kernel(ax, ay);
}

// ---- spectra.cpp:10-130 (same expressions, same operation order) ----
OCN_HD double alpha(const ocn_spectrum_params& p) {
  return 0.076 * pow(p.wind_speed * p.wind_speed / (p.fetch * p.gravity), 0.22);
}
OCN_HD double peak_omega(const ocn_spectrum_params& p) {
  if (p.has_peak_omega_override) return p.peak_omega_override;
  return 22.0 * p.gravity * p.gravity / (p.wind_speed * p.fetch);
}
OCN_HD double standard_peak_omega(const ocn_spectrum_params& p) {
  return 22.0 * cbrt(p.gravity * p.gravity / (p.wind_speed * p.fetch));
}
// returns false (DomainError) for omega <= 0
OCN_HD bool jonswap(double omega, const ocn_spectrum_params& p, double* out) {
  if (!(omega > 0.0)) return false;
  double g = p.gravity;
  double wp = peak_omega(p);
  double sigma = omega <= wp ? 0.07 : 0.09;
  double d = (omega - wp) / (sigma * wp);
  double r = exp(-0.5 * d * d);
  double ratio = wp / omega;
  double ratio4 = ratio * ratio * ratio * ratio;
  *out = alpha(p) * g * g / pow(omega, 5.0) * exp(-1.25 * ratio4) * pow(3.3, r);
  return true;
}
OCN_HD double beta_s(double r) {
  if (r < 0.95) return 2.61 * pow(r, 1.3);
  if (r < 1.6) return 2.28 * pow(r, -1.3);
  double eps = 0.8393 * exp(-0.567 * log(r * r)) - 0.4;
  return pow(10.0, eps);
}
OCN_HD double directional_kernel(double beta, double theta) {
  double sech = 1.0 / cosh(beta * theta);
  return 0.5 * beta * sech * sech / tanh(beta * kPiD);
}
OCN_HD double donelan_banner(double omega, double theta, double omega_p) {
  return directional_kernel(beta_s(omega / omega_p), theta);
}
OCN_HD double swell_spread(double omega, double theta, double omega_p, double xi) {
  double r = omega / omega_p;
  double s = 16.0 * tanh(1.0 / r) * xi * xi;
  if (s == 0.0) return 1.0;
  double c = fabs(cos(0.5 * theta));
  if (c == 0.0) return 0.0;
  return pow(c, 2.0 * s);
}
OCN_HD double q_dbxi_approx(double r) {
  if (r < 0.94) return 7.1467551 * r * r - 13.4662001 * r + 7.75651088;
  if (r < 5.0) return -0.69906109 * r * r + 0.77975933 * r + 0.10169164;
  if (r < 100.0) return -2.1860997 * r * r + 0.0269209 * r + 0.00016283;
  return 1.2038847 * r + 0.0008147;
}
OCN_HD double directional(double omega, double theta, const ocn_spectrum_params& p) {
  double uniform = 1.0 / (2.0 * kPiD);
  double delta = p.direction_mix;
  if (delta == 0.0) return uniform;
  double wp = peak_omega(p);
  double d = q_dbxi_approx(omega / wp) * donelan_banner(omega, theta, wp) *
             swell_spread(omega, theta, wp, p.swell);
  if (d < 0.0) d = 0.0;
  return (1.0 - delta) * uniform + delta * d;
}
OCN_HD double h0_variance(double kx, double kz, double k, double omega, double L,
                          const ocn_spectrum_params& p) {
  if (k <= 0.0) return 0.0;
  double dk = 2.0 * kPiD / L;
  double theta = atan2(kz, kx) - p.wind_direction;
  double s = 0.0;
  jonswap(omega, p, &s);
  double d = directional(omega, theta, p);
  double domega_dk = p.gravity / (2.0 * omega);
  return s * d * domega_dk * dk * dk / k;
}

// velocity.cpp:10 — E(k, y)
OCN_HD double attenuation(double k, double y) { return y > 0.0 ? 1.0 + k * y : exp(k * y); }

OCN_HD double damping_factor(double speed, double d0, double d_max, double v_max) {
  double u = speed / v_max;
  u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
  return (1.0 - u) * d0 + u * d_max;
}

}  // namespace sm
}  // namespace ocn
