// samplers.cuh — device samplers over the fp32 maps / slices (fp64 coordinates
// and weights, fp32 taps): bilinear_periodic (surface.cpp:107-121),
// sample_displacement / height_at (surface.cpp:131-151), sample_slice /
// velocity_at (velocity.cpp:203-265), FdmZone::sample (interactive.cpp:120-129).
#pragma once

#include "objects.cuh"

namespace ocn {

struct SurfView {
  int n, C;
  double length[kMaxCascades];
  const float* fields;  // [C][8][n][n]
  __device__ __forceinline__ const float* f(int c, int field) const {
    return fields + ((size_t)c * 8 + field) * (size_t)n * n;
  }
};

struct SliceView {
  int n, C, D;
  double length[kMaxCascades];
  double y_min, y_max;
  const double* depths;  // [D] sorted
  const float* fields;   // [D][C][3][n][n]
  __device__ __forceinline__ const float* f(int d, int c, int comp) const {
    return fields + (((size_t)d * C + c) * 3 + comp) * (size_t)n * n;
  }
};

struct ZoneView {
  int n;
  double delta, ox, oz;
  const float* curr;
};

constexpr int kMaxZones = 16;

struct ZoneList {
  int count;
  ZoneView z[kMaxZones];
};

SurfView make_surf_view(ocn_maps* m);
SliceView make_slice_view(ocn_slices* s);

// Tap indices and weights of the periodic bilinear stencil (fp64).
struct Bilin {
  size_t q00, q10, q01, q11;
  double w00, w10, w01, w11;
};

__device__ __forceinline__ Bilin bilin_setup(int n, double length, double x, double z) {
  const double u = x / length * n;
  const double v = z / length * n;
  const double fu0 = floor(u), fv0 = floor(v);
  const double fu = u - fu0, fv = v - fv0;
  int i0 = (int)fu0 % n;
  if (i0 < 0) i0 += n;
  int j0 = (int)fv0 % n;
  if (j0 < 0) j0 += n;
  const int i1 = (i0 + 1) % n, j1 = (j0 + 1) % n;
  Bilin b;
  b.q00 = (size_t)i0 * n + j0;
  b.q10 = (size_t)i1 * n + j0;
  b.q01 = (size_t)i0 * n + j1;
  b.q11 = (size_t)i1 * n + j1;
  b.w00 = (1 - fu) * (1 - fv);
  b.w10 = fu * (1 - fv);
  b.w01 = (1 - fu) * fv;
  b.w11 = fu * fv;
  return b;
}

__device__ __forceinline__ double bilin_tap(const Bilin& b, const float* __restrict__ f) {
  return (double)__ldg(f + b.q00) * b.w00 + (double)__ldg(f + b.q10) * b.w10 +
         (double)__ldg(f + b.q01) * b.w01 + (double)__ldg(f + b.q11) * b.w11;
}

__device__ __forceinline__ double sample_field(const SurfView& s, int field, double x, double z) {
  double acc = 0.0;
#pragma unroll 4  // the cascades' taps issue together (latency-bound gathers)
  for (int c = 0; c < s.C; ++c) acc += bilin_tap(bilin_setup(s.n, s.length[c], x, z), s.f(c, field));
  return acc;
}

__device__ __forceinline__ void sample_disp(const SurfView& s, double x, double z, double* dx,
                                            double* h, double* dz) {
  double a = 0.0, b = 0.0, c2 = 0.0;
#pragma unroll 4
  for (int c = 0; c < s.C; ++c) {
    const Bilin w = bilin_setup(s.n, s.length[c], x, z);
    a += bilin_tap(w, s.f(c, OCN_FIELD_DX));
    b += bilin_tap(w, s.f(c, OCN_FIELD_H));
    c2 += bilin_tap(w, s.f(c, OCN_FIELD_DZ));
  }
  *dx = a, *h = b, *dz = c2;
}

// Algorithm 1 (surface.cpp:141-151), kHeightRetrievalIters = 4; also returns
// the final parametric point p (for the assembly outputs).
__device__ __forceinline__ double height_at_dev(const SurfView& s, double x, double z,
                                                double* px = nullptr, double* pz = nullptr,
                                                double* odx = nullptr, double* odz = nullptr) {
  double wx = 0.0, wz = 0.0, h = 0.0, dx, dz, hh;
  double qx = x, qz = z;
#pragma unroll 1
  for (int it = 0; it < 4; ++it) {
    qx = x - wx;
    qz = z - wz;
    sample_disp(s, qx, qz, &dx, &hh, &dz);
    wx = dx;
    wz = dz;
    h = hh;
  }
  if (px) *px = qx, *pz = qz;
  if (odx) *odx = wx, *odz = wz;
  return h;
}

// FdmZone::sample, interactive.cpp:120-129
__device__ __forceinline__ double zone_sample(const ZoneView& z, double x, double zc) {
  const int n = z.n;
  const double u = (x - z.ox) / z.delta;
  const double v = (zc - z.oz) / z.delta;
  if (u < 0.0 || v < 0.0 || u > n - 1 || v > n - 1) return 0.0;
  const int i0 = min((int)u, n - 2), j0 = min((int)v, n - 2);
  const double fu = u - i0, fv = v - j0;
  const float* f = z.curr;
  return (double)f[(size_t)i0 * n + j0] * (1 - fu) * (1 - fv) +
         (double)f[(size_t)(i0 + 1) * n + j0] * fu * (1 - fv) +
         (double)f[(size_t)i0 * n + j0 + 1] * (1 - fu) * fv +
         (double)f[(size_t)(i0 + 1) * n + j0 + 1] * fu * fv;
}

__device__ __forceinline__ void sample_slice_dev(const SliceView& s, int d, double x, double z,
                                                 double v[3]) {
  v[0] = v[1] = v[2] = 0.0;
#pragma unroll 4
  for (int c = 0; c < s.C; ++c) {
    const Bilin w = bilin_setup(s.n, s.length[c], x, z);
    v[0] += bilin_tap(w, s.f(d, c, 0));
    v[1] += bilin_tap(w, s.f(d, c, 1));
    v[2] += bilin_tap(w, s.f(d, c, 2));
  }
}

__device__ __forceinline__ double exp_interp_dev(double a, double fa, double b, double fb,
                                                 double x) {
  const bool degenerate = fabs(fa) < 1e-12 || fabs(fb) < 1e-12 || ((fa < 0.0) != (fb < 0.0));
  if (degenerate) {
    const double u = (x - a) / (b - a);
    return fa + (fb - fa) * u;
  }
  const double beta = (log(fabs(fb)) - log(fabs(fa))) / (b - a);
  return fa * exp(beta * (x - a));
}

__device__ __forceinline__ double wrap_angle_dev(double a) {
  const double pi = 3.14159265358979323846;
  a = fmod(a + pi, 2.0 * pi);
  if (a <= 0.0) a += 2.0 * pi;
  return a - pi;
}

// velocity_at (velocity.cpp:213-265). Returns false for y outside
// [y_min, y_max] (DomainError) unless clamp (Simulation::water_velocity).
// velocity_at split for lane-parallel callers: the depth bracket, the partial
// slice sums over cascades c = c0, c0 + cstep, ..., and the combination.
struct VelBracket {
  int kind;  // 0 out of range, 1 below the first slice, 2 above the last, 3 interior
  int il, ih;
  double u;  // kinds 1 / 2: the linear weight
};

__device__ __forceinline__ VelBracket velocity_bracket(const SliceView& s, double& y, int clamp) {
  VelBracket r{0, 0, 0, 0.0};
  if (clamp) y = y < s.y_min ? s.y_min : (s.y_max < y ? s.y_max : y);
  if (y < s.y_min || y > s.y_max) return r;
  const double* dep = s.depths;
  const int D = s.D;
  if (y <= dep[0]) {
    r.kind = 1, r.il = r.ih = 0;
    r.u = (y - s.y_min) / (dep[0] - s.y_min);
    return r;
  }
  if (y >= dep[D - 1]) {
    r.kind = 2, r.il = D - 2, r.ih = D - 1;
    r.u = (y - dep[D - 2]) / (dep[D - 1] - dep[D - 2]);
    return r;
  }
  int lo = 0, hi = D;  // upper_bound
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (y < dep[mid]) hi = mid;
    else lo = mid + 1;
  }
  r.kind = 3, r.il = lo - 1, r.ih = lo;
  return r;
}

__device__ __forceinline__ void sample_slice_part(const SliceView& s, int d, double x, double z,
                                                  int c0, int cstep, double v[3]) {
  v[0] = v[1] = v[2] = 0.0;
  for (int c = c0; c < s.C; c += cstep) {
    const Bilin w = bilin_setup(s.n, s.length[c], x, z);
    v[0] += bilin_tap(w, s.f(d, c, 0));
    v[1] += bilin_tap(w, s.f(d, c, 1));
    v[2] += bilin_tap(w, s.f(d, c, 2));
  }
}

static __device__ void velocity_combine(const SliceView& s, const VelBracket& br, double y,
                                        int interp, const double va[3], const double vb[3],
                                        double out[3]);

__device__ __forceinline__ bool velocity_at_dev(const SliceView& s, double x, double z, double y,
                                                int interp, int clamp, double out[3]) {
  const VelBracket br = velocity_bracket(s, y, clamp);
  if (br.kind == 0) {
    out[0] = out[1] = out[2] = 0.0;
    return false;
  }
  double va[3] = {0.0, 0.0, 0.0}, vb[3];
  if (br.kind != 1) sample_slice_dev(s, br.il, x, z, va);
  sample_slice_dev(s, br.ih, x, z, vb);
  velocity_combine(s, br, y, interp, va, vb, out);
  return true;
}

static __device__ __noinline__ void velocity_combine(const SliceView& s, const VelBracket& br,
                                                     double y, int interp, const double va[3],
                                                     const double vb[3], double out[3]) {
  if (br.kind == 1) {
    out[0] = vb[0] * br.u, out[1] = vb[1] * br.u, out[2] = vb[2] * br.u;
    return;
  }
  if (br.kind == 2) {
    for (int m = 0; m < 3; ++m) out[m] = va[m] + (vb[m] - va[m]) * br.u;
    return;
  }
  const double a = s.depths[br.il], b = s.depths[br.ih];
  const double u_lin = (y - a) / (b - a);
  if (interp == OCN_INTERP_LINEAR) {
    for (int m = 0; m < 3; ++m) out[m] = va[m] + (vb[m] - va[m]) * u_lin;
    return;
  }
  const double mag_a = hypot(va[0], va[2]);
  const double mag_b = hypot(vb[0], vb[2]);
  const double mag = exp_interp_dev(a, mag_a, b, mag_b, y);
  const double vy = exp_interp_dev(a, va[1], b, vb[1], y);
  const double ang_a = atan2(va[2], va[0]);
  const double ang_b = atan2(vb[2], vb[0]);
  const double dphi = wrap_angle_dev(ang_b - ang_a);
  double hx, hz;
  if (fabs(dphi) > 3.14159265358979323846 - 0.1) {
    hx = (1.0 - u_lin) * va[0] + u_lin * vb[0];
    hz = (1.0 - u_lin) * va[2] + u_lin * vb[2];
  } else {
    double u = u_lin;
    if (mag_a > 1e-12 && mag_b > 1e-12) {
      const double beta = (log(mag_b) - log(mag_a)) / (b - a);
      if (fabs(beta) > 1e-12) u = expm1(beta * (y - a)) / expm1(beta * (b - a));
    }
    const double phi = ang_a + dphi * u;
    double sp, cp;
    sincos(phi, &sp, &cp);
    hx = mag * cp;
    hz = mag * sp;
  }
  out[0] = hx, out[1] = vy, out[2] = hz;
}


}  // namespace ocn
