// spectral_kernels.cuh — the device side of the spectral step: K1 (spectrum
// init) and its tables, the time evolution, the row kernels (k_rows, the
// warp-synchronous k_rows_w), the column kernels (k_cols, the persistent
// TMA-fed k_cols_tma) and the small conversion
// kernels of the plain-FFT entry points. Included by spectral.cu inside
// namespace ocn::{anonymous}; the host side (plans, groups, graphs, C-ABI)
// stays in spectral.cu.
#pragma once

// ------------------------------------------------------------------ K1
// generate_h0, spectra.cpp:150-169, one thread per mode of every grid (fp64,
// bit-exact Philox and band mask; per-grid spectrum parameters).
__global__ void __launch_bounds__(256) k_spectrum_init(int n, int count, const GridConst* gc,
                                                       double2* h0_f64, float2* h0,
                                                       uint8_t* in_band) {
  const size_t nn = (size_t)n * n;
  const size_t total = nn * count;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / nn);
    const size_t q = idx - (size_t)c * nn;
    const int i = (int)(q / n), j = (int)(q - (size_t)i * n);
    const GridConst& G = gc[c];
    const double dk = G.dk;
    const double kx = dk * (i - n / 2);
    const double kz = dk * (j - n / 2);
    const double k = sm::hypot_ref(kx, kz);
    const double omega = sqrt(G.p.gravity * k);
    const bool banded = k > 0.0 && k >= G.band_min && k < G.band_max;
    double hr = 0.0, hi = 0.0;
    if (banded) {
      double gr, gi;
      sm::gaussian_complex(G.p.rng_seed, G.cindex, (uint32_t)i, (uint32_t)j, &gr, &gi);
      const double amp = sqrt(sm::h0_variance(kx, kz, k, omega, G.length, G.p));
      hr = gr * amp;
      hi = gi * amp;
    }
    h0_f64[idx] = make_double2(hr, hi);
    h0[idx] = make_float2((float)hr, (float)hi);
    in_band[idx] = banded ? 1 : 0;
  }
}

// WaveGrid accessors: h0_conj_neg (spectra.cpp:171-177) and wave vectors.
__global__ void k_grid_extras(int n, double dk, double g, const double2* h0, double2* h0cn,
                              double4* waves) {
  const size_t nn = (size_t)n * n;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < nn;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / n), j = (int)(q % n);
    if (h0cn) {
      const int ni = i == 0 ? 0 : n - i, nj = j == 0 ? 0 : n - j;
      const double2 v = h0[(size_t)ni * n + nj];
      h0cn[q] = make_double2(v.x, -v.y);
    }
    if (waves) {
      const double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
      const double k = sm::hypot_ref(kx, kz);
      waves[q] = make_double4(kx, kz, k, sqrt(g * k));
    }
  }
}

// assemble_coefficients (surface.cpp:39-68) in fp64 for the drop-in API
__global__ void k_assemble_coef(int n, double dk, double g, double t, double chop,
                                const double2* h0, const uint8_t* band, double2* out) {
  const size_t nn = (size_t)n * n;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < nn;
       q += (size_t)gridDim.x * blockDim.x) {
    double2 f[8];
    for (int m = 0; m < 8; ++m) f[m] = make_double2(0.0, 0.0);
    if (band[q]) {
      const int i = (int)(q / n), j = (int)(q % n);
      const int ni = i == 0 ? 0 : n - i, nj = j == 0 ? 0 : n - j;
      const double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
      const double k = sm::hypot_ref(kx, kz);
      const double w = sqrt(g * k);
      double sn, cs;
      sincos(w * t, &sn, &cs);
      const double2 a = h0[q], bm = h0[(size_t)ni * n + nj];
      const double2 b = make_double2(bm.x, -bm.y);  // conj(h0(-k))
      const double htr = (a.x * cs - a.y * sn) + (b.x * cs + b.y * sn);
      const double hti = (a.x * sn + a.y * cs) + (b.y * cs - b.x * sn);
      const double ux = kx / k, uz = kz / k;
      const double2 dx = make_double2(-ux * hti * chop, ux * htr * chop);
      const double2 dz = make_double2(-uz * hti * chop, uz * htr * chop);
      f[0] = make_double2(htr, hti);
      f[1] = dx;
      f[2] = dz;
      f[3] = make_double2(kx * dx.y, -kx * dx.x);   // (0, -kx) * Dx
      f[4] = make_double2(kx * dz.y, -kx * dz.x);   // (0, -kx) * Dz
      f[5] = make_double2(kz * dz.y, -kz * dz.x);   // (0, -kz) * Dz
      f[6] = make_double2(-kx * hti, kx * htr);     // (0, kx) * h~
      f[7] = make_double2(-kz * hti, kz * htr);     // (0, kz) * h~
    }
    for (int m = 0; m < 8; ++m) out[(size_t)m * nn + q] = f[m];
  }
}

// ------------------------------------------------------------------ evolve
// h~ and G (surface.cpp:49-50; velocity.cpp:16-20) at time t, one cascade.
// d_time = {t, dt}: grid g of a time-batched set (GridConst::frame) is
// evaluated at t + frame dt.
__global__ void k_set_time(double* d_time, double t, double dt) {
  d_time[0] = t;
  d_time[1] = dt;
}

// Per-frame tables built once at spectrum creation: h0p = (h0(k), conj(h0(-k)))
// as one float4 (no mirror gather per frame, spectra.cpp:171-177) and the fp64
// dispersion w(k) = sqrt(g |k|) (spectra.hpp:44-46), so the frame's evolve is
// two streaming loads and one or two stores per mode.
__global__ void __launch_bounds__(256) k_evolve_tables(int n, int count, const GridConst* gc,
                                                       const float2* __restrict__ h0,
                                                       float4* h0p, double* omega) {
  const size_t nn = (size_t)n * n;
  const size_t total = nn * count;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / nn);
    const int q = (int)(idx - (size_t)c * nn);
    const int i = q / n, j = q - i * n;
    const int ni = i == 0 ? 0 : n - i, nj = j == 0 ? 0 : n - j;
    const float2* h = h0 + (size_t)c * nn;
    const float2 a = h[q], m = h[ni * n + nj];
    h0p[idx] = make_float4(a.x, a.y, m.x, -m.y);
    const double dk = gc[c].dk;
    const double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
    omega[idx] = sqrt(gc[c].p.gravity * sqrt(kx * kx + kz * kz));
  }
}

// h~ = h0 e^{iwt} + conj(h0(-k)) e^{-iwt} -> spec_h, and (velocity plans)
// G = h0 e^{iwt} - conj(h0(-k)) e^{-iwt} -> spec_g (surface.cpp:49-50;
// velocity.cpp:16-20); the fp64 phase is reduced mod 2 pi before the fp32 sincos.
// One work item per mode of a table grid (`base` grids x N^2): its (h0,
// conj h0(-k)) and w are loaded once and evolved for every frame of a
// time-batched set (grid f * base + c at t + f dt; frames = 1 otherwise).
// With skip_rows (band skipping), only the rows a row pass can read are
// evolved: |i - N/2| < GridConst::row_half.
template <bool WITH_G>
__global__ void __launch_bounds__(256) k_evolve(size_t total, int logn, int base, int frames,
                                                const double* d_time,
                                                const float4* __restrict__ h0p,
                                                const double* __restrict__ omega, float2* spec_h,
                                                float2* spec_g, const GridConst* gc, int skip_rows) {
  const double t0 = d_time[0], dt = d_time[1];
  const int n = 1 << logn, lognn = 2 * logn;
  const size_t qmask = ((size_t)1 << lognn) - 1;
  const size_t stride_f = (size_t)base << lognn;  // elements between frames
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int g = (int)(idx >> lognn);
    const size_t q = idx & qmask;
    if (skip_rows) {
      const int i = (int)(q >> logn);
      if (abs(i - n / 2) >= __ldg(&gc[g].row_half)) continue;
    }
    const float4 hp = __ldg(h0p + idx);
    const double w = __ldg(omega + idx);
    for (int f = 0; f < frames; ++f) {
      double ph = w * (t0 + (double)f * dt);
      ph -= 6.283185307179586476925 * rint(ph * 0.15915494309189533577);
      float s, cs;
      sincosf((float)ph, &s, &cs);
      // A = a e^{i ph}, B = b e^{-i ph}
      const float ar = hp.x * cs - hp.y * s, ai = hp.x * s + hp.y * cs;
      const float br = hp.z * cs + hp.w * s, bi = hp.w * cs - hp.z * s;
      const size_t o = idx + (size_t)f * stride_f;
      __stcg(spec_h + o, make_float2(ar + br, ai + bi));
      if constexpr (WITH_G) __stcg(spec_g + o, make_float2(ar - br, ai - bi));
    }
  }
}

// North-star item 3 per texel of every grid: the slope
// normal n = (-Hx, 1, -Hz) / |.| and the Jacobian of X = p + D,
// J = (1 - DxDx)(1 - DzDz) - DzDx^2 (stored DxDx / DzDx / DzDz are -dD/d(.)),
// from the grid's maps -> out [grid][4][N][N] (nx, ny, nz, J), 4 texels per thread.
__global__ void __launch_bounds__(256) k_assemble_grid(int count, size_t nn, const float* maps,
                                                       float* out) {
  const size_t quads = nn / 4;
  const size_t total = quads * count;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t g = idx / quads, q = idx - g * quads;
    const float4* f = reinterpret_cast<const float4*>(maps + g * 8 * nn) + q;
    const float4 hx = __ldcs(f + OCN_FIELD_HX * quads), hz = __ldcs(f + OCN_FIELD_HZ * quads);
    const float4 xx = __ldcs(f + OCN_FIELD_DXDX * quads), zx = __ldcs(f + OCN_FIELD_DZDX * quads);
    const float4 zz = __ldcs(f + OCN_FIELD_DZDZ * quads);
    float4 nx, ny, nz, jac;
    auto one = [](float a, float b, float dxx, float dzx, float dzz, float& ox, float& oy, float& oz,
                  float& oj) {
      const float inv = 1.0f / sqrtf(fmaf(a, a, fmaf(b, b, 1.0f)));
      ox = -a * inv;
      oy = inv;
      oz = -b * inv;
      oj = (1.0f - dxx) * (1.0f - dzz) - dzx * dzx;
    };
    one(hx.x, hz.x, xx.x, zx.x, zz.x, nx.x, ny.x, nz.x, jac.x);
    one(hx.y, hz.y, xx.y, zx.y, zz.y, nx.y, ny.y, nz.y, jac.y);
    one(hx.z, hz.z, xx.z, zx.z, zz.z, nx.z, ny.z, nz.z, jac.z);
    one(hx.w, hz.w, xx.w, zx.w, zz.w, nx.w, ny.w, nz.w, jac.w);
    float4* o = reinterpret_cast<float4*>(out + g * 4 * nn) + q;
    __stcs(o, nx);
    __stcs(o + quads, ny);
    __stcs(o + 2 * quads, nz);
    __stcs(o + 3 * quads, jac);
  }
}

// ------------------------------------------------------------------ rows
// kCentreByShift: the reference centres its inverse FFT by multiplying the
// output by (-1)^(i+j) (fft.cpp:73-75). For power-of-two N that equals the
// transform of the input shifted by N/2 in both axes:
//   sum_k X[k ^ N/2] e^{+2 pi i n k / N} = (-1)^n sum_k X[k] e^{+2 pi i n k / N},
// so the row pass reads mode (i, j ^ N/2) for FFT input j and writes its
// result to scratch row i ^ N/2; the column pass then needs no sign multiply.
// (Same values up to fp32 rounding order; the slab path keeps the explicit sign.)
struct RowArgs {
  int items;  // N * G (generic kernel)
  int G;
  int rpc = 1;  // warp kernel, surface family: rows per CTA
  const XformDesc* desc;   // group descriptors
  const GroupSeg* segs;    // per-grid segments of the group (warp kernel)
  const float2* spec_h;    // h~ of every grid, [grid][N][N]
  const float2* spec_g;    // G of every grid (velocity plans)
  const GridConst* gc;     // per-grid constants
  float chop;
  const float2* src;  // plain mode: [G][N][N] complex input
  float2* scratch;    // [G][N][N]
  const float2* tw;
  // rows outside a grid's band (GridConst::row_half) are exactly zero: skip
  // them (set only when the column pass treats them as zero without reading)
  int skip_zero_rows;
  int stage_f4;  // warp row kernel: float4 slots of the per-row staging area
  // fused evolve (warp row kernel): h~ / G of the staged rows are evaluated
  // from the h0p / omega tables at d_time (k_evolve's arithmetic) instead of
  // being read from spec_h / spec_g
  const float4* h0p;
  const double* omega;
  const double* d_time;
};

// h~ (surface, A + B) or G (velocity, A - B) of one mode at time t from its
// (h0(k), conj h0(-k)) pair and w(k) -- k_evolve's arithmetic, bit for bit
template <bool G_FORM>
__device__ __forceinline__ float2 evolve_mode(float4 hp, double w, double t) {
  double ph = w * t;
  ph -= 6.283185307179586476925 * rint(ph * 0.15915494309189533577);
  float s, cs;
  sincosf((float)ph, &s, &cs);
  const float ar = hp.x * cs - hp.y * s, ai = hp.x * s + hp.y * cs;
  const float br = hp.z * cs + hp.w * s, bi = hp.w * cs - hp.z * s;
  return G_FORM ? make_float2(ar - br, ai - bi) : make_float2(ar + br, ai + bi);
}

// packed coefficient X + iY of transform `d` at mode (i, j)
__device__ __forceinline__ float2 packed_coef(const XformDesc& d, float2 s, int i, int j, int n,
                                              float dk, float g, float chop) {
  const float kx = dk * (float)(i - n / 2);
  const float kz = dk * (float)(j - n / 2);
  const float k2 = kx * kx + kz * kz;
  if (k2 == 0.0f) return make_float2(0.f, 0.f);
  const float k = sqrtf(k2);
  const float inv_k = 1.0f / k;
  float mr, mi;
  float2 base;
  switch (d.kind) {
    case kSurfHDx: {  // h~ (1 - ux chop)
      mr = 1.0f - kx * inv_k * chop;
      mi = 0.f;
      base = s;
      break;
    }
    case kSurfDzDxDx: {  // i chop (uz + kx ux) h~
      mr = 0.f;
      mi = chop * (kz * inv_k + kx * kx * inv_k);
      base = s;
      break;
    }
    case kSurfDzDxDzDz: {  // chop uz (kx + i kz) h~
      const float f = chop * kz * inv_k;
      mr = f * kx;
      mi = f * kz;
      base = s;
      break;
    }
    case kSurfHxHz: {  // (-kz + i kx) h~
      mr = -kz;
      mi = kx;
      base = s;
      break;
    }
    case kVelXZ: {  // -(g/w) E(y0) (kx + i kz) G
      const float w = sqrtf(g * k);
      const float e = d.y0 > 0.f ? 1.0f + k * d.y0 : expf(k * d.y0);
      const float f = -(g / w) * e;
      mr = f * kx;
      mi = f * kz;
      base = s;
      break;
    }
    case kVelYPair: {  // w (-E(y1) + i E(y0)) G
      const float w = sqrtf(g * k);
      const float e0 = d.y0 > 0.f ? 1.0f + k * d.y0 : expf(k * d.y0);
      const float e1 = d.y1 > 0.f ? 1.0f + k * d.y1 : expf(k * d.y1);
      mr = -w * e1;
      mi = w * e0;
      base = s;
      break;
    }
    default: {  // kVelYSingle: i w E(y0) G
      const float w = sqrtf(g * k);
      const float e0 = d.y0 > 0.f ? 1.0f + k * d.y0 : expf(k * d.y0);
      mr = 0.f;
      mi = w * e0;
      base = s;
      break;
    }
  }
  return make_float2(base.x * mr - base.y * mi, base.x * mi + base.y * mr);
}

template <int N, bool PLAIN>
__global__ void __launch_bounds__(Launch<N>::THREADS) k_rows(const RowArgs a) {
  using L = Launch<N>;
  extern __shared__ float2 smem[];
  const int local = threadIdx.x / L::T;
  const int t = threadIdx.x - local * L::T;
  const int item = blockIdx.x * L::PER_CTA + local;
  const bool valid = item < a.items;
  const int row = valid ? item / a.G : 0;
  const int gi = valid ? item - row * a.G : 0;
  float2* sm = smem + local * L::ROW_STRIDE;
  constexpr int H = N / 2;  // centring half-shift (see kCentreByShift)
  float2* out = a.scratch + ((size_t)gi * N + (row ^ H)) * N;
  if constexpr (PLAIN) {
    const float2* in = a.src + ((size_t)gi * N + row) * N;
    fft::cta_fft<N>(
        t, sm, a.tw, [&](int j) { return valid ? __ldg(in + (j ^ H)) : make_float2(0.f, 0.f); },
        [&](int k, float2 x) {
          if (valid) out[k] = x;
        });
  } else {
    const XformDesc d = a.desc[gi];
    const float2* srow =
        (d.kind <= kSurfHxHz ? a.spec_h : a.spec_g) + ((size_t)d.cascade * N + row) * N;
    const float dk = (float)a.gc[d.cascade].dk, g = (float)a.gc[d.cascade].p.gravity;
    fft::cta_fft<N>(
        t, sm, a.tw,
        [&](int j) {
          if (!valid) return make_float2(0.f, 0.f);
          return packed_coef(d, __ldg(srow + (j ^ H)), row, j ^ H, N, dk, g, a.chop);
        },
        [&](int k, float2 x) {
          if (valid) out[k] = x;
        });
  }
}

struct ColArgs {
  const float2* scratch;  // [G][N][N]
  const XformDesc* desc;  // split outputs per transform
  const GridConst* gc;    // band-limited skipping (nullptr: every row is read)
  float2* out_c;          // complex mode: [G][N][N]
  const float2* tw;
  const CUtensorMap* out_maps;  // TMA-store column pass: Re / Im store maps per transform
};

// ------------------------------------------------------------------ rows (N <= 1024)
// Warp-synchronous variant: one CTA per row handles every transform of the
// group (warp w takes transform slots w, w + W, ...). The row's (h~, G) and
// the per-mode kz, |k|, 1/|k|, omega are staged once in shared memory; the
// per-transform multiplier is selected once per warp (no per-element switch),
// coefficients are written to the warp's FFT buffer and transformed with
// __syncwarp-only exchanges.
template <int N>
struct WarpLaunch {
  using PL = fft::Plan<N>;
  static_assert(PL::T <= 32, "warp kernels need T <= 32");
  static constexpr int T = PL::T;
  static constexpr int TPW = 32 / T;  // transforms per warp
  static constexpr int STRIDE = Launch<N>::ROW_STRIDE;
  static constexpr int TWN = (PL::tw_size() + 15) / 16 * 16;  // shared twiddle slots
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

enum RowMode : int { kRowPlain = 0, kRowSurface = 1, kRowVelocity = 2 };

#ifndef OCN_ROWS_MINB_SMALL
#define OCN_ROWS_MINB_SMALL 2
#endif
template <int N, int MODE, bool FUSED = false>
__global__ void __launch_bounds__(256, N >= 1024 ? 2 : OCN_ROWS_MINB_SMALL) k_rows_w(const RowArgs a) {
  constexpr bool PLAIN = MODE == kRowPlain;
  using W = WarpLaunch<N>;
  constexpr int T = W::T;
  constexpr int H = N / 2;  // centring half-shift (see kCentreByShift)
  extern __shared__ float4 smem4[];
  // Per mode of this row, shared by every transform of the group (SoA):
  //   sht = h~,  sv0 = V0 = G (-g / w)(kx + i kz),  sw0 = W0 = G w,  sk = |k|,
  //   sinv = 1/|k| (0 at k = 0). A velocity coefficient is then V0 E(y) or
  //   W0 (-E(y1) + i E(y0)), E(y) = exp(|k| y) (y <= 0) or 1 + |k| y.
  // Surface CTAs take a.rpc rows: a grid has only 4 surface transforms, so
  // one row keeps only 4 warps busy for a short CTA whose staging latency is
  // then poorly hidden. N >= 1024: up to 4 rows with only h~ staged (1/|k|
  // recomputed per element, MUFU); smaller N: up to 2 rows with h~ and 1/|k|
  // staged (measured best for each: config 3 / config 4).
  constexpr bool SURF_INV_INLINE = N >= 1024;
  const int rpc = MODE == kRowSurface ? a.rpc : 1;
  float2* sht = reinterpret_cast<float2*>(smem4);
  float* sinv = reinterpret_cast<float*>(sht + rpc * N);
  float2* sv0 = reinterpret_cast<float2*>(smem4);
  float2* sw0 = sv0 + N;
  float* sk = reinterpret_cast<float*>(sw0 + N);
  // inter-pass twiddles in shared memory (no global loads in the FFT passes)
  float2* stw = PLAIN ? reinterpret_cast<float2*>(smem4) : reinterpret_cast<float2*>(smem4 + a.stage_f4);
  float2* bufs = stw + W::TWN;
  for (int i = threadIdx.x; i < fft::Plan<N>::tw_size(); i += blockDim.x) stw[i] = __ldg(a.tw + i);
  const int row0 = blockIdx.x * rpc;
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / T, t = lane - sub * T;
  // this CTA: one row of one grid, the transforms [first, first + count) of the group
  int seg_first = 0, seg_count = a.G, grid = 0;
  if constexpr (!PLAIN) {
    const GroupSeg sg = a.segs[blockIdx.y];
    seg_first = sg.first, seg_count = sg.count, grid = sg.grid;
  }
  const float dkf = PLAIN ? 0.f : (float)a.gc[grid].dk;
  int row_half = N;  // |row - N/2| < row_half may be nonzero
  if constexpr (!PLAIN) {
    if (a.skip_zero_rows) {
      row_half = a.gc[grid].row_half;
      if (abs(row0 - N / 2) >= row_half && abs(row0 + rpc - 1 - N / 2) >= row_half &&
          (row0 - N / 2) * (row0 + rpc - 1 - N / 2) > 0)
        return;  // every row of this CTA is outside the band (uniform exit)
    }
  }
  if constexpr (!PLAIN) {
    const float2* srow =
        (MODE == kRowSurface ? a.spec_h : a.spec_g) + ((size_t)grid * N + row0) * N;
    const float g = (float)a.gc[grid].p.gravity;
    const size_t tab = FUSED ? ((size_t)a.gc[grid].src * N + row0) * N : 0;
    const double tt = FUSED ? a.d_time[0] + (double)a.gc[grid].frame * a.d_time[1] : 0.0;
    // MUFU reciprocal square roots (no IEEE slow-path calls, so the row's
    // loads issue back to back); only the arrays this family reads
#pragma unroll 4
    for (int j = threadIdx.x; j < rpc * N; j += blockDim.x) {
      // h~ (surface) or G (velocity)
      float2 sp;
      if constexpr (FUSED)
        sp = evolve_mode<MODE == kRowVelocity>(__ldg(a.h0p + tab + j), __ldg(a.omega + tab + j), tt);
      else
        sp = __ldg(srow + j);
      const float kx = dkf * (float)(row0 + j / N - N / 2);
      const float kz = dkf * (float)((j & (N - 1)) - N / 2);
      const float k2 = kx * kx + kz * kz;
      const bool zero = k2 == 0.f;  // k = 0: every coefficient vanishes
      const float inv = zero ? 0.f : rsqrtf(k2);
      const float k = k2 * inv;
      if constexpr (MODE == kRowSurface) {
        sht[j] = sp;
        if constexpr (!SURF_INV_INLINE) sinv[j] = inv;
      } else {
        const float rw = zero ? 0.f : rsqrtf(g * k);  // 1 / w
        const float w = g * k * rw, f = -g * rw;     // w, -g / w
        sv0[j] = make_float2(f * (sp.x * kx - sp.y * kz), f * (sp.x * kz + sp.y * kx));
        sw0[j] = make_float2(sp.x * w, sp.y * w);
        sk[j] = k;
      }
    }
  }
  __syncthreads();
  const int slots = (seg_count + W::TPW - 1) / W::TPW;
  const int items = slots * rpc;  // (row of the CTA, transform slot)
  float2* buf = bufs + (size_t)(warp * W::TPW + sub) * W::STRIDE;
  // the (kind, y0, y1) of this warp's next transform are loaded one slot ahead
  auto desc_of = [&](int item) {
    const int li = (item % slots) * W::TPW + sub;
    const XformDesc* d = a.desc + seg_first + (li < seg_count ? li : 0);
    return make_float4(__int_as_float(__ldg(&d->kind)), __ldg(&d->y0), __ldg(&d->y1),
                       __int_as_float(__ldg(&d->row_half)));
  };
  float4 dnext = make_float4(0.f, 0.f, 0.f, 0.f);
  if constexpr (!PLAIN) dnext = desc_of(warp < items ? warp : 0);
  for (int item = warp; item < items; item += warps) {
    const int rr = item / slots, slot = item - rr * slots;
    const int row = row0 + rr;
    const float kx = dkf * (float)(row - N / 2);
    const int li = slot * W::TPW + sub;
    const bool valid = li < seg_count;
    const int gi = seg_first + (valid ? li : 0);  // transform index within the group
    const float4 dcur = dnext;
    if constexpr (!PLAIN)
      if (item + warps < items) dnext = desc_of(item + warps);
    if (abs(row - N / 2) >= row_half) continue;  // exactly zero: not written, not read
    bool edge_row = false;  // the row's nonzero inputs are j < T and j >= N - T
    if constexpr (!PLAIN)
      if (a.skip_zero_rows) {  // this transform's own band (depth attenuation)
        const int rt = __float_as_int(dcur.w);
        if (rt > 0 && abs(row - N / 2) >= rt) continue;
        // |kz| < band as well: input j (mode j ^ N/2) is zero unless j < rt or j > N - rt
        edge_row = rt > 0 && rt <= fft::Plan<N>::T;
      }
    float2* out = a.scratch + ((size_t)gi * N + (row ^ H)) * N;
    auto store = [&](int k, float2 x) {
      if (valid) out[k] = x;
    };
    if constexpr (PLAIN) {
      const float2* in = a.src + ((size_t)gi * N + row) * N;
      for (int j = t; j < N; j += T)
        buf[fft::pad32(j)] = valid ? __ldg(in + (j ^ H)) : make_float2(0.f, 0.f);
      __syncwarp();
      fft::cta_fft<N, true, true, false, true>(
          t, buf, stw, [&](int j) { return buf[fft::pad32(j)]; }, store);
    } else {
      const int dkind = __float_as_int(dcur.x);
      // One branch-free FFT body per transform kind (selected once per
      // transform, warp-uniform): no per-element kind tests in pass 0.
      if constexpr (MODE == kRowSurface) {
        // surface pairs: X + iY = h~ M(kx, kz) (surface.cpp:77-80 packing),
        // every kind written as one branch-free form with per-transform
        // constants (a per-kind body let the compiler hoist the shared loads
        // of all four and spill):
        //   Re M = c0 + c3 kz + kx / |k| (c1 + c2 kz)
        //   Im M = c4 + (c5 (kz + kx^2) + c6 kz^2) / |k|
        // h~ = 0 at k = 0 (K1 masks it), so that mode needs no special case
        const float chop = a.chop, dk = dkf;
        float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, c5 = 0.f, c6 = 0.f;
        if (dkind == kSurfHDx) c0 = 1.f, c1 = -chop;             // 1 - chop kx / k
        else if (dkind == kSurfDzDxDx) c5 = chop;                 // i chop (kz + kx^2) / k
        else if (dkind == kSurfDzDxDzDz) c2 = chop, c6 = chop;    // chop kz (kx + i kz) / k
        else c3 = -1.f, c4 = kx;                                  // -kz + i kx
        const float kx2 = kx * kx;
        fft::cta_fft<N, true, false, false, true, 0, 0, (fft::Plan<N>::P > 1)>(
            t, buf, stw,
            [&](int j) {
              const int jj = j ^ H;
              const float2 h = sht[rr * N + jj];
              const float kz = dk * (float)(jj - N / 2);
              float inv;
              if constexpr (SURF_INV_INLINE) {
                const float k2 = fmaf(kz, kz, kx2);
                inv = k2 > 0.f ? rsqrtf(k2) : 0.f;
              } else {
                inv = sinv[rr * N + jj];
              }
              const float mr = fmaf(inv * kx, fmaf(c2, kz, c1), fmaf(c3, kz, c0));
              const float mi = fmaf(inv, fmaf(c6 * kz, kz, c5 * (kz + kx2)), c4);
              return make_float2(h.x * mr - h.y * mi, h.x * mi + h.y * mr);
            },
            store, fft::NoHook{}, edge_row);
      } else {
        static_assert(MODE == kRowVelocity, "row mode");
        // velocity: Z (re + i im) with Z = V0 (x/z pair) or W0 (vy pair);
        // E(y) = 1 + |k| y above the mean surface, else exp(|k| y) (selected,
        // not branched: the depth is per transform)
        const float2* Z = dkind == kVelXZ ? sv0 : sw0;
        constexpr float kLog2e = 1.4426950408889634f;
        const float y0 = dcur.y, y1 = dcur.z, y0l = y0 * kLog2e, y1l = y1 * kLog2e;
        const bool up0 = y0 > 0.f, up1 = y1 > 0.f;
        auto run = [&](auto kind_c) {
          constexpr int KIND = decltype(kind_c)::value;
          fft::cta_fft<N, true, false, false, true, 0, 0, (fft::Plan<N>::P > 1)>(
              t, buf, stw,
              [&](int j) {
                const int jj = j ^ H;
                const float2 z = Z[jj];
                const float k = sk[jj];
                const float l0 = fmaf(k, y0, 1.0f), x0 = ex2_approx(k * y0l);
                const float e0 = up0 ? l0 : x0;
                if constexpr (KIND == kVelXZ) {
                  return make_float2(z.x * e0, z.y * e0);
                } else if constexpr (KIND == kVelYPair) {
                  const float l1 = fmaf(k, y1, 1.0f), x1 = ex2_approx(k * y1l);
                  const float mr = -(up1 ? l1 : x1), mi = e0;
                  return make_float2(z.x * mr - z.y * mi, z.x * mi + z.y * mr);
                } else {
                  return make_float2(-z.y * e0, z.x * e0);
                }
              },
              store, fft::NoHook{}, edge_row);
        };
        switch (dkind) {
          case kVelXZ: run(std::integral_constant<int, kVelXZ>{}); break;
          case kVelYPair: run(std::integral_constant<int, kVelYPair>{}); break;
          default: run(std::integral_constant<int, kVelYSingle>{}); break;
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ columns

template <int N, bool COMPLEX_OUT>
__global__ void __launch_bounds__(Launch<N>::THREADS) k_cols(const ColArgs a) {
  using L = Launch<N>;
  extern __shared__ float2 smem[];
  const int c = threadIdx.x % L::PER_CTA;  // column within the tile (fastest)
  const int t = threadIdx.x / L::PER_CTA;
  const int col = blockIdx.x * L::PER_CTA + c;
  const int xf = blockIdx.y;
  const bool valid = col < N;
  float2* sm = smem + c * L::COL_STRIDE;
  const float2* in = a.scratch + (size_t)xf * N * N + (valid ? col : 0);
  if constexpr (COMPLEX_OUT) {
    float2* out = a.out_c + (size_t)xf * N * N;
    fft::cta_fft<N>(
        t, sm, a.tw, [&](int i) { return __ldg(in + (size_t)i * N); },
        [&](int r, float2 x) {
          if (!valid) return;
          out[(size_t)r * N + col] = x;
        });
  } else {
    const XformDesc d = a.desc[xf];
    fft::cta_fft<N>(
        t, sm, a.tw, [&](int i) { return __ldg(in + (size_t)i * N); },
        [&](int r, float2 x) {
          if (!valid) return;
          // streaming stores: the fields are not re-read by this step
          __stcs(d.out_re + (size_t)r * N + col, x.x);  // fft.cpp:93-99 split
          if (d.out_im) __stcs(d.out_im + (size_t)r * N + col, x.y);
        });
  }
}

// Column pass, persistent and TMA-fed (128 <= N <= 4096). A CTA walks the
// column tiles [N rows][PC columns] (tile = transform x column block) with a
// ring of STAGES shared buffers: one elected thread keeps STAGES - 1 tiles in
// flight with one 4-D cp.async.bulk.tensor load each (completion on an
// mbarrier) while the CTA transforms the landed tile in place (dense
// [row][column] layout read by pass 0, padded per-column layout for the
// exchange) and refills the buffer as soon as its last shared reads are done.
// Twiddles live in shared memory. The epilogue splits Re / Im: by default into
// shared staging planes written out by TMA stores (2 load stages fit beside
// them), otherwise with evict-first stores from the warps (3 load stages).
// Measured on B200 (config 3): 8-column tiles with one CTA per SM beat a
// 4-column ring with 2 CTAs / SM (1.36 vs 2.06 ms spectral per frame).
template <int N>
struct ColTma {
  using PL = fft::Plan<N>;
  static constexpr int T = PL::T;
  static constexpr int THREADS = T > 256 ? T : 256;
  static constexpr int PC = THREADS / T;  // columns per tile
  static constexpr int STRIDE = fft::col_stride(PL::SMEM, PC);
  static constexpr int DENSE = N * PC;  // float2 per tile
  static constexpr int PADDED = PC * STRIDE;
  static constexpr int STAGE = ((DENSE > PADDED ? DENSE : PADDED) + 15) / 16 * 16;
  static constexpr int TW = PL::tw_size();
  static constexpr int STAGES = (227 * 1024 - TW * 8 - 64) / (STAGE * 8) >= 3 ? 3 : 2;
  static constexpr uint32_t TILE_BYTES = (uint32_t)DENSE * 8;
  static constexpr size_t smem(int stages, bool tma_store = false) {
    return ((size_t)stages * STAGE + (tma_store ? DENSE : 0) + TW) * 8 + stages * 8;
  }
  static constexpr size_t SMEM = smem(STAGES);
  static constexpr int BR = N < 256 ? N : 256;  // rows per box dimension
  static constexpr bool OK = PL::P > 1 && N >= 128 && N <= 4096 && SMEM <= 227 * 1024;
};

// columns per tile of the TMA column kernel, 0 outside its range
int cols_tma_pc(int n) { return n >= 128 && n <= 4096 ? 8192 / n : 0; }

// TMA_STORE (split mode): the final pass writes Re / Im into fp32 staging
// planes and one elected thread stores them with two tiled TMA stores (no STG
// from the warps); the staging is reused once the previous tile's stores have
// read it (cp.async.bulk.wait_group.read in the refill point).
// Band-limited grids (GridConst::row_half, a.gc != nullptr): only the scratch
// rows that can be nonzero are loaded, as 32-row chunks through `src_chunk`;
// the others are exactly zero (the row pass skipped them) and pass 0 reads
// them as zero. Scratch row r holds spectrum row r ^ N/2, so the nonzero rows
// are [0, row_half) and (N - row_half, N).
// WARP_STORE (with TMA_STORE): every warp stores its own outputs -- thread t
// of column c ends with rows t + T r', so a warp's outputs are one 3-D box
// {PC, 32 / PC, 32} of the plane viewed as [N / T][T][N] (plane_warp_map_for)
// -- from its own 8 KB of the staging, after a per-thread fence and a
// __syncwarp: no CTA barrier and no CTA-wide fence in the epilogue.
template <int N, bool COMPLEX_OUT, int S, bool TMA_STORE = false, bool WARP_STORE = false>
__global__ void __launch_bounds__(ColTma<N>::THREADS, 1)
    k_cols_tma(const __grid_constant__ CUtensorMap src, const __grid_constant__ CUtensorMap src_chunk,
               const ColArgs a, int tiles_x, int ntiles) {
  using CT = ColTma<N>;
  constexpr int PC = CT::PC;
  constexpr int H = N / 2, CH = 32, NCH = N / CH;  // 32-row chunks
  auto row_half_of = [&](int xf) {
    const int rh = a.gc ? __ldg(&a.desc[xf].row_half) : 0;
    return rh > 0 ? rh : H + 1;
  };
  extern __shared__ __align__(128) float2 smem[];
  float* sre = reinterpret_cast<float*>(smem + S * CT::STAGE);  // TMA_STORE staging
  float* sim = sre + CT::DENSE;
  float2* stw = smem + S * CT::STAGE + (TMA_STORE ? CT::DENSE : 0);
  const uint32_t bar0 = tma::smem_u32(stw + CT::TW);
  const int c = threadIdx.x % PC, t = threadIdx.x / PC;
  auto issue = [&](int tile, int s) {
    const int xf = tile / tiles_x, col0 = (tile - xf * tiles_x) * PC;
    const int rh = row_half_of(xf);
    const int lo = (rh + CH - 1) / CH;        // chunks [0, lo) hold rows [0, rh)
    const int hi = (N - rh + 1) / CH;         // chunks [hi, NCH) hold rows (N - rh, N)
    if (rh > H || lo >= hi) {
      tma::mbar_arrive_expect_tx(bar0 + 8 * s, CT::TILE_BYTES);
      tma::load_4d(tma::smem_u32(smem + s * CT::STAGE), &src, 2 * col0, 0, 0, xf, bar0 + 8 * s);
    } else {
      const int nch = lo + (NCH - hi);
      tma::mbar_arrive_expect_tx(bar0 + 8 * s, (uint32_t)nch * CH * PC * 8);
      for (int k = 0; k < NCH; ++k) {
        if (k >= lo && k < hi) continue;
        tma::load_4d(tma::smem_u32(smem + s * CT::STAGE + k * CH * PC), &src_chunk, 2 * col0, 0, k,
                     xf, bar0 + 8 * s);
      }
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) tma::mbar_init(bar0 + 8 * s, 1);
    tma::fence_mbar_init();
    for (int s = 0; s < S; ++s) {
      const int tile = blockIdx.x + s * gridDim.x;
      if (tile < ntiles) issue(tile, s);
    }
  }
  for (int i = threadIdx.x; i < CT::TW; i += CT::THREADS) stw[i] = __ldg(a.tw + i);
  __syncthreads();
  int s = 0;
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int xf = tile / tiles_x;
    const int col = (tile - xf * tiles_x) * PC + c;
    float2* buf = smem + s * CT::STAGE;
    tma::mbar_wait(bar0 + 8 * s, phase);
    auto refill = [&] {
      if (TMA_STORE && (WARP_STORE ? (threadIdx.x & 31) == 0 : threadIdx.x == 0))
        tma::bulk_wait_read();  // staging free again
      __syncthreads();  // every thread's shared reads of this buffer are done
      if (threadIdx.x == 0) {
        const int next = tile + S * gridDim.x;
        if (next < ntiles) {
          tma::fence_proxy_async_smem();
          issue(next, s);
        }
      }
    };
    const float2* dense = buf;
    const int rh = row_half_of(xf);
    const bool edge_only = rh <= N / 32;  // band within the first / last T rows
    // pass-0 element i of column `col`: zero outside the band rows
    auto load_band = [&](int i) {
      return abs((i ^ H) - H) < rh ? dense[i * PC + c] : make_float2(0.f, 0.f);
    };
    if constexpr (COMPLEX_OUT) {
      float2* out = a.out_c + (size_t)xf * N * N;
      fft::cta_fft<N, false, true, false, true, 0, 0, true>(
          t, buf + c * CT::STRIDE, stw, load_band,
          [&](int r, float2 x) {
            out[(size_t)r * N + col] = x;
          },
          refill, edge_only);
    } else if constexpr (TMA_STORE && WARP_STORE) {
      constexpr int T = CT::T;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      float* my_re = sre + warp * 1024;  // 32 r' x 32 lanes
      float* my_im = sim + warp * 1024;
      fft::cta_fft<N, false, true, false, true, 0, 0, true>(
          t, buf + c * CT::STRIDE, stw, load_band,
          [&](int r, float2 x) {
            my_re[(r / T) * 32 + lane] = x.x;  // box order {c, t, r'}; fft.cpp:93-99 split
            my_im[(r / T) * 32 + lane] = x.y;
          },
          refill, edge_only);
      tma::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int col0 = col - c, t0 = (warp * 32) / PC;
        tma::store_3d(a.out_maps + 2 * xf, tma::smem_u32(my_re), col0, t0, 0);
        if (a.desc[xf].out_im) tma::store_3d(a.out_maps + 2 * xf + 1, tma::smem_u32(my_im), col0, t0, 0);
        tma::bulk_commit();
      }
    } else if constexpr (TMA_STORE) {
      fft::cta_fft<N, false, true, false, true, 0, 0, true>(
          t, buf + c * CT::STRIDE, stw, load_band,
          [&](int r, float2 x) {
            sre[r * PC + c] = x.x;  // fft.cpp:93-99 split
            sim[r * PC + c] = x.y;
          },
          refill, edge_only);
      tma::fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int col0 = col - c;
        tma::store_3d(a.out_maps + 2 * xf, tma::smem_u32(sre), col0, 0, 0);
        if (a.desc[xf].out_im) tma::store_3d(a.out_maps + 2 * xf + 1, tma::smem_u32(sim), col0, 0, 0);
        tma::bulk_commit();
      }
    } else {
      const XformDesc d = a.desc[xf];
      fft::cta_fft<N, false, true, false, true, 0, 0, true>(
          t, buf + c * CT::STRIDE, stw, load_band,
          [&](int r, float2 x) {
            __stcs(d.out_re + (size_t)r * N + col, x.x);  // fft.cpp:93-99 split
            if (d.out_im) __stcs(d.out_im + (size_t)r * N + col, x.y);
          },
          refill, edge_only);
    }
    if (++s == S) s = 0, phase ^= 1;
  }
  if (TMA_STORE && (WARP_STORE ? (threadIdx.x & 31) == 0 : threadIdx.x == 0)) tma::bulk_wait();
}

// fp64 interleaved pair -> fp32 X + iY (fft.cpp:88-91)
__global__ void k_pack_pair(size_t nn, const double2* x, const double2* y, float2* out) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < nn;
       q += (size_t)gridDim.x * blockDim.x) {
    const double2 a = x[q];
    const double2 b = y ? y[q] : make_double2(0.0, 0.0);
    out[q] = make_float2((float)(a.x - b.y), (float)(a.y + b.x));
  }
}

__global__ void k_f32_to_f64(size_t n, const float* in, double* out) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x)
    out[q] = (double)in[q];
}

__global__ void k_c32_to_c64(size_t n, const float2* in, double2* out) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x)
    out[q] = make_double2(in[q].x, in[q].y);
}

