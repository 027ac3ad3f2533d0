// slab.cu — one very large surface grid split across ranks (SURVEY 8d/8e
// config 5): rank r owns spectrum rows [r R, (r+1) R), R = N / ranks.
//
//   ocn_slab_rows : evolve the owned rows (h0 of the owned rows and of their
//                   mirror rows -i are generated locally: the counter-based
//                   Philox makes h0(i, j) a pure function of (i, j), so no
//                   exchange is needed for conj(h0(-k))), build the 4 packed
//                   surface coefficients (surface.cpp:77-80 pairs) and run the
//                   row FFTs; the result is written straight into the all-to-all
//                   send layout [dest][pair][row][col in dest's column slab].
//   (caller)      : all-to-all of the N/ranks x N/ranks tiles (NCCL over
//                   NVLink: torch.distributed.all_to_all_single in bench.py).
//   ocn_slab_cols : column FFTs of the owned column slab from the receive
//                   layout [src][pair][row][col], (-1)^(i+j), Re/Im split into
//                   8 fp32 fields kept in the transposed (column-slab) layout.
//                   For N >= 4096 a column (N x 8 B) is too long to stage
//                   several of them in shared memory, and one column per CTA
//                   reads one 8-byte element per 32-byte sector; the pass is
//                   then a four-step FFT over N = N1 x 128 on 8-column tiles:
//                   k_slab_colsA: length-N1 DFTs over rows i1 * 128 + i2
//                   (fixed i2), twiddle w_N^(i2 k1), written back in place;
//                   k_slab_colsB: length-128 DFTs over the contiguous rows
//                   k1 * 128 + i2, output row k1 + N1 k2, sign and split.
#include <algorithm>
#include <cmath>
#include <memory>

#include "fft_core.cuh"
#include "objects.cuh"
#include "spectrum_math.cuh"

struct ocn_slab {
  ocn_ctx* ctx = nullptr;
  int n = 0, ranks = 1, rank = 0, rows = 0, cols = 0;
  ocn::GridConst gc{};
  ocn::DevBuf<float2> h0, h0m;   // [rows][N]: h0 of owned rows, h0 of rows neg(i)
  ocn::DevBuf<float2> spec;      // [rows][N]: h~ (the slab builds surface fields only)
  ocn::DevBuf<float2> twiddle;
  ocn::DevBuf<float2> tw1, tw2, wn;  // four-step column pass: inner tables, w_N^m
  ocn::DevBuf<float2> tw128, w_hi, w_lo;  // four-step row pass (N = 16384): w_N^(128 h), w_N^l
  ocn::DevBuf<double> d_time;
  ocn::DevBuf<float> fields;     // [8][N][cols]
  ocn::DevBuf<float2> ring;      // fused four-step columns: step A results, kFsRing column blocks
  ocn::DevBuf<int> fs_sync;      // fused four-step columns: dispatch counter, per-block A / B counts
};

namespace ocn {
namespace {

constexpr int kSlabThreads = 256;

template <int N>
using SlabLaunch = fft::CtaLaunch<N, kSlabThreads>;

// h0 at (i, j) (spectra.cpp:150-169), fp64, same math as K1
__device__ double2 h0_mode(const GridConst& G, int n, int i, int j) {
  const double dk = G.dk;
  const double kx = dk * (i - n / 2), kz = dk * (j - n / 2);
  const double k = sm::hypot_ref(kx, kz);
  const double omega = sqrt(G.p.gravity * k);
  if (!(k > 0.0 && k >= G.band_min && k < G.band_max)) return make_double2(0.0, 0.0);
  double gr, gi;
  sm::gaussian_complex(G.p.rng_seed, G.cindex, (uint32_t)i, (uint32_t)j, &gr, &gi);
  const double amp = sqrt(sm::h0_variance(kx, kz, k, omega, G.length, G.p));
  return make_double2(gr * amp, gi * amp);
}

__global__ void k_slab_init(int n, int row0, int rows, GridConst G, float2* h0, float2* h0m) {
  const size_t total = (size_t)rows * n;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
       q += (size_t)gridDim.x * blockDim.x) {
    const int li = (int)(q / n), j = (int)(q % n);
    const int i = row0 + li, ni = i == 0 ? 0 : n - i;
    const double2 a = h0_mode(G, n, i, j), b = h0_mode(G, n, ni, j);
    h0[q] = make_float2((float)a.x, (float)a.y);
    h0m[q] = make_float2((float)b.x, (float)b.y);
  }
}

// sqrt in fp64 from the fp32 MUFU estimate plus one Newton step (relative
// error ~1e-14, ~5 instructions against the ~20 of the IEEE fp64 sqrt): the
// dispersion w = sqrt(g |k|) only enters the fp64 phase w t, where 1e-14 of
// ~1e2 rad is far below the fp32 sincos it feeds
__device__ __forceinline__ double sqrt_nr(double x) {
  if (!(x > 0.0)) return 0.0;
  const double r = (double)rsqrtf((float)x);
  const double y = x * r;
  return fma(0.5 * r, fma(-y, y, x), y);
}

// h~ (surface.cpp:49-50) of the owned rows; conj(h0(-k)) from the mirror rows
__global__ void __launch_bounds__(256) k_slab_evolve(int logn, int row0, int rows, GridConst G,
                                                     const double* d_time,
                                                     const float2* __restrict__ h0,
                                                     const float2* __restrict__ h0m,
                                                     float2* spec) {
  const int n = 1 << logn;
  const size_t total = (size_t)rows << logn;
  const double t = *d_time;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
       q += (size_t)gridDim.x * blockDim.x) {
    const int li = (int)(q >> logn), j = (int)(q & (n - 1));
    const int i = row0 + li, nj = j == 0 ? 0 : n - j;
    const float2 a = __ldcs(h0 + q);
    const float2 m = __ldcs(h0m + ((size_t)li << logn) + nj);
    const float2 b = make_float2(m.x, -m.y);
    const double kx = G.dk * (i - n / 2), kz = G.dk * (j - n / 2);
    const double omega = sqrt_nr(G.p.gravity * sqrt_nr(kx * kx + kz * kz));
    double ph = omega * t;
    ph -= 6.283185307179586476925 * rint(ph * 0.15915494309189533577);
    float s, c;
    sincosf((float)ph, &s, &c);
    const float ar = a.x * c - a.y * s, ai = a.x * s + a.y * c;
    const float br = b.x * c + b.y * s, bi = b.y * c - b.x * s;
    spec[q] = make_float2(ar + br, ai + bi);
  }
}

struct SlabRowArgs {
  int row0, rows, cols;
  float dk, chop;
  const float2* spec;
  float2* send;  // [dest][4][rows][cols]
  const float2* tw;
  int p0, np;    // packed pairs [p0, p0 + np) of this launch
};

// packed surface pair p at mode (i, j): h~ M_p (surface.cpp:77-80)
__device__ __forceinline__ float2 surface_pair(int p, float2 s, float kx, float kz, float chop) {
  const float k2 = kx * kx + kz * kz;
  if (k2 == 0.f) return make_float2(0.f, 0.f);
  const float inv = rsqrtf(k2);
  float mr, mi;
  if (p == 0) mr = 1.0f - kx * inv * chop, mi = 0.f;
  else if (p == 1) mr = 0.f, mi = chop * (kz + kx * kx) * inv;
  else if (p == 2) mr = chop * kz * inv * kx, mi = chop * kz * inv * kz;
  else mr = -kz, mi = kx;
  return make_float2(s.x * mr - s.y * mi, s.x * mi + s.y * mr);
}

template <int N>
__global__ void __launch_bounds__(SlabLaunch<N>::THREADS) k_slab_rows(const SlabRowArgs a) {
  using L = SlabLaunch<N>;
  extern __shared__ float2 smem[];
  const int local = threadIdx.x / L::T, t = threadIdx.x - local * L::T;
  const int item = blockIdx.x * L::PER_CTA + local;  // (row, pair)
  const bool valid = item < a.rows * a.np;
  const int li = valid ? item / a.np : 0, p = a.p0 + item % a.np;
  const float kx = a.dk * (float)(a.row0 + li - N / 2);
  const float2* srow = a.spec + (size_t)li * N;
  // surface_pair as one branch-free form with per-pair constants (as k_rows_w):
  //   Re M = c0 + c3 kz + kx / |k| (c1 + c2 kz),  Im M = c4 + (c5 (kz + kx^2) + c6 kz^2) / |k|
  const float chop = a.chop, kx2 = kx * kx;
  float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, c5 = 0.f, c6 = 0.f;
  if (p == 0) c0 = 1.f, c1 = -chop;
  else if (p == 1) c5 = chop;
  else if (p == 2) c2 = chop, c6 = chop;
  else c3 = -1.f, c4 = kx;
  const int cols_log2 = __ffs(a.cols) - 1;  // cols = N / ranks, a power of two
  fft::cta_fft<N>(
      t, smem + local * L::ROW_STRIDE, a.tw,
      [&](int j) {
        if (!valid) return make_float2(0.f, 0.f);
        const float2 h = __ldg(srow + j);
        const float kz = a.dk * (float)(j - N / 2);
        const float k2 = fmaf(kz, kz, kx2);
        const float inv = k2 > 0.f ? rsqrtf(k2) : 0.f;
        const float mr = fmaf(inv * kx, fmaf(c2, kz, c1), fmaf(c3, kz, c0));
        const float mi = fmaf(inv, fmaf(c6 * kz, kz, c5 * (kz + kx2)), c4);
        return make_float2(h.x * mr - h.y * mi, h.x * mi + h.y * mr);
      },
      [&](int k, float2 x) {
        if (!valid) return;
        const int dest = k >> cols_log2, kc = k & (a.cols - 1);
        a.send[(((size_t)dest * 4 + p) * a.rows + li) * a.cols + kc] = x;
      });
}

// Row pass for N = 16384 = 128 x 128: one 512-thread CTA per (row, pair), the
// row's FFT as a four-step inside shared memory with warp-synchronous
// 128-point FFTs (4 threads each) -- two CTA barriers per row instead of the
// generic 3-pass CTA FFT's four, and every twiddle from shared memory:
//   step 1 (group g = i2): Y[k1] = sum_i1 x[128 i1 + i2] w_128^(i1 k1), times
//          w_N^(i2 k1) (= hi[m >> 7] lo[m & 127], m = i2 k1), written
//          transposed to X[k1][i2];
//   step 2 (group g = k1, in place): out[k1 + 128 k2] = sum_i2 X[k1][i2] w_128^(i2 k2).
// x[j] is the packed coefficient of the pair at mode (row, j) (surface.cpp:77-80),
// generated in step 1's loads from h~ (as k_slab_rows).
constexpr int kRow4sThreads = 512;
template <int N>
__global__ void __launch_bounds__(kRow4sThreads, 1)
    k_slab_rows_4s(const SlabRowArgs a, const float2* __restrict__ tw128,
                   const float2* __restrict__ w_hi, const float2* __restrict__ w_lo) {
  constexpr int M = 128;
  static_assert(N == M * M, "four-step row pass is for N = 16384");
  using PL = fft::Plan<M>;
  constexpr int T = PL::T, S = PL::SMEM;
  extern __shared__ float2 smem[];
  float2* X = smem;              // [128][S]
  float2* stw = X + M * S;       // Plan<128> twiddles
  float2* hi = stw + PL::tw_size();
  float2* lo = hi + M;
  for (int i = threadIdx.x; i < PL::tw_size(); i += kRow4sThreads) stw[i] = __ldg(tw128 + i);
  for (int i = threadIdx.x; i < M; i += kRow4sThreads) hi[i] = __ldg(w_hi + i), lo[i] = __ldg(w_lo + i);
  const int li = blockIdx.x / a.np, p = a.p0 + blockIdx.x % a.np;
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const float kx = a.dk * (float)(a.row0 + li - N / 2);
  const float2* srow = a.spec + (size_t)li * N;
  const float chop = a.chop, kx2 = kx * kx;
  float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, c5 = 0.f, c6 = 0.f;
  if (p == 0) c0 = 1.f, c1 = -chop;
  else if (p == 1) c5 = chop;
  else if (p == 2) c2 = chop, c6 = chop;
  else c3 = -1.f, c4 = kx;
  __syncthreads();  // tables staged
  // step 1: the 128 DFTs over i1 (stride-128 elements), group g = i2
  fft::cta_fft<M, true, false, false, true>(
      t, X + g * S, stw,
      [&](int i1) {
        const int j = M * i1 + g;
        const float2 h = __ldg(srow + j);
        const float kz = a.dk * (float)(j - N / 2);
        const float k2 = fmaf(kz, kz, kx2);
        const float inv = k2 > 0.f ? rsqrtf(k2) : 0.f;
        const float mr = fmaf(inv * kx, fmaf(c2, kz, c1), fmaf(c3, kz, c0));
        const float mi = fmaf(inv, fmaf(c6 * kz, kz, c5 * (kz + kx2)), c4);
        return make_float2(h.x * mr - h.y * mi, h.x * mi + h.y * mr);
      },
      [&](int k1, float2 y) {
        const int m = g * k1;
        X[k1 * S + g] = fft::cmul(y, fft::cmul(hi[m >> 7], lo[m & (M - 1)]));
      },
      [] { __syncthreads(); });  // every group's exchange reads done: X may be overwritten
  __syncthreads();
  // step 2: the 128 DFTs over i2 (rows of X), group g = k1, in place
  const int cols_log2 = __ffs(a.cols) - 1;
  fft::cta_fft<M, true, true, false, true>(
      t, X + g * S, stw, [&](int i2) { return X[g * S + i2]; },
      [&](int k2, float2 x) {
        const int k = g + M * k2;
        const int dest = k >> cols_log2, kc = k & (a.cols - 1);
        a.send[(((size_t)dest * 4 + p) * a.rows + li) * a.cols + kc] = x;
      });
}

struct SlabColArgs {
  int rows, cols, col0;
  int rows_log2;  // rows = N / ranks is a power of two
  const float2* recv;  // [src][4][rows][cols]
  float* fields;       // [8][N][cols]
  const float2* tw;
  int p0;              // first packed pair of this launch (grid y / z = pairs)
};

template <int N>
__global__ void __launch_bounds__(SlabLaunch<N>::THREADS) k_slab_cols(const SlabColArgs a) {
  using L = SlabLaunch<N>;
  extern __shared__ float2 smem[];
  const int c = threadIdx.x % L::PER_CTA, t = threadIdx.x / L::PER_CTA;
  const int p = a.p0 + blockIdx.y;
  const int kc = blockIdx.x * L::PER_CTA + c;
  const bool valid = kc < a.cols;
  const int col = a.col0 + (valid ? kc : 0);
  float* re = a.fields + (size_t)(2 * p) * N * a.cols;
  float* im = a.fields + (size_t)(2 * p + 1) * N * a.cols;
  fft::cta_fft<N>(
      t, smem + c * L::COL_STRIDE, a.tw,
      [&](int i) {
        if (!valid) return make_float2(0.f, 0.f);
        const int src = i >> a.rows_log2, li = i & (a.rows - 1);
        return __ldg(a.recv + (((size_t)src * 4 + p) * a.rows + li) * a.cols + kc);
      },
      [&](int i, float2 x) {
        if (!valid) return;
        const float s = ((i + col) & 1) ? -1.f : 1.f;  // fft.cpp:73-75
        re[(size_t)i * a.cols + kc] = s * x.x;         // fft.cpp:93-99
        im[(size_t)i * a.cols + kc] = s * x.y;
      });
}

// ---------------------------------------------------------------- four-step columns
// Stride between the 64 transform buffers of a four-step CTA: the FFT's own
// (conflict-free for its exchanges); an odd stride, which spreads the
// cooperative column-major tile loads over more banks, measured slower (config 5
// 18.7 vs 17.4 ms).
template <int SMEM>
constexpr int kFsStride = SMEM;
constexpr int kFsN2 = 128;  // inner length of the second step
constexpr int kFsPC = 32;   // columns per tile (256-byte row segments: DRAM page locality)
constexpr int kFsB = 2;     // i2 (step A) or k1 (step B) values per CTA (64 transforms)

// element (row i, column kc) of pair p in the receive layout [src][4][R][R]:
// ((src 4 + p) R + li) cols + kc = (i + 3 R src) cols + (p R cols + kc)
__device__ __forceinline__ size_t recv_index(const SlabColArgs& a, int p, int i, int kc) {
  const int src = i >> a.rows_log2;
  return (size_t)(i + 3 * a.rows * src) * a.cols + ((size_t)p * a.rows * a.cols + kc);
}

// step A: for each i2 of the tile, Y[k1] = sum_i1 x[128 i1 + i2] w_N1^(i1 k1),
// times w_N^(i2 k1), stored back at row 128 k1 + i2 (the same rows)
template <int N>
__global__ void __launch_bounds__(kFsB * kFsPC * (N / kFsN2) / 32) k_slab_colsA(const SlabColArgs a, float2* recv,
                                                             const float2* __restrict__ tw1,
                                                             const float2* __restrict__ wn) {
  constexpr int N1 = N / kFsN2, NT = kFsB * kFsPC;
  using PL = fft::Plan<N1>;
  constexpr int T = PL::T, TPW = 32 / T, S = kFsStride<PL::SMEM>;
  extern __shared__ float2 smem[];  // [NT][S]
  const int p = a.p0 + blockIdx.z, kc0 = blockIdx.x * kFsPC, i20 = blockIdx.y * kFsB;
  // each thread moves one (column, i2) lane: fixed across the rows it visits
  constexpr int STEP = kFsB * kFsPC * N1 / 32 / NT;  // i1 per iteration (blockDim / NT)
  const int c = threadIdx.x % kFsPC, i2l = (threadIdx.x / kFsPC) % kFsB, i10 = threadIdx.x / NT;
  float2* lane_sm = smem + (i2l * kFsPC + c) * S;
#pragma unroll 8
  for (int i1 = i10; i1 < N1; i1 += STEP)
    lane_sm[fft::pad32(i1)] = __ldg(recv + recv_index(a, p, kFsN2 * i1 + i20 + i2l, kc0 + c));
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tr = warp * TPW + lane / T, t = lane % T;
  float2* buf = smem + tr * S;
  const int i2 = i20 + tr / kFsPC;
  fft::cta_fft<N1, true, true, true>(
      t, buf, tw1, [&](int n) { return buf[fft::pad32(n)]; },
      [&](int k1, float2 x) { buf[fft::pad32(k1)] = fft::cmul(x, __ldg(wn + i2 * k1)); });
  __syncthreads();
#pragma unroll 8
  for (int k1 = i10; k1 < N1; k1 += STEP)
    recv[recv_index(a, p, kFsN2 * k1 + i20 + i2l, kc0 + c)] = lane_sm[fft::pad32(k1)];
}

// step B: for each k1 of the tile, X[k1 + N1 k2] = sum_i2 Y[128 k1 + i2] w_128^(i2 k2);
// (-1)^(k + col) and the Re / Im split into the field planes
template <int N>
__global__ void __launch_bounds__(kFsB * kFsPC * kFsN2 / 32) k_slab_colsB(const SlabColArgs a, const float2* recv,
                                                        const float2* __restrict__ tw2) {
  constexpr int N1 = N / kFsN2, NT = kFsB * kFsPC;
  using PL = fft::Plan<kFsN2>;
  constexpr int T = PL::T, TPW = 32 / T, S = kFsStride<PL::SMEM>;
  extern __shared__ float2 smem[];  // [NT][S]
  const int p = a.p0 + blockIdx.z, kc0 = blockIdx.x * kFsPC, k10 = blockIdx.y * kFsB;
  constexpr int STEP = kFsB * kFsPC * kFsN2 / 32 / NT;
  const int c = threadIdx.x % kFsPC, k1l = (threadIdx.x / kFsPC) % kFsB, i20 = threadIdx.x / NT;
  float2* lane_sm = smem + (k1l * kFsPC + c) * S;
  const float2* lane_src = recv + recv_index(a, p, kFsN2 * (k10 + k1l), kc0 + c);
  // rows 128 (k10 + k1l) + i2 stay inside one source block (R >= 128)
#pragma unroll 8
  for (int i2 = i20; i2 < kFsN2; i2 += STEP) lane_sm[fft::pad32(i2)] = __ldg(lane_src + (size_t)i2 * a.cols);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tr = warp * TPW + lane / T, t = lane % T;
  float2* buf = smem + tr * S;
  fft::cta_fft<kFsN2, true, true, true>(
      t, buf, tw2, [&](int n) { return buf[fft::pad32(n)]; },
      [&](int k2, float2 x) { buf[fft::pad32(k2)] = x; });
  __syncthreads();
  float* re = a.fields + (size_t)(2 * p) * N * a.cols;
  float* im = a.fields + (size_t)(2 * p + 1) * N * a.cols;
  const int kc = kc0 + c;
#pragma unroll 8
  for (int k2 = i20; k2 < kFsN2; k2 += STEP) {
    const int k = k10 + k1l + N1 * k2;
    const float2 x = lane_sm[fft::pad32(k2)];
    const float sg = ((k + a.col0 + kc) & 1) ? -1.f : 1.f;  // fft.cpp:73-75
    __stcs(re + (size_t)k * a.cols + kc, sg * x.x);          // fft.cpp:93-99
    __stcs(im + (size_t)k * a.cols + kc, sg * x.y);
  }
}

// ---------------------------------------------------------------- fused four-step columns
// Steps A and B of the four-step column pass in ONE persistent kernel over a
// work list ordered by 32-column block: the block's N1 / kFsB... A items (pairs
// of i2, as k_slab_colsA) then its B items (pairs of k1, as k_slab_colsB). A
// writes its results to a ring of kFsRing block slots instead of back into
// `recv`; B reads them from there. A block's intermediate (N x 32 x 8 B, 4 MB at
// N = 16384) is consumed while it is still in L2 and the ring slot is
// overwritten before its lines are evicted: the column pass moves recv once and
// the fields once instead of recv three times and the fields once.
//   B items of block b wait until A_done[b] = nA (A never waits for B of its
//   own block); A items of block b >= kFsRing wait, before writing, until
//   B_done[b - kFsRing] = nB (that slot's readers are done). Items are taken
//   in list order (one atomic per item), so every item waits only on items
//   taken earlier: no deadlock whatever the residency.
constexpr int kFsRing = 8;
constexpr int kFsLag = 3;  // B items of a block run this many blocks after its A items

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const int* p, int target) {
  while (ld_acquire(p) < target) __nanosleep(64);
}

template <int N>
__global__ void __launch_bounds__(kFsB * kFsPC * kFsN2 / 32) k_slab_cols_fused(
    const SlabColArgs a, const float2* __restrict__ recv, float2* ring, int* sync, int nblocks,
    const float2* __restrict__ tw1, const float2* __restrict__ wn, const float2* __restrict__ tw2) {
  constexpr int N1 = N / kFsN2, NT = kFsB * kFsPC;
  constexpr int nA = kFsN2 / kFsB, nB = N1 / kFsB, PER = nA + nB;
  static_assert(kFsB * kFsPC * N1 / 32 == kFsB * kFsPC * kFsN2 / 32 || N1 <= kFsN2,
                "step A uses at most the CTA's threads");
  constexpr int THREADS = kFsB * kFsPC * kFsN2 / 32;
  constexpr int THREADS_A = kFsB * kFsPC * N1 / 32;
  constexpr size_t SLOT = (size_t)N * kFsPC;  // float2 per ring slot
  extern __shared__ float2 smem[];
  __shared__ int s_item;
  int* dispatch = sync;
  int* a_done = sync + 1;
  int* b_done = sync + 1 + nblocks;
  const int ncb = a.cols / kFsPC;
  // work list by step st: A items of block st, then B items of block st - kFsLag
  // (B of a block is taken kFsLag blocks after its A items, which are then long
  // done: no spinning on a block still being produced)
  const int total = (nblocks + kFsLag) * PER;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(dispatch, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= total) return;
    const int st = item / PER, r = item - st * PER;
    const int blk = r < nA ? st : st - kFsLag;
    if (blk < 0 || blk >= nblocks) {
      __syncthreads();  // s_item is rewritten by the next iteration
      continue;
    }
    const int p = a.p0 + blk / ncb, kc0 = (blk % ncb) * kFsPC;
    float2* slot = ring + (size_t)(blk % kFsRing) * SLOT;
    if (r < nA) {
      // ---- step A (k_slab_colsA): i2 = 2 r, 2 r + 1
      using PL = fft::Plan<N1>;
      constexpr int T = PL::T, TPW = 32 / T, S = kFsStride<PL::SMEM>;
      constexpr int STEP = THREADS_A / NT;
      const int i20 = r * kFsB;
      if (threadIdx.x < THREADS_A) {
        const int c = threadIdx.x % kFsPC, i2l = (threadIdx.x / kFsPC) % kFsB, i10 = threadIdx.x / NT;
        float2* lane_sm = smem + (i2l * kFsPC + c) * S;
#pragma unroll 8
        for (int i1 = i10; i1 < N1; i1 += STEP)
          lane_sm[fft::pad32(i1)] = __ldg(recv + recv_index(a, p, kFsN2 * i1 + i20 + i2l, kc0 + c));
      }
      __syncthreads();
      if (threadIdx.x < THREADS_A) {
        const int tr = warp * TPW + lane / T, t = lane % T;
        float2* buf = smem + tr * S;
        const int i2 = i20 + tr / kFsPC;
        fft::cta_fft<N1, true, true, true>(
            t, buf, tw1, [&](int n) { return buf[fft::pad32(n)]; },
            [&](int k1, float2 x) { buf[fft::pad32(k1)] = fft::cmul(x, __ldg(wn + i2 * k1)); });
      }
      if (blk >= kFsRing && threadIdx.x == 0) spin_until(b_done + blk - kFsRing, nB);
      __syncthreads();
      if (threadIdx.x < THREADS_A) {
        const int c = threadIdx.x % kFsPC, i2l = (threadIdx.x / kFsPC) % kFsB, i10 = threadIdx.x / NT;
        const float2* lane_sm = smem + (i2l * kFsPC + c) * S;
#pragma unroll 8
        for (int k1 = i10; k1 < N1; k1 += STEP)
          __stcg(slot + (size_t)(kFsN2 * k1 + i20 + i2l) * kFsPC + c, lane_sm[fft::pad32(k1)]);
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(a_done + blk, 1);
    } else {
      // ---- step B (k_slab_colsB): k1 = 2 (r - nA), + 1
      using PL = fft::Plan<kFsN2>;
      constexpr int T = PL::T, TPW = 32 / T, S = kFsStride<PL::SMEM>;
      constexpr int STEP = THREADS / NT;
      const int k10 = (r - nA) * kFsB;
      const int c = threadIdx.x % kFsPC, k1l = (threadIdx.x / kFsPC) % kFsB, i20 = threadIdx.x / NT;
      float2* lane_sm = smem + (k1l * kFsPC + c) * S;
      if (threadIdx.x == 0) spin_until(a_done + blk, nA);
      __syncthreads();
      const float2* lane_src = slot + (size_t)(kFsN2 * (k10 + k1l)) * kFsPC + c;
#pragma unroll 8
      for (int i2 = i20; i2 < kFsN2; i2 += STEP)
        lane_sm[fft::pad32(i2)] = __ldcg(lane_src + (size_t)i2 * kFsPC);
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(b_done + blk, 1);  // the slot's reads of this item are done
      const int tr = warp * TPW + lane / T, t = lane % T;
      float2* buf = smem + tr * S;
      fft::cta_fft<kFsN2, true, true, true>(
          t, buf, tw2, [&](int n) { return buf[fft::pad32(n)]; },
          [&](int k2, float2 x) { buf[fft::pad32(k2)] = x; });
      __syncthreads();
      float* re = a.fields + (size_t)(2 * p) * N * a.cols;
      float* im = a.fields + (size_t)(2 * p + 1) * N * a.cols;
      const int kc = kc0 + c;
#pragma unroll 8
      for (int k2 = i20; k2 < kFsN2; k2 += STEP) {
        const int k = k10 + k1l + N1 * k2;
        const float2 x = lane_sm[fft::pad32(k2)];
        const float sg = ((k + a.col0 + kc) & 1) ? -1.f : 1.f;  // fft.cpp:73-75
        __stcs(re + (size_t)k * a.cols + kc, sg * x.x);          // fft.cpp:93-99
        __stcs(im + (size_t)k * a.cols + kc, sg * x.y);
      }
    }
    __syncthreads();  // shared memory is reused by the next item
  }
}

static bool fused_cols_enabled() {
  static const bool on = [] {
    const char* e = getenv("OCN_SLAB_NO_FUSED_COLS");
    return !(e && *e && *e != '0');
  }();
  return on;
}

template <int N>
bool slab_fourstep(ocn_slab* sl, const SlabColArgs& a, float2* recv, int np) {
  if constexpr (N >= 4096) {
    if (a.cols % kFsPC) return false;
    constexpr int N1 = N / kFsN2;
    const size_t smemA = (size_t)kFsB * kFsPC * kFsStride<fft::Plan<N1>::SMEM> * sizeof(float2);
    const size_t smemB = (size_t)kFsB * kFsPC * kFsStride<fft::Plan<kFsN2>::SMEM> * sizeof(float2);
    smem_opt_in(k_slab_colsA<N>, smemA);
    smem_opt_in(k_slab_colsB<N>, smemB);
    if (fused_cols_enabled() && N1 <= kFsN2) {
      const int nblocks = np * (a.cols / kFsPC);
      sl->ring.ensure((size_t)kFsRing * N * kFsPC);
      sl->fs_sync.ensure(1 + 2 * (size_t)nblocks);
      OCN_CUDA(cudaMemsetAsync(sl->fs_sync.p, 0, (1 + 2 * (size_t)nblocks) * sizeof(int),
                               sl->ctx->stream));
      const size_t smemF = std::max(smemA, smemB);
      smem_opt_in(k_slab_cols_fused<N>, smemF);
      int per_sm = 0;
      OCN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, k_slab_cols_fused<N>, kFsB * kFsPC * kFsN2 / 32, smemF));
      const int grid = std::max(1, per_sm) * sl->ctx->sm_count;
      k_slab_cols_fused<N><<<grid, kFsB * kFsPC * kFsN2 / 32, smemF, sl->ctx->stream>>>(
          a, recv, sl->ring.p, sl->fs_sync.p, nblocks, sl->tw1.p, sl->wn.p, sl->tw2.p);
      OCN_LAUNCHED(sl->ctx);
      return true;
    }
    const dim3 ga(a.cols / kFsPC, kFsN2 / kFsB, np), gb(a.cols / kFsPC, N1 / kFsB, np);
    k_slab_colsA<N><<<ga, kFsB * kFsPC * N1 / 32, smemA, sl->ctx->stream>>>(a, recv, sl->tw1.p, sl->wn.p);
    OCN_LAUNCHED(sl->ctx);
    k_slab_colsB<N><<<gb, kFsB * kFsPC * kFsN2 / 32, smemB, sl->ctx->stream>>>(a, recv, sl->tw2.p);
    OCN_LAUNCHED(sl->ctx);
    return true;
  } else {
    (void)sl, (void)a, (void)recv, (void)np;
    return false;
  }
}

template <int N>
void slab_rows_launch(ocn_slab* sl, const SlabRowArgs& a) {  // pairs [a.p0, a.p0 + a.np)
  if constexpr (N == 16384) {
    using PL = fft::Plan<128>;
    const size_t smem = ((size_t)128 * PL::SMEM + PL::tw_size() + 2 * 128) * sizeof(float2);
    smem_opt_in(k_slab_rows_4s<N>, smem);
    k_slab_rows_4s<N><<<a.rows * a.np, kRow4sThreads, smem, sl->ctx->stream>>>(
        a, sl->tw128.p, sl->w_hi.p, sl->w_lo.p);
    OCN_LAUNCHED(sl->ctx);
    return;
  }
  using L = SlabLaunch<N>;
  if (L::SMEM_BYTES > 48 * 1024) {
    smem_opt_in(k_slab_rows<N>, L::SMEM_BYTES);
    smem_opt_in(k_slab_cols<N>, L::SMEM_BYTES);
  }
  const int blocks = (a.rows * a.np + L::PER_CTA - 1) / L::PER_CTA;
  k_slab_rows<N><<<blocks, L::THREADS, L::SMEM_BYTES, sl->ctx->stream>>>(a);
  OCN_LAUNCHED(sl->ctx);
}

template <int N>
void slab_cols_launch(ocn_slab* sl, const SlabColArgs& a, float2* recv, int np) {
  if (slab_fourstep<N>(sl, a, recv, np)) return;
  using L = SlabLaunch<N>;
  if (L::SMEM_BYTES > 48 * 1024) {
    smem_opt_in(k_slab_rows<N>, L::SMEM_BYTES);
    smem_opt_in(k_slab_cols<N>, L::SMEM_BYTES);
  }
  dim3 grid((a.cols + L::PER_CTA - 1) / L::PER_CTA, np);
  k_slab_cols<N><<<grid, L::THREADS, L::SMEM_BYTES, sl->ctx->stream>>>(a);
  OCN_LAUNCHED(sl->ctx);
}

#define OCN_SLAB_DISPATCH(n, MACRO)                       \
  switch (n) {                                            \
    case 64: MACRO(64); break;                            \
    case 128: MACRO(128); break;                          \
    case 256: MACRO(256); break;                          \
    case 512: MACRO(512); break;                          \
    case 1024: MACRO(1024); break;                        \
    case 2048: MACRO(2048); break;                        \
    case 4096: MACRO(4096); break;                        \
    case 8192: MACRO(8192); break;                        \
    case 16384: MACRO(16384); break;                      \
    default: fail(OCN_ERR_CONFIG, "slab size %d not supported (64..16384)", n); \
  }

int grid_cap(ocn_ctx* ctx, size_t n) {
  size_t b = (n + 255) / 256, cap = (size_t)ctx->sm_count * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

__global__ void k_set_time_slab(double* d, double t) { *d = t; }
__global__ void k_f32_f64_slab(size_t n, const float* in, double* out) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x)
    out[q] = in[q];
}

}  // namespace

std::vector<float2> make_twiddles(int n);  // spectral.cu

// Row pass of packed pairs [p0, p0 + np) (evolve: also advance h~ to t first).
void slab_rows_pairs(ocn_slab* sl, double t, double choppiness, void* dev_send, int p0, int np,
                     bool evolve) {
  NvtxRange nv("slab.rows");
  ocn_ctx* ctx = sl->ctx;
  ProfWindow pw(ctx, OCN_PROF_ROWS);
  if (evolve) {
    k_set_time_slab<<<1, 1, 0, ctx->stream>>>(sl->d_time.p, t);
    OCN_LAUNCHED(ctx);
    const size_t slab = (size_t)sl->rows * sl->n;
    int logn = 0;
    while ((1 << logn) < sl->n) ++logn;
    k_slab_evolve<<<grid_cap(ctx, slab), 256, 0, ctx->stream>>>(
        logn, sl->rank * sl->rows, sl->rows, sl->gc, sl->d_time.p, sl->h0.p, sl->h0m.p, sl->spec.p);
    OCN_LAUNCHED(ctx);
  }
  SlabRowArgs a{sl->rank * sl->rows, sl->rows, sl->cols, (float)sl->gc.dk, (float)choppiness,
                sl->spec.p, (float2*)dev_send, sl->twiddle.p, p0, np};
#define OCN_SR(NN) slab_rows_launch<NN>(sl, a)
  OCN_SLAB_DISPATCH(sl->n, OCN_SR)
#undef OCN_SR
}

// Column pass of packed pairs [p0, p0 + np) from the receive layout.
void slab_cols_pairs(ocn_slab* sl, void* dev_recv, int p0, int np) {
  NvtxRange nv("slab.cols");
  ProfWindow pw(sl->ctx, OCN_PROF_COLS);
  int lg = 0;
  while ((1 << lg) < sl->rows) ++lg;
  SlabColArgs a{sl->rows, sl->cols, sl->rank * sl->cols, lg, (const float2*)dev_recv, sl->fields.p,
                sl->twiddle.p, p0};
#define OCN_SC(NN) slab_cols_launch<NN>(sl, a, (float2*)dev_recv, np)
  OCN_SLAB_DISPATCH(sl->n, OCN_SC)
#undef OCN_SC
}

void slab_geometry(const ocn_slab* sl, ocn_ctx** ctx, int* n, int* ranks, int* rank, int* rows) {
  *ctx = sl->ctx;
  *n = sl->n;
  *ranks = sl->ranks;
  *rank = sl->rank;
  *rows = sl->rows;
}

}  // namespace ocn

using namespace ocn;

extern "C" {

int ocn_slab_create(ocn_ctx* ctx, int n, int ranks, int rank, double length, double band_min,
                    double band_max, uint32_t cascade_index, const ocn_spectrum_params* params,
                    ocn_slab** out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && params && out, "null argument");
    if (!is_pow2(n) || n < 64 || n > 16384) fail(OCN_ERR_CONFIG, "slab grid must be 64..16384, pow2");
    OCN_REQUIRE(ranks >= 1 && n % ranks == 0 && (n / ranks) >= 1 && rank >= 0 && rank < ranks,
                "bad slab decomposition %d / %d", rank, ranks);
    if (!(length > 0.0)) fail(OCN_ERR_CONFIG, "cascade length must be > 0");
    if (!(band_min >= 0.0) || !(band_max > band_min))
      fail(OCN_ERR_CONFIG, "cascade band must satisfy 0 <= band_min < band_max");
    int st = ocn_spectrum_validate(params);
    if (st) fail(st, "%s", global_error().c_str());
    DeviceScope ds(ctx);
    auto sl = std::make_unique<ocn_slab>();
    sl->ctx = ctx;
    sl->n = n;
    sl->ranks = ranks;
    sl->rank = rank;
    sl->rows = sl->cols = n / ranks;
    sl->gc.dk = 2.0 * kPi / length;
    sl->gc.length = length;
    sl->gc.band_min = band_min;
    sl->gc.band_max = band_max;
    sl->gc.cindex = cascade_index;
    sl->gc.p = *params;
    const size_t slab = (size_t)sl->rows * n;
    sl->h0.alloc(slab);
    sl->h0m.alloc(slab);
    sl->spec.alloc(slab);
    sl->fields.alloc(8 * slab);
    sl->d_time.alloc(1);
    k_slab_init<<<grid_cap(ctx, slab), 256, 0, ctx->stream>>>(n, rank * sl->rows, sl->rows, sl->gc,
                                                            sl->h0.p, sl->h0m.p);
    OCN_LAUNCHED(ctx);
    std::vector<float2> tw = make_twiddles(n);
    sl->twiddle.alloc(tw.size());
    OCN_CUDA(cudaMemcpyAsync(sl->twiddle.p, tw.data(), tw.size() * sizeof(float2),
                             cudaMemcpyHostToDevice, ctx->stream));
    if (n >= 4096) {  // four-step column pass tables
      auto up = [&](DevBuf<float2>& b, const std::vector<float2>& h) {
        b.alloc(h.size());
        OCN_CUDA(cudaMemcpy(b.p, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice));
      };
      up(sl->tw1, make_twiddles(n / kFsN2));
      up(sl->tw2, make_twiddles(kFsN2));
      std::vector<float2> w(n);
      for (int m = 0; m < n; ++m) {
        const double ang = 2.0 * kPi * m / n;  // synthesis sign, fft.hpp:10-17
        w[m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
      up(sl->wn, w);
      if (n == 16384) {  // w_N^m = w_hi[m >> 7] w_lo[m & 127] for m < N
        std::vector<float2> hi(128), lo(128);
        for (int m = 0; m < 128; ++m) {
          const double ah = 2.0 * kPi * (128.0 * m) / n, al = 2.0 * kPi * m / n;
          hi[m] = make_float2((float)std::cos(ah), (float)std::sin(ah));
          lo[m] = make_float2((float)std::cos(al), (float)std::sin(al));
        }
        up(sl->tw128, make_twiddles(128));
        up(sl->w_hi, hi);
        up(sl->w_lo, lo);
      }
    }
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx_retain(ctx);
    *out = sl.release();
  });
}

int ocn_slab_destroy(ocn_slab* sl) {
  if (!sl) return OCN_OK;
  ocn_ctx* ctx = sl->ctx;
  {
    DeviceScope ds(ctx);
    cudaStreamSynchronize(ctx->stream);
    delete sl;
  }
  ctx_release(ctx);
  return OCN_OK;
}

int ocn_slab_info(const ocn_slab* sl, int* rows, int* cols, size_t* exchange_bytes) {
  if (!sl) return OCN_ERR_ARG;
  if (rows) *rows = sl->rows;
  if (cols) *cols = sl->cols;
  if (exchange_bytes) *exchange_bytes = (size_t)4 * sl->rows * sl->n * sizeof(float2);
  return OCN_OK;
}

int ocn_slab_rows(ocn_slab* sl, double t, double choppiness, void* dev_send) {
  return api_call(sl ? sl->ctx : nullptr, [&] {
    OCN_REQUIRE(sl && dev_send, "null argument");
    DeviceScope ds(sl->ctx);
    slab_rows_pairs(sl, t, choppiness, dev_send, 0, 4, true);
  });
}

int ocn_slab_cols(ocn_slab* sl, void* dev_recv) {
  return api_call(sl ? sl->ctx : nullptr, [&] {
    OCN_REQUIRE(sl && dev_recv, "null argument");
    DeviceScope ds(sl->ctx);
    slab_cols_pairs(sl, dev_recv, 0, 4);
  });
}

int ocn_slab_download(ocn_slab* sl, int field, double* host_out) {
  return api_call(sl ? sl->ctx : nullptr, [&] {
    OCN_REQUIRE(sl && host_out && field >= 0 && field < 8, "bad arguments");
    ocn_ctx* ctx = sl->ctx;
    DeviceScope ds(ctx);
    const size_t cnt = (size_t)sl->n * sl->cols;
    DevBuf<double> tmp(cnt);
    k_f32_f64_slab<<<grid_cap(ctx, cnt), 256, 0, ctx->stream>>>(cnt, sl->fields.p + field * cnt, tmp.p);
    OCN_LAUNCHED(ctx);
    OCN_CUDA(cudaMemcpyAsync(host_out, tmp.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
