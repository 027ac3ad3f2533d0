// direct.cu — DirectVelocityEvaluator (velocity.hpp:24-37, velocity.cpp:24-59)
// on the device: the exact spectral sum of the water velocity at arbitrary
// points, O(modes × points), that the interpolation studies compare the
// slices against (bench.cpp:94-210).
//
// Construction keeps the reference's mode list exactly: every in-band mode
// with G(k, t) != 0, in (cascade, i, j) order, with the same fp64 coefficients
// cx = G·(−kx g/ω), cy = G·iω, cz = G·(−kz g/ω). It is two passes over the
// h0 table (one warp per spectrum row: count, then a ballot-ordered emit into
// the host-scanned row offsets), so the list is deterministic.
//
// Evaluation: points × modes, one thread per point, modes streamed through
// shared memory in tiles (every warp reads the same mode: broadcast). The
// phase kx x + kz z is fp64 (in turns) and reduced to [-1/2, 1/2] in fp64;
// cos / sin of the reduced phase and the e^{ky} attenuation are fp32 SFU ops;
// the sums are fp64. When there are too few points to fill the GPU, the mode list is split
// into chunks whose partial sums are added in chunk order by a second kernel
// (deterministic for a given device).
#include <vector>

#include "objects.cuh"
#include "spectrum_math.cuh"

struct ocn_direct {
  ocn_ctx* ctx = nullptr;
  double time = 0.0;
  int64_t modes = 0;
  // SoA mode table: kx, kz, k, cx.re, cx.im, cy.re, cy.im, cz.re, cz.im
  ocn::DevBuf<double> m;
  ocn::DevBuf<double> partial;  // [chunks][n][3] scratch of the split evaluation
};

namespace ocn {
namespace {

constexpr int kModeFields = 9;
constexpr int kTile = 128;  // modes per shared-memory tile
constexpr int kEvalThreads = 256;

struct RowMode {
  bool live;
  double kx, kz, k, cx[2], cy[2], cz[2];
};

// The mode at (c, i, j): in_band and G = h0 e^{iωt} − conj(h0(−k)) e^{−iωt}
// (velocity.cpp:16-20, 27-43; h0_conj_neg from spectra.cpp:170-176).
__device__ __forceinline__ RowMode make_mode(const GridConst& G, int n, const double2* h0,
                                             const uint8_t* band, int i, int j, double t) {
  RowMode r{};
  const size_t idx = (size_t)i * n + j;
  if (!band[idx]) return r;
  const double kx = G.dk * (i - n / 2);
  const double kz = G.dk * (j - n / 2);
  const double k = sm::hypot_ref(kx, kz);
  const double omega = sqrt(G.p.gravity * k);
  const double cr = cos(omega * t), sr = sin(omega * t);
  const int ni = i == 0 ? 0 : n - i, nj = j == 0 ? 0 : n - j;
  const double2 a = h0[idx];
  const double2 bn = h0[(size_t)ni * n + nj];
  const double br = bn.x, bi = -bn.y;  // conj(h0(-k))
  // a * (cr + i sr) - b * (cr - i sr)
  const double gre = (a.x * cr - a.y * sr) - (br * cr + bi * sr);
  const double gim = (a.x * sr + a.y * cr) - (bi * cr - br * sr);
  if (gre == 0.0 && gim == 0.0) return r;
  r.live = true;
  r.kx = kx, r.kz = kz, r.k = k;
  const double g = G.p.gravity;
  const double fx = -kx * g / omega, fz = -kz * g / omega;
  r.cx[0] = gre * fx, r.cx[1] = gim * fx;
  r.cy[0] = gre * 0.0 - gim * omega, r.cy[1] = gre * omega + gim * 0.0;
  r.cz[0] = gre * fz, r.cz[1] = gim * fz;
  return r;
}

// One warp per spectrum row (c, i): the live-mode count of the row.
__global__ void k_direct_count(const GridConst* gc, int n, int C, const double2* h0,
                               const uint8_t* band, double t, int32_t* row_count) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= C * n) return;
  const int c = row / n, i = row % n;
  const GridConst G = gc[c];
  const size_t nn = (size_t)n * n;
  int cnt = 0;
  for (int j = lane; j < n; j += 32)
    cnt += make_mode(G, n, h0 + c * nn, band + c * nn, i, j, t).live ? 1 : 0;
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) row_count[row] = cnt;
}

// Same walk; live modes written in j order at the row's offset (ballot rank).
__global__ void k_direct_emit(const GridConst* gc, int n, int C, const double2* h0,
                              const uint8_t* band, double t, const int64_t* row_off, double* m,
                              int64_t stride) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= C * n) return;
  const int c = row / n, i = row % n;
  const GridConst G = gc[c];
  const size_t nn = (size_t)n * n;
  int64_t base = row_off[row];
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int j = j0 + lane;
    RowMode r{};
    if (j < n) r = make_mode(G, n, h0 + c * nn, band + c * nn, i, j, t);
    const unsigned live = __ballot_sync(0xffffffffu, r.live);
    if (r.live) {
      const int64_t q = base + __popc(live & ((1u << lane) - 1u));
      const double v[kModeFields] = {r.kx, r.kz, r.k, r.cx[0], r.cx[1], r.cy[0], r.cy[1], r.cz[0], r.cz[1]};
#pragma unroll
      for (int f = 0; f < kModeFields; ++f) m[f * stride + q] = v[f];
    }
    base += __popc(live);
  }
}

// Sum over modes [m0, m1) at each point; out[p*3 + comp] (+ chunk offset).
// Staging converts each mode once per CTA into the form the inner loop wants:
// wave numbers in turns (kx / 2π, fp64) so the phase reduction is one rint,
// and k log2 e as fp32 for the attenuation. Per mode-point the inner loop is
// then phase (DMUL + DFMA), reduction (rint + DADD), fp32 sin / cos / ex2 with
// the attenuation folded into sin and cos, and 6 DFMA accumulations.
__global__ void __launch_bounds__(kEvalThreads) k_direct_eval(const double* __restrict__ m,
                                                              int64_t stride, int64_t modes,
                                                              int64_t chunk, int64_t n,
                                                              const double* __restrict__ xzy,
                                                              double* __restrict__ out) {
  __shared__ double s_kt[2][kTile];  // kx / 2π, kz / 2π
  __shared__ double s_c[6][kTile];   // cx, cy, cz (re, im)
  __shared__ float s_kl[kTile];      // k log2 e
  const int64_t p = blockIdx.x * (int64_t)kEvalThreads + threadIdx.x;
  const int64_t m0 = blockIdx.y * chunk;
  const int64_t m1 = min(modes, m0 + chunk);
  double x = 0.0, z = 0.0, y = 0.0;
  if (p < n) x = xzy[3 * p], z = xzy[3 * p + 1], y = xzy[3 * p + 2];
  // attenuation (velocity.cpp:10): e^{ky} = 2^{(k log2e) y} below, 1 + ky = 1 + (k log2e)(y ln 2) above
  const bool above = y > 0.0;
  const float ya = above ? (float)(y * 0.6931471805599453) : (float)y;
  double vx = 0.0, vy = 0.0, vz = 0.0;
  constexpr double kInvTwoPi = 0.15915494309189535;
  constexpr float kTwoPiF = 6.28318530717958648f;
  for (int64_t t0 = m0; t0 < m1; t0 += kTile) {
    const int cnt = (int)min((int64_t)kTile, m1 - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += kEvalThreads) {
      const int64_t q = t0 + e;
      s_kt[0][e] = m[q] * kInvTwoPi;
      s_kt[1][e] = m[stride + q] * kInvTwoPi;
      s_kl[e] = (float)(m[2 * stride + q] * 1.4426950408889634);
    }
    for (int q = threadIdx.x; q < 6 * kTile; q += kEvalThreads) {
      const int f = q / kTile, e = q % kTile;
      if (e < cnt) s_c[f][e] = m[(3 + f) * stride + t0 + e];
    }
    __syncthreads();
#pragma unroll 4
    for (int e = 0; e < cnt; ++e) {
      const double u = fma(s_kt[0][e], x, s_kt[1][e] * z);  // phase in turns
      const float r = (float)(u - rint(u));                 // |r| <= 1/2
      float sf, cf;
      __sincosf(r * kTwoPiF, &sf, &cf);
      const float kl = s_kl[e];
      const float att = above ? fmaf(kl, ya, 1.0f) : exp2f(kl * ya);
      const double s = (double)(sf * att), c = (double)(cf * att);
      // Re((a + i b)(c + i s)) = a c - b s, velocity.cpp:51-55
      vx = fma(s_c[0][e], c, fma(-s_c[1][e], s, vx));
      vy = fma(s_c[2][e], c, fma(-s_c[3][e], s, vy));
      vz = fma(s_c[4][e], c, fma(-s_c[5][e], s, vz));
    }
  }
  if (p < n) {
    double* o = out + ((size_t)blockIdx.y * n + p) * 3;
    o[0] = vx, o[1] = vy, o[2] = vz;
  }
}

// out[p] = Σ_chunk partial[chunk][p] in chunk order.
__global__ void k_direct_sum(const double* partial, int chunks, int64_t n3, double* out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n3;
       q += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += partial[(size_t)c * n3 + q];
    out[q] = s;
  }
}

}  // namespace
}  // namespace ocn

using namespace ocn;

extern "C" {

int ocn_direct_create(ocn_cascades* cas, double t, ocn_direct** out) {
  return api_call(cas ? cas->ctx : nullptr, [&] {
    OCN_REQUIRE(cas && out, "null argument");
    if (cas->frames > 1) fail(OCN_ERR_CONFIG, "the direct evaluator takes one frame's cascade set");
    ocn_ctx* ctx = cas->ctx;
    DeviceScope ds(ctx);
    const int n = cas->n, C = cas->count, rows = C * n;
    DevBuf<int32_t> d_cnt((size_t)rows);
    const int wpb = 8;
    const int blocks = (rows + wpb - 1) / wpb;
    k_direct_count<<<blocks, 32 * wpb, 0, ctx->stream>>>(cas->gconst.p, n, C, cas->h0_f64.p,
                                                         cas->in_band.p, t, d_cnt.p);
    OCN_LAUNCHED(ctx);
    std::vector<int32_t> cnt((size_t)rows);
    OCN_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt.p, rows * sizeof(int32_t), cudaMemcpyDeviceToHost,
                             ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<int64_t> off((size_t)rows);
    int64_t total = 0;
    for (int r = 0; r < rows; ++r) off[r] = total, total += cnt[r];
    auto d = std::make_unique<ocn_direct>();
    d->ctx = ctx;
    d->time = t;
    d->modes = total;
    if (total > 0) {
      DevBuf<int64_t> d_off((size_t)rows);
      OCN_CUDA(cudaMemcpyAsync(d_off.p, off.data(), rows * sizeof(int64_t), cudaMemcpyHostToDevice,
                               ctx->stream));
      d->m.alloc((size_t)kModeFields * total);
      k_direct_emit<<<blocks, 32 * wpb, 0, ctx->stream>>>(cas->gconst.p, n, C, cas->h0_f64.p,
                                                          cas->in_band.p, t, d_off.p, d->m.p, total);
      OCN_LAUNCHED(ctx);
      OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    ctx_retain(ctx);
    *out = d.release();
  });
}

int ocn_direct_destroy(ocn_direct* d) {
  if (!d) return OCN_OK;
  ocn_ctx* ctx = d->ctx;
  {
    DeviceScope ds(ctx);
    cudaStreamSynchronize(ctx->stream);
    delete d;
  }
  ctx_release(ctx);
  return OCN_OK;
}

int ocn_direct_modes(const ocn_direct* d, int64_t* count) {
  if (!d || !count) return OCN_ERR_ARG;
  *count = d->modes;
  return OCN_OK;
}

int ocn_direct_evaluate(ocn_direct* d, int64_t n, const double* xzy, double* out) {
  return api_call(d ? d->ctx : nullptr, [&] {
    OCN_REQUIRE(d && n >= 0 && (n == 0 || (xzy && out)), "bad direct evaluation arguments");
    if (n == 0) return;
    ocn_ctx* ctx = d->ctx;
    DeviceScope ds(ctx);
    InStage si(ctx, xzy, (size_t)n * 3 * sizeof(double));
    OutStage so(ctx, out, (size_t)n * 3 * sizeof(double));
    const int64_t pblocks = (n + kEvalThreads - 1) / kEvalThreads;
    // Split the mode list into ordered chunks so that points x chunks fills whole
    // waves of resident CTAs (few points: many chunks; a ragged last wave costs
    // up to half the time otherwise).
    static int per_sm = 0;
    if (!per_sm) {
      OCN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_direct_eval, kEvalThreads, 0));
      per_sm = std::max(per_sm, 1);
    }
    const int64_t slots = (int64_t)ctx->sm_count * per_sm;
    const int64_t max_chunks = std::min<int64_t>(65535, std::max<int64_t>(1, d->modes / (16 * kTile)));
    int64_t chunks = 1;
    double best = -1.0;
    for (int64_t c = 1; c <= std::min<int64_t>(max_chunks, 4 * slots); ++c) {
      const int64_t ctas = pblocks * c;
      const double eff = (double)ctas / (double)(((ctas + slots - 1) / slots) * slots);
      if (eff > best + 1e-3) best = eff, chunks = c;
      if (ctas >= 4 * slots) break;
    }
    const int64_t chunk = chunks > 1 ? (d->modes + chunks - 1) / chunks : std::max<int64_t>(d->modes, 1);
    chunks = chunks > 1 ? (d->modes + chunk - 1) / chunk : 1;
    double* dst = (double*)so.dev;
    if (chunks > 1) {
      d->partial.ensure((size_t)chunks * n * 3);
      dst = d->partial.p;
    }
    k_direct_eval<<<dim3((unsigned)pblocks, (unsigned)chunks), kEvalThreads, 0, ctx->stream>>>(
        d->m.p, d->modes, d->modes, chunk, n, (const double*)si.dev, dst);
    OCN_LAUNCHED(ctx);
    if (chunks > 1) {
      const int64_t n3 = n * 3;
      const int sb = (int)std::min<int64_t>((n3 + 255) / 256, (int64_t)ctx->sm_count * 8);
      k_direct_sum<<<sb, 256, 0, ctx->stream>>>(d->partial.p, (int)chunks, n3, (double*)so.dev);
      OCN_LAUNCHED(ctx);
    }
    so.finish();
  });
}

}  // extern "C"
