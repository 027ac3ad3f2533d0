// samplers.cu — batched point samplers (the FluidQuery samplers of
// hydro.hpp:38-49 as bulk device kernels) and the north-star item 3
// assembly of displacement, normal and Jacobian at query points.
#include <cstring>

#include "samplers.cuh"

namespace ocn {

SurfView make_surf_view(ocn_maps* m) {
  if (m->cas->frames > 1)
    fail(OCN_ERR_CONFIG, "samplers need one frame's maps (this set batches %d frames)",
         m->cas->frames);
  if (m->cas->count > kMaxCascades)
    fail(OCN_ERR_CONFIG, "samplers sum at most %d cascades (maps of a %d-grid set)", kMaxCascades,
         m->cas->count);
  SurfView v{};
  v.n = m->cas->n;
  v.C = m->cas->count;
  for (int c = 0; c < v.C; ++c) v.length[c] = m->cas->lengths[c];
  v.fields = m->fields.p;
  return v;
}

SliceView make_slice_view(ocn_slices* s) {
  if (s->cas->frames > 1)
    fail(OCN_ERR_CONFIG, "samplers need one frame's slices (this set batches %d frames)",
         s->cas->frames);
  if (s->cas->count > kMaxCascades)
    fail(OCN_ERR_CONFIG, "samplers sum at most %d cascades (slices of a %d-grid set)", kMaxCascades,
         s->cas->count);
  SliceView v{};
  v.n = s->cas->n;
  v.C = s->cas->count;
  v.D = s->cfg.count;
  for (int c = 0; c < v.C; ++c) v.length[c] = s->cas->lengths[c];
  v.y_min = s->cfg.y_min;
  v.y_max = s->cfg.y_max;
  v.depths = s->d_depths.p;
  v.fields = s->fields.p;
  return v;
}

namespace {

__global__ void k_maps_sample(SurfView s, int field, int64_t n, const double* xz, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sample_field(s, field, xz[2 * i], xz[2 * i + 1]);
}

__global__ void k_sample_disp(SurfView s, int64_t n, const double* xz, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    sample_disp(s, xz[2 * i], xz[2 * i + 1], &out[3 * i], &out[3 * i + 1], &out[3 * i + 2]);
}

__global__ void k_height_at(SurfView s, int64_t n, const double* xz, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = height_at_dev(s, xz[2 * i], xz[2 * i + 1]);
}

// height_at_tolerance, surface.cpp:153-169
__global__ void k_height_tol(SurfView s, int64_t n, const double* xz, double tol, int max_iters,
                             double* out, int32_t* iters) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double wx = 0.0, wz = 0.0, h_prev = 0.0, dx, h, dz;
    int used = max_iters;
    double res = 0.0;
    bool done = false;
    for (int it = 1; it <= max_iters; ++it) {
      sample_disp(s, xz[2 * i] - wx, xz[2 * i + 1] - wz, &dx, &h, &dz);
      wx = dx, wz = dz;
      if (fabs(h - h_prev) < tol) {
        res = h;
        used = it;
        done = true;
        break;
      }
      h_prev = h;
    }
    out[i] = done ? res : h_prev;
    if (iters) iters[i] = used;
  }
}

// displacement, normal, Jacobian at the Algorithm-1 point
__global__ void k_assemble(SurfView s, int64_t n, const double* xz, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double px, pz, dx, dz;
    const double h = height_at_dev(s, xz[2 * i], xz[2 * i + 1], &px, &pz, &dx, &dz);
    double hx = 0, hz = 0, dxdx = 0, dzdx = 0, dzdz = 0;
#pragma unroll 4
    for (int c = 0; c < s.C; ++c) {
      const Bilin w = bilin_setup(s.n, s.length[c], px, pz);
      hx += bilin_tap(w, s.f(c, OCN_FIELD_HX));
      hz += bilin_tap(w, s.f(c, OCN_FIELD_HZ));
      dxdx += bilin_tap(w, s.f(c, OCN_FIELD_DXDX));
      dzdx += bilin_tap(w, s.f(c, OCN_FIELD_DZDX));
      dzdz += bilin_tap(w, s.f(c, OCN_FIELD_DZDZ));
    }
    const double inv = rsqrt(hx * hx + 1.0 + hz * hz);
    double* o = out + 10 * i;
    o[0] = dx;
    o[1] = h;
    o[2] = dz;
    o[3] = -hx * inv;
    o[4] = inv;
    o[5] = -hz * inv;
    o[6] = (1.0 - dxdx) * (1.0 - dzdz) - dzdx * dzdx;
    o[7] = dxdx;
    o[8] = dzdx;
    o[9] = dzdz;
  }
}

__global__ void k_sample_slice(SliceView s, int d, int64_t n, const double* xz, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    sample_slice_dev(s, d, xz[2 * i], xz[2 * i + 1], out + 3 * i);
}

__global__ void k_velocity_at(SliceView s, int64_t n, const double* xzy, int interp, int clamp,
                              double* out, int* domain_err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!velocity_at_dev(s, xzy[3 * i], xzy[3 * i + 1], xzy[3 * i + 2], interp, clamp, out + 3 * i))
      atomicOr(domain_err, 1);
  }
}

int blocks_for(ocn_ctx* ctx, int64_t n) {
  int64_t b = (n + 127) / 128;
  int64_t cap = (int64_t)ctx->sm_count * 32;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

template <typename F>
int sample_call(ocn_ctx* ctx, int64_t n, const double* in, size_t in_per, double* out,
                size_t out_per, F&& launch) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && n >= 0 && (n == 0 || (in && out)), "bad sampler arguments");
    if (n == 0) return;
    DeviceScope ds(ctx);
    InStage si(ctx, in, (size_t)n * in_per * sizeof(double));
    OutStage so(ctx, out, (size_t)n * out_per * sizeof(double));
    launch((const double*)si.dev, (double*)so.dev);
    OCN_LAUNCHED(ctx);
    so.finish();
  });
}

}  // namespace
}  // namespace ocn

using namespace ocn;

extern "C" {

int ocn_maps_sample(ocn_maps* m, int field, int64_t n, const double* xz, double* out) {
  if (!m || field < 0 || field >= 8) return OCN_ERR_ARG;
  ocn_ctx* ctx = m->cas->ctx;
  return sample_call(ctx, n, xz, 2, out, 1, [&](const double* i, double* o) {
    const SurfView v = make_surf_view(m);
    k_maps_sample<<<blocks_for(ctx, n), 128, 0, ctx->stream>>>(v, field, n, i, o);
  });
}

int ocn_sample_displacement(ocn_maps* m, int64_t n, const double* xz, double* out) {
  if (!m) return OCN_ERR_ARG;
  ocn_ctx* ctx = m->cas->ctx;
  return sample_call(ctx, n, xz, 2, out, 3, [&](const double* i, double* o) {
    const SurfView v = make_surf_view(m);
    k_sample_disp<<<blocks_for(ctx, n), 128, 0, ctx->stream>>>(v, n, i, o);
  });
}

int ocn_height_at(ocn_maps* m, int64_t n, const double* xz, double* out) {
  if (!m) return OCN_ERR_ARG;
  ocn_ctx* ctx = m->cas->ctx;
  return sample_call(ctx, n, xz, 2, out, 1, [&](const double* i, double* o) {
    const SurfView v = make_surf_view(m);
    k_height_at<<<blocks_for(ctx, n), 128, 0, ctx->stream>>>(v, n, i, o);
  });
}

int ocn_height_at_tolerance(ocn_maps* m, int64_t n, const double* xz, double tol, int max_iters,
                            double* out, int32_t* iterations) {
  if (!m) return OCN_ERR_ARG;
  ocn_ctx* ctx = m->cas->ctx;
  return api_call(ctx, [&] {
    const SurfView v = make_surf_view(m);
    OCN_REQUIRE(n >= 0 && (n == 0 || (xz && out)), "bad sampler arguments");
    if (n == 0) return;
    DeviceScope ds(ctx);
    InStage si(ctx, xz, (size_t)n * 2 * sizeof(double));
    OutStage so(ctx, out, (size_t)n * sizeof(double));
    std::unique_ptr<OutStage> sit;
    if (iterations) sit = std::make_unique<OutStage>(ctx, iterations, (size_t)n * sizeof(int32_t));
    k_height_tol<<<blocks_for(ctx, n), 128, 0, ctx->stream>>>(
        v, n, (const double*)si.dev, tol, max_iters, (double*)so.dev,
        sit ? (int32_t*)sit->dev : nullptr);
    OCN_LAUNCHED(ctx);
    so.finish();
    if (sit) sit->finish();
  });
}

int ocn_surface_assemble(ocn_maps* m, int64_t n, const double* xz, double* out) {
  if (!m) return OCN_ERR_ARG;
  ocn_ctx* ctx = m->cas->ctx;
  return sample_call(ctx, n, xz, 2, out, 10, [&](const double* i, double* o) {
    const SurfView v = make_surf_view(m);
    k_assemble<<<blocks_for(ctx, n), 128, 0, ctx->stream>>>(v, n, i, o);
  });
}

int ocn_sample_slice(ocn_slices* s, int depth, int64_t n, const double* xz, double* out) {
  if (!s || depth < 0 || depth >= s->cfg.count) return OCN_ERR_ARG;
  ocn_ctx* ctx = s->cas->ctx;
  return sample_call(ctx, n, xz, 2, out, 3, [&](const double* i, double* o) {
    const SliceView v = make_slice_view(s);
    k_sample_slice<<<blocks_for(ctx, n), 128, 0, ctx->stream>>>(v, depth, n, i, o);
  });
}

int ocn_velocity_at(ocn_slices* s, int64_t n, const double* xzy, int interp, int clamp,
                    double* out) {
  if (!s) return OCN_ERR_ARG;
  ocn_ctx* ctx = s->cas->ctx;
  return api_call(ctx, [&] {
    const SliceView v = make_slice_view(s);
    OCN_REQUIRE(n >= 0 && (n == 0 || (xzy && out)), "bad sampler arguments");
    if (n == 0) return;
    DeviceScope ds(ctx);
    InStage si(ctx, xzy, (size_t)n * 3 * sizeof(double));
    OutStage so(ctx, out, (size_t)n * 3 * sizeof(double));
    DevBuf<int> err(1);
    OCN_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), ctx->stream));
    k_velocity_at<<<blocks_for(ctx, n), 128, 0, ctx->stream>>>(v, n, (const double*)si.dev, interp,
                                                              clamp, (double*)so.dev, err.p);
    OCN_LAUNCHED(ctx);
    int h_err = 0;
    OCN_CUDA(cudaMemcpyAsync(&h_err, err.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    so.finish();
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h_err) fail(OCN_ERR_DOMAIN, "velocity_at: depth outside [y_min, y_max]");
  });
}

}  // extern "C"
