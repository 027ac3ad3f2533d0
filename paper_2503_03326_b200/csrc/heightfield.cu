// heightfield.cu — the composed free surface and the ABHF heightfield writer
// fed straight from device fields.
//
// Simulation::compose_height (sim.cpp:44-51) = height_at over the maps plus
// FdmZone::sample of every other body's zone, evaluated here in bulk on the
// device; dump_fields (main.cpp:59-90) samples it on a resolution² grid over
// the first cascade's tile and writes ABHF files (heightfield_io.hpp:11-16,
// heightfield_io.cpp:30-45). The per-cascade fields are fp32 on the device
// already, so a field file is one D2H of the plane behind the 16-byte header.
#include <cstdio>
#include <cstring>

#include "samplers.cuh"

namespace ocn {

ZoneView zone_view(ocn_zone* z);  // fdm.cu

namespace {

// Simulation::compose_height, sim.cpp:44-51 (the excluded body's zone is
// simply not in the list).
__device__ __forceinline__ double compose_dev(const SurfView& s, const ZoneList& zl, double x,
                                              double z) {
  double h = height_at_dev(s, x, z);
  for (int k = 0; k < zl.count; ++k) h += zone_sample(zl.z[k], x, z);
  return h;
}

__global__ void k_compose_height(SurfView s, ZoneList zl, int64_t n, const double* xz,
                                 double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = compose_dev(s, zl, xz[2 * i], xz[2 * i + 1]);
}

// dump_fields' composed grid (main.cpp:62-67): point (extent*i/res, extent*j/res)
// into [i][j] row-major. The point coordinates are generated in the kernel
// (no query upload); F is double for the API download, float for the file.
template <typename F>
__global__ void k_compose_grid(SurfView s, ZoneList zl, int res, double extent, F* out) {
  const int64_t total = (int64_t)res * res;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / res), j = (int)(q % res);
    const double x = extent * i / res;
    const double z = extent * j / res;
    out[q] = (F)compose_dev(s, zl, x, z);
  }
}

int grid_blocks(ocn_ctx* ctx, int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)ctx->sm_count * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

ZoneList zone_list(int n_zones, ocn_zone* const* zones) {
  OCN_REQUIRE(n_zones >= 0 && n_zones <= kMaxZones, "zone count %d out of range [0, %d]", n_zones,
              kMaxZones);
  OCN_REQUIRE(n_zones == 0 || zones, "null zone list");
  ZoneList zl{};
  zl.count = n_zones;
  for (int k = 0; k < n_zones; ++k) {
    OCN_REQUIRE(zones[k], "null zone %d", k);
    zl.z[k] = zone_view(zones[k]);
  }
  return zl;
}

// Pinned staging of one float plane for the file writers.
struct PinnedF32 {
  float* p = nullptr;
  explicit PinnedF32(size_t n) { OCN_CUDA(cudaMallocHost(&p, n * sizeof(float))); }
  ~PinnedF32() {
    if (p) cudaFreeHost(p);
  }
};

// write_heightfield (heightfield_io.cpp:30-45): "ABHF", u32 N, i32 cascade,
// f32 time, N*N f32 row-major, all little-endian (the host is x86-64 / aarch64 LE).
void write_abhf(const char* path, uint32_t res, int32_t cascade, float time, const float* data) {
  OCN_REQUIRE(path, "null path");
  FILE* f = std::fopen(path, "wb");
  if (!f) fail(OCN_ERR_IO, "cannot open for writing: %s", path);
  unsigned char hdr[16];
  std::memcpy(hdr, "ABHF", 4);
  std::memcpy(hdr + 4, &res, 4);
  std::memcpy(hdr + 8, &cascade, 4);
  std::memcpy(hdr + 12, &time, 4);
  const size_t nn = (size_t)res * res;
  const bool ok = std::fwrite(hdr, 1, 16, f) == 16 && std::fwrite(data, sizeof(float), nn, f) == nn;
  const bool closed = std::fclose(f) == 0;
  if (!ok || !closed) fail(OCN_ERR_IO, "heightfield: write failed");
}

}  // namespace
}  // namespace ocn

using namespace ocn;

extern "C" {

int ocn_compose_height(ocn_maps* m, int n_zones, ocn_zone* const* zones, int64_t n,
                       const double* xz, double* out) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && n >= 0 && (n == 0 || (xz && out)), "bad compose_height arguments");
    const ZoneList zl = zone_list(n_zones, zones);
    if (n == 0) return;
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const SurfView v = make_surf_view(m);
    InStage si(ctx, xz, (size_t)n * 2 * sizeof(double));
    OutStage so(ctx, out, (size_t)n * sizeof(double));
    k_compose_height<<<grid_blocks(ctx, n), 256, 0, ctx->stream>>>(v, zl, n, (const double*)si.dev,
                                                                   (double*)so.dev);
    OCN_LAUNCHED(ctx);
    so.finish();
  });
}

int ocn_compose_grid(ocn_maps* m, int n_zones, ocn_zone* const* zones, int resolution,
                     double extent, double* out) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && out, "null argument");
    if (resolution <= 0) fail(OCN_ERR_CONFIG, "composed grid resolution %d must be positive", resolution);
    const ZoneList zl = zone_list(n_zones, zones);
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const SurfView v = make_surf_view(m);
    const int64_t total = (int64_t)resolution * resolution;
    OutStage so(ctx, out, (size_t)total * sizeof(double));
    k_compose_grid<double><<<grid_blocks(ctx, total), 256, 0, ctx->stream>>>(v, zl, resolution,
                                                                             extent, (double*)so.dev);
    OCN_LAUNCHED(ctx);
    so.finish();
  });
}

int ocn_heightfield_write_field(ocn_maps* m, int cascade, int field, float time, const char* path) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && path && cascade >= 0 && cascade < m->cas->count && field >= 0 && field < 8,
                "bad heightfield field arguments");
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const int n = m->cas->n;
    const size_t nn = (size_t)n * n;
    PinnedF32 host(nn);
    OCN_CUDA(cudaMemcpyAsync(host.p, m->field(cascade, field), nn * sizeof(float),
                             cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    write_abhf(path, (uint32_t)n, cascade, time, host.p);
  });
}

int ocn_heightfield_write_composed(ocn_maps* m, int n_zones, ocn_zone* const* zones,
                                   int resolution, double extent, float time, const char* path) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && path, "null argument");
    if (resolution <= 0 || resolution > (1 << 16))
      fail(OCN_ERR_CONFIG, "composed grid resolution %d out of range", resolution);
    const ZoneList zl = zone_list(n_zones, zones);
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const SurfView v = make_surf_view(m);
    const int64_t total = (int64_t)resolution * resolution;
    DevBuf<float> dev((size_t)total);
    k_compose_grid<float><<<grid_blocks(ctx, total), 256, 0, ctx->stream>>>(v, zl, resolution,
                                                                            extent, dev.p);
    OCN_LAUNCHED(ctx);
    PinnedF32 host((size_t)total);
    OCN_CUDA(cudaMemcpyAsync(host.p, dev.p, (size_t)total * sizeof(float), cudaMemcpyDeviceToHost,
                             ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    write_abhf(path, (uint32_t)resolution, -1, time, host.p);
  });
}

}  // extern "C"
