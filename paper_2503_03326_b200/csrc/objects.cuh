// objects.cuh — the opaque handle types behind the C-ABI, and the API guard.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace ocn {

constexpr int kMaxCascades = 16;   // cascades summed by one sampler (maps / slices)
constexpr int kMaxGrids = 1 << 16;  // grids of one spectral set (cascades x instances)

// Per-grid constants of a spectral set (device array).
struct GridConst {
  double dk, length, band_min, band_max;
  uint32_t cindex;
  // spectrum rows i with |i - N/2| >= row_half hold no mode of the band
  // (|k| >= |kx| >= band_max): exactly zero h0, so their row transforms are
  // exactly zero. N/2 + 1 when every row can carry the band.
  int32_t row_half;
  ocn_spectrum_params p;
  // time-batched sets: grid g reads the h0 / w tables of
  // grid `src` and is evaluated at t + frame dt (src = g, frame = 0 otherwise)
  int32_t src;
  int32_t frame;
};

// A run of consecutive transforms of one grid inside a transform group.
struct GroupSeg {
  int grid;   // cascade / grid index
  int first;  // first transform, relative to the group
  int count;
  int pad;
};

// One packed C2C transform of the spectral step (X + iY of one field pair).
enum XformKind : int {
  kSurfHDx = 0,     // (H, Dx)        surface.cpp:77
  kSurfDzDxDx = 1,  // (Dz, DxDx)     surface.cpp:78
  kSurfDzDxDzDz = 2,// (DzDx, DzDz)   surface.cpp:79
  kSurfHxHz = 3,    // (Hx, Hz)       surface.cpp:80
  kVelXZ = 4,       // (vx_d, vz_d)   velocity.cpp:156-161
  kVelYPair = 5,    // (vy_d, vy_d+1) velocity.cpp:163-167
  kVelYSingle = 6,  // (vy_d, 0)      velocity.cpp:168-172
};

struct XformDesc {
  int cascade;
  int kind;
  float y0, y1;   // slice depths for the velocity kinds
  float* out_re;  // fp32 plane [N][N] receiving Re
  float* out_im;  // fp32 plane receiving Im (nullptr: dropped)
  // spectrum rows i with |i - N/2| >= row_half have an exactly zero
  // coefficient row: outside the grid's band, or (velocity) attenuated below
  // fp32 at this depth. <= 0: unknown (every row is transformed).
  int row_half = 0;
};

struct SpectralPlan {
  DevBuf<XformDesc> desc;
  DevBuf<CUtensorMap> out_maps;  // TMA-store column pass: Re / Im maps per transform
  // transform groups (G consecutive transforms, possibly spanning grids) and
  // their per-grid segments
  struct Group {
    int first, count, seg0, nseg, max_seg;
    int family;  // 0: surface pairs, 1: velocity
  };
  std::vector<Group> groups;
  DevBuf<GroupSeg> segs;
  // CUDA graph of the whole step (everything but the time upload), captured on
  // the second use of the plan; rebuilt when the choppiness changes.
  cudaGraphExec_t exec = nullptr;
  double graph_chop = 0.0;
  uint64_t graph_kernels = 0;
  int uses = 0;
  ~SpectralPlan() {
    if (exec) cudaGraphExecDestroy(exec);
  }
  std::vector<XformDesc> host_desc;
  std::vector<ocn_xform_info> info;  // every transform of the step, incl. the dropped ones
  std::vector<int> first;  // per cascade: first transform index
  std::vector<int> count;  // per cascade: number of transforms
  bool need_surface = false, need_velocity = false;
  int zero_transforms = 0;  // velocity transforms dropped as exactly zero (planes zeroed once)
  bool assembly = false;    // the captured graph includes the per-texel assembly
};

}  // namespace ocn

struct ocn_cascades {
  ocn_ctx* ctx = nullptr;
  int refs = 1;  // owner + every maps / slices built on it (freed at zero)
  int n = 0, count = 0;
  std::vector<double> lengths, band_min, band_max;
  std::vector<uint32_t> cascade_index;
  ocn_spectrum_params params{};             // of grid 0 (all grids for plain cascade sets)
  std::vector<ocn_spectrum_params> grid_params;
  ocn::DevBuf<ocn::GridConst> gconst;      // [count]
  ocn::DevBuf<double2> h0_f64;  // [C][N][N] fp64 amplitudes (API download)
  ocn::DevBuf<float2> h0;       // [C][N][N] fp32 hot-path table
  ocn::DevBuf<uint8_t> in_band; // [C][N][N]
  ocn::DevBuf<float2> twiddle;  // per-N inter-pass twiddles (fft_core.cuh)
  ocn::DevBuf<float4> h0p;      // [C][N][N] (h0(k), conj(h0(-k))), built once
  ocn::DevBuf<double> omega;    // [C][N][N] dispersion w(k), built once
  ocn::DevBuf<float2> spec_h;   // [C][N][N] evolved h~ at the current frame
  ocn::DevBuf<float2> spec_g;   // [C][N][N] evolved G (written by velocity plans only)
  ocn::DevBuf<float2> scratch;  // row-pass intermediates of one transform group
  ocn::DevBuf<double> d_time;   // frame time read by k_evolve (set per frame)
  int group = 1;                // transforms per group
  int base = 0;                 // grids holding tables (count / frames)
  int frames = 1;               // time-batched set: count = base x frames
  double frame_dt = 0.0;        // default frame spacing of a time-batched set
  CUtensorMap cols_map;         // TMA source map of the scratch (column pass)
  CUtensorMap cols_chunk_map;   // same, 32-row chunks (band-limited loads)
  bool cols_map_ok = false;
  std::map<std::pair<const void*, const void*>, std::unique_ptr<ocn::SpectralPlan>> plans;
};

struct ocn_maps {
  ocn_cascades* cas = nullptr;
  double time = 0.0;
  double choppiness = 1.0;
  ocn::DevBuf<float> fields;  // [C][8][N][N]
  float* field(int c, int f) { return fields.p + ((size_t)c * 8 + f) * (size_t)cas->n * cas->n; }
  // per-texel normal + Jacobian planes [C][4][N][N] (ocn_maps_set_assembly)
  bool assembly = false;
  ocn::DevBuf<float> assembled;
};

struct ocn_slices {
  ocn_cascades* cas = nullptr;
  ocn_slice_config cfg{};
  std::vector<double> depths;
  double time = 0.0;
  ocn::DevBuf<double> d_depths;
  ocn::DevBuf<float> fields;  // [D][C][3][N][N]
  float* field(int d, int c, int comp) {
    size_t nn = (size_t)cas->n * cas->n;
    return fields.p + (((size_t)d * cas->count + c) * 3 + comp) * nn;
  }
};

namespace ocn {

// Per-thread fallback error slot for calls without a context.
std::string& global_error();

template <typename F>
int api_call(ocn_ctx* ctx, F&& f) {
  try {
    f();
    return OCN_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.what();
    global_error() = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "out of host memory";
    global_error() = "out of host memory";
    return OCN_ERR_CUDA;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    global_error() = e.what();
    return OCN_ERR_ARG;
  }
}

#define OCN_REQUIRE(cond, ...)                         \
  do {                                                 \
    if (!(cond)) ::ocn::fail(OCN_ERR_ARG, __VA_ARGS__); \
  } while (0)

void ctx_retain(ocn_ctx* ctx);
void ctx_release(ocn_ctx* ctx);

// Spectral engine (spectral.cu)
// dt < 0: the set's own frame spacing (time-batched sets, ocn_cascades_create_frames)
void spectral_step(ocn_cascades* cas, ocn_maps* maps, ocn_slices* slices, double t,
                   double choppiness, double dt = -1.0);

}  // namespace ocn
