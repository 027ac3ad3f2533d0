// spectral.cu — K1 (spectrum init), time evolution, and the fused
// coefficient + batched packed 2D inverse FFT (K2 + K3 + K4) on sm_100a.
//
// Reference path replaced: generate_h0 (spectra.cpp:132-179), CascadeSet
// (surface.cpp:22-37), assemble_coefficients + generate_maps
// (surface.cpp:39-103), build_slices (velocity.cpp:104-179),
// ifft2_centered / ifft2_hermitian_pair (fft.cpp:39-101).
//
// Per frame, for every grid of the set:
//   k_evolve     : h~(k,t) = h0 e^{iwt} + conj(h0(-k)) e^{-iwt} and
//                  G(k,t) = h0 e^{iwt} - conj(h0(-k)) e^{-iwt}  (fp64 phase,
//                  reduced mod 2pi before the fp32 sincos) -> spec_h / spec_g
//   k_rows_w<N>  : (128 <= N <= 1024; k_rows<N> otherwise) per (row, grid
//                  segment of a transform group): the row's h~ or G-derived
//                  arrays staged in shared memory, each packed coefficient
//                  X + iY generated in the FFT's pass-0 load (no coefficient
//                  arrays in HBM), then the row FFT -> scratch (input
//                  half-shifted: the (-1)^(i+j) centring, kCentreByShift)
//   k_cols_tma<N>: persistent column FFT of scratch fed by TMA (k_cols<N>
//                  with direct loads outside 128 <= N <= 4096), Re -> field X,
//                  Im -> field Y (fp32, row-major [i][j])
// Transforms run in groups sharing one scratch buffer (group * N^2 * 8 B, 768 MB
// budget, equal-sized groups per family; see group_for / get_plan).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <set>
#include <tuple>

#include "fft_core.cuh"
#include "objects.cuh"
#include "spectrum_math.cuh"
#include "tma.cuh"

namespace ocn {

std::string& global_error() {
  static thread_local std::string e;
  return e;
}

// Handles keep their context (and maps / slices their cascades) alive, so
// destruction order from garbage-collected front ends never matters.
void ctx_retain(ocn_ctx* ctx) { ctx->refs.fetch_add(1); }
void ctx_release(ocn_ctx* ctx) {
  if (!ctx || ctx->refs.fetch_sub(1) != 1) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
  delete ctx;
}
bool tma::encode_f32(CUtensorMap* map, int rank, void* base, const uint64_t* dims,
                     const uint64_t* strides, const uint32_t* box) {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!fn) return false;
  const cuuint32_t elem[5] = {1, 1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, base, dims, strides, box, elem,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void smem_opt_in(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int>> done;
  int dev = 0;
  OCN_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert({dev, func, bytes}).second) return;
  OCN_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

static void cascades_release(ocn_cascades* c) {
  if (!c || --c->refs != 0) return;
  ocn_ctx* ctx = c->ctx;
  {
    DeviceScope ds(ctx);
    cudaStreamSynchronize(ctx->stream);
    delete c;
  }
  ctx_release(ctx);
}

namespace {

constexpr int kThreads = 256;

template <int N>
using Launch = fft::CtaLaunch<N, kThreads>;

#include "spectral_kernels.cuh"

int grid_for(ocn_ctx* ctx, size_t n, int threads = 256) {
  size_t b = (n + threads - 1) / threads;
  size_t cap = (size_t)ctx->sm_count * 16;
  return (int)(b < cap ? (b ? b : 1) : cap);
}

#define OCN_DISPATCH_N(n, MACRO)                            \
  switch (n) {                                              \
    case 2: MACRO(2); break;                                \
    case 4: MACRO(4); break;                                \
    case 8: MACRO(8); break;                                \
    case 16: MACRO(16); break;                              \
    case 32: MACRO(32); break;                              \
    case 64: MACRO(64); break;                              \
    case 128: MACRO(128); break;                            \
    case 256: MACRO(256); break;                            \
    case 512: MACRO(512); break;                            \
    case 1024: MACRO(1024); break;                          \
    case 2048: MACRO(2048); break;                          \
    case 4096: MACRO(4096); break;                          \
    case 8192: MACRO(8192); break;                          \
    case 16384: MACRO(16384); break;                        \
    default: fail(OCN_ERR_CONFIG, "FFT size %d is not a supported power of two", n); \
  }

template <int N>
void set_smem_attrs() {
  using L = Launch<N>;
  if (L::SMEM_BYTES > 48 * 1024) {
    smem_opt_in(k_rows<N, false>, L::SMEM_BYTES);
    smem_opt_in(k_rows<N, true>, L::SMEM_BYTES);
    smem_opt_in(k_cols<N, false>, L::SMEM_BYTES);
    smem_opt_in(k_cols<N, true>, L::SMEM_BYTES);
  }
}

// Column kernel epilogue of the spectral step: per-warp TMA stores (default;
// 0.507 vs 0.518 ms config-3 spectral) or, with OCN_COLS=tma, one CTA-wide
// TMA store per tile behind a fence and a CTA barrier. Measured and removed
// (config 3 spectral, ms): direct loads with 2 CTAs / SM 0.572; 2 persistent
// CTAs / SM with one TMA stage each and warp stores 0.538; a compact chunk
// ring with double-buffered exchange 0.661.
static int cols_variant() {
  static const int v = [] {
    const char* e = getenv("OCN_COLS");
    if (e && !strcmp(e, "tma")) return 0;
    return 4;
  }();
  return v;
}

template <int N>
constexpr bool use_warp_kernels() {
  return N >= 128 && N <= 1024;
}

template <int N>
void launch_rows(ocn_ctx* ctx, const RowArgs& a, bool plain, cudaStream_t st, int nseg,
                 int max_seg, int family) {
  if constexpr (use_warp_kernels<N>()) {
    using W = WarpLaunch<N>;
    const int slots = (max_seg + W::TPW - 1) / W::TPW;
    const int cap = 8;
    // surface rows per CTA: a grid has only 4 surface transforms, so several
    // rows keep the CTA's 8 warps busy and amortise its twiddle / staging set-up
    static constexpr int kMaxRpc = N >= 1024 ? 4 : 2;  // 8 at N = 256 measured slower (config 1: 1.15 vs 1.10 ms)
    static const int max_rpc = [] {  // experiment override: OCN_ROWS_RPC=1|2|4|8
      const char* e = getenv("OCN_ROWS_RPC");
      return e && atoi(e) > 0 ? std::min(atoi(e), kMaxRpc) : kMaxRpc;
    }();
    int rpc = 1;
    if (!plain && family == 0)
      while (2 * rpc <= max_rpc && 2 * rpc * slots <= 2 * cap) rpc *= 2;
    const int warps = slots * rpc < cap ? slots * rpc : cap;
    RowArgs ar = a;
    ar.rpc = rpc;
    // staging: velocity (V0, W0, |k|) 20 B per mode of one row; surface h~ (8 B)
    // plus 1/|k| (4 B, N < 1024) per mode of each of the rpc rows
    auto stage_f4 = [](int r) {
      const size_t surf = (size_t)r * N * (N >= 1024 ? 8 : 12);
      return (int)((std::max<size_t>(surf, (size_t)N * 20) + 15) / 16);
    };
    ar.stage_f4 = plain ? 0 : stage_f4(family == 0 ? rpc : 1);
    const size_t smem = (size_t)ar.stage_f4 * sizeof(float4) + W::TWN * sizeof(float2) +
                        (size_t)warps * W::TPW * W::STRIDE * sizeof(float2);
    {
      const size_t smax = (size_t)stage_f4(kMaxRpc) * sizeof(float4) + W::TWN * sizeof(float2) +
                          (size_t)8 * W::TPW * W::STRIDE * sizeof(float2);
      smem_opt_in(k_rows_w<N, kRowPlain>, smax);
      smem_opt_in(k_rows_w<N, kRowSurface>, smax);
      smem_opt_in(k_rows_w<N, kRowVelocity>, smax);
      smem_opt_in(k_rows_w<N, kRowSurface, true>, smax);
      smem_opt_in(k_rows_w<N, kRowVelocity, true>, smax);
    }
    const dim3 grid(N / rpc, plain ? 1 : nseg);
    const bool fused = a.h0p != nullptr;
    if (plain)
      k_rows_w<N, kRowPlain><<<grid, 32 * warps, smem, st>>>(ar);
    else if (family == 0 && fused)
      k_rows_w<N, kRowSurface, true><<<grid, 32 * warps, smem, st>>>(ar);
    else if (family == 0)
      k_rows_w<N, kRowSurface><<<grid, 32 * warps, smem, st>>>(ar);
    else if (fused)
      k_rows_w<N, kRowVelocity, true><<<grid, 32 * warps, smem, st>>>(ar);
    else
      k_rows_w<N, kRowVelocity><<<grid, 32 * warps, smem, st>>>(ar);
    OCN_LAUNCHED(ctx);
    return;
  }
  using L = Launch<N>;
  set_smem_attrs<N>();
  const int blocks = (a.items + L::PER_CTA - 1) / L::PER_CTA;
  if (plain)
    k_rows<N, true><<<blocks, L::THREADS, L::SMEM_BYTES, st>>>(a);
  else
    k_rows<N, false><<<blocks, L::THREADS, L::SMEM_BYTES, st>>>(a);
  OCN_LAUNCHED(ctx);
}

template <int N>
void launch_cols(ocn_ctx* ctx, const ColArgs& a, int G, bool complex_out, cudaStream_t st,
                 const CUtensorMap* map, const CUtensorMap* chunk_map) {
  if constexpr (ColTma<N>::OK) {
    if (map) {
      using CT = ColTma<N>;
      smem_opt_in(k_cols_tma<N, false, CT::STAGES>, CT::SMEM);
      smem_opt_in(k_cols_tma<N, true, CT::STAGES>, CT::SMEM);
      if (CT::smem(2, true) <= 227 * 1024) smem_opt_in(k_cols_tma<N, false, 2, true>, CT::smem(2, true));
      const int tiles_x = N / CT::PC, ntiles = tiles_x * G;
      // persistent: one CTA per SM; on a low-priority context (the spectral
      // side of a frame pipeline) one SM is left free. The concurrent
      // high-priority stream's kernels (hull / mask / FDM chain) fit beside a
      // column CTA (<= 20 K registers, <= 17 KB shared memory each) except
      // the single-CTA ones (waterline chain, mask preparation, block scan),
      // which take the free SM instead of waiting for the whole column pass.
      // Measured (config 3, one box): frame 0.578 -> 0.546-0.552 ms device,
      // e2e 0.578 -> 0.534-0.536; the spectral step alone 0.4665 -> 0.4669.
      // OCN_COLS_GRID overrides the CTA count.
      static const int cap = [] {
        const char* e = getenv("OCN_COLS_GRID");
        return e && atoi(e) > 0 ? atoi(e) : 0;
      }();
      const int per_sm_grid = cap ? std::min(cap, ctx->sm_count)
                                  : std::max(1, ctx->sm_count - (ctx->priority < 0 ? 1 : 0));
      const int grid = std::min(ntiles, per_sm_grid);
      if constexpr (N >= 256 && N <= 1024 && CT::smem(2, true) <= 227 * 1024) {
        if (!complex_out && a.out_maps && cols_variant() == 4) {
          smem_opt_in(k_cols_tma<N, false, 2, true, true>, CT::smem(2, true));
          k_cols_tma<N, false, 2, true, true><<<grid, CT::THREADS, CT::smem(2, true), st>>>(
              *map, *chunk_map, a, tiles_x, ntiles);
          OCN_LAUNCHED(ctx);
          return;
        }
      }
      if (complex_out)
        k_cols_tma<N, true, CT::STAGES><<<grid, CT::THREADS, CT::SMEM, st>>>(*map, *chunk_map, a, tiles_x, ntiles);
      else if (a.out_maps && CT::smem(2, true) <= 227 * 1024)
        k_cols_tma<N, false, 2, true><<<grid, CT::THREADS, CT::smem(2, true), st>>>(*map, *chunk_map, a, tiles_x, ntiles);
      else
        k_cols_tma<N, false, CT::STAGES><<<grid, CT::THREADS, CT::SMEM, st>>>(*map, *chunk_map, a, tiles_x, ntiles);
      OCN_LAUNCHED(ctx);
      return;
    }
  }
  using L = Launch<N>;
  set_smem_attrs<N>();
  dim3 grid((N + L::PER_CTA - 1) / L::PER_CTA, G);
  if (complex_out)
    k_cols<N, true><<<grid, L::THREADS, L::SMEM_BYTES, st>>>(a);
  else
    k_cols<N, false><<<grid, L::THREADS, L::SMEM_BYTES, st>>>(a);
  OCN_LAUNCHED(ctx);
}

void rows_dispatch(ocn_ctx* ctx, int n, const RowArgs& a, bool plain, cudaStream_t st,
                   int nseg = 1, int max_seg = 0, int family = 0) {
  if (max_seg <= 0) max_seg = a.G;
#define OCN_ROWS(NN) launch_rows<NN>(ctx, a, plain, st, nseg, max_seg, family)
  OCN_DISPATCH_N(n, OCN_ROWS)
#undef OCN_ROWS
}
void cols_dispatch(ocn_ctx* ctx, int n, const ColArgs& a, int G, bool complex_out, cudaStream_t st,
                   const CUtensorMap* map = nullptr, const CUtensorMap* chunk_map = nullptr) {
#define OCN_COLS(NN) launch_cols<NN>(ctx, a, G, complex_out, st, map, chunk_map ? chunk_map : map)
  OCN_DISPATCH_N(n, OCN_COLS)
#undef OCN_COLS
}

template <int N>
int tw_size_of() {
  return fft::Plan<N>::tw_size();
}

}  // namespace

// Inter-pass twiddle table for length n (layout of fft_core.cuh), fp64 -> fp32.
std::vector<float2> make_twiddles(int n) {
  std::vector<float2> out;
  int E = n >= 32 ? 32 : n;
  int logn = ilog2(n), loge = ilog2(E);
  int P = loge ? 1 + (logn - loge + loge - 1) / loge : 1;
  auto ipow = [](int b, int e) {
    int r = 1;
    while (e--) r *= b;
    return r;
  };
  for (int p = 1; p < P; ++p) {
    int R = p < P - 1 ? E : n / ipow(E, P - 1);
    int NS = ipow(E, p);
    for (int r = 0; r < R; ++r)
      for (int b = 0; b < NS; ++b) {
        // exp(+2 pi i b r / (NS R)) via an exact integer reduction of the angle
        long long num = (long long)b * r % ((long long)NS * R);
        double ang = 2.0 * kPi * (double)num / (double)((long long)NS * R);
        out.push_back(make_float2((float)cos(ang), (float)sin(ang)));
      }
  }
  if (out.empty()) out.push_back(make_float2(1.f, 0.f));
  return out;
}

namespace {


// Column-pass source map over a scratch buffer [G][N][N] complex64, viewed as
// fp32 [G][N / BR][BR][2N] so one box {2 PC, BR, N / BR, 1} is a whole column
// tile. Returns false (-> direct-load kernel) outside the TMA kernel's range
// or when OCN_COLS_LDG=1 asks for the direct-load column kernel.
static bool cols_ldg() {
  static const bool on = [] {
    const char* e = getenv("OCN_COLS_LDG");
    return e && *e && *e != '0';
  }();
  return on;
}

// chunk: the 32-row chunk map of the band-limited loads (box {2 PC, 32, 1, 1})
bool cols_map_for(int n, int G, const float2* scratch, CUtensorMap* map, bool chunk = false) {
  const int pc = cols_tma_pc(n);
  const int br = chunk ? std::min(32, n) : (n < 256 ? n : 256);
  if (!pc || cols_ldg()) return false;
  const uint64_t dims[4] = {2ull * n, (uint64_t)br, (uint64_t)(n / br), (uint64_t)G};
  const uint64_t strides[3] = {2ull * n * 4, (uint64_t)br * 2 * n * 4, (uint64_t)n * n * 8};
  const uint32_t box[4] = {2u * pc, (uint32_t)br, chunk ? 1u : (uint32_t)(n / br), 1u};
  if (!tma::encode_f32(map, 4, const_cast<float2*>(scratch), dims, strides, box))
    fail(OCN_ERR_CUDA, "cuTensorMapEncodeTiled failed for the column pass (N=%d, G=%d)", n, G);
  return true;
}

// Store map of one fp32 output plane [N][N] viewed as [N / BR][BR][N]: box
// {PC, BR, N / BR} is the plane's share of one column tile.
static void plane_map_for(int n, float* plane, CUtensorMap* map) {
  const int pc = cols_tma_pc(n), br = n < 256 ? n : 256;
  const uint64_t dims[3] = {(uint64_t)n, (uint64_t)br, (uint64_t)(n / br)};
  const uint64_t strides[2] = {(uint64_t)n * 4, (uint64_t)br * n * 4};
  const uint32_t box[3] = {(uint32_t)pc, (uint32_t)br, (uint32_t)(n / br)};
  *map = CUtensorMap{};
  if (plane && !tma::encode_f32(map, 3, plane, dims, strides, box))
    fail(OCN_ERR_CUDA, "cuTensorMapEncodeTiled failed for an output plane (N=%d)", n);
}

// TMA-store column pass (default; OCN_COLS_STG=1 selects direct evict-first
// stores from the warps, 3 load stages): measured 1.122 vs 1.128 ms spectral
// per frame (config 3); the column pass then runs at ~94% of the measured HBM
// copy bandwidth on its real traffic (ncu, 96-transform groups).
static bool cols_tma_store() {
  static const bool on = [] {
    const char* e = getenv("OCN_COLS_STG");
    return !(e && *e && *e != '0');
  }();
  return on;
}

// Store map of one fp32 output plane for the ring column kernel's per-warp
// boxes: the plane viewed as [N / T][T][N] (row = t + T r'), box {PC, 32 / PC, 32}.
static void plane_warp_map_for(int n, float* plane, CUtensorMap* map) {
  const int pc = cols_tma_pc(n), T = n / 32;
  const uint64_t dims[3] = {(uint64_t)n, (uint64_t)T, 32};
  const uint64_t strides[2] = {(uint64_t)n * 4, (uint64_t)T * n * 4};
  const uint32_t box[3] = {(uint32_t)pc, (uint32_t)(32 / pc), 32};
  *map = CUtensorMap{};
  if (plane && !tma::encode_f32(map, 3, plane, dims, strides, box))
    fail(OCN_ERR_CUDA, "cuTensorMapEncodeTiled failed for an output plane (N=%d)", n);
}

static void build_out_maps(int n, const XformDesc* desc, int count, DevBuf<CUtensorMap>& out) {
  const bool warp_boxes = cols_variant() == 4 && n >= 256 && n <= 1024;
  std::vector<CUtensorMap> h((size_t)2 * count);
  for (int i = 0; i < count; ++i) {
    auto mk = warp_boxes ? plane_warp_map_for : plane_map_for;
    mk(n, desc[i].out_re, &h[2 * i]);
    mk(n, desc[i].out_im, &h[2 * i + 1]);
  }
  out.alloc(h.size());
  OCN_CUDA(cudaMemcpy(out.p, h.data(), h.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
}

static bool band_skip_enabled() {
  static const bool on = [] {
    const char* e = getenv("OCN_NO_BAND_SKIP");
    return !(e && *e && *e != '0');
  }();
  return on;
}

bool fused_evolve_enabled() {
  static const bool on = [] {
    const char* e = getenv("OCN_NO_FUSED_EVOLVE");
    return !(e && *e && *e != '0');
  }();
  return on;
}

bool merged_cols_enabled() {
  static const bool on = [] {
    const char* e = getenv("OCN_NO_MERGED_COLS");
    return !(e && *e && *e != '0');
  }();
  return on;
}

size_t group_for(int n, int total) {
  // Scratch budget of the transform groups. Larger groups amortise the row
  // kernel's per-row staging over more transforms and keep the persistent
  // column kernel's tile ring full: measured on B200 at N = 1024 (config 3,
  // spectral ms / frame, first TMA column kernel) 64 MB 1.75, 256 MB 1.46,
  // 512 MB 1.39, 1 GB 1.36, 2 GB 1.33; with balanced family groups (get_plan)
  // 384 MB 1.100, 512 MB 1.123, 768 MB 1.095, 1 GB 1.124. With the current
  // kernels (f32x2 FFT, per-warp TMA stores) 768 MB 0.492 / 0.949 (configs 3 /
  // 4), 1200 MB 0.473 / 0.949, 1536 MB 0.473 / 0.937: every config's
  // transforms fit in one scratch at 1536 MB (config 3: 164 x 8 MB; config 4:
  // 768 x 2 MB; config 1: 2400 x 512 KB), which also lets the column pass run
  // as one launch (enqueue_spectral). OCN_SCRATCH_MB overrides.
  static const size_t budget = [] {
    const char* e = getenv("OCN_SCRATCH_MB");
    return (size_t)(e && atoi(e) > 0 ? atoi(e) : 1536) << 20;
  }();
  size_t per = (size_t)n * n * sizeof(float2);
  size_t g = budget / per;
  if (g < 1) g = 1;
  if (g > (size_t)total) g = total;
  return g;
}

}  // namespace

// Builds (or fetches) the transform list of one spectral step.
static SpectralPlan* get_plan(ocn_cascades* cas, ocn_maps* maps, ocn_slices* slices) {
  auto key = std::make_pair((const void*)maps, (const void*)slices);
  auto it = cas->plans.find(key);
  if (it != cas->plans.end()) return it->second.get();
  auto plan = std::make_unique<SpectralPlan>();
  plan->need_surface = maps != nullptr;
  plan->need_velocity = slices != nullptr;
  // Surface transforms of every grid first, then the velocity transforms, so
  // that every transform group is of one family (one row-kernel variant each).
  if (maps) {
    static const int pairs[4][2] = {{OCN_FIELD_H, OCN_FIELD_DX},
                                    {OCN_FIELD_DZ, OCN_FIELD_DXDX},
                                    {OCN_FIELD_DZDX, OCN_FIELD_DZDZ},
                                    {OCN_FIELD_HX, OCN_FIELD_HZ}};
    for (int c = 0; c < cas->count; ++c)
      for (int p = 0; p < 4; ++p) {
        plan->host_desc.push_back({c, p, 0.f, 0.f, maps->field(c, pairs[p][0]),
                                   maps->field(c, pairs[p][1])});
        plan->info.push_back({c, p, pairs[p][0], pairs[p][1], 0, 1, 0.0, 0.0});
      }
  }
  if (slices) {
    const int D = slices->cfg.count;
    for (int c = 0; c < cas->count; ++c) {
      for (int d = 0; d < D; ++d) {
        plan->host_desc.push_back({c, kVelXZ, (float)slices->depths[d], 0.f,
                                   slices->field(d, c, 0), slices->field(d, c, 2)});
        plan->info.push_back({c, kVelXZ, d, d, 0, 1, slices->depths[d], 0.0});
      }
      for (int d0 = 0; d0 < D; d0 += 2) {
        if (d0 + 1 < D) {
          plan->host_desc.push_back({c, kVelYPair, (float)slices->depths[d0],
                                     (float)slices->depths[d0 + 1], slices->field(d0, c, 1),
                                     slices->field(d0 + 1, c, 1)});
          plan->info.push_back({c, kVelYPair, d0, d0 + 1, 0, 1, slices->depths[d0],
                                slices->depths[d0 + 1]});
        } else {
          plan->host_desc.push_back({c, kVelYSingle, (float)slices->depths[d0], 0.f,
                                     slices->field(d0, c, 1), nullptr});
          plan->info.push_back({c, kVelYSingle, d0, -1, 0, 1, slices->depths[d0], 0.0});
        }
      }
    }
  }
  // Depth-attenuated velocity transforms that are exactly zero: every mode of
  // grid c has |k| >= band_min (others have h0 = 0), so at depth y < 0 the
  // attenuation 2^(|k| y log2 e) of every mode is at most 2^(band_min y log2 e);
  // below 2^-132 the row pass's ex2.approx.ftz returns 0 for all of them and
  // the whole transform is 0. Such transforms are dropped from the step and
  // their output planes zeroed once here (OCN_NO_DEPTH_SKIP=1 keeps them).
  // At config 3 this drops 31 of the 48 velocity transforms of the 4 m grid
  // and 13 of the 16 m grid.
  {
    static const bool skip = [] {
      const char* e = getenv("OCN_NO_DEPTH_SKIP");
      return !(e && *e && *e != '0');
    }();
    auto dead = [&](int c, float y) {
      const double bmin = cas->band_min[c] * (1.0 - 1e-5);
      return y < 0.f && bmin * (-(double)y) * 1.4426950408889634 >= 132.0;
    };
    // Per-transform row band: the grid's, narrowed at depth y < 0 to the modes
    // whose attenuation survives fp32: |kx| < 132 / (|y| log2 e) (the pair
    // transforms take the shallower of their two depths).
    auto depth_rows = [&](int c, float y) {
      if (!(y < 0.f)) return cas->n / 2 + 1;
      const double kmax = 132.0 / ((-(double)y) * 1.4426950408889634) * (1.0 + 1e-5);
      const double rh = std::ceil(kmax / (2.0 * kPi / cas->lengths[c]));
      return rh > cas->n / 2 ? cas->n / 2 + 1 : (int)rh;
    };
    std::vector<XformDesc> keep;
    for (size_t xi = 0; xi < plan->host_desc.size(); ++xi) {
      XformDesc d = plan->host_desc[xi];
      {
        const double rg = std::ceil(cas->band_max[d.cascade] * (1.0 + 1e-9) /
                                    (2.0 * kPi / cas->lengths[d.cascade]));
        d.row_half = rg > cas->n / 2 ? cas->n / 2 + 1 : (int)rg;  // = GridConst::row_half
        if (d.kind == kVelXZ || d.kind == kVelYSingle)
          d.row_half = std::min(d.row_half, depth_rows(d.cascade, d.y0));
        else if (d.kind == kVelYPair)
          d.row_half = std::min(d.row_half, std::max(depth_rows(d.cascade, d.y0),
                                                     depth_rows(d.cascade, d.y1)));
      }
      plan->info[xi].row_half = d.row_half;
      bool zero = false;
      if (skip && d.kind == kVelXZ) zero = dead(d.cascade, d.y0);
      else if (skip && d.kind == kVelYPair) zero = dead(d.cascade, d.y0) && dead(d.cascade, d.y1);
      else if (skip && d.kind == kVelYSingle) zero = dead(d.cascade, d.y0);
      if (!zero) {
        keep.push_back(d);
        continue;
      }
      plan->info[xi].executed = 0;
      const size_t bytes = (size_t)cas->n * cas->n * sizeof(float);
      OCN_CUDA(cudaMemsetAsync(d.out_re, 0, bytes, cas->ctx->stream));
      if (d.out_im) OCN_CUDA(cudaMemsetAsync(d.out_im, 0, bytes, cas->ctx->stream));
      ++plan->zero_transforms;
    }
    plan->host_desc.swap(keep);
  }
  // (16-byte store boxes: PC >= 4 columns, i.e. N <= 2048)
  if (cas->cols_map_ok && cols_tma_store() && cols_tma_pc(cas->n) >= 4)
    build_out_maps(cas->n, plan->host_desc.data(), (int)plan->host_desc.size(), plan->out_maps);
  plan->desc.alloc(plan->host_desc.size());
  OCN_CUDA(cudaMemcpy(plan->desc.p, plan->host_desc.data(),
                      plan->host_desc.size() * sizeof(XformDesc), cudaMemcpyHostToDevice));
  // groups of G consecutive transforms (spanning grids), split into per-grid segments
  std::vector<GroupSeg> segs;
  const int total = (int)plan->host_desc.size();
  auto family = [&](int i) { return plan->host_desc[i].kind <= kSurfHxHz ? 0 : 1; };
  for (int g0 = 0; g0 < total;) {
    // the family's remaining run, split into equal groups of <= cas->group
    // (balanced groups: 96 + 96 beat 128 + 64 at config 3, 1.11 vs 1.16 ms)
    int run = 1;
    while (g0 + run < total && family(g0 + run) == family(g0)) ++run;
    const int ngroups = (run + cas->group - 1) / cas->group;
    const int cnt = (run + ngroups - 1) / ngroups;
    SpectralPlan::Group gr{g0, cnt, (int)segs.size(), 0, 0, family(g0)};
    for (int i = 0; i < gr.count; ++i) {
      const int c = plan->host_desc[g0 + i].cascade;
      if (gr.nseg == 0 || segs.back().grid != c) {
        segs.push_back({c, i, 0, 0});
        ++gr.nseg;
      }
      ++segs.back().count;
      gr.max_seg = std::max(gr.max_seg, segs.back().count);
    }
    plan->groups.push_back(gr);
    g0 += cnt;
  }
  plan->segs.alloc(std::max<size_t>(segs.size(), 1));
  if (!segs.empty())
    OCN_CUDA(cudaMemcpy(plan->segs.p, segs.data(), segs.size() * sizeof(GroupSeg),
                        cudaMemcpyHostToDevice));
  SpectralPlan* raw = plan.get();
  cas->plans[key] = std::move(plan);
  return raw;
}

static void forget_plans(ocn_cascades* cas, const void* obj) {
  for (auto it = cas->plans.begin(); it != cas->plans.end();) {
    if (it->first.first == obj || it->first.second == obj)
      it = cas->plans.erase(it);
    else
      ++it;
  }
}

static void assemble_grids(ocn_maps* m, cudaStream_t st) {
  ocn_ctx* ctx = m->cas->ctx;
  const size_t nn = (size_t)m->cas->n * m->cas->n;
  OCN_REQUIRE(nn % 4 == 0 && m->assembled.p, "assembly planes missing");
  k_assemble_grid<<<grid_for(ctx, nn / 4 * m->cas->count), 256, 0, st>>>(m->cas->count, nn,
                                                                         m->fields.p, m->assembled.p);
  OCN_LAUNCHED(ctx);
}

static void enqueue_spectral(ocn_cascades* cas, SpectralPlan* plan, ocn_maps* maps,
                             double choppiness) {
  ocn_ctx* ctx = cas->ctx;
  const int n = cas->n;
  const size_t nn = (size_t)n * n;
  cudaStream_t A = ctx->stream;
  ProfWindow whole(ctx, OCN_PROF_SPECTRAL);
  // Time-batched frame sets with N in the warp row kernel's range: the row pass
  // evaluates h~ / G itself (no spectrum round trip through memory, no evolve
  // launch). Measured on B200: config 1 0.998 -> 0.953 ms per 10 frames; for
  // single-frame sets the extra per-row table loads cost more than the evolve
  // pass saves (config 3 0.491 -> 0.514, config 4 0.947 -> 0.971), so those keep
  // k_evolve. OCN_NO_FUSED_EVOLVE=1 keeps it everywhere.
  const bool fused = n >= 128 && n <= 1024 && cas->frames > 1 && fused_evolve_enabled();
  if (!fused) {
    ProfWindow pw(ctx, OCN_PROF_EVOLVE);  // every grid in one launch
    // skip never-read rows only where every reader is a band-aware warp row kernel
    const int skip = n >= 128 && n <= 1024 && cas->cols_map_ok && band_skip_enabled() ? 1 : 0;
    const size_t total = nn * cas->base;  // table modes; each evolved for every frame
    if (plan->need_velocity)
      k_evolve<true><<<grid_for(ctx, total), 256, 0, A>>>(
          total, ilog2(n), cas->base, cas->frames, cas->d_time.p, cas->h0p.p, cas->omega.p,
          cas->spec_h.p, cas->spec_g.p, cas->gconst.p, skip);
    else
      k_evolve<false><<<grid_for(ctx, total), 256, 0, A>>>(
          total, ilog2(n), cas->base, cas->frames, cas->d_time.p, cas->h0p.p, cas->omega.p,
          cas->spec_h.p, nullptr, cas->gconst.p, skip);
    OCN_LAUNCHED(ctx);
  }
  // When every transform of the step fits in the scratch at once, the family
  // groups' row passes write disjoint scratch ranges and ONE column launch
  // covers all of them (config 3: 7 -> 4 launches, no per-group column-pass
  // tail; measured 0.473 -> see DESIGN.md). OCN_NO_MERGED_COLS=1 keeps one
  // column launch per group.
  int all = 0;
  for (const auto& gr : plan->groups) all += gr.count;
  const bool merged = plan->groups.size() > 1 && all <= cas->group && merged_cols_enabled();
  const bool band = cas->cols_map_ok && band_skip_enabled();
  auto run_cols = [&](int first, int count) {
    ColArgs ca{};
    ca.scratch = cas->scratch.p;
    ca.desc = plan->desc.p + first;
    ca.tw = cas->twiddle.p;
    ca.out_maps = plan->out_maps.p ? plan->out_maps.p + 2 * first : nullptr;
    ca.gc = band ? cas->gconst.p : nullptr;
    ProfWindow pw(ctx, OCN_PROF_COLS);
    cols_dispatch(ctx, n, ca, count, false, A, cas->cols_map_ok ? &cas->cols_map : nullptr,
                  cas->cols_map_ok ? &cas->cols_chunk_map : nullptr);
  };
  size_t off = 0;  // merged: this group's first scratch slot
  for (size_t gidx = 0; gidx < plan->groups.size(); ++gidx) {
    const SpectralPlan::Group& gr = plan->groups[gidx];
    float2* scratch = cas->scratch.p + (merged ? off * nn : 0);
    off += gr.count;
    RowArgs ra{};
    ra.items = n * gr.count;
    ra.G = gr.count;
    ra.desc = plan->desc.p + gr.first;
    ra.segs = plan->segs.p + gr.seg0;
    ra.spec_h = cas->spec_h.p;
    ra.spec_g = cas->spec_g.p;
    ra.gc = cas->gconst.p;
    ra.chop = (float)choppiness;
    ra.scratch = scratch;
    ra.tw = cas->twiddle.p;
    // band-limited grids: the row pass skips the exactly-zero rows and the
    // TMA column pass reads only the band rows (off with OCN_NO_BAND_SKIP=1)
    ra.skip_zero_rows = band ? 1 : 0;
    if (fused) {
      ra.h0p = cas->h0p.p;
      ra.omega = cas->omega.p;
      ra.d_time = cas->d_time.p;
    }
    {
      ProfWindow pw(ctx, OCN_PROF_ROWS);
      rows_dispatch(ctx, n, ra, false, A, gr.nseg, gr.max_seg, gr.family);
    }
    if (!merged) run_cols(gr.first, gr.count);
  }
  if (merged) run_cols(plan->groups[0].first, all);
  if (plan->assembly && maps) assemble_grids(maps, A);
}

static bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("OCN_NO_GRAPH");
    return !(e && *e && *e != '0');
  }();
  return on;
}

void spectral_step(ocn_cascades* cas, ocn_maps* maps, ocn_slices* slices, double t,
                   double choppiness, double dt) {
  NvtxRange nv(slices ? (maps ? "surface+velocity" : "velocity") : "surface");
  ocn_ctx* ctx = cas->ctx;
  DeviceScope ds(ctx);
  OCN_REQUIRE(cas->h0.p, "these maps carry no spectrum (ocn_maps_create_bare)");
  SpectralPlan* plan = get_plan(cas, maps, slices);
  const bool assembly = maps && maps->assembly;
  if (plan->assembly != assembly) {  // the captured graph has (or lacks) the assembly node
    if (plan->exec) cudaGraphExecDestroy(plan->exec), plan->exec = nullptr;
    plan->assembly = assembly;
  }
  k_set_time<<<1, 1, 0, ctx->stream>>>(cas->d_time.p, t, dt < 0.0 ? cas->frame_dt : dt);
  OCN_LAUNCHED(ctx);
  // profiling mode 1 = per-kernel windows (eager launches); mode 2 = stage
  // windows only, the step still replays its graph
  const bool use_graph = graphs_enabled() && ctx->prof_mode != 1 && plan->uses > 0;
  if (use_graph && (!plan->exec || plan->graph_chop != choppiness)) {
    if (plan->exec) cudaGraphExecDestroy(plan->exec), plan->exec = nullptr;
    const uint64_t before = ctx->launches.load();
    cudaGraph_t graph;
    const bool prof = ctx->profiling;
    ctx->profiling = false;  // no event windows inside the captured graph
    OCN_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
    try {
      enqueue_spectral(cas, plan, maps, choppiness);
      ctx->profiling = prof;
    } catch (...) {
      ctx->profiling = prof;
      cudaStreamEndCapture(ctx->stream, &graph);
      throw;
    }
    OCN_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
    cudaError_t e = cudaGraphInstantiate(&plan->exec, graph, 0);
    cudaGraphDestroy(graph);
    OCN_CUDA(e);
    plan->graph_kernels = ctx->launches.load() - before;
    ctx->launches.fetch_sub(plan->graph_kernels);  // captured, not executed
    plan->graph_chop = choppiness;
  }
  if (use_graph) {
    ProfWindow pw(ctx, OCN_PROF_SPECTRAL);
    OCN_CUDA(cudaGraphLaunch(plan->exec, ctx->stream));
    ctx->launches.fetch_add(plan->graph_kernels);
  } else {
    enqueue_spectral(cas, plan, maps, choppiness);
  }
  ++plan->uses;
  if (maps) {
    maps->time = t;
    maps->choppiness = choppiness;
  }
  if (slices) slices->time = t;
}

// Plain packed transform(s) on device buffers: src [G][n][n] -> split or complex.
static void plain_ifft(ocn_ctx* ctx, int n, int G, const float2* src, float2* scratch,
                       const float2* tw, const XformDesc* d_desc, float2* out_c) {
  RowArgs ra{};
  ra.items = n * G;
  ra.G = G;
  ra.src = src;
  ra.scratch = scratch;
  ra.tw = tw;
  rows_dispatch(ctx, n, ra, true, ctx->stream);
  ColArgs ca{};
  ca.scratch = scratch;
  ca.desc = d_desc;
  ca.out_c = out_c;
  ca.tw = tw;
  CUtensorMap map;
  const bool tma_ok = cols_map_for(n, G, scratch, &map);
  cols_dispatch(ctx, n, ca, G, out_c != nullptr, ctx->stream, tma_ok ? &map : nullptr);
}

}  // namespace ocn

using namespace ocn;

// =========================================================================== C-ABI
extern "C" {

int ocn_abi_version(void) { return OCN_ABI_VERSION; }

int ocn_ctx_create_priority(int device, int priority, ocn_ctx** out) {
  return api_call(nullptr, [&] {
    OCN_REQUIRE(out, "ocn_ctx_create: out is NULL");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      fail(OCN_ERR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    }
    OCN_REQUIRE(device >= 0 && device < ndev, "ocn_ctx_create: device %d out of range", device);
    auto ctx = std::make_unique<ocn_ctx>();
    ctx->device = device;
    OCN_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    OCN_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(OCN_ERR_CUDA, "libocean_b200 is built for sm_100a; device %d is sm_%d%d", device,
           prop.major, prop.minor);
    ctx->sm_count = prop.multiProcessorCount;
    OCN_REQUIRE(priority >= -1 && priority <= 1, "ocn_ctx_create_priority: priority %d", priority);
    int lo = 0, hi = 0;  // CUDA: lower numbers are higher priorities
    OCN_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const int prio = priority > 0 ? hi : (priority < 0 ? lo : 0);
    ctx->priority = priority;
    OCN_CUDA(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, prio));
    *out = ctx.release();
  });
}

int ocn_ctx_create(int device, ocn_ctx** out) { return ocn_ctx_create_priority(device, 0, out); }

int ocn_ctx_destroy(ocn_ctx* ctx) {
  ocn::ctx_release(ctx);
  return OCN_OK;
}

const char* ocn_last_error(const ocn_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : ocn::global_error().c_str();
}

int ocn_ctx_synchronize(ocn_ctx* ctx) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx, "null context");
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ocn_ctx_profile(ocn_ctx* ctx, int mode) {
  if (!ctx) return OCN_ERR_ARG;
  ctx->profiling = mode != 0;
  ctx->prof_mode = mode;
  return OCN_OK;
}

static void prof_resolve(ocn_ctx* ctx) {
  OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto& w : ctx->prof_pending) {
    float ms = 0.f;
    OCN_CUDA(cudaEventElapsedTime(&ms, w.start, w.stop));
    ctx->prof_ms[w.cat] += ms;
    ctx->prof_count[w.cat] += 1;
    ctx->prof_pool.push_back(w.start);
    ctx->prof_pool.push_back(w.stop);
  }
  ctx->prof_pending.clear();
}

int ocn_ctx_profile_read(ocn_ctx* ctx, int category, double* total_ms, uint64_t* count) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && category >= 0 && category < OCN_PROF_COUNT, "bad profile category");
    DeviceScope ds(ctx);
    prof_resolve(ctx);
    if (total_ms) *total_ms = ctx->prof_ms[category];
    if (count) *count = ctx->prof_count[category];
  });
}

int ocn_ctx_profile_reset(ocn_ctx* ctx) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx, "null context");
    DeviceScope ds(ctx);
    prof_resolve(ctx);
    for (int k = 0; k < OCN_PROF_COUNT; ++k) ctx->prof_ms[k] = 0.0, ctx->prof_count[k] = 0;
  });
}

void* ocn_ctx_stream(ocn_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

uint64_t ocn_ctx_kernel_launches(const ocn_ctx* ctx) {
  return ctx ? ctx->launches.load(std::memory_order_relaxed) : 0;
}

// ---- spectrum scalars (host evaluation of the same __host__ __device__ code)
int ocn_spectrum_validate(const ocn_spectrum_params* p) {
  return api_call(nullptr, [&] {
    OCN_REQUIRE(p, "null params");
    if (!(p->wind_speed > 0.0)) fail(OCN_ERR_CONFIG, "wind_speed must be > 0");
    if (!(p->fetch > 0.0)) fail(OCN_ERR_CONFIG, "fetch must be > 0");
    if (p->swell < 0.0 || p->swell > 1.0) fail(OCN_ERR_CONFIG, "swell must be in [0, 1]");
    if (p->direction_mix < 0.0 || p->direction_mix > 1.0)
      fail(OCN_ERR_CONFIG, "direction_mix must be in [0, 1]");
    if (!(p->gravity > 0.0)) fail(OCN_ERR_CONFIG, "gravity must be > 0");
    if (p->has_peak_omega_override && !(p->peak_omega_override > 0.0))
      fail(OCN_ERR_CONFIG, "peak_omega_override must be > 0");
  });
}
double ocn_alpha(const ocn_spectrum_params* p) { return sm::alpha(*p); }
double ocn_peak_omega(const ocn_spectrum_params* p) { return sm::peak_omega(*p); }
double ocn_standard_peak_omega(const ocn_spectrum_params* p) { return sm::standard_peak_omega(*p); }
double ocn_dispersion(double k, double g) { return sqrt(g * k); }
int ocn_jonswap(double omega, const ocn_spectrum_params* p, double* out) {
  return api_call(nullptr, [&] {
    if (!sm::jonswap(omega, *p, out)) fail(OCN_ERR_DOMAIN, "jonswap: omega must be > 0");
  });
}
double ocn_beta_s(double r) { return sm::beta_s(r); }
double ocn_directional_kernel(double b, double t) { return sm::directional_kernel(b, t); }
double ocn_donelan_banner(double w, double t, double wp) { return sm::donelan_banner(w, t, wp); }
double ocn_swell_spread(double w, double t, double wp, double xi) {
  return sm::swell_spread(w, t, wp, xi);
}
double ocn_q_dbxi_approx(double r) { return sm::q_dbxi_approx(r); }
double ocn_q_dbxi_quadrature(double r, double xi, int panels) {
  // composite Simpson over [-pi, pi] (spectra.cpp:84-98)
  double beta = sm::beta_s(r);
  double s = 16.0 * tanh(1.0 / r) * xi * xi;
  auto f = [&](double th) {
    double c = fabs(cos(0.5 * th));
    double spread = (s == 0.0) ? 1.0 : (c == 0.0 ? 0.0 : pow(c, 2.0 * s));
    return sm::directional_kernel(beta, th) * spread;
  };
  double h = 2.0 * kPi / panels;
  double acc = f(-kPi) + f(kPi);
  for (int i = 1; i < panels; ++i) acc += f(-kPi + h * i) * ((i & 1) ? 4.0 : 2.0);
  return 1.0 / (acc * h / 3.0);
}
double ocn_directional(double w, double t, const ocn_spectrum_params* p) {
  return sm::directional(w, t, *p);
}
double ocn_h0_variance(double kx, double kz, double k, double omega, double L,
                       const ocn_spectrum_params* p) {
  return sm::h0_variance(kx, kz, k, omega, L, *p);
}
double ocn_damping_factor(double speed, double d0, double d_max, double v_max) {
  return sm::damping_factor(speed, d0, d_max, v_max);
}
double ocn_attenuation(double k, double y) { return sm::attenuation(k, y); }
int ocn_log_distribution(double y, double y_min, double* out) {
  return api_call(nullptr, [&] {
    if (!(y_min < 0.0)) fail(OCN_ERR_DOMAIN, "log_distribution: y_min must be negative");
    const double alpha = 0.0001;
    double beta = -y_min / (2.0 * log(alpha * y_min * y_min + 1.0));
    double v = beta * log(alpha * y * y + 1.0);
    *out = y > 0.0 ? v : -v;
  });
}
int ocn_exp_interp(double a, double fa, double b, double fb, double x, double* out) {
  return api_call(nullptr, [&] {
    if (a == b) fail(OCN_ERR_DOMAIN, "exp_interp: endpoints coincide");
    bool degenerate = fabs(fa) < 1e-12 || fabs(fb) < 1e-12 || ((fa < 0.0) != (fb < 0.0));
    if (degenerate) {
      *out = fa + (fb - fa) * ((x - a) / (b - a));
      return;
    }
    double beta = (log(fabs(fb)) - log(fabs(fa))) / (b - a);
    *out = fa * exp(beta * (x - a));
  });
}
int ocn_slice_depths(const ocn_slice_config* cfg, double* depths) {
  return api_call(nullptr, [&] {
    OCN_REQUIRE(cfg && depths, "null argument");
    if (!(cfg->y_min < cfg->y_max)) fail(OCN_ERR_CONFIG, "slice interval requires y_min < y_max");
    if (cfg->count < 2) fail(OCN_ERR_CONFIG, "at least two depth slices are required");
    if (cfg->distribution == OCN_DEPTH_LOGARITHMIC && !(cfg->y_min < 0.0))
      fail(OCN_ERR_CONFIG, "logarithmic distribution requires y_min < 0");
    std::vector<double> d(cfg->count);
    for (int i = 0; i < cfg->count; ++i) {
      double pre = cfg->y_min + (cfg->y_max - cfg->y_min) * i / (cfg->count - 1);
      if (cfg->distribution == OCN_DEPTH_LOGARITHMIC)
        ocn_log_distribution(pre, cfg->y_min, &d[i]);
      else
        d[i] = pre;
    }
    std::sort(d.begin(), d.end());
    std::memcpy(depths, d.data(), d.size() * sizeof(double));
  });
}

// ---- cascades (K1)
// `count` grids with tables (spectrum init, h0 / w tables), each repeated for
// `frames` frames (time-batched sets; frames = 1 otherwise): grid f * count + c
// evaluates grid c's spectrum at t + f dt.
static void cascades_create(ocn_ctx* ctx, int resolution, int count, const double* lengths,
                            const double* band_min, const double* band_max,
                            const uint32_t* cascade_index, const ocn_spectrum_params* params,
                            int frames, double frame_dt, ocn_cascades** out) {
  OCN_REQUIRE(ctx && out && lengths && band_min && band_max && params, "null argument");
  OCN_REQUIRE(count >= 1 && count <= kMaxGrids, "grid count %d out of range", count);
  OCN_REQUIRE(frames >= 1 && (size_t)frames * count <= (size_t)kMaxGrids,
              "frames x grids %d x %d out of range", frames, count);
  if (!is_pow2(resolution) || resolution < 2)
    fail(OCN_ERR_CONFIG, "grid resolution must be a power of two >= 2");
  if (resolution > 16384) fail(OCN_ERR_CONFIG, "grid resolution above 16384 is not supported");
  for (int c = 0; c < count; ++c) {
    if (!(lengths[c] > 0.0)) fail(OCN_ERR_CONFIG, "cascade length must be > 0");
    if (!(band_min[c] >= 0.0) || !(band_max[c] > band_min[c]))
      fail(OCN_ERR_CONFIG, "cascade band must satisfy 0 <= band_min < band_max");
    int st = ocn_spectrum_validate(params + c);
    if (st) fail(st, "%s", global_error().c_str());
  }
  DeviceScope ds(ctx);
  auto cas = std::make_unique<ocn_cascades>();
  const int total = count * frames;
  cas->ctx = ctx;
  cas->n = resolution;
  cas->count = total;
  cas->base = count;
  cas->frames = frames;
  cas->frame_dt = frame_dt;
  for (int f = 0; f < frames; ++f) {
    cas->lengths.insert(cas->lengths.end(), lengths, lengths + count);
    cas->band_min.insert(cas->band_min.end(), band_min, band_min + count);
    cas->band_max.insert(cas->band_max.end(), band_max, band_max + count);
    for (int c = 0; c < count; ++c)
      cas->cascade_index.push_back(cascade_index ? cascade_index[c] : (uint32_t)c);
    cas->grid_params.insert(cas->grid_params.end(), params, params + count);
  }
  cas->params = params[0];
  const size_t nn = (size_t)resolution * resolution;
  cas->h0_f64.alloc(nn * count);
  cas->h0.alloc(nn * count);
  cas->in_band.alloc(nn * count);
  cas->h0p.alloc(nn * count);
  cas->omega.alloc(nn * count);
  cas->spec_h.alloc(nn * total);
  cas->spec_g.alloc(nn * total);
  std::vector<GridConst> gc(total);
  for (int g = 0; g < total; ++g) {
    const int c = g % count;
    gc[g].dk = 2.0 * kPi / lengths[c];
    gc[g].length = lengths[c];
    gc[g].band_min = band_min[c];
    gc[g].band_max = band_max[c];
    gc[g].cindex = cas->cascade_index[c];
    gc[g].p = params[c];
    // rows with |kx| >= band_max (1 + 1e-9) are outside the band whatever kz
    // (hypot(kx, kz) >= |kx|; the margin covers rounding)
    const double rh = std::ceil(band_max[c] * (1.0 + 1e-9) / gc[g].dk);
    gc[g].row_half = rh > resolution / 2 ? resolution / 2 + 1 : (int)rh;
    gc[g].src = c;
    gc[g].frame = g / count;
  }
  cas->gconst.alloc(total);
  OCN_CUDA(cudaMemcpyAsync(cas->gconst.p, gc.data(), total * sizeof(GridConst),
                           cudaMemcpyHostToDevice, ctx->stream));
  k_spectrum_init<<<grid_for(ctx, nn * count), 256, 0, ctx->stream>>>(
      resolution, count, cas->gconst.p, cas->h0_f64.p, cas->h0.p, cas->in_band.p);
  OCN_LAUNCHED(ctx);
  k_evolve_tables<<<grid_for(ctx, nn * count), 256, 0, ctx->stream>>>(
      resolution, count, cas->gconst.p, cas->h0.p, cas->h0p.p, cas->omega.p);
  OCN_LAUNCHED(ctx);
  std::vector<float2> tw = make_twiddles(resolution);
  cas->twiddle.alloc(tw.size());
  OCN_CUDA(cudaMemcpyAsync(cas->twiddle.p, tw.data(), tw.size() * sizeof(float2),
                           cudaMemcpyHostToDevice, ctx->stream));
  cas->group = (int)group_for(resolution, 1 << 30);
  cas->d_time.alloc(2);
  cas->scratch.alloc((size_t)cas->group * nn);
  cas->cols_map_ok = cols_map_for(resolution, cas->group, cas->scratch.p, &cas->cols_map);
  if (cas->cols_map_ok)
    cols_map_for(resolution, cas->group, cas->scratch.p, &cas->cols_chunk_map, true);
  OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx_retain(ctx);
  *out = cas.release();
}

int ocn_cascades_create_multi(ocn_ctx* ctx, int resolution, int count, const double* lengths,
                              const double* band_min, const double* band_max,
                              const uint32_t* cascade_index, const ocn_spectrum_params* params,
                              ocn_cascades** out) {
  return api_call(ctx, [&] {
    cascades_create(ctx, resolution, count, lengths, band_min, band_max, cascade_index, params, 1,
                    0.0, out);
  });
}

int ocn_cascades_create_frames(ocn_ctx* ctx, int resolution, int count, const double* lengths,
                               const double* band_min, const double* band_max,
                               const uint32_t* cascade_index, const ocn_spectrum_params* params,
                               int frames, double dt, ocn_cascades** out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(params, "null argument");
    std::vector<ocn_spectrum_params> ps(count > 0 ? count : 0, *params);
    cascades_create(ctx, resolution, count, lengths, band_min, band_max, cascade_index, ps.data(),
                    frames, dt, out);
  });
}

int ocn_cascades_create(ocn_ctx* ctx, int resolution, int count, const double* lengths,
                        const double* band_min, const double* band_max,
                        const uint32_t* cascade_index, const ocn_spectrum_params* params,
                        ocn_cascades** out) {
  if (!params || count < 1 || count > kMaxGrids) {
    global_error() = "bad cascade arguments";
    if (ctx) ctx->last_error = global_error();
    return OCN_ERR_ARG;
  }
  std::vector<ocn_spectrum_params> ps(count, *params);
  return ocn_cascades_create_multi(ctx, resolution, count, lengths, band_min, band_max,
                                   cascade_index, ps.data(), out);
}

int ocn_cascades_destroy(ocn_cascades* c) {
  cascades_release(c);
  return OCN_OK;
}

int ocn_cascades_info(const ocn_cascades* c, int* resolution, int* count) {
  if (!c) return OCN_ERR_ARG;
  if (resolution) *resolution = c->n;
  if (count) *count = c->count;
  return OCN_OK;
}

int ocn_cascades_download(ocn_cascades* c, int grid, double* h0, double* h0cn, uint8_t* in_band,
                          double* waves) {
  return api_call(c ? c->ctx : nullptr, [&] {
    OCN_REQUIRE(c && grid >= 0 && grid < c->count, "bad cascade handle / index");
    ocn_ctx* ctx = c->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)c->n * c->n;
    grid %= c->base;  // time-batched sets: one table per cascade
    const double2* src = c->h0_f64.p + (size_t)grid * nn;
    if (h0)
      OCN_CUDA(cudaMemcpyAsync(h0, src, nn * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    if (in_band)
      OCN_CUDA(cudaMemcpyAsync(in_band, c->in_band.p + (size_t)grid * nn, nn,
                               cudaMemcpyDeviceToHost, ctx->stream));
    if (h0cn || waves) {
      DevBuf<double2> d_cn(h0cn ? nn : 0);
      DevBuf<double4> d_w(waves ? nn : 0);
      k_grid_extras<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(
          c->n, 2.0 * kPi / c->lengths[grid], c->grid_params[grid].gravity, src, d_cn.p, d_w.p);
      OCN_LAUNCHED(ctx);
      if (h0cn)
        OCN_CUDA(cudaMemcpyAsync(h0cn, d_cn.p, nn * sizeof(double2), cudaMemcpyDeviceToHost,
                                 ctx->stream));
      if (waves)
        OCN_CUDA(cudaMemcpyAsync(waves, d_w.p, nn * sizeof(double4), cudaMemcpyDeviceToHost,
                                 ctx->stream));
      OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ocn_assemble_coefficients(ocn_cascades* c, int grid, double t, double chop, double* out) {
  return api_call(c ? c->ctx : nullptr, [&] {
    OCN_REQUIRE(c && out && grid >= 0 && grid < c->count, "bad arguments");
    ocn_ctx* ctx = c->ctx;
    DeviceScope ds(ctx);
    grid %= c->base;
    const size_t nn = (size_t)c->n * c->n;
    DevBuf<double2> d(8 * nn);
    k_assemble_coef<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(
        c->n, 2.0 * kPi / c->lengths[grid], c->grid_params[grid].gravity, t, chop,
        c->h0_f64.p + (size_t)grid * nn, c->in_band.p + (size_t)grid * nn, d.p);
    OCN_LAUNCHED(ctx);
    OCN_CUDA(cudaMemcpyAsync(out, d.p, 8 * nn * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---- maps
int ocn_maps_create(ocn_cascades* c, ocn_maps** out) {
  return api_call(c ? c->ctx : nullptr, [&] {
    OCN_REQUIRE(c && out, "null argument");
    DeviceScope ds(c->ctx);
    auto m = std::make_unique<ocn_maps>();
    m->cas = c;
    const size_t nn = (size_t)c->n * c->n;
    m->fields.alloc(nn * 8 * c->count);
    OCN_CUDA(cudaMemsetAsync(m->fields.p, 0, m->fields.bytes(), c->ctx->stream));
    ++c->refs;
    *out = m.release();
  });
}

int ocn_maps_destroy(ocn_maps* m) {
  if (!m) return OCN_OK;
  ocn_cascades* c = m->cas;
  {
    DeviceScope ds(c->ctx);
    cudaStreamSynchronize(c->ctx->stream);
    forget_plans(c, m);
    delete m;
  }
  cascades_release(c);
  return OCN_OK;
}

int ocn_surface_generate(ocn_maps* m, double t, double choppiness) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m, "null maps");
    spectral_step(m->cas, m, nullptr, t, choppiness);
  });
}

int ocn_maps_time(const ocn_maps* m, double* t) {
  if (!m || !t) return OCN_ERR_ARG;
  *t = m->time;
  return OCN_OK;
}

int ocn_maps_download(ocn_maps* m, int cascade, int field, double* out) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && out && cascade >= 0 && cascade < m->cas->count && field >= 0 && field < 8,
                "bad maps download arguments");
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)m->cas->n * m->cas->n;
    DevBuf<double> tmp(nn);
    k_f32_to_f64<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(nn, m->field(cascade, field), tmp.p);
    OCN_LAUNCHED(ctx);
    OCN_CUDA(cudaMemcpyAsync(out, tmp.p, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ocn_surface_generate_batch(ocn_maps* m, double t0, double dt, double choppiness) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m, "ocn_surface_generate_batch: maps is NULL");
    spectral_step(m->cas, m, nullptr, t0, choppiness, dt);
  });
}

int ocn_maps_set_assembly(ocn_maps* m, int enable) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m, "ocn_maps_set_assembly: maps is NULL");
    const size_t nn = (size_t)m->cas->n * m->cas->n;
    if (!m->cas->h0.p) fail(OCN_ERR_CONFIG, "maps without a spectrum have no spectral step");
    if (nn % 4) fail(OCN_ERR_CONFIG, "per-texel assembly needs N >= 2");
    m->assembly = enable != 0;
    if (m->assembly && !m->assembled.p) {
      DeviceScope ds(m->cas->ctx);
      m->assembled.alloc(nn * 4 * m->cas->count);
      OCN_CUDA(cudaMemsetAsync(m->assembled.p, 0, m->assembled.bytes(), m->cas->ctx->stream));
    }
  });
}

int ocn_maps_download_assembly(ocn_maps* m, int cascade, int component, float* out) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && out && cascade >= 0 && cascade < m->cas->count && component >= 0 &&
                    component < 4,
                "bad assembly download arguments");
    if (!m->assembled.p) fail(OCN_ERR_CONFIG, "assembly is not enabled on these maps");
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)m->cas->n * m->cas->n;
    OCN_CUDA(cudaMemcpyAsync(out, m->assembled.p + ((size_t)cascade * 4 + component) * nn,
                             nn * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ocn_maps_download_f32(ocn_maps* m, int cascade, int field, float* out) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && out && cascade >= 0 && cascade < m->cas->count && field >= 0 && field < 8,
                "bad maps download arguments");
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)m->cas->n * m->cas->n;
    OCN_CUDA(cudaMemcpyAsync(out, m->field(cascade, field), nn * sizeof(float),
                             cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

__global__ void k_f64_to_f32_s(size_t n, const double* in, float* out) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x)
    out[q] = (float)in[q];
}

int ocn_maps_create_bare(ocn_ctx* ctx, int n, int count, const double* lengths, ocn_maps** out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && lengths && out, "null argument");
    OCN_REQUIRE(count >= 1 && count <= kMaxCascades, "cascade count %d out of range", count);
    if (!is_pow2(n) || n < 2) fail(OCN_ERR_CONFIG, "grid resolution must be a power of two >= 2");
    DeviceScope ds(ctx);
    // a spectrum-less cascade set carrying only the tile geometry
    auto cas = std::make_unique<ocn_cascades>();
    cas->ctx = ctx;
    cas->n = n;
    cas->count = count;
    cas->base = count;
    cas->lengths.assign(lengths, lengths + count);
    cas->band_min.assign(count, 0.0);
    cas->band_max.assign(count, 1e300);
    for (int c = 0; c < count; ++c) cas->cascade_index.push_back((uint32_t)c);
    cas->params.gravity = kGravity;
    ctx_retain(ctx);
    auto m = std::make_unique<ocn_maps>();
    m->cas = cas.release();
    m->fields.alloc((size_t)n * n * 8 * count);
    OCN_CUDA(cudaMemsetAsync(m->fields.p, 0, m->fields.bytes(), ctx->stream));
    ++m->cas->refs;
    ocn_cascades* bare = m->cas;
    *out = m.release();
    ocn_cascades_destroy(bare);  // the maps now hold the only reference
  });
}

int ocn_maps_upload(ocn_maps* m, int cascade, int field, const double* in) {
  return api_call(m ? m->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(m && in && cascade >= 0 && cascade < m->cas->count && field >= 0 && field < 8,
                "bad maps upload arguments");
    ocn_ctx* ctx = m->cas->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)m->cas->n * m->cas->n;
    DevBuf<double> tmp(nn);
    OCN_CUDA(cudaMemcpyAsync(tmp.p, in, nn * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    k_f64_to_f32_s<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(nn, tmp.p, m->field(cascade, field));
    OCN_LAUNCHED(ctx);
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ocn_maps_device_field(ocn_maps* m, int cascade, int field, const float** dev_out) {
  if (!m || !dev_out || cascade < 0 || cascade >= m->cas->count || field < 0 || field >= 8)
    return OCN_ERR_ARG;
  *dev_out = m->field(cascade, field);
  return OCN_OK;
}

// ---- slices
int ocn_slices_create(ocn_cascades* c, const ocn_slice_config* cfg, ocn_slices** out) {
  return api_call(c ? c->ctx : nullptr, [&] {
    OCN_REQUIRE(c && cfg && out, "null argument");
    std::vector<double> d(cfg->count > 0 ? cfg->count : 1);
    int st = ocn_slice_depths(cfg, d.data());
    if (st) fail(st, "%s", global_error().c_str());
    DeviceScope ds(c->ctx);
    auto s = std::make_unique<ocn_slices>();
    s->cas = c;
    s->cfg = *cfg;
    s->depths = d;
    s->d_depths.alloc(d.size());
    OCN_CUDA(cudaMemcpy(s->d_depths.p, d.data(), d.size() * sizeof(double), cudaMemcpyHostToDevice));
    const size_t nn = (size_t)c->n * c->n;
    s->fields.alloc(nn * 3 * c->count * cfg->count);
    OCN_CUDA(cudaMemsetAsync(s->fields.p, 0, s->fields.bytes(), c->ctx->stream));
    ++c->refs;
    *out = s.release();
  });
}

int ocn_slices_destroy(ocn_slices* s) {
  if (!s) return OCN_OK;
  ocn_cascades* c = s->cas;
  {
    DeviceScope ds(c->ctx);
    cudaStreamSynchronize(c->ctx->stream);
    forget_plans(c, s);
    delete s;
  }
  cascades_release(c);
  return OCN_OK;
}

int ocn_velocity_build(ocn_slices* s, double t) {
  return api_call(s ? s->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(s, "null slices");
    spectral_step(s->cas, nullptr, s, t, 1.0);
  });
}

int ocn_slices_depths(const ocn_slices* s, int* count, double* depths) {
  if (!s) return OCN_ERR_ARG;
  if (count) *count = s->cfg.count;
  if (depths) std::memcpy(depths, s->depths.data(), s->depths.size() * sizeof(double));
  return OCN_OK;
}

int ocn_slices_download(ocn_slices* s, int depth, int cascade, int comp, double* out) {
  return api_call(s ? s->cas->ctx : nullptr, [&] {
    OCN_REQUIRE(s && out && depth >= 0 && depth < s->cfg.count && cascade >= 0 &&
                    cascade < s->cas->count && comp >= 0 && comp < 3,
                "bad slices download arguments");
    ocn_ctx* ctx = s->cas->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)s->cas->n * s->cas->n;
    DevBuf<double> tmp(nn);
    k_f32_to_f64<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(nn, s->field(depth, cascade, comp),
                                                            tmp.p);
    OCN_LAUNCHED(ctx);
    OCN_CUDA(cudaMemcpyAsync(out, tmp.p, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ocn_spectral_step(ocn_maps* m, ocn_slices* s, double t, double choppiness) {
  ocn_cascades* cas = m ? m->cas : (s ? s->cas : nullptr);
  return api_call(cas ? cas->ctx : nullptr, [&] {
    OCN_REQUIRE(cas, "ocn_spectral_step: maps and slices are both NULL");
    OCN_REQUIRE(!m || !s || m->cas == s->cas, "maps and slices belong to different cascades");
    spectral_step(cas, m, s, t, choppiness);
  });
}

int ocn_spectral_plan_info(ocn_maps* m, ocn_slices* s, int capacity, ocn_xform_info* out,
                           int* count) {
  ocn_cascades* cas = m ? m->cas : (s ? s->cas : nullptr);
  return api_call(cas ? cas->ctx : nullptr, [&] {
    OCN_REQUIRE(cas, "ocn_spectral_plan_info: maps and slices are both NULL");
    OCN_REQUIRE(!m || !s || m->cas == s->cas, "maps and slices belong to different cascades");
    OCN_REQUIRE(count, "ocn_spectral_plan_info: count is NULL");
    DeviceScope ds(cas->ctx);
    const SpectralPlan* plan = get_plan(cas, m, s);
    *count = (int)plan->info.size();
    if (out)
      for (int i = 0; i < capacity && i < *count; ++i) out[i] = plan->info[i];
  });
}

// ---- standalone FFT (fp64 host buffers in and out)
static void host_ifft(ocn_ctx* ctx, int n, const double* x, const double* y, double* re,
                      double* im, double* complex_out) {
  if (n < 2 || !is_pow2(n))
    fail(OCN_ERR_CONFIG, "FFT field size must be a power of two >= 2, got %d", n);
  if (n > 16384) fail(OCN_ERR_CONFIG, "FFT size %d above 16384 is not supported", n);
  DeviceScope ds(ctx);
  const size_t nn = (size_t)n * n;
  DevBuf<double2> dx(nn), dy(y ? nn : 0);
  DevBuf<float2> packed(nn), scratch(nn), outc(complex_out ? nn : 0);
  DevBuf<float> dre(complex_out ? 0 : nn), dim(complex_out ? 0 : nn);
  OCN_CUDA(cudaMemcpyAsync(dx.p, x, nn * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  if (y)
    OCN_CUDA(cudaMemcpyAsync(dy.p, y, nn * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  k_pack_pair<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(nn, dx.p, dy.p, packed.p);
  OCN_LAUNCHED(ctx);
  std::vector<float2> tw = make_twiddles(n);
  DevBuf<float2> dtw(tw.size());
  OCN_CUDA(cudaMemcpyAsync(dtw.p, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice,
                           ctx->stream));
  XformDesc hd{0, 0, 0.f, 0.f, dre.p, dim.p};
  DevBuf<XformDesc> dd(1);
  OCN_CUDA(cudaMemcpyAsync(dd.p, &hd, sizeof(hd), cudaMemcpyHostToDevice, ctx->stream));
  plain_ifft(ctx, n, 1, packed.p, scratch.p, dtw.p, dd.p, complex_out ? outc.p : nullptr);
  if (complex_out) {
    DevBuf<double2> o64(nn);
    k_c32_to_c64<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(nn, outc.p, o64.p);
    OCN_LAUNCHED(ctx);
    OCN_CUDA(cudaMemcpyAsync(complex_out, o64.p, nn * sizeof(double2), cudaMemcpyDeviceToHost,
                             ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    DevBuf<double> o64(nn);
    if (re) {
      k_f32_to_f64<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(nn, dre.p, o64.p);
      OCN_LAUNCHED(ctx);
      OCN_CUDA(cudaMemcpyAsync(re, o64.p, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (im) {
      k_f32_to_f64<<<grid_for(ctx, nn), 256, 0, ctx->stream>>>(nn, dim.p, o64.p);
      OCN_LAUNCHED(ctx);
      OCN_CUDA(cudaMemcpyAsync(im, o64.p, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  }
  OCN_CUDA(cudaStreamSynchronize(ctx->stream));
}

int ocn_ifft2_centered(ocn_ctx* ctx, int n, const double* in, double* out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && in && out, "null argument");
    host_ifft(ctx, n, in, nullptr, nullptr, nullptr, out);
  });
}

int ocn_ifft2_pair(ocn_ctx* ctx, int n, const double* x, const double* y, double* re, double* im) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && x && y, "null argument");
    host_ifft(ctx, n, x, y, re, im, nullptr);
  });
}

}  // extern "C"
