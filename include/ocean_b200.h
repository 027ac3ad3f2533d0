/*
 * ocean_b200.h — C-ABI of the B200 (sm_100a) implementation of the Arc Blanc
 * per-frame hot path (arXiv 2503.03326).
 *
 * Every entry point returns an int status (OCN_OK = 0) and never throws. The
 * status values mirror the reference's exception taxonomy
 * (proj/include/ocean/core.hpp:21-35) and the CLI's exit-code mapping
 * (proj/tools/main.cpp:303-320): the C++ drop-in layer (the ocean headers under include/ocean)
 * re-throws ConfigError / MeshError / NumericError / IoError / DomainError with
 * the message from ocn_last_error().
 *
 * Handles are opaque. All device work of one handle family runs on the stream
 * owned by its ocn_ctx; calls marked (async) only enqueue work, calls that
 * return data to host memory synchronize that stream first.
 *
 * Pointers named host_* are host memory. Pointers to sampled positions /
 * outputs of the batched samplers may be host or device memory (the library
 * inspects them with cudaPointerGetAttributes).
 *
 * Which reference interface each entry point replaces is cited per function
 * (file:line relative to the reference tree's proj/ directory).
 */
#ifndef OCEAN_B200_H
#define OCEAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCN_ABI_VERSION 2

#if defined(__GNUC__)
#define OCN_API __attribute__((visibility("default")))
#else
#define OCN_API
#endif

/* ---- status codes (core.hpp:21-35 error types; main.cpp:303-320 exits) ---- */
#define OCN_OK 0
#define OCN_ERR_CONFIG 2  /* ConfigError  */
#define OCN_ERR_MESH 3    /* MeshError    */
#define OCN_ERR_NUMERIC 4 /* NumericError */
#define OCN_ERR_IO 5      /* IoError      */
#define OCN_ERR_DOMAIN 6  /* DomainError  */
#define OCN_ERR_CUDA 7    /* CUDA runtime failure / no device / missing kernel image */
#define OCN_ERR_ARG 8     /* null handle or bad argument (programming error) */

/* ---- surface field order: surface.hpp:43-53 (enum SurfaceField) ---- */
#define OCN_FIELD_H 0
#define OCN_FIELD_DX 1
#define OCN_FIELD_DZ 2
#define OCN_FIELD_DXDX 3
#define OCN_FIELD_DZDX 4
#define OCN_FIELD_DZDZ 5
#define OCN_FIELD_HX 6
#define OCN_FIELD_HZ 7
#define OCN_FIELD_COUNT 8

/* ---- velocity.hpp:48-49 ---- */
#define OCN_DEPTH_LOGARITHMIC 0
#define OCN_DEPTH_UNIFORM 1
#define OCN_INTERP_EXPONENTIAL 0
#define OCN_INTERP_LINEAR 1

/* SpectrumParams, spectra.hpp:17-34. peak_omega_override is used when
 * has_peak_omega_override != 0 (std::optional in the reference). */
typedef struct ocn_spectrum_params {
  double wind_speed;     /* U, m/s (default 5)        */
  double fetch;          /* F, m (default 1e5)        */
  double wind_direction; /* theta0, rad               */
  double swell;          /* xi in [0,1]               */
  double direction_mix;  /* delta in [0,1]            */
  double gravity;        /* default 9.80665           */
  uint64_t rng_seed;
  int32_t has_peak_omega_override;
  int32_t reserved0;
  double peak_omega_override;
} ocn_spectrum_params;

/* SliceConfig, velocity.hpp:51-58. */
typedef struct ocn_slice_config {
  double y_min; /* -125 */
  double y_max; /* 4.5  */
  int32_t count;
  int32_t distribution; /* OCN_DEPTH_* */
  int32_t single_precision;
  int32_t reserved0;
} ocn_slice_config;

/* BodyPose, hydro.hpp:17-35. orientation = (w, x, y, z), body -> world. */
typedef struct ocn_pose {
  double position[3];
  double orientation[4];
  double linear_velocity[3];
  double angular_velocity[3];
  double com_body[3];
} ocn_pose;

/* A host water-velocity sampler (FluidQuery::water_velocity, hydro.hpp:38-49,
 * called per submerged state at hydro.cpp:276-282): the library calls it once per
 * evaluation with every submerged TriangleState centroid as (x, z, y) triples in
 * state order (xzy[3 n]) and reads the medium velocities (vx, vy, vz) from
 * out[3 n]. */
typedef void (*ocn_velocity_fn)(void* user, int64_t n, const double* host_xzy, double* host_out);

/* DragCoefficients hydro.hpp:92-95 + medium constants of FluidQuery
 * hydro.hpp:38-49. The surface / velocity samplers of FluidQuery are the
 * device-resident maps / slices / zones named in ocn_fluid, or host callbacks:
 * a host surface sampler enters as ocn_hydro_aggregate's host_vertex_depth, a
 * host velocity sampler as host_velocity (used when slices is NULL). */
typedef struct ocn_fluid {
  void* maps;          /* ocn_maps*   : height_at sampler (required unless depths are overridden) */
  void* slices;        /* ocn_slices* : velocity_at sampler, or NULL for still water            */
  int32_t velocity_clamp; /* 1: clamp y into [y_min, y_max] as Simulation::water_velocity
                              (sim.cpp:39-42); 0: DomainError outside (velocity.cpp:214-215) */
  int32_t n_zones;     /* FdmZone::sample terms added to the height (sim.cpp:44-51)            */
  void* const* zones;  /* ocn_zone* [n_zones]                                                  */
  double wind[3];
  double water_density; /* 1025  */
  double air_density;   /* 1.204 */
  double cd_water;      /* 1 */
  double cd_air;        /* 1 */
  int32_t n_profile;    /* density_profile entries (depth, rho), hydro.cpp:11-23 */
  int32_t reserved0;
  const double* host_profile; /* 2 * n_profile doubles, or NULL */
  ocn_velocity_fn host_velocity; /* host water_velocity sampler, or NULL (ABI 2) */
  void* host_velocity_user;
} ocn_fluid;

/* HydroReport, hydro.hpp:97-109, plus the composed rigid-body load of
 * sim.cpp:114-122 / rigid_body.cpp:36-39 (thrust excluded). */
typedef struct ocn_hydro_report {
  double submerged_volume;
  double center_of_immersion[3];
  double buoyancy_force[3];
  double water_drag[3];
  double air_drag[3];
  double water_center[3];
  double air_center[3];
  double submerged_area;
  double dry_area;
  double force[3];  /* F_b + F_w (if immersed) + F_a */
  double torque[3]; /* about pose.position                  */
  int32_t volume_clamped;
  int32_t has_center_of_immersion;
  int32_t state_count;
  int32_t degenerate_skipped;
  int32_t waterline_loops;
  int32_t waterline_points;
  int32_t nonfinite; /* device NaN/Inf flag over the report */
  int32_t reserved0;
} ocn_hydro_report;

/* TriangleState, hydro.hpp:53-60 (status 0 = Submerged, 1 = Dry). */
typedef struct ocn_triangle_state {
  int32_t parent;
  int32_t status;
  double area;
  double centroid[3];
  double depth;
  double normal[3];
} ocn_triangle_state;

/* FdmConfig + DampingParams, interactive.hpp:16-33. */
typedef struct ocn_fdm_config {
  int32_t grid_size; /* 512 */
  int32_t margin;    /* 16  */
  double delta_min;  /* 0 = derive from body size */
  double delta_max;  /* 0 = 10 x delta_min        */
  double delta_rate_limit; /* 0.05 */
  double d0;    /* 0.98  */
  double d_max; /* 0.999 */
  double v_max; /* 5     */
} ocn_fdm_config;

/* MaskParams / MaskFrame, interactive.hpp:35-49. */
typedef struct ocn_mask_params {
  double back_height;
  double intensity;
  double amplitude;
} ocn_mask_params;

typedef struct ocn_mask_frame {
  double center_x;
  double half_beam;
  double z_min;
  double z_max;
  double mesh_height;
  double volume_ratio; /* ignored by ocn_zone_mask_from_hydro (taken from the device report) */
} ocn_mask_frame;

/* Scalar state of an FdmZone (interactive.hpp:65-104). */
typedef struct ocn_zone_state {
  int32_t grid_size;
  int32_t margin;
  double spacing;
  double wave_speed;
  double damping;
  double origin[2];
  double pos_curr[2];
  double carry[2];
  int32_t last_shift[2];
  int32_t dropped_wake;
  int32_t reserved0;
  double delta_min;
  double delta_max;
} ocn_zone_state;

typedef struct ocn_ctx ocn_ctx;
typedef struct ocn_cascades ocn_cascades;
typedef struct ocn_maps ocn_maps;
typedef struct ocn_slices ocn_slices;
typedef struct ocn_mesh ocn_mesh;
typedef struct ocn_zone ocn_zone;
typedef struct ocn_slab ocn_slab;
typedef struct ocn_direct ocn_direct;

/* ================================ context ================================ */
OCN_API int ocn_abi_version(void);
OCN_API int ocn_ctx_create(int device, ocn_ctx** out);
/* As ocn_ctx_create with a stream priority: 1 highest, -1 lowest, 0 default.
 * Objects of contexts on the same device may be passed to each other's calls
 * (device memory is shared); ordering between two contexts is the caller's,
 * with events on their ocn_ctx_stream streams. That is how bench.py overlaps
 * frame f's forces / mask / FDM (high priority) with frame f+1's spectral
 * step (low priority) on double-buffered maps and slices. */
OCN_API int ocn_ctx_create_priority(int device, int priority, ocn_ctx** out);
OCN_API int ocn_ctx_destroy(ocn_ctx* ctx);
/* Last error message of this context (or the global one when ctx == NULL). */
OCN_API const char* ocn_last_error(const ocn_ctx* ctx);
OCN_API int ocn_ctx_synchronize(ocn_ctx* ctx);
/* The cudaStream_t all work of this context is enqueued on. */
OCN_API void* ocn_ctx_stream(ocn_ctx* ctx);
/* Number of kernels this library has launched on the context (graph launches
 * count every kernel node). Used by bench.py for "gpu_launches". */
OCN_API uint64_t ocn_ctx_kernel_launches(const ocn_ctx* ctx);

/* Per-stage device timing with CUDA events on the context stream (used by
 * bench.py for the roofline of the dominant kernels). Categories: */
#define OCN_PROF_EVOLVE 0   /* k_evolve (time evolution h~, G)          */
#define OCN_PROF_ROWS 1     /* k_rows (coefficients + row FFT)          */
#define OCN_PROF_COLS 2     /* k_cols (column FFT + sign + Re/Im split) */
#define OCN_PROF_HYDRO 3    /* whole ocn_hydro_aggregate pipeline        */
#define OCN_PROF_MASK 4     /* compute_mask (+ apply)                    */
#define OCN_PROF_FDM 5      /* FdmZone::step stencil                     */
#define OCN_PROF_SPECTRAL 6 /* whole spectral step (evolve+rows+cols)    */
#define OCN_PROF_COUNT 8
/* mode 0: off; 1: per-kernel windows (spectral step launched eagerly, every
 * category valid); 2: stage windows only (spectral / hydro / mask / fdm; the
 * spectral step keeps replaying its CUDA graph). */
OCN_API int ocn_ctx_profile(ocn_ctx* ctx, int mode);
/* Synchronizes, then returns the accumulated milliseconds and launch count of
 * a category since the last reset. */
OCN_API int ocn_ctx_profile_read(ocn_ctx* ctx, int category, double* total_ms, uint64_t* count);
OCN_API int ocn_ctx_profile_reset(ocn_ctx* ctx);

/* ============================ spectrum scalars =========================== */
/* Scalar spectrum model, spectra.cpp:10-130. Same __host__ __device__ code
 * as the device kernels; exposed for the C++ drop-in of spectra.hpp:37-79. */
OCN_API int ocn_spectrum_validate(const ocn_spectrum_params* p);
OCN_API double ocn_alpha(const ocn_spectrum_params* p);
OCN_API double ocn_peak_omega(const ocn_spectrum_params* p);
OCN_API double ocn_standard_peak_omega(const ocn_spectrum_params* p);
OCN_API double ocn_dispersion(double k, double g);
OCN_API int ocn_jonswap(double omega, const ocn_spectrum_params* p, double* out);
OCN_API double ocn_beta_s(double r_omega);
OCN_API double ocn_directional_kernel(double beta, double theta);
OCN_API double ocn_donelan_banner(double omega, double theta, double omega_p);
OCN_API double ocn_swell_spread(double omega, double theta, double omega_p, double xi);
OCN_API double ocn_q_dbxi_approx(double r_omega);
OCN_API double ocn_q_dbxi_quadrature(double r_omega, double xi, int panels);
OCN_API double ocn_directional(double omega, double theta, const ocn_spectrum_params* p);
OCN_API double ocn_h0_variance(double kx, double kz, double k, double omega, double tile_length,
                       const ocn_spectrum_params* p);
OCN_API double ocn_damping_factor(double speed, double d0, double d_max, double v_max);
OCN_API double ocn_attenuation(double k, double y);
OCN_API int ocn_log_distribution(double y, double y_min, double* out);
OCN_API int ocn_exp_interp(double a, double f_a, double b, double f_b, double x, double* out);
OCN_API int ocn_slice_depths(const ocn_slice_config* cfg, double* host_depths);

/* ============================ cascades (K1) ============================== */
/* generate_h0 (spectra.cpp:132-179) for `count` grids of one resolution, run
 * as one sm_100a kernel (fp64 spectrum, bit-exact Philox and band mask).
 * CascadeSet (surface.cpp:22-37) is count = lengths.size() with bands from
 * the cutoffs; generate_h0 alone is count = 1. */
OCN_API int ocn_cascades_create(ocn_ctx* ctx, int resolution, int count, const double* host_lengths,
                        const double* host_band_min, const double* host_band_max,
                        const uint32_t* host_cascade_index, const ocn_spectrum_params* params,
                        ocn_cascades** out);
/* Batched spectral sets (independent instances): `count`
 * grids with their own spectrum parameters (params has count entries). One
 * spectral step then evolves and transforms every grid. Samplers over maps of
 * such a set sum at most 16 grids (a set of instances is for synthesis). */
OCN_API int ocn_cascades_create_multi(ocn_ctx* ctx, int resolution, int count,
                                      const double* host_lengths, const double* host_band_min,
                                      const double* host_band_max,
                                      const uint32_t* host_cascade_index,
                                      const ocn_spectrum_params* params, ocn_cascades** out);
/* Time-batched spectral set (generate_maps is a pure function
 * of t, surface.cpp:70-103): `frames` copies of a `count`-grid cascade set; grid
 * f * count + c is grid c evaluated at t + f dt. The spectrum tables exist once
 * per grid c. Maps of the set are laid out [frames][count][8][N][N]; dt is the
 * spacing ocn_surface_generate / ocn_spectral_step use (ocn_surface_generate_batch
 * passes its own). Info / download / assemble calls take any grid index
 * (frame f's grid c downloads grid c's spectrum). Samplers reject such maps. */
OCN_API int ocn_cascades_create_frames(ocn_ctx* ctx, int resolution, int count,
                                       const double* host_lengths, const double* host_band_min,
                                       const double* host_band_max,
                                       const uint32_t* host_cascade_index,
                                       const ocn_spectrum_params* params, int frames, double dt,
                                       ocn_cascades** out);
OCN_API int ocn_cascades_destroy(ocn_cascades* c);
OCN_API int ocn_cascades_info(const ocn_cascades* c, int* resolution, int* count);
/* WaveGrid accessors (spectra.hpp:95-104): h0 / h0_conj_neg as interleaved
 * complex (2*N*N doubles), in_band (N*N bytes), waves (4*N*N doubles:
 * kx, kz, k, omega per mode). Any pointer may be NULL. */
OCN_API int ocn_cascades_download(ocn_cascades* c, int grid, double* host_h0, double* host_h0cn,
                          uint8_t* host_in_band, double* host_waves);

/* assemble_coefficients (surface.cpp:39-68) of one grid at time t on the
 * device (fp64): out = 8 interleaved complex fields (8 * 2*N*N doubles) in
 * SurfaceField order. Not on the per-frame path (the spectral step generates
 * its packed coefficients in registers); provided for the drop-in API. */
OCN_API int ocn_assemble_coefficients(ocn_cascades* c, int grid, double t, double choppiness,
                                      double* host_out);

/* =========================== surface maps (K2+K4) ========================= */
/* SurfaceMaps (surface.hpp:65-80): 8 fp32 fields per cascade, device-resident. */
OCN_API int ocn_maps_create(ocn_cascades* c, ocn_maps** out);
OCN_API int ocn_maps_destroy(ocn_maps* m);
/* generate_maps (surface.cpp:70-103), (async). Same pairing as
 * surface.cpp:77-80; each pair is one C2C inverse FFT of X + iY. */
OCN_API int ocn_surface_generate(ocn_maps* m, double t, double choppiness);
/* generate_maps of every frame of a time-batched set at t0 + f dt, (async). On an
 * ordinary set it equals ocn_surface_generate(m, t0, choppiness). */
OCN_API int ocn_surface_generate_batch(ocn_maps* m, double t0, double dt, double choppiness);
/* North-star item 3 on the grid: with enable != 0 every
 * spectral step of these maps also writes, per texel of every grid, the slope
 * normal (-Hx, 1, -Hz)/|.| and the Jacobian J = (1 - DxDx)(1 - DzDz) - DzDx^2
 * of X = p + D into fp32 planes [grid][4][N][N] (nx, ny, nz, J). */
OCN_API int ocn_maps_set_assembly(ocn_maps* m, int enable);
OCN_API int ocn_maps_download_assembly(ocn_maps* m, int cascade, int component, float* host_out);
OCN_API int ocn_maps_time(const ocn_maps* m, double* t);
OCN_API int ocn_maps_download(ocn_maps* m, int cascade, int field, double* host_out);
OCN_API int ocn_maps_download_f32(ocn_maps* m, int cascade, int field, float* host_out);
OCN_API int ocn_maps_device_field(ocn_maps* m, int cascade, int field, const float** dev_out);
/* Maps not produced by a spectral step (e.g. SurfaceMaps assembled by the
 * caller): `count` cascades of tile lengths host_lengths at resolution n,
 * filled with ocn_maps_upload; usable by every sampler. */
OCN_API int ocn_maps_create_bare(ocn_ctx* ctx, int resolution, int count,
                                 const double* host_lengths, ocn_maps** out);
OCN_API int ocn_maps_upload(ocn_maps* m, int cascade, int field, const double* host_in);

/* ========================= velocity slices (K3+K4) ======================== */
OCN_API int ocn_slices_create(ocn_cascades* c, const ocn_slice_config* cfg, ocn_slices** out);
OCN_API int ocn_slices_destroy(ocn_slices* s);
/* build_slices (velocity.cpp:104-179), (async). (vx, vz) packed per depth,
 * vy packed across adjacent depths, zero partner for an odd count. */
OCN_API int ocn_velocity_build(ocn_slices* s, double t);
OCN_API int ocn_slices_depths(const ocn_slices* s, int* count, double* host_depths);
/* component: 0 = vx, 1 = vy, 2 = vz */
OCN_API int ocn_slices_download(ocn_slices* s, int depth, int cascade, int component, double* host_out);

/* Fused per-frame spectral step: maps and (optional) slices at time t in one
 * enqueued graph (async). Equivalent to ocn_surface_generate + ocn_velocity_build. */
OCN_API int ocn_spectral_step(ocn_maps* m, ocn_slices* s, double t, double choppiness);

/* One packed transform of the spectral step of (maps, slices), in plan order:
 * the surface pairs of every grid (surface.cpp:77-80), then per grid the
 * (vx, vz) transform of every depth and the vy transforms across adjacent
 * depths (velocity.cpp:145-172). */
typedef struct ocn_xform_info {
  int32_t cascade;
  int32_t kind;     /* 0..3 surface pairs; 4 (vx, vz)_d; 5 (vy_d, vy_d+1); 6 (vy_d, 0) */
  int32_t index0;   /* surface: field of Re; velocity: depth index d of Re             */
  int32_t index1;   /* surface: field of Im; velocity: depth index of Im (-1: none)     */
  int32_t row_half; /* spectrum rows |i - N/2| >= row_half are exactly zero in fp32 and
                       skipped (band edge, or attenuation below 2^-132 at the depth)    */
  int32_t executed; /* 0: the whole transform is exactly zero at its depth(s): its
                       planes are zeroed once when the plan is built, never per frame */
  double y0, y1;    /* slice depths of the velocity kinds                              */
} ocn_xform_info;
/* The transform list of ocn_spectral_step(m, s) (builds the plan if needed).
 * count = total transforms; the first min(capacity, count) are copied to out. */
OCN_API int ocn_spectral_plan_info(ocn_maps* m, ocn_slices* s, int capacity, ocn_xform_info* out,
                                   int* count);

/* ============================= standalone FFT ============================= */
/* ifft2_centered (fft.cpp:69-77) and ifft2_hermitian_pair (fft.cpp:79-101) on
 * host fp64 interleaved complex buffers (2*N*N doubles); device math is fp32. */
OCN_API int ocn_ifft2_centered(ocn_ctx* ctx, int n, const double* host_in, double* host_out);
OCN_API int ocn_ifft2_pair(ocn_ctx* ctx, int n, const double* host_x, const double* host_y,
                   double* host_re, double* host_im);

/* ============================ batched samplers ============================ */
/* SurfaceMaps::sample (surface.cpp:125-129): out[i] = sum_c bilinear(field_c, x_i). */
OCN_API int ocn_maps_sample(ocn_maps* m, int field, int64_t n, const double* xz, double* out);
/* SurfaceMaps::sample_displacement (surface.cpp:131-139): out = (dx, h, dz) per point. */
OCN_API int ocn_sample_displacement(ocn_maps* m, int64_t n, const double* xz, double* out);
/* height_at (surface.cpp:141-151), Algorithm 1 with 4 rounds. */
OCN_API int ocn_height_at(ocn_maps* m, int64_t n, const double* xz, double* out);
/* height_at_tolerance (surface.cpp:153-169). */
OCN_API int ocn_height_at_tolerance(ocn_maps* m, int64_t n, const double* xz, double tol,
                            int max_iters, double* out, int32_t* iterations);
/* North-star item 3 (no reference function): at each query
 * point x, the composed displaced surface after Algorithm 1:
 * out[10*i + 0..9] = (X - x)_x, h, (X - x)_z, normal(3), jacobian,
 *                    sum DxDx, sum DzDx, sum DzDz.
 * normal ∝ (-Hx, 1, -Hz), J = (1 - DxDx)(1 - DzDz) - DzDx^2 (SURVEY sign convention). */
OCN_API int ocn_surface_assemble(ocn_maps* m, int64_t n, const double* xz, double* out);
/* VelocitySlices::sample_slice (velocity.cpp:203-211), out = 3 per point. */
OCN_API int ocn_sample_slice(ocn_slices* s, int depth, int64_t n, const double* xz, double* out);
/* velocity_at (velocity.cpp:213-265). xzy = (x, z, y) per point; out = 3 per point.
 * clamp != 0 clamps y into [y_min, y_max] first (sim.cpp:39-42). */
OCN_API int ocn_velocity_at(ocn_slices* s, int64_t n, const double* xzy, int interp, int clamp,
                    double* out);

/* ============================== hydro (K5-K8) ============================== */
/* A validated, outward-oriented TriMesh (mesh.cpp:48-116 is load-time host
 * code in the C++ layer); normals / areas per triangle as the reference computes. */
OCN_API int ocn_mesh_create(ocn_ctx* ctx, int n_vertices, const double* host_vertices, int n_triangles,
                    const int32_t* host_triangles, const double* host_normals,
                    const double* host_areas, double volume, ocn_mesh** out);
OCN_API int ocn_mesh_destroy(ocn_mesh* mesh);
/* aggregate (hydro.cpp:253-306) incl. classify_clip (hydro.cpp:63-215).
 * host_vertex_depth may be NULL (depths from the fluid's maps + zones); when
 * given, it replaces the surface sampler (signed depth per vertex, e.g. from a
 * user sampler). report may be NULL: the evaluation then stays asynchronous
 * and the report is fetched with ocn_hydro_report_get. */
OCN_API int ocn_hydro_aggregate(ocn_mesh* mesh, const ocn_pose* pose, const ocn_fluid* fluid,
                        const double* host_vertex_depth, ocn_hydro_report* report);
/* aggregate for n <= 16 bodies as ONE launch set (Simulation::step's body loop,
 * sim.cpp:74-83): meshes[i] at poses[i] against fluids[i] -- each with its own
 * zone list and drag coefficients; all fluids share maps / slices and all meshes
 * one context. reports may be NULL (async; ocn_hydro_report_get per mesh). */
OCN_API int ocn_hydro_aggregate_batch(int n, ocn_mesh* const* meshes, const ocn_pose* poses,
                                      const ocn_fluid* fluids, ocn_hydro_report* reports);
OCN_API int ocn_hydro_report_get(ocn_mesh* mesh, ocn_hydro_report* report);
/* The reports of n evaluated meshes of one context with one synchronisation. */
OCN_API int ocn_hydro_reports_get(int n, ocn_mesh* const* meshes, ocn_hydro_report* reports);
/* Per-vertex world positions (3 doubles) and signed depths of the last evaluation. */
OCN_API int ocn_hydro_vertices(ocn_mesh* mesh, double* host_world, double* host_depth);
/* TriangleStates of the last evaluation in parent order (ClipResult::states). */
OCN_API int ocn_hydro_states(ocn_mesh* mesh, int capacity, ocn_triangle_state* host_states, int* count);
/* Waterline loops of the last evaluation: loop_offsets has n_loops + 1 entries;
 * points are xyz triples (closed loops repeat their first point, hydro.cpp:208-209). */
OCN_API int ocn_hydro_waterline(ocn_mesh* mesh, int* n_loops, int* n_points, int32_t* host_loop_offsets,
                        double* host_points);

/* ============================ FDM zone (K9-K10) ============================ */
OCN_API int ocn_zone_create(ocn_ctx* ctx, const ocn_fdm_config* cfg, double body_size, double body_x,
                    double body_z, double dt, ocn_zone** out);
OCN_API int ocn_zone_destroy(ocn_zone* z);
OCN_API int ocn_zone_get_state(const ocn_zone* z, ocn_zone_state* out);
/* FdmZone::update_stability (interactive.cpp:54-65). */
OCN_API int ocn_zone_update_stability(ocn_zone* z, double body_speed, double dt);
/* FdmZone::step (interactive.cpp:67-111), (async). */
OCN_API int ocn_zone_step(ocn_zone* z, double dt, double body_x, double body_z);
/* FdmZone::apply_mask (interactive.cpp:113-118) for an explicit cell list. */
OCN_API int ocn_zone_apply_cells(ocn_zone* z, int n, const int32_t* host_ij, const double* host_h);
/* compute_mask (interactive.cpp:146-195) against explicit host loops
 * (loop_offsets: n_loops + 1 entries, points xyz). apply != 0 also performs
 * apply_mask. The cell list is kept on the device; n_cells returns its size. */
OCN_API int ocn_zone_compute_mask(ocn_zone* z, int n_loops, const int32_t* host_loop_offsets,
                          const double* host_points, double body_yaw, double body_x,
                          double body_z, double body_speed, const ocn_mask_frame* frame,
                          const ocn_mask_params* params, int apply, int* n_cells);
/* compute_mask + apply_mask from the device-resident waterline and submerged
 * volume of mesh's last ocn_hydro_aggregate (sim.cpp:86-109), (async). */
OCN_API int ocn_zone_mask_from_hydro(ocn_zone* z, ocn_mesh* mesh, double body_yaw, double body_x,
                             double body_z, double body_speed, const ocn_mask_frame* frame,
                             const ocn_mask_params* params);
/* As ocn_zone_mask_from_hydro without apply_mask: Simulation::step computes
 * every body's mask before any is applied (sim.cpp:73-109), since other bodies'
 * hull depths read this zone. ocn_zone_apply_last_mask applies it (async). */
OCN_API int ocn_zone_mask_from_hydro_deferred(ocn_zone* z, ocn_mesh* mesh, double body_yaw,
                                              double body_x, double body_z, double body_speed,
                                              const ocn_mask_frame* frame,
                                              const ocn_mask_params* params);
OCN_API int ocn_zone_apply_last_mask(ocn_zone* z);
/* One body of a Simulation step (sim.cpp:73-109): its mesh and zone handles,
 * pose, drag coefficients, speed |v|, yaw (BodyPose::yaw) and mask inputs. */
typedef struct ocn_body_frame {
  void* mesh; /* ocn_mesh* */
  void* zone; /* ocn_zone* */
  ocn_pose pose;
  double cd_water, cd_air;
  double speed, yaw;
  ocn_mask_frame frame;
  ocn_mask_params mask;
} ocn_body_frame;
/* The per-body stages of Simulation::step for every body, in sim.cpp's order:
 * per body aggregate (fluid = maps / slices / medium; the zone list is every
 * OTHER body's zone), update_stability, deferred mask; then per body
 * apply_mask + FdmZone::step at the given position; then the reports
 * (reports[n_bodies], synchronous). reports == NULL leaves the stages
 * enqueued (async); read them with ocn_hydro_report_get. */
OCN_API int ocn_bodies_step(int n_bodies, const ocn_body_frame* bodies, const ocn_fluid* fluid,
                            double dt, ocn_hydro_report* reports);
/* ================= Simulation on device-resident state ====================
 * Simulation (sim.hpp:16-60, sim.cpp:15-131) in C++ behind the C-ABI: the spectral
 * surface and slices, every body's hull in one batched launch set with sim.cpp's
 * zone order (ocn_bodies_step), deferred masks, zone steps, and the rigid-body
 * integration (rigid_body.cpp:6-61) on the host. pipelined != 0 (with
 * rebuild_stride 1) prefetches step f+1's spectral step into a second map /
 * slice buffer on a low-priority context while step f's bodies run. */
typedef struct ocn_sim_config {
  int32_t resolution;
  int32_t count;         /* cascades (<= 16) */
  double lengths[16];    /* CascadeConfig (surface.hpp:18-25) */
  double cutoffs[16];    /* count - 1 band edges */
  ocn_spectrum_params spectrum;
  ocn_slice_config slices;
  double choppiness;
  double dt;
  double wind[3];
  int32_t rebuild_stride; /* VelocityScenarioConfig::rebuild_stride */
  int32_t pipelined;
} ocn_sim_config;
/* BodyConfig (scenario.hpp:30-47) with the hull's TriMesh properties (the mesh is
 * built and validated by the caller: ocn_mesh_create on the sim's context). */
typedef struct ocn_sim_body {
  ocn_mesh* mesh;
  double volume;
  double centroid[3];
  double bbox_min[3];
  double bbox_max[3];
  double unit_inertia[9]; /* TriMesh::unit_inertia, row-major */
  double density;         /* kg / m^3, or mass when has_mass */
  double mass;
  int32_t has_mass;
  int32_t box_inertia;
  double position[3];
  double yaw;
  double initial_velocity[3];
  double cd_water, cd_air, angular_damping;
  int32_t n_thrust;
  int32_t reserved0;
  const double* thrust;   /* n_thrust x (until, fx, fy, fz), body frame (sim.cpp:53-57) */
  ocn_fdm_config fdm;
  ocn_mask_params mask;
} ocn_sim_body;
typedef struct ocn_sim ocn_sim;
OCN_API int ocn_sim_create(ocn_ctx* ctx, const ocn_sim_config* cfg, int n_bodies,
                           const ocn_sim_body* bodies, ocn_sim** out);
OCN_API int ocn_sim_destroy(ocn_sim* sim);
/* Simulation::step, `steps` times (synchronous: each step reads the reports). */
OCN_API int ocn_sim_step(ocn_sim* sim, int steps);
/* Body state: position, orientation (w x y z), linear and angular velocity (13
 * doubles) and its last hydro report; either pointer may be NULL. */
OCN_API int ocn_sim_body_state(const ocn_sim* sim, int body, double* host_state13,
                               ocn_hydro_report* report);
/* Cumulative stage times in seconds in Simulation::Timing order (sim.hpp:50-54):
 * [0] surface, [1] velocity, [2] hydro, [3] zones, [4] integrate. [0] is the
 * device time of the whole spectral step -- maps and velocity slices are one
 * fused step (one graph) here, so [1] stays 0 -- [2] / [3] the device time of
 * the batched hulls / of the masks + FDM steps (CUDA events on their streams;
 * overlapping in pipelined mode), [4] the host time of the rigid integration.
 * Informational, as in the reference; collected while ocn_sim_set_timing is on. */
OCN_API int ocn_sim_timing(const ocn_sim* sim, double* seconds5);
/* Stage timing is collected only while enabled (off at creation: the events
 * and clock reads cost host time in a host-synchronous step). */
OCN_API int ocn_sim_set_timing(ocn_sim* sim, int enabled);
/* time, step index, the current maps / slices and the bodies' zones (any may be NULL). */
OCN_API int ocn_sim_info(const ocn_sim* sim, double* time, int* step_index, ocn_maps** maps,
                         ocn_slices** slices, ocn_zone** zones);

/* Cells of the last mask in row-major order (MaskCell, interactive.hpp:56-59). */
OCN_API int ocn_zone_mask_download(ocn_zone* z, int capacity, int32_t* host_ij, double* host_h,
                           int* n_cells);
/* FdmZone::sample (interactive.cpp:120-129). */
OCN_API int ocn_zone_sample(ocn_zone* z, int64_t n, const double* xz, double* out);
OCN_API int ocn_zone_download(ocn_zone* z, double* host_curr, double* host_prev);
OCN_API int ocn_zone_upload(ocn_zone* z, const double* host_curr, const double* host_prev);

/* ========================= slab-decomposed grid (config 5) ================= */
/* One cascade of resolution n split over `ranks` ranks by rows:
 * rank `rank` owns spectrum rows and output columns [rank R, (rank+1) R),
 * R = n / ranks. Per frame: ocn_slab_rows writes this rank's 4 packed row
 * transforms into the all-to-all send buffer laid out [dest][4][R][R]
 * complex64 (dev_send, exchange_bytes); the caller exchanges it (NCCL
 * all-to-all; dest tile d goes to rank d); ocn_slab_cols consumes the receive
 * buffer [src][4][R][R] and writes the 8 surface fields of the owned column
 * slab ([field][n][R] fp32, transposed-slab layout). Both are async. For
 * n >= 4096 the column pass is a four-step FFT that works in place in the
 * receive buffer (its contents are overwritten). */
OCN_API int ocn_slab_create(ocn_ctx* ctx, int n, int ranks, int rank, double length,
                            double band_min, double band_max, uint32_t cascade_index,
                            const ocn_spectrum_params* params, ocn_slab** out);
OCN_API int ocn_slab_destroy(ocn_slab* s);
OCN_API int ocn_slab_info(const ocn_slab* s, int* rows, int* cols, size_t* exchange_bytes);
OCN_API int ocn_slab_rows(ocn_slab* s, double t, double choppiness, void* dev_send);
OCN_API int ocn_slab_cols(ocn_slab* s, void* dev_recv);
/* Column slab of one field: n x R doubles, row-major [i][column - rank R]. */
OCN_API int ocn_slab_download(ocn_slab* s, int field, double* host_out);

/* ------ the exchange over NVLink: an NCCL
 * communicator of the library's own (NCCL is loaded at run time, sharing a copy
 * the process already has). Rank 0 makes the unique id (128 bytes), the caller
 * distributes it (MPI, torch.distributed, a file, ...), every rank creates its
 * communicator on its context's device. */
typedef struct ocn_comm ocn_comm;
OCN_API int ocn_comm_unique_id(char* host_id_128);
OCN_API int ocn_comm_create(ocn_ctx* ctx, const char* host_id_128, int nranks, int rank,
                            ocn_comm** out);
OCN_API int ocn_comm_destroy(ocn_comm* comm);
OCN_API int ocn_comm_info(const ocn_comm* comm, int* nranks, int* rank);
/* The all-to-all of the R x R tiles of packed pair `pair` (-1: all four) between
 * dev_send ([dest][4][R][R]) and dev_recv ([src][4][R][R]) as grouped
 * ncclSend / ncclRecv on the slab's stream (async); the rank's own tile is a
 * device copy. */
OCN_API int ocn_slab_exchange(ocn_slab* s, ocn_comm* comm, int pair, void* dev_send, void* dev_recv);
/* One frame (async): per packed pair p, the row pass, then its exchange on the
 * communicator's stream, then its column pass once its tiles arrived -- the
 * NVLink transfer of pair p overlaps the row pass of p + 1 and the column pass
 * of p - 1. comm may be NULL for a 1-rank slab. dev_send == dev_recv is allowed
 * for 1 rank. */
OCN_API int ocn_slab_frame(ocn_slab* s, ocn_comm* comm, double t, double choppiness,
                           void* dev_send, void* dev_recv);

/* ================= composed surface and ABHF heightfields ================== */
/* Simulation::compose_height (sim.cpp:44-51) in bulk: height_at over the maps
 * plus FdmZone::sample of each listed zone (pass every body's zone except the
 * excluded one). xz / out may be host or device pointers. */
OCN_API int ocn_compose_height(ocn_maps* m, int n_zones, ocn_zone* const* zones, int64_t n,
                               const double* xz, double* out);
/* dump_fields' composed grid (main.cpp:62-67): out[i*res + j] =
 * compose_height(extent*i/res, extent*j/res); points generated on the device. */
OCN_API int ocn_compose_grid(ocn_maps* m, int n_zones, ocn_zone* const* zones, int resolution,
                             double extent, double* out);
/* write_heightfield_file (heightfield_io.hpp:11-16, heightfield_io.cpp:30-45,
 * 73-78) of one device field, header {N, cascade, time}; OCN_ERR_IO when the
 * file cannot be written (IoError). */
OCN_API int ocn_heightfield_write_field(ocn_maps* m, int cascade, int field, float time,
                                        const char* path);
/* The composed-surface file of dump_fields (main.cpp:68-75): header
 * {resolution, -1, time}, samples rounded to fp32 on the device. */
OCN_API int ocn_heightfield_write_composed(ocn_maps* m, int n_zones, ocn_zone* const* zones,
                                           int resolution, double extent, float time,
                                           const char* path);

/* ===================== direct spectral velocity (K11) ====================== */
/* DirectVelocityEvaluator (velocity.hpp:24-37, velocity.cpp:24-59): the mode
 * list of the cascade set at time t (every in-band mode with G != 0, in
 * (cascade, i, j) order, fp64 coefficients), kept on the device. */
OCN_API int ocn_direct_create(ocn_cascades* c, double t, ocn_direct** out);
OCN_API int ocn_direct_destroy(ocn_direct* d);
OCN_API int ocn_direct_modes(const ocn_direct* d, int64_t* count);
/* operator()(x, y) at n points: xzy = (x, z, y) per point, out = (vx, vy, vz)
 * per point (host or device pointers). fp64 phases and sums, fp32 sin / cos /
 * exp of the reduced phase and attenuation (max relative error <= 1e-6 of the
 * summed magnitude, tests/test_gpu_direct.py). */
OCN_API int ocn_direct_evaluate(ocn_direct* d, int64_t n, const double* xzy, double* out);

#ifdef __cplusplus
}
#endif

#endif /* OCEAN_B200_H */
