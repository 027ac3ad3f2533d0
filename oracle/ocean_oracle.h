/*
 * ocean_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64, single-threaded restatement of the reference CPU algorithm
 * of the Arc Blanc hot path (reference tree /root/reference/proj). It is the
 * checker for the CUDA product path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it. The product library
 * (libocean_b200.so) never links or calls it.
 *
 * Parity pin: tests/test_oracle_vs_ref.py compares every function here with
 * the reference itself (oracle/_ref/libocean_ref.so, compiled from the
 * reference sources by oracle/Makefile) and with the committed golden
 * fixtures in tests/golden/ generated from that build.
 *
 * Arrays: complex fields are interleaved (re, im) doubles, row-major [i][j]
 * with storage index s <-> wave index s - N/2 (fft.hpp:10-16).
 * Return values: OCN_* status codes from include/ocean_b200.h.
 */
#ifndef OCEAN_ORACLE_H
#define OCEAN_ORACLE_H

#include "../include/ocean_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:14-76 ---- */
void orc_philox(uint64_t key_lo, uint64_t key_hi, uint64_t ctr_lo, uint64_t ctr_hi, uint32_t out[4]);
void orc_gaussian_complex(uint64_t seed, uint32_t stream, uint32_t i, uint32_t j, double out[2]);

/* ---- spectra.cpp:10-130 ---- */
int orc_spectrum_validate(const ocn_spectrum_params* p);
double orc_alpha(const ocn_spectrum_params* p);
double orc_peak_omega(const ocn_spectrum_params* p);
double orc_standard_peak_omega(const ocn_spectrum_params* p);
double orc_dispersion(double k, double g);
int orc_jonswap(double omega, const ocn_spectrum_params* p, double* out);
double orc_beta_s(double r);
double orc_directional_kernel(double beta, double theta);
double orc_donelan_banner(double omega, double theta, double omega_p);
double orc_swell_spread(double omega, double theta, double omega_p, double xi);
double orc_q_dbxi_approx(double r);
double orc_q_dbxi_quadrature(double r, double xi, int panels);
double orc_directional(double omega, double theta, const ocn_spectrum_params* p);
double orc_h0_variance(double kx, double kz, double k, double omega, double tile_length,
                       const ocn_spectrum_params* p);

/* generate_h0, spectra.cpp:132-179. Outputs may be NULL except h0. */
int orc_generate_h0(int n, double length, double band_min, double band_max,
                    const ocn_spectrum_params* p, uint32_t cascade, double* h0, double* h0cn,
                    uint8_t* in_band, double* waves);

/* ---- fft.cpp ---- */
int orc_ifft2_centered(int n, double* data);
int orc_ifft2_pair(int n, const double* x, const double* y, double* re, double* im);

/* ---- surface.cpp ---- */
/* assemble_coefficients surface.cpp:39-68: out = 8 complex fields (8 * 2n^2). */
int orc_assemble_coefficients(int n, double length, double gravity, const double* h0,
                              const double* h0cn, const uint8_t* in_band, double t,
                              double choppiness, double* out);
/* generate_maps surface.cpp:70-103; maps = [C][8][n*n]. */
/* One packed surface pair of a grid too large for generate_maps on the host
 * (16384^2): h0 per mode on the fly, surface.cpp:45-66 coefficients of pair
 * `pair` (surface.cpp:77-80 order), fft.cpp:79-101 packed transform with rows /
 * columns over `threads` OpenMP threads; optional direct sums of the packed
 * spectrum at npts grid nodes ab = (a, b) pairs -> direct (re, im). */
int orc_surface_pair_large(int n, double length, double band_min, double band_max,
                           const ocn_spectrum_params* p, uint32_t cascade, double t, double chop,
                           int pair, int threads, int npts, const int32_t* ab, double* direct,
                           double* re, double* im);
int orc_generate_maps(int n, int C, const double* lengths, double gravity, const double* h0,
                      const double* h0cn, const uint8_t* in_band, double t, double choppiness,
                      int single_precision, double* maps);

/* ---- velocity.cpp ---- */
double orc_attenuation(double k, double y);
int orc_log_distribution(double y, double y_min, double* out);
int orc_exp_interp(double a, double fa, double b, double fb, double x, double* out);
int orc_slice_depths(const ocn_slice_config* cfg, double* depths);
/* build_slices velocity.cpp:104-179; slices = [D][C][3][n*n] (vx, vy, vz). */
int orc_build_slices(int n, int C, const double* lengths, double gravity, const double* h0,
                     const double* h0cn, const uint8_t* in_band, double t,
                     const ocn_slice_config* cfg, double* depths, double* slices);
/* DirectVelocityEvaluator velocity.cpp:24-59 at points xzy = (x, z, y). */
int orc_direct_velocity(int n, int C, const double* lengths, double gravity, const double* h0,
                        const double* h0cn, const uint8_t* in_band, double t, int64_t npts,
                        const double* xzy, double* out);

/* ---- samplers ---- */
typedef struct orc_surface {
  int n, C;
  const double* lengths; /* [C] */
  const double* maps;    /* [C][8][n*n] */
} orc_surface;

typedef struct orc_slices {
  int n, C, D;
  const double* lengths; /* [C] */
  const double* depths;  /* [D] sorted */
  double y_min, y_max;
  const double* data; /* [D][C][3][n*n] */
} orc_slices;

int orc_maps_sample(const orc_surface* s, int field, int64_t npts, const double* xz, double* out);
int orc_sample_displacement(const orc_surface* s, int64_t npts, const double* xz, double* out);
int orc_height_at(const orc_surface* s, int64_t npts, const double* xz, double* out);
int orc_height_at_tolerance(const orc_surface* s, int64_t npts, const double* xz, double tol,
                            int max_iters, double* out, int32_t* iterations);
int orc_sample_slice(const orc_slices* s, int depth, int64_t npts, const double* xz, double* out);
int orc_velocity_at(const orc_slices* s, int64_t npts, const double* xzy, int interp, int clamp,
                    double* out);

/* ---- mesh.cpp:18-116 (TriMesh constructor) ----
 * tris is rewritten in place when the mesh is re-oriented.
 * props: volume, centroid[3], unit_inertia[9], bbox_min[3], bbox_max[3],
 *        total_area, degenerate_count  (19 doubles). */
int orc_mesh_build(int nv, const double* verts, int nt, int32_t* tris, double* normals,
                   double* areas, double* props);

/* ---- interactive.cpp ---- */
typedef struct orc_zone {
  ocn_fdm_config cfg; /* after derivation of delta_min / delta_max */
  int n, margin;
  double delta, c, damping;
  double origin[2], pos_curr[2], carry[2];
  int last_shift[2];
  int dropped_wake;
  double* curr; /* n*n */
  double* prev; /* n*n */
} orc_zone;

double orc_damping_factor(double speed, double d0, double d_max, double v_max);
int orc_zone_create(const ocn_fdm_config* cfg, double body_size, double bx, double bz, double dt,
                    orc_zone** out);
void orc_zone_destroy(orc_zone* z);
int orc_zone_update_stability(orc_zone* z, double speed, double dt);
int orc_zone_step(orc_zone* z, double dt, double bx, double bz);
int orc_zone_apply_cells(orc_zone* z, int n, const int32_t* ij, const double* h);
double orc_zone_sample(const orc_zone* z, double x, double zc);
int orc_mask_height(double x, double z, const ocn_mask_frame* f, double speed,
                    const ocn_mask_params* p, double* out);
/* point_in_loops on 2D loops (loop_offsets n_loops+1, points xz pairs). */
int orc_point_in_loops(double px, double pz, int n_loops, const int32_t* offsets,
                       const double* pts_xz);
/* compute_mask interactive.cpp:146-195; loops as xyz triples. Returns the
 * number of cells in *n_cells (up to capacity written). */
int orc_compute_mask(const orc_zone* z, int n_loops, const int32_t* loop_offsets,
                     const double* points, double yaw, double bx, double bz, double speed,
                     const ocn_mask_frame* frame, const ocn_mask_params* params, int capacity,
                     int32_t* ij, double* h, int* n_cells);

/* ---- hydro.cpp ---- */
typedef struct orc_fluid {
  const orc_surface* surface; /* NULL: flat sea at y = 0 */
  const orc_slices* slices;   /* NULL: still water       */
  int velocity_clamp;
  int n_zones;
  const orc_zone* const* zones;
  double wind[3];
  double water_density, air_density, cd_water, cd_air;
  int n_profile;
  const double* profile; /* (depth, rho) pairs */
} orc_fluid;

typedef struct orc_clip_out {
  int capacity_states;
  ocn_triangle_state* states;
  int n_states;
  int capacity_loops;
  int32_t* loop_offsets; /* n_loops + 1 */
  int capacity_points;
  double* points; /* xyz */
  int n_loops, n_points;
  double submerged_area, dry_area;
  int degenerate_skipped;
} orc_clip_out;

/* World positions + vertex depths (hydro.cpp:69-76), surface = height_at +
 * zone samples. */
int orc_vertex_depths(int nv, const double* verts, const ocn_pose* pose, const orc_fluid* fluid,
                      double* wpos, double* depth);
/* classify_clip hydro.cpp:63-215 from explicit world positions / depths. */
int orc_classify_clip(int nv, const double* wpos, const double* depth, int nt,
                      const int32_t* tris, const double* normals, const double* areas,
                      const ocn_pose* pose, orc_clip_out* out);
/* aggregate hydro.cpp:253-306; vertex_depth may be NULL (sampled from fluid). */
int orc_aggregate(int nv, const double* verts, int nt, const int32_t* tris,
                  const double* normals, const double* areas, double mesh_volume,
                  const ocn_pose* pose, const orc_fluid* fluid, const double* vertex_depth,
                  ocn_hydro_report* report, orc_clip_out* clip);

#ifdef __cplusplus
}
#endif

#endif
