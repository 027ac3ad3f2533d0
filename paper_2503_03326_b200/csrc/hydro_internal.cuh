// hydro_internal.cuh — device records and handle types of the hydro / FDM stages.
#pragma once

#include "objects.cuh"
#include "samplers.cuh"

namespace ocn {

struct PoseDev {
  double p[3], q[4], v[3], w[3], com[3];
};

struct FluidDev {
  double wind[3];
  double water_density, air_density, cd_water, cd_air;
  int n_profile;
  const double* profile;
};

// TriangleState (hydro.hpp:53-60); status 0 = Submerged, 1 = Dry
struct StateDev {
  int parent, status;
  double area;
  double3 centroid;
  double depth;
  double3 normal;
};

// one waterline crossing segment of a partial triangle: edge keys (min, max)
// of the two crossed edges and their crossing points (hydro.cpp:204-209)
struct SegDev {
  int2 ka, kb;
  double3 pa, pb;
};

struct ReportDev {
  ocn_hydro_report r;
};

// One hull evaluation of a (possibly batched) aggregate launch set: the mesh,
// this evaluation's pose / medium / zones / samplers, and the mesh's buffers.
struct HydroJob {
  const double* verts;
  const int3* tris;
  const double* normals;
  const double* areas;
  int nv, nt, degenerate, hcap;
  double volume;
  PoseDev P;
  FluidDev F;
  int clamp;                      // velocity_at clamps y into [y_min, y_max]
  const double* override_depth;   // host-sampled vertex depths, or nullptr
  const double* ext_vel;          // host-sampled medium velocity per state, or nullptr
  ZoneList zones;                 // FdmZone::sample terms (sim.cpp:44-51)
  double *wpos, *depth;
  int2 *counts, *offsets, *block_sums, *total;
  StateDev* states;
  SegDev* segs;
  double* block_out;
  ReportDev* report;
  int* flags;
  int* ticket;
  unsigned long long* hkeys;
  int *hvals, *partner;
  unsigned char* used;
  int *loop_off, *point_ref, *loop_counts;
  double* loop_points;
};

// NB jobs sharing the surface / velocity samplers, passed by value (one
// kernel-parameter block per launch: no upload); blockIdx.y = job.
constexpr int kMaxBatch = 16;
template <int NB>
struct HydroBatch {
  int n;
  int have_surf, have_vel;
  SurfView surf;
  SliceView vel;
  HydroJob job[NB];
};

}  // namespace ocn

struct ocn_mesh {
  ocn_ctx* ctx = nullptr;
  int nv = 0, nt = 0, degenerate = 0;
  double volume = 0.0;
  bool evaluated = false;
  ocn::DevBuf<double> verts, normals, areas;
  ocn::DevBuf<int3> tris;
  ocn::DevBuf<double> wpos, depth, override_depth, d_profile;
  ocn::DevBuf<double> ext_vel;           // host water_velocity results per state
  std::vector<double> ext_vel_host;
  ocn::DevBuf<int2> counts, offsets, block_sums, total;
  ocn::DevBuf<ocn::StateDev> states;
  ocn::DevBuf<ocn::SegDev> segs;
  ocn::DevBuf<double> block_out;
  ocn::DevBuf<ocn::ReportDev> report;
  ocn::DevBuf<int> flags;  // [0] velocity domain error, [1] non-manifold waterline
  ocn::DevBuf<int> ticket;  // k_forces last-block counter (0 between evaluations)
  int hcap = 0;
  ocn::DevBuf<unsigned long long> hkeys;
  ocn::DevBuf<int> hvals, partner;
  ocn::DevBuf<unsigned char> used;
  ocn::DevBuf<int> loop_off, point_ref, loop_counts;
  ocn::DevBuf<double> loop_points;
  // pinned host staging of the report and flags (one synchronisation per read)
  ocn::ReportDev* h_report = nullptr;
  int* h_flags = nullptr;
  ~ocn_mesh() {
    if (h_report) cudaFreeHost(h_report);
    if (h_flags) cudaFreeHost(h_flags);
  }
};

// FdmZone (interactive.hpp:61-104): host scalars + device fp32 fields
struct ocn_zone {
  ocn_ctx* ctx = nullptr;
  ocn_fdm_config cfg{};  // delta_min / delta_max resolved at construction
  int n = 0, margin = 0;
  double delta = 0, c = 0, damping = 0;
  double origin[2] = {0, 0}, pos_curr[2] = {0, 0}, carry[2] = {0, 0};
  int last_shift[2] = {0, 0};
  int dropped_wake = 0;
  ocn::DevBuf<float> buf[3];  // curr, prev, next rotate
  int icurr = 0, iprev = 1;
  // mask state (interactive.cpp:146-195)
  ocn::DevBuf<double> mask_h;         // heights over the candidate box
  ocn::DevBuf<unsigned char> mask_f;  // inside flags over the candidate box
  ocn::DevBuf<int> mask_box;          // i0, i1, j0, j1, n_edges_ok
  ocn::DevBuf<double> loops_xz;       // de-rotated loop points (2 per point)
  ocn::DevBuf<int> loops_off;
  ocn::DevBuf<double> loop_bbox;      // lo.x, lo.z, hi.x, hi.z
  ocn::DevBuf<int> mask_count;
  ocn::DevBuf<int> bin_off, bin_edges;  // x-binned loop edges (k_mask_prepare)
  float* curr() { return buf[icurr].p; }
  float* prev() { return buf[iprev].p; }
};

namespace ocn {
ZoneView zone_view(ocn_zone* z);
}
