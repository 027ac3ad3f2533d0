// bodies.cu — the per-body part of Simulation::step (sim.cpp:73-109) for all
// bodies in one C-ABI call, with every body's hull evaluated by ONE batched
// launch set (hydro.cu: HydroBatch, blockIdx.y = body).
//
// Order is sim.cpp's: body i's hull senses every other body's zone with the
// spacing that zone has at body i's turn -- zones j < i are past their
// update_stability (sim.cpp:74-99). update_stability is host scalar bookkeeping
// (the zone's field is untouched), so the jobs are built in body order with
// the stabilities updated in between, each job capturing its zone views as
// they stand, and the whole batch then runs at once. The masks are computed
// (not applied) per body, then per body apply_mask + FdmZone::step at the
// pre-integration position, then the reports are read (one synchronisation).
#include <vector>

#include "hydro_internal.cuh"

namespace ocn {
HydroJob make_job(ocn_mesh* m, const ocn_pose* pose, const ocn_fluid* fluid, const double* host_depth);
void fill_samplers_batch(HydroBatch<kMaxBatch>& B, const ocn_fluid* fluid);
void hydro_evaluate_jobs(int n, ocn_mesh* const* meshes, const HydroBatch<kMaxBatch>& B);
void hydro_reports_read(int n, ocn_mesh* const* meshes, ocn_hydro_report* out);
void zones_step_batch(int nz, ocn_zone* const* zones, double dt, const double* bx, const double* bz);
void zones_apply_last_mask_batch(int nz, ocn_zone* const* zones);
void zones_mask_from_hydro_batch(int nz, ocn_zone* const* zones, ocn_mesh* const* meshes,
                                 const double* yaw, const double* bx, const double* bz,
                                 const double* speed, const ocn_mask_frame* frames,
                                 const ocn_mask_params* params);
}  // namespace ocn

using namespace ocn;

namespace ocn {
// ocn_bodies_step; `mid` (optional) is recorded on the bodies' stream between
// the hulls and the zone passes (ocn_sim's hydro / zones stage timing)
void bodies_step(int n_bodies, const ocn_body_frame* bodies, const ocn_fluid* fluid, double dt,
                 ocn_hydro_report* reports, cudaEvent_t mid) {
  ocn_mesh* m0 = n_bodies > 0 && bodies ? (ocn_mesh*)bodies[0].mesh : nullptr;
  {
    OCN_REQUIRE(n_bodies >= 0 && n_bodies <= kMaxBatch, "ocn_bodies_step: %d bodies (0..%d)",
                n_bodies, kMaxBatch);
    if (n_bodies == 0) return;
    OCN_REQUIRE(bodies && fluid, "null argument");
    auto check = [](int st) {
      if (st != OCN_OK) fail(st, "%s", global_error().c_str());
    };
    std::vector<ocn_mesh*> meshes(n_bodies);
    HydroBatch<kMaxBatch> B{};
    B.n = n_bodies;
    std::vector<void*> others;
    for (int i = 0; i < n_bodies; ++i) {
      const ocn_body_frame& b = bodies[i];
      OCN_REQUIRE(b.mesh && b.zone, "body %d: null mesh / zone", i);
      meshes[i] = (ocn_mesh*)b.mesh;
      OCN_REQUIRE(meshes[i]->ctx == m0->ctx, "bodies must share one context");
      others.clear();
      for (int k = 0; k < n_bodies; ++k)
        if (k != i) others.push_back(bodies[k].zone);
      ocn_fluid f = *fluid;
      f.n_zones = (int32_t)others.size();
      f.zones = others.empty() ? nullptr : others.data();
      f.cd_water = b.cd_water;
      f.cd_air = b.cd_air;
      f.host_velocity = nullptr;
      if (i == 0) fill_samplers_batch(B, &f);
      B.job[i] = make_job(meshes[i], &b.pose, &f, nullptr);
      check(ocn_zone_update_stability((ocn_zone*)b.zone, b.speed, dt));
    }
    hydro_evaluate_jobs(n_bodies, meshes.data(), B);
    if (mid) OCN_CUDA(cudaEventRecord(mid, m0->ctx->stream));
    NvtxRange nv("zones");
    // every body's mask, apply and FDM step as one launch each (zones are
    // independent: batching keeps sim.cpp's per-body results)
    std::vector<ocn_zone*> zones(n_bodies);
    std::vector<double> yaw(n_bodies), bx(n_bodies), bz(n_bodies), speed(n_bodies);
    std::vector<ocn_mask_frame> frames(n_bodies);
    std::vector<ocn_mask_params> params(n_bodies);
    for (int i = 0; i < n_bodies; ++i) {
      const ocn_body_frame& b = bodies[i];
      zones[i] = (ocn_zone*)b.zone;
      yaw[i] = b.yaw;
      bx[i] = b.pose.position[0];
      bz[i] = b.pose.position[2];
      speed[i] = b.speed;
      frames[i] = b.frame;
      params[i] = b.mask;
    }
    zones_mask_from_hydro_batch(n_bodies, zones.data(), meshes.data(), yaw.data(), bx.data(),
                                bz.data(), speed.data(), frames.data(), params.data());
    zones_apply_last_mask_batch(n_bodies, zones.data());
    zones_step_batch(n_bodies, zones.data(), dt, bx.data(), bz.data());
    if (!reports) return;  // asynchronous: reports via ocn_hydro_report_get
    hydro_reports_read(n_bodies, meshes.data(), reports);
  }
}
}  // namespace ocn

extern "C" {

int ocn_bodies_step(int n_bodies, const ocn_body_frame* bodies, const ocn_fluid* fluid, double dt,
                    ocn_hydro_report* reports) {
  ocn_mesh* m0 = n_bodies > 0 && bodies ? (ocn_mesh*)bodies[0].mesh : nullptr;
  return api_call(m0 ? m0->ctx : nullptr,
                  [&] { bodies_step(n_bodies, bodies, fluid, dt, reports, nullptr); });
}

}  // extern "C"
