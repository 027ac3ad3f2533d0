// bodies.cu — the per-body part of Simulation::step (sim.cpp:73-109) for all
// bodies in one C-ABI call: host orchestration of the device stages, so a
// multi-body step costs one library call instead of five per body.
//
// Order is sim.cpp's: per body i, aggregate against height_at plus every other
// body's zone (compose_height, sim.cpp:44-51), update_stability (spacing
// changes at once, so body i+1 sees it), and the mask computed but not applied;
// then per body apply_mask + FdmZone::step at the pre-integration position;
// then the reports are read (one stream synchronisation).
#include <vector>

#include "objects.cuh"

using namespace ocn;

extern "C" {

int ocn_bodies_step(int n_bodies, const ocn_body_frame* bodies, const ocn_fluid* fluid, double dt,
                    ocn_hydro_report* reports) {
  if (n_bodies < 0 || (n_bodies > 0 && (!bodies || !fluid))) return OCN_ERR_ARG;
  if (n_bodies == 0) return OCN_OK;
  std::vector<void*> others;
  others.reserve(n_bodies);
  for (int i = 0; i < n_bodies; ++i) {
    const ocn_body_frame& b = bodies[i];
    others.clear();
    for (int k = 0; k < n_bodies; ++k)
      if (k != i) others.push_back(bodies[k].zone);
    ocn_fluid f = *fluid;
    f.n_zones = (int32_t)others.size();
    f.zones = others.empty() ? nullptr : others.data();
    f.cd_water = b.cd_water;
    f.cd_air = b.cd_air;
    int st = ocn_hydro_aggregate((ocn_mesh*)b.mesh, &b.pose, &f, nullptr, nullptr);
    if (st != OCN_OK) return st;
    st = ocn_zone_update_stability((ocn_zone*)b.zone, b.speed, dt);
    if (st != OCN_OK) return st;
    st = ocn_zone_mask_from_hydro_deferred((ocn_zone*)b.zone, (ocn_mesh*)b.mesh, b.yaw,
                                           b.pose.position[0], b.pose.position[2], b.speed,
                                           &b.frame, &b.mask);
    if (st != OCN_OK) return st;
  }
  for (int i = 0; i < n_bodies; ++i) {
    int st = ocn_zone_apply_last_mask((ocn_zone*)bodies[i].zone);
    if (st != OCN_OK) return st;
    st = ocn_zone_step((ocn_zone*)bodies[i].zone, dt, bodies[i].pose.position[0],
                       bodies[i].pose.position[2]);
    if (st != OCN_OK) return st;
  }
  if (!reports) return OCN_OK;  // asynchronous: reports via ocn_hydro_report_get
  for (int i = 0; i < n_bodies; ++i) {
    const int st = ocn_hydro_report_get((ocn_mesh*)bodies[i].mesh, &reports[i]);
    if (st != OCN_OK) return st;
  }
  return OCN_OK;
}

}  // extern "C"
