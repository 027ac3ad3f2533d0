// sim.cu — Simulation::step (sim.cpp:15-131) over device-resident state, in
// C++ behind the C-ABI (ocn_sim): the spectral surface and velocity slices,
// every body's hull in one batched launch set with sim.cpp's zone order
// (ocn_bodies_step), the deferred masks, the zone steps, and the rigid-body
// integration (rigid_body.cpp:6-61, 13 host doubles per body).
//
// Pipelined (default when rebuild_stride == 1): the spectral step of step f+1
// is a pure function of time, so it is enqueued on a low-priority context into
// the second of two map / slice buffers right after step f's bodies, and runs
// beside them; CUDA events order the buffers (ready: its spectral step done;
// consumed: the last body stage reading it done). Only the hydro reports come
// back to the host each step, for the integration.
#include <chrono>
#include <cmath>
#include <memory>
#include <vector>

#include "hydro_internal.cuh"

namespace ocn {
void bodies_step(int n_bodies, const ocn_body_frame* bodies, const ocn_fluid* fluid, double dt,
                 ocn_hydro_report* reports, cudaEvent_t mid);  // bodies.cu
}

namespace ocn {
void hydro_reports_read(int n, ocn_mesh* const* meshes, ocn_hydro_report* out);
}

namespace {

struct V3 {
  double x = 0, y = 0, z = 0;
};
V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double norm(V3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
V3 v3(const double* p) { return {p[0], p[1], p[2]}; }

struct M3 {
  double m[3][3]{};
};
V3 mul(const M3& A, V3 v) {
  return {A.m[0][0] * v.x + A.m[0][1] * v.y + A.m[0][2] * v.z,
          A.m[1][0] * v.x + A.m[1][1] * v.y + A.m[1][2] * v.z,
          A.m[2][0] * v.x + A.m[2][1] * v.y + A.m[2][2] * v.z};
}
M3 mul(const M3& A, const M3& B) {
  M3 C;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k) C.m[i][j] += A.m[i][k] * B.m[k][j];
  return C;
}
M3 transpose(const M3& A) {
  M3 T;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T.m[i][j] = A.m[j][i];
  return T;
}
// Mat3::inverse (core.hpp:119-137): adjugate / determinant
M3 inverse(const M3& A) {
  const auto& m = A.m;
  const double det = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                     m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                     m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  if (std::fabs(det) < 1e-300) ocn::fail(OCN_ERR_NUMERIC, "singular matrix");
  const double id = 1.0 / det;
  M3 r;
  r.m[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) * id;
  r.m[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) * id;
  r.m[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) * id;
  r.m[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) * id;
  r.m[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) * id;
  r.m[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) * id;
  r.m[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) * id;
  r.m[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) * id;
  r.m[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) * id;
  return r;
}

// quaternion (w, x, y, z), core.hpp:142-186
struct Q {
  double w = 1, x = 0, y = 0, z = 0;
};
Q qmul(Q a, Q b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
Q qnormalized(Q q) {
  const double n = std::sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  return {q.w / n, q.x / n, q.y / n, q.z / n};
}
Q qaxis(V3 axis, double angle) {
  const double n = norm(axis);
  if (n < 1e-300) return {};
  const double h = 0.5 * angle, s = std::sin(h) / n;
  return {std::cos(h), axis.x * s, axis.y * s, axis.z * s};
}
V3 qrotate(Q q, V3 v) {
  const V3 u{q.x, q.y, q.z};
  const V3 t = cross(u, v) * 2.0;
  return (v + t * q.w) + cross(u, t);
}
M3 qmatrix(Q q) {
  const double w = q.w, x = q.x, y = q.y, z = q.z;
  M3 r;
  r.m[0][0] = 1 - 2 * (y * y + z * z), r.m[0][1] = 2 * (x * y - w * z), r.m[0][2] = 2 * (x * z + w * y);
  r.m[1][0] = 2 * (x * y + w * z), r.m[1][1] = 1 - 2 * (x * x + z * z), r.m[1][2] = 2 * (y * z - w * x);
  r.m[2][0] = 2 * (x * z - w * y), r.m[2][1] = 2 * (y * z + w * x), r.m[2][2] = 1 - 2 * (x * x + y * y);
  return r;
}
double qyaw(Q q) {  // BodyPose::yaw, hydro.hpp:31-34
  const V3 bow = qrotate(q, {0, 0, 1});
  return std::atan2(bow.x, bow.z);
}

// RigidBody (rigid_body.cpp:6-61)
struct Rigid {
  double mass = 1;
  M3 ib, ib_inv;
  V3 p, v, w, com, L, F, T;
  Q q;
  void apply_force_at(V3 f, V3 at) {  // rigid_body.cpp:36-39
    F = F + f;
    T = T + cross(at - p, f);
  }
  void integrate(V3 g, double dt, double damping) {  // rigid_body.cpp:41-61
    v = v + (F * (1.0 / mass) + g) * dt;
    L = L + T * dt;
    if (damping > 0.0) L = L * (1.0 - damping * dt);
    const M3 r = qmatrix(q);
    w = mul(mul(mul(r, ib_inv), transpose(r)), L);
    p = p + v * dt;
    const double wn = norm(w);
    if (wn > 1e-300) q = qnormalized(qmul(qaxis(w * (1.0 / wn), wn * dt), q));
    F = {};
    T = {};
  }
};

struct SimBody {
  ocn_mesh* mesh = nullptr;
  ocn_zone* zone = nullptr;
  Rigid rigid;
  double cd_water = 1, cd_air = 1, damping = 0;
  V3 bbox_min, bbox_max;
  ocn_mask_params mask{};
  std::vector<double> thrust;  // (until, fx, fy, fz) per phase, body frame
  ocn_hydro_report report{};
};

}  // namespace

struct ocn_sim {
  ocn_ctx* ctx = nullptr;   // bodies (high priority when pipelined)
  ocn_ctx* sctx = nullptr;  // spectral step (low priority when pipelined; else == ctx)
  bool own_sctx = false;
  ocn_cascades* cas = nullptr;
  ocn_maps* maps[2]{};
  ocn_slices* slices[2]{};
  int nbuf = 1, cur = 0;
  bool pipelined = false, prefetched = false;
  cudaEvent_t ready[2]{}, consumed[2]{};
  double dt = 1.0 / 60.0, time = 0.0, chop = 1.0, gravity = 9.80665;
  int step_index = 0, rebuild_stride = 1;
  double wind[3]{};
  std::vector<SimBody> bodies;
  // Simulation::Timing (sim.hpp:50-54): device time of the spectral step
  // (surface and velocity are one fused graph), of the hulls and of the zone
  // passes (CUDA events on their streams), host time of the integration
  struct Stage {
    cudaEvent_t a = nullptr, b = nullptr;
    bool pending = false;
    double seconds = 0.0;
  };
  Stage spec[2], hyd, zon;    // spec: one pair per buffer (settled when reused)
  cudaEvent_t mid = nullptr;  // hulls -> zones split (recorded inside the bodies step)
  double integrate_s = 0.0;
  bool timing = false;        // ocn_sim_set_timing (off: no events, no host clock reads)
};

namespace {

using namespace ocn;

void check(int st) {
  if (st != OCN_OK) fail(st, "%s", global_error().c_str());
}

// the step's surface / slices for time t into buffer k (sim.cpp:63-70)
void spectral(ocn_sim* s, int k, double t, bool slices) {
  if (slices)
    check(ocn_spectral_step(s->maps[k], s->slices[k], t, s->chop));
  else
    check(ocn_surface_generate(s->maps[k], t, s->chop));
}

void stage_settle(ocn_sim::Stage& st);

// spectral() between a pair of timing events on the spectral stream
void timed_spectral(ocn_sim* s, int k, double t, bool slices) {
  ocn_sim::Stage& st = s->spec[k];
  stage_settle(st);  // this buffer's previous step (complete by now)
  if (s->timing) OCN_CUDA(cudaEventRecord(st.a, s->sctx->stream));
  spectral(s, k, t, slices);
  if (s->timing) {
    OCN_CUDA(cudaEventRecord(st.b, s->sctx->stream));
    st.pending = true;
  }
}

void stage_settle(ocn_sim::Stage& st) {  // fold a completed event pair into the total
  if (!st.pending) return;
  OCN_CUDA(cudaEventSynchronize(st.b));
  float ms = 0.f;
  OCN_CUDA(cudaEventElapsedTime(&ms, st.a, st.b));
  st.seconds += 1e-3 * ms;
  st.pending = false;
}

void destroy(ocn_sim* s) {
  if (!s) return;
  for (auto* e : {s->spec[0].a, s->spec[0].b, s->spec[1].a, s->spec[1].b, s->hyd.a, s->zon.b, s->mid})
    if (e) cudaEventDestroy(e);
  for (auto& b : s->bodies)
    if (b.zone) ocn_zone_destroy(b.zone);
  for (int k = 0; k < 2; ++k) {
    if (s->maps[k]) ocn_maps_destroy(s->maps[k]);
    if (s->slices[k]) ocn_slices_destroy(s->slices[k]);
    if (s->ready[k]) cudaEventDestroy(s->ready[k]);
    if (s->consumed[k]) cudaEventDestroy(s->consumed[k]);
  }
  if (s->cas) ocn_cascades_destroy(s->cas);
  if (s->own_sctx) ocn_ctx_destroy(s->sctx);
  delete s;
}

}  // namespace

extern "C" {

int ocn_sim_create(ocn_ctx* ctx, const ocn_sim_config* cfg, int n_bodies,
                   const ocn_sim_body* bodies, ocn_sim** out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && cfg && out && (n_bodies == 0 || bodies), "null argument");
    OCN_REQUIRE(n_bodies >= 0 && n_bodies <= 16, "%d bodies (0..16)", n_bodies);
    OCN_REQUIRE(cfg->count >= 1 && cfg->count <= 16, "cascade count %d", cfg->count);
    if (!(cfg->dt > 0.0)) fail(OCN_ERR_CONFIG, "dt must be > 0");
    if (cfg->rebuild_stride < 1) fail(OCN_ERR_CONFIG, "velocity rebuild_stride must be >= 1");
    DeviceScope ds(ctx);
    std::unique_ptr<ocn_sim, void (*)(ocn_sim*)> s(new ocn_sim, destroy);
    s->ctx = ctx;
    s->dt = cfg->dt;
    s->chop = cfg->choppiness;
    s->gravity = cfg->spectrum.gravity;
    s->rebuild_stride = cfg->rebuild_stride;
    for (int k = 0; k < 3; ++k) s->wind[k] = cfg->wind[k];
    s->pipelined = cfg->pipelined != 0 && cfg->rebuild_stride == 1;
    if (s->pipelined) {
      check(ocn_ctx_create_priority(ctx->device, -1, &s->sctx));
      s->own_sctx = true;
    } else {
      s->sctx = ctx;
    }
    // CascadeSet (surface.cpp:22-37): band c = [cutoffs[c-1], cutoffs[c])
    std::vector<double> bmin(cfg->count), bmax(cfg->count);
    for (int c = 0; c < cfg->count; ++c) {
      bmin[c] = c == 0 ? 0.0 : cfg->cutoffs[c - 1];
      bmax[c] = c + 1 < cfg->count ? cfg->cutoffs[c] : 1e300;
    }
    check(ocn_cascades_create(s->sctx, cfg->resolution, cfg->count, cfg->lengths, bmin.data(),
                              bmax.data(), nullptr, &cfg->spectrum, &s->cas));
    s->nbuf = s->pipelined ? 2 : 1;
    for (int k = 0; k < s->nbuf; ++k) {
      check(ocn_maps_create(s->cas, &s->maps[k]));
      check(ocn_slices_create(s->cas, &cfg->slices, &s->slices[k]));
      OCN_CUDA(cudaEventCreateWithFlags(&s->ready[k], cudaEventDisableTiming));
      OCN_CUDA(cudaEventCreateWithFlags(&s->consumed[k], cudaEventDisableTiming));
    }
    for (auto* e : {&s->spec[0].a, &s->spec[0].b, &s->spec[1].a, &s->spec[1].b, &s->hyd.a,
                    &s->zon.b, &s->mid})
      OCN_CUDA(cudaEventCreate(e));
    s->hyd.b = s->zon.a = s->mid;
    spectral(s.get(), 0, 0.0, true);  // sim.cpp:18-20
    if (s->pipelined) OCN_CUDA(cudaEventRecord(s->ready[0], s->sctx->stream));
    for (int i = 0; i < n_bodies; ++i) {  // sim.cpp:22-36
      const ocn_sim_body& c = bodies[i];
      OCN_REQUIRE(c.mesh, "body %d: null mesh", i);
      OCN_REQUIRE(c.mesh->ctx == ctx, "body %d: mesh of another context", i);
      SimBody b;
      b.mesh = c.mesh;
      b.cd_water = c.cd_water;
      b.cd_air = c.cd_air;
      b.damping = c.angular_damping;
      b.mask = c.mask;
      b.bbox_min = v3(c.bbox_min), b.bbox_max = v3(c.bbox_max);
      b.thrust.assign(c.thrust, c.thrust + 4 * (size_t)std::max(c.n_thrust, 0));
      const double density = c.has_mass ? c.mass / c.volume : c.density;
      Rigid& r = b.rigid;
      r.q = qaxis({0, 1, 0}, c.yaw);  // Quat::yaw
      r.com = v3(c.centroid);
      r.p = v3(c.position) + qrotate(r.q, r.com);
      r.v = v3(c.initial_velocity);
      // RigidBody::from_mesh (rigid_body.cpp:16-34)
      r.mass = density * c.volume;
      if (!(r.mass > 0.0)) fail(OCN_ERR_CONFIG, "rigid body mass must be > 0");
      if (c.box_inertia) {
        const V3 e = b.bbox_max - b.bbox_min;
        r.ib.m[0][0] = r.mass / 12.0 * (e.y * e.y + e.z * e.z);
        r.ib.m[1][1] = r.mass / 12.0 * (e.x * e.x + e.z * e.z);
        r.ib.m[2][2] = r.mass / 12.0 * (e.x * e.x + e.y * e.y);
      } else {
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < 3; ++k) r.ib.m[a][k] = c.unit_inertia[3 * a + k] * density;
      }
      r.ib_inv = inverse(r.ib);
      r.q = qnormalized(r.q);
      r.L = {};  // angular velocity 0 at start
      const V3 ext = b.bbox_max - b.bbox_min;
      check(ocn_zone_create(ctx, &c.fdm, std::max(ext.x, ext.z), r.p.x, r.p.z, s->dt, &b.zone));
      s->bodies.push_back(b);
    }
    OCN_CUDA(cudaStreamSynchronize(s->sctx->stream));
    *out = s.release();
  });
}

int ocn_sim_destroy(ocn_sim* s) {
  if (!s) return OCN_OK;
  DeviceScope ds(s->ctx);
  cudaStreamSynchronize(s->ctx->stream);
  cudaStreamSynchronize(s->sctx->stream);
  destroy(s);
  return OCN_OK;
}

int ocn_sim_step(ocn_sim* s, int steps) {
  return api_call(s ? s->ctx : nullptr, [&] {
    OCN_REQUIRE(s && steps >= 0, "bad arguments");
    DeviceScope ds(s->ctx);
    const int nb = (int)s->bodies.size();
    std::vector<ocn_body_frame> frames(nb);
    std::vector<ocn_hydro_report> reports(nb);
    for (int it = 0; it < steps; ++it) {
      const double t_next = s->time + s->dt;  // sim.cpp:61
      int k = 0;
      if (!s->pipelined) {
        timed_spectral(s, 0, t_next, s->step_index % s->rebuild_stride == 0);
      } else {
        k = 1 - s->cur;
        if (!s->prefetched) {  // first step: nothing prefetched yet
          OCN_CUDA(cudaStreamWaitEvent(s->sctx->stream, s->consumed[k], 0));
          timed_spectral(s, k, t_next, true);
          OCN_CUDA(cudaEventRecord(s->ready[k], s->sctx->stream));
        }
        s->cur = k;
        OCN_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->ready[k], 0));
      }
      // sense + clip + mask, zone updates (sim.cpp:73-109)
      ocn_fluid fluid{};
      fluid.maps = s->maps[k];
      fluid.slices = s->slices[k];
      fluid.velocity_clamp = 1;  // Simulation::water_velocity, sim.cpp:39-42
      for (int q = 0; q < 3; ++q) fluid.wind[q] = s->wind[q];
      fluid.water_density = 1025.0;
      fluid.air_density = 1.204;
      for (int i = 0; i < nb; ++i) {
        const SimBody& b = s->bodies[i];
        const Rigid& r = b.rigid;
        ocn_body_frame& f = frames[i];
        f = ocn_body_frame{};
        f.mesh = b.mesh;
        f.zone = b.zone;
        const double pv[][3] = {{r.p.x, r.p.y, r.p.z}, {r.v.x, r.v.y, r.v.z},
                                {r.w.x, r.w.y, r.w.z}, {r.com.x, r.com.y, r.com.z}};
        for (int q = 0; q < 3; ++q) {
          f.pose.position[q] = pv[0][q];
          f.pose.linear_velocity[q] = pv[1][q];
          f.pose.angular_velocity[q] = pv[2][q];
          f.pose.com_body[q] = pv[3][q];
        }
        f.pose.orientation[0] = r.q.w, f.pose.orientation[1] = r.q.x;
        f.pose.orientation[2] = r.q.y, f.pose.orientation[3] = r.q.z;
        f.cd_water = b.cd_water;
        f.cd_air = b.cd_air;
        f.speed = norm(r.v);
        f.yaw = qyaw(r.q);
        const V3 ext = b.bbox_max - b.bbox_min;  // sim.cpp:88-97
        f.frame.center_x = 0.0;
        f.frame.half_beam = ext.x;
        f.frame.z_min = b.bbox_min.z;
        f.frame.z_max = b.bbox_max.z;
        f.frame.mesh_height = ext.y;
        f.mask = b.mask;
      }
      if (s->timing) OCN_CUDA(cudaEventRecord(s->hyd.a, s->ctx->stream));
      {
        NvtxRange nv("hydro+zones");
        bodies_step(nb, frames.data(), &fluid, s->dt, nullptr, s->timing ? s->mid : nullptr);
      }
      if (s->timing) OCN_CUDA(cudaEventRecord(s->zon.b, s->ctx->stream));
      if (s->pipelined) {
        // the next step's spectral step (a function of time only) goes into the
        // other buffer, whose last readers were the PREVIOUS step's bodies
        OCN_CUDA(cudaEventRecord(s->consumed[k], s->ctx->stream));
        OCN_CUDA(cudaStreamWaitEvent(s->sctx->stream, s->consumed[1 - k], 0));
        timed_spectral(s, 1 - k, t_next + s->dt, true);
        OCN_CUDA(cudaEventRecord(s->ready[1 - k], s->sctx->stream));
        s->prefetched = true;
      }
      std::vector<ocn_mesh*> meshes(nb);
      for (int i = 0; i < nb; ++i) meshes[i] = s->bodies[i].mesh;
      hydro_reports_read(nb, meshes.data(), reports.data());  // the bodies' stream is idle now
      if (s->timing) {
        s->hyd.pending = s->zon.pending = true;
        stage_settle(s->hyd);
        stage_settle(s->zon);
      }
      // forces and integration (sim.cpp:112-125)
      NvtxRange nv_int("integrate");
      const auto t_int = s->timing ? std::chrono::steady_clock::now()
                                   : std::chrono::steady_clock::time_point{};
      for (int i = 0; i < nb; ++i) {
        SimBody& b = s->bodies[i];
        const ocn_hydro_report& rp = reports[i];
        b.report = rp;
        Rigid& r = b.rigid;
        if (rp.has_center_of_immersion) {
          r.apply_force_at(v3(rp.buoyancy_force), v3(rp.water_center));
          r.apply_force_at(v3(rp.water_drag), v3(rp.water_center));
        }
        r.apply_force_at(v3(rp.air_drag), v3(rp.air_center));
        for (size_t ph = 0; ph < b.thrust.size() / 4; ++ph)  // thrust_force, sim.cpp:53-57
          if (s->time < b.thrust[4 * ph]) {
            r.F = r.F + qrotate(r.q, v3(&b.thrust[4 * ph + 1]));
            break;
          }
        r.integrate({0.0, -s->gravity, 0.0}, s->dt, b.damping);
      }
      if (s->timing)
        s->integrate_s +=
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_int).count();
      s->time = t_next;
      ++s->step_index;
      for (int i = 0; i < nb; ++i) {  // check_finite, sim.cpp:133-142
        const Rigid& r = s->bodies[i].rigid;
        const double probe = r.p.x + r.p.y + r.p.z + r.v.x + r.v.y + r.v.z;
        if (!std::isfinite(probe))
          fail(OCN_ERR_NUMERIC, "non-finite body state (body %d, step %d)", i, s->step_index);
      }
    }
  });
}

int ocn_sim_set_timing(ocn_sim* s, int enabled) {
  if (!s) return OCN_ERR_ARG;
  s->timing = enabled != 0;
  return OCN_OK;
}

int ocn_sim_timing(const ocn_sim* sc, double* seconds5) {
  if (!sc || !seconds5) return OCN_ERR_ARG;
  ocn_sim* s = const_cast<ocn_sim*>(sc);
  return api_call(s->ctx, [&] {
    DeviceScope ds(s->ctx);
    stage_settle(s->spec[0]);
    stage_settle(s->spec[1]);
    seconds5[0] = s->spec[0].seconds + s->spec[1].seconds;  // surface + velocity (one fused step)
    seconds5[1] = 0.0;
    seconds5[2] = s->hyd.seconds;
    seconds5[3] = s->zon.seconds;
    seconds5[4] = s->integrate_s;
  });
}

int ocn_sim_body_state(const ocn_sim* s, int body, double* host_state13, ocn_hydro_report* report) {
  if (!s || body < 0 || body >= (int)s->bodies.size()) return OCN_ERR_ARG;
  const Rigid& r = s->bodies[body].rigid;
  if (host_state13) {
    const double v[13] = {r.p.x, r.p.y, r.p.z, r.q.w, r.q.x, r.q.y, r.q.z,
                          r.v.x, r.v.y, r.v.z, r.w.x, r.w.y, r.w.z};
    for (int k = 0; k < 13; ++k) host_state13[k] = v[k];
  }
  if (report) *report = s->bodies[body].report;
  return OCN_OK;
}

int ocn_sim_info(const ocn_sim* s, double* time, int* step_index, ocn_maps** maps,
                 ocn_slices** slices, ocn_zone** zones) {
  if (!s) return OCN_ERR_ARG;
  if (time) *time = s->time;
  if (step_index) *step_index = s->step_index;
  if (maps) *maps = s->maps[s->cur];
  if (slices) *slices = s->slices[s->cur];
  if (zones)
    for (size_t i = 0; i < s->bodies.size(); ++i) zones[i] = s->bodies[i].zone;
  return OCN_OK;
}

}  // extern "C"
