// C++ drop-in API test: exercises include/ocean/*.hpp the way reference callers
// do (Simulation::step, the bench studies, the CLI dump) and checks the
// SPEC.md known answers. argv[1]: directory where it writes raw fp64 outputs
// for tests/test_gpu_cpp_api.py to compare against the CPU oracle.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "ocean/heightfield_io.hpp"
#include "ocean/hydro.hpp"
#include "ocean/interactive.hpp"
#include "ocean/surface.hpp"
#include "ocean/velocity.hpp"

using namespace ocean;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static void dump(const std::string& path, const double* p, size_t n) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(p), n * sizeof(double));
}

int main(int argc, char** argv) {
  const std::string out = argc > 1 ? argv[1] : ".";
  // ---- spectrum scalars (SPEC.md known answers)
  CHECK(std::fabs(dispersion(1.0) - 3.131557) < 1e-6);
  CHECK(std::fabs(beta_s(1.0) - 2.28) < 1e-12);
  CHECK(std::fabs(damping_factor(2.5) - 0.9895) < 1e-12);
  SpectrumParams sp;
  sp.wind_speed = 20.0;
  sp.wind_direction = 0.4;
  sp.swell = 0.5;
  sp.direction_mix = 0.5;
  sp.rng_seed = 42;
  sp.peak_omega_override = sp.standard_peak_omega();
  bool threw = false;
  try {
    jonswap(0.0, sp);
  } catch (const DomainError&) {
    threw = true;
  }
  CHECK(threw);
  // ---- cascades, maps, coefficients (config-2 spectrum at N = 64)
  CascadeConfig cc;
  cc.resolution = 64;
  cc.lengths = {1024.0, 256.0, 16.0, 4.0};
  cc.cutoffs = {12 * kPi / 256, 12 * kPi / 16, 12 * kPi / 4};
  CascadeSet cs(cc, sp);
  SurfaceMaps maps = generate_maps(cs, 1.5);
  CHECK(maps.cascades.size() == 4 && maps.cascades[0].fields[kFieldH].size() == 64);
  // maps vs the standalone packed transform of assemble_coefficients (surface.cpp:77-80)
  auto coef = assemble_coefficients(cs.grids()[2], 1.5);
  auto [re, im] = ifft2_hermitian_pair(coef[kFieldH], coef[kFieldDx]);
  double err = 0.0, mx = 0.0;
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) {
      err = std::max(err, std::fabs(re.at(i, j) - maps.cascades[2].fields[kFieldH].at(i, j)));
      mx = std::max(mx, std::fabs(re.at(i, j)));
    }
  CHECK(err <= 1e-4 * mx);
  for (int c = 0; c < 4; ++c)
    for (int f = 0; f < kFieldCount; ++f)
      dump(out + "/maps_" + std::to_string(c) + "_" + std::to_string(f) + ".bin",
           maps.cascades[c].fields[f].data(), 64 * 64);
  // WaveGrid accessors
  const WaveGrid& g0 = cs.grids()[0];
  CHECK(g0.resolution() == 64 && !g0.in_band(32, 32));
  CHECK(std::fabs(g0.wave(10, 20).k - std::hypot(g0.wave(10, 20).kx, g0.wave(10, 20).kz)) < 1e-12);
  // samplers: single-point == batched
  std::vector<Vec2> xs = {{3.0, 7.0}, {-100.5, 33.25}, {512.0, -4.0}};
  auto hb = height_at(maps, xs);
  for (size_t i = 0; i < xs.size(); ++i) CHECK(hb[i] == height_at(maps, xs[i]));
  dump(out + "/heights.bin", hb.data(), hb.size());
  // caller-assembled maps are uploaded on first sampling
  SurfaceMaps copy;
  copy.cascades = maps.cascades;
  CHECK(std::fabs(height_at(copy, xs[1]) - hb[1]) < 1e-9);
  // ---- velocity
  SliceConfig sc;
  sc.count = 8;
  VelocitySlices vs = build_slices(cs, 1.5, sc);
  CHECK(vs.depths().size() == 8 && vs.depths().front() < vs.depths().back());
  Vec3 v = velocity_at(vs, {3.0, 7.0}, -2.0);
  double vv[3] = {v.x, v.y, v.z};
  dump(out + "/velocity.bin", vv, 3);
  threw = false;
  try {
    velocity_at(vs, {0, 0}, -500.0);
  } catch (const DomainError&) {
    threw = true;
  }
  CHECK(threw);
  // ---- hull forces: unit cube known answers, flat water
  std::istringstream cube(
      "v -0.5 -0.5 -0.5\nv -0.5 -0.5 0.5\nv -0.5 0.5 -0.5\nv -0.5 0.5 0.5\n"
      "v 0.5 -0.5 -0.5\nv 0.5 -0.5 0.5\nv 0.5 0.5 -0.5\nv 0.5 0.5 0.5\n"
      "f 1 2 4\nf 1 4 3\nf 5 7 8\nf 5 8 6\nf 1 5 6\nf 1 6 2\nf 3 4 8\nf 3 8 7\n"
      "f 1 3 7\nf 1 7 5\nf 2 6 8\nf 2 8 4\n");
  TriMesh box = load_obj(cube, "cube");
  CHECK(std::fabs(box.volume() - 1.0) < 1e-12);
  BodyPose pose;
  pose.position = {0, -10, 0};
  HydroReport r = aggregate(box, pose, FluidQuery::still_water());
  CHECK(std::fabs(r.submerged_volume - 1.0) < 1e-9 && std::fabs(r.submerged_area - 6.0) < 1e-9);
  pose.position = {0, 1e-7, 0};
  r = aggregate(box, pose, FluidQuery::still_water());
  CHECK(std::fabs(r.submerged_volume - 0.5) < 1e-6);
  CHECK(r.waterline.size() == 1);
  CHECK(std::fabs(r.buoyancy_force.y - 1025 * kGravity * 0.5) < 1e-2);
  // icosphere in the wavy sea with device samplers
  TriMesh ico = make_icosphere(6.0, 3);
  BodyPose bp;
  bp.position = {3.0, 0.5, 7.0};
  bp.orientation = Quat::yaw(0.3);
  bp.linear_velocity = {1, 0, 4};
  bp.com_body = ico.centroid();
  FluidQuery fq;
  fq.maps = &maps;
  fq.slices = &vs;
  fq.wind = {5, 0, 2};
  HydroReport wave = aggregate(ico, bp, fq);
  CHECK(wave.center_of_immersion.has_value());
  ClipResult clip = classify_clip(ico, bp, fq);
  CHECK(!clip.states.empty() && clip.waterline.size() >= 1);
  CHECK(std::fabs(submerged_volume(clip.states) - wave.submerged_volume) < 1e-6 * (1 + wave.submerged_volume));
  double rep[6] = {wave.submerged_volume, wave.buoyancy_force.y, wave.water_drag.x, wave.water_drag.y,
                   wave.water_drag.z, wave.air_drag.x};
  dump(out + "/report.bin", rep, 6);
  // host std::function sampler path (depths evaluated by the caller's sampler)
  FluidQuery host_fq;
  host_fq.surface_height = [&](Vec2 x) { return height_at(maps, x); };
  HydroReport via_host = aggregate(ico, bp, host_fq);
  CHECK(std::fabs(via_host.submerged_volume - wave.submerged_volume) <= 1e-9 * wave.submerged_volume);
  // ---- FDM zone: CFL pinned at 0.49, mask + step
  FdmConfig fc;
  fc.grid_size = 256;
  FdmZone zone(fc, 12.0, {3.0, 7.0}, 1.0 / 60.0);
  zone.update_stability(4.1, 1.0 / 60.0);
  CHECK(std::fabs(zone.cfl_ratio(1.0 / 60.0) - 0.49) < 1e-12);
  MaskFrame frame;
  frame.half_beam = 12.0;
  frame.z_min = -6.0;
  frame.z_max = 6.0;
  frame.mesh_height = 12.0;
  frame.volume_ratio = wave.submerged_volume / ico.volume();
  auto cells = compute_mask(zone, wave.waterline, bp.yaw(), bp.position.xz(), 4.1, frame, {});
  CHECK(!cells.empty());
  zone.apply_mask(cells);
  zone.step(1.0 / 60.0, {3.0 + 1.0 / 60.0, 7.0 + 4.0 / 60.0});
  const RealField& fld = zone.field();
  double energy = 0.0;
  for (double x : fld) energy += x * x;
  CHECK(std::isfinite(energy) && energy > 0.0);
  // ---- heightfields (heightfield_io.hpp) and the composed surface (sim.cpp:44-51)
  {
    const std::string hf = out + "/h_dev.abhf", hh = out + "/h_host.abhf";
    write_heightfield_file(hf, maps, 1, kFieldH, 1.5);
    write_heightfield_file(hh, {64u, 1, 1.5f}, maps.cascades[1].fields[kFieldH]);
    std::ifstream a(hf, std::ios::binary), b(hh, std::ios::binary);
    std::stringstream sa, sb;
    sa << a.rdbuf();
    sb << b.rdbuf();
    CHECK(sa.str().size() == 16 + 4 * 64 * 64 && sa.str() == sb.str());  // device fp32 == host f64->f32
    HeightfieldHeader hdr;
    RealField back = read_heightfield_file(hf, &hdr);
    CHECK(hdr.resolution == 64 && hdr.cascade == 1 && hdr.time == 1.5f);
    CHECK(back.at(5, 9) == maps.cascades[1].fields[kFieldH].at(5, 9));
    bool io_threw = false;
    try {
      read_heightfield_file(out + "/missing.abhf");
    } catch (const IoError&) {
      io_threw = true;
    }
    CHECK(io_threw);
    std::vector<Vec2> pts = {{3.5, 7.25}, {10.0, 2.0}, {-4.0, 30.0}};
    auto ch = compose_height(maps, {&zone}, pts);
    for (size_t i = 0; i < pts.size(); ++i)
      CHECK(std::fabs(ch[i] - (height_at(maps, pts[i]) + zone.sample(pts[i]))) <= 1e-9);
    write_composed_heightfield_file(out + "/composed.abhf", maps, {&zone}, 32, 1024.0, 1.5);
    RealField comp = read_heightfield_file(out + "/composed.abhf", &hdr);
    CHECK(hdr.resolution == 32 && hdr.cascade == -1 && comp.size() == 32);
    const double want = height_at(maps, Vec2{1024.0 * 3 / 32, 1024.0 * 5 / 32}) +
                        zone.sample(Vec2{1024.0 * 3 / 32, 1024.0 * 5 / 32});
    CHECK(std::fabs(comp.at(3, 5) - want) <= 1e-6 * (1.0 + std::fabs(want)));
  }
  // ---- DirectVelocityEvaluator (velocity.hpp:24-37) on the device
  {
    DirectVelocityEvaluator dv(cs, 1.5);
    CHECK(dv.mode_count() > 0);
    Vec3 a = dv(Vec2{3.0, 7.0}, -2.0);
    auto batch = dv(std::vector<Vec3>{{3.0, 7.0, -2.0}, {10.0, -4.0, 1.0}});
    CHECK(batch.size() == 2 && std::fabs(batch[0].x - a.x) <= 1e-12 * (1 + std::fabs(a.x)));
    Vec3 b = velocity_direct(cs, Vec2{3.0, 7.0}, -2.0, 1.5);
    CHECK(std::fabs(b.y - a.y) <= 1e-12 * (1 + std::fabs(a.y)));
    dump(out + "/direct.bin", &a.x, 3);
  }
  std::printf("cpp api: %d failures (cells %zu, v_w %.6f)\n", failures, cells.size(),
              wave.submerged_volume);
  return failures ? 1 : 0;
}
