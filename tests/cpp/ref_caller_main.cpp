// The reference's own caller, run on the drop-in: a driver of the reference
// Simulation (proj/include/ocean/sim.hpp, proj/src/sim.cpp:15-131) built from a
// JSON scenario by the reference parser (proj/src/scenario.cpp:149-212).
//
// oracle/Makefile builds it twice from this one file:
//   ref_caller_b200 : sim.cpp, rigid_body.cpp and scenario.cpp of the reference,
//                     UNMODIFIED, compiled against this repo's include/ (the
//                     hot-path headers) and linked with libocean_api.so /
//                     libocean_b200.so: every hot-path call of Simulation::step
//                     lands on the B200 path, with the step's host samplers
//                     (FluidQuery lambdas, sim.cpp:77-80) called back from it;
//   ref_caller_cpu  : the same sources against the reference library itself.
// tests/test_gpu_dropin.py runs both and compares the trajectories.
//
//   ref_caller_<x> <scenario: twobody | box | hull> <steps>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>

#include "ocean/sim.hpp"

namespace {
const char* kTwoBody = R"({
  "seed": 11, "dt": 0.016666666666666666, "duration": 10.0, "wind": [5.0, 0.0, 2.0],
  "spectrum": {"wind_speed": 9.0, "fetch": 100000.0, "wind_direction": 0.3, "swell": 0.2,
               "direction_mix": 0.3, "peak_omega": "standard"},
  "cascades": {"resolution": 64, "lengths": [256.0, 16.0, 4.0],
               "cutoffs": [2.356194490192345, 9.42477796076938]},
  "velocity": {"count": 8, "distribution": "logarithmic"},
  "bodies": [
    {"name": "a", "mesh": {"type": "icosphere", "radius": 1.5, "segments": 2},
     "density": 600.0, "position": [0.0, 0.2, 0.0], "yaw": 0.3, "velocity": [1.0, 0.0, 2.0],
     "fdm": {"grid_size": 128, "margin": 8}},
    {"name": "b", "mesh": {"type": "icosphere", "radius": 1.0, "segments": 2},
     "density": 500.0, "position": [3.0, 0.0, 1.5], "yaw": -0.4, "velocity": [-0.5, 0.0, 1.0],
     "fdm": {"grid_size": 128, "margin": 8}}
  ]
})";

std::string with_primitive(const char* type) {
  std::string s = kTwoBody;
  const std::string from = "\"type\": \"icosphere\", \"radius\": 1.5";
  const std::string to = std::string("\"type\": \"") + type + "\", \"size\": [3.0, 1.5, 2.0]";
  s.replace(s.find(from), from.size(), to);
  return s;
}
}  // namespace

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "twobody";
  const int steps = argc > 2 ? std::atoi(argv[2]) : 12;
  try {
    const std::string json = which == "twobody" ? std::string(kTwoBody) : with_primitive(which.c_str());
    ocean::Scenario sc = ocean::parse_scenario(json, which);
    ocean::Simulation sim(sc);
    for (int k = 0; k < steps; ++k) {
      sim.step();
      for (size_t b = 0; b < sim.bodies().size(); ++b) {
        const auto& body = *sim.bodies()[b];
        const auto& p = body.rigid.pose();
        const auto& r = body.report;
        std::printf("%d %zu %.17g  %.17g %.17g %.17g  %.17g %.17g %.17g  %.17g %.17g %.17g %.17g"
                    "  %.17g %.17g %.17g  %.17g %.17g %.17g  %.17g %.17g %.17g  %zu\n",
                    k, b, sim.time(), p.position.x, p.position.y, p.position.z,
                    p.linear_velocity.x, p.linear_velocity.y, p.linear_velocity.z,
                    p.orientation.w, p.orientation.x, p.orientation.y, p.orientation.z,
                    r.submerged_volume, r.buoyancy_force.y, r.water_drag.x,
                    r.water_drag.y, r.water_drag.z, r.air_drag.x, r.air_drag.y, r.air_drag.z,
                    r.air_drag.z == 0.0 ? 0.0 : 1.0, body.mask.size());
      }
    }
    // the composed surface the bodies sensed (sim.cpp:44-51)
    const double xs[4][2] = {{0.0, 0.0}, {3.0, 1.5}, {1.2, -0.7}, {-20.5, 13.25}};
    for (const auto& x : xs)
      std::printf("H %.17g %.17g %.17g\n", x[0], x[1], sim.compose_height({x[0], x[1]}));
  } catch (const ocean::MeshError& e) {
    std::printf("MeshError %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::printf("ERROR %s\n", e.what());
    return 1;
  }
  return 0;
}
