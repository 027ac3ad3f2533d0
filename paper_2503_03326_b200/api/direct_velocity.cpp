// direct_velocity.cpp — DirectVelocityEvaluator / velocity_direct of the
// drop-in velocity.hpp (reference velocity.cpp:24-63) over ocn_direct_*.
#include "ocean/velocity.hpp"
#include "ocean_b200.h"

namespace ocean {

void throw_on_status(int st, const char* where);  // ocean_api.cpp

DirectVelocityEvaluator::DirectVelocityEvaluator(const CascadeSet& cascades, double t) {
  ocn_direct* d = nullptr;
  throw_on_status(ocn_direct_create(cascades.device_handle(), t, &d), "DirectVelocityEvaluator");
  dev_ = std::shared_ptr<ocn_direct>(d, [](ocn_direct* p) { ocn_direct_destroy(p); });
}

Vec3 DirectVelocityEvaluator::operator()(Vec2 x, double y) const {
  const double xzy[3] = {x.x, x.z, y};
  double v[3];
  throw_on_status(ocn_direct_evaluate(dev_.get(), 1, xzy, v), "DirectVelocityEvaluator");
  return {v[0], v[1], v[2]};
}

std::vector<Vec3> DirectVelocityEvaluator::operator()(const std::vector<Vec3>& xzy) const {
  std::vector<double> in(3 * xzy.size()), out(3 * xzy.size());
  for (size_t i = 0; i < xzy.size(); ++i)
    in[3 * i] = xzy[i].x, in[3 * i + 1] = xzy[i].y, in[3 * i + 2] = xzy[i].z;
  throw_on_status(ocn_direct_evaluate(dev_.get(), static_cast<int64_t>(xzy.size()), in.data(),
                                      out.data()),
                  "DirectVelocityEvaluator");
  std::vector<Vec3> v(xzy.size());
  for (size_t i = 0; i < v.size(); ++i) v[i] = {out[3 * i], out[3 * i + 1], out[3 * i + 2]};
  return v;
}

long long DirectVelocityEvaluator::mode_count() const {
  int64_t n = 0;
  throw_on_status(ocn_direct_modes(dev_.get(), &n), "DirectVelocityEvaluator");
  return n;
}

Vec3 velocity_direct(const CascadeSet& cascades, Vec2 x, double y, double t) {
  return DirectVelocityEvaluator(cascades, t)(x, y);
}

}  // namespace ocean
