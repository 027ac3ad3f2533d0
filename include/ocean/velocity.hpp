// ocean/velocity.hpp — drop-in for proj/include/ocean/velocity.hpp.
//
// build_slices generates the (vx, vz) and paired vy depth slices on the B200
// (fused with the surface spectrum when built through the same CascadeSet);
// sampling and depth interpolation run on the device.
#ifndef OCEAN_B200_VELOCITY_HPP
#define OCEAN_B200_VELOCITY_HPP

#include <memory>
#include <vector>

#include "ocean/surface.hpp"

struct ocn_slices;
struct ocn_direct;

namespace ocean {

double attenuation(double k, double y);
double log_distribution(double y, double y_min);
double exp_interp(double a, double f_a, double b, double f_b, double x);

enum class DepthDistribution { Logarithmic, Uniform };
enum class DepthInterp { Exponential, Linear };

struct SliceConfig {
  double y_min = -125.0;
  double y_max = 4.5;
  int count = 8;
  DepthDistribution distribution = DepthDistribution::Logarithmic;
  bool single_precision = false;
  void validate() const;
};

std::vector<double> slice_depths(const SliceConfig& config);

// Precomputed time-rotated coefficients for repeated direct evaluations at
// one instant (velocity.hpp:24-37). The mode list lives on the device
// (ocn_direct_*); a single-point call is one launch, the batched overload
// (B200 extension) evaluates every point in one launch.
class DirectVelocityEvaluator {
 public:
  DirectVelocityEvaluator(const CascadeSet& cascades, double t);
  Vec3 operator()(Vec2 x, double y) const;
  // B200 extension: points packed (x, z, y) as the batched velocity_at
  std::vector<Vec3> operator()(const std::vector<Vec3>& xzy) const;
  long long mode_count() const;                                      // B200 extension

 private:
  std::shared_ptr<ocn_direct> dev_;
};

Vec3 velocity_direct(const CascadeSet& cascades, Vec2 x, double y, double t);

namespace detail {
struct SlicesHandle;
}

class VelocitySlices {
 public:
  VelocitySlices() = default;
  const std::vector<double>& depths() const { return depths_; }
  double y_min() const { return y_min_; }
  double y_max() const { return y_max_; }
  Vec3 sample_slice(size_t i, Vec2 x) const;
  ocn_slices* device_handle() const;  // B200 extension

  friend VelocitySlices build_slices(const CascadeSet& cascades, double t,
                                     const SliceConfig& config);

 private:
  double y_min_ = 0.0, y_max_ = 0.0;
  std::vector<double> depths_;
  std::shared_ptr<detail::SlicesHandle> dev_;
};

VelocitySlices build_slices(const CascadeSet& cascades, double t, const SliceConfig& config);
Vec3 velocity_at(const VelocitySlices& slices, Vec2 x, double y,
                 DepthInterp interp = DepthInterp::Exponential);
// B200 extension: batched velocity_at (one launch)
std::vector<Vec3> velocity_at(const VelocitySlices& slices, const std::vector<Vec3>& xzy,
                              DepthInterp interp = DepthInterp::Exponential, bool clamp = false);

}  // namespace ocean

#endif
