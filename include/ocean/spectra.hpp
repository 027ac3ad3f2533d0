// ocean/spectra.hpp — drop-in for proj/include/ocean/spectra.hpp.
//
// Scalar spectrum functions evaluate the same __host__ __device__ fp64 code the
// K1 kernel runs; generate_h0 builds the amplitude tables on the B200
// (bit-exact Philox and band mask) and materialises them on first access.
#ifndef OCEAN_B200_SPECTRA_HPP
#define OCEAN_B200_SPECTRA_HPP

#include <memory>
#include <optional>
#include <vector>

#include "ocean/core.hpp"

struct ocn_cascades;

namespace ocean {

struct SpectrumParams {
  double wind_speed = 5.0;      // U
  double fetch = 100000.0;      // F
  double wind_direction = 0.0;  // theta0
  double swell = 0.0;           // xi
  double direction_mix = 0.0;   // delta
  double gravity = kGravity;
  uint64_t rng_seed = 0;
  std::optional<double> peak_omega_override;

  double alpha() const;
  double peak_omega() const;
  double standard_peak_omega() const;
  void validate() const;
};

struct WaveVector {
  double kx = 0.0, kz = 0.0, k = 0.0, omega = 0.0;
};

double dispersion(double k, double g = kGravity);
double jonswap(double omega, const SpectrumParams& params);
double beta_s(double r_omega);
double directional_kernel(double beta, double theta);
double donelan_banner(double omega, double theta, double omega_p);
double swell_spread(double omega, double theta, double omega_p, double xi);
double q_dbxi_approx(double r_omega);
double q_dbxi_quadrature(double r_omega, double xi, int panels = 4096);
double directional(double omega, double theta, const SpectrumParams& params);

struct GridConfig {
  int resolution = 256;
  double length = 256.0;
  double band_min = 0.0;
  double band_max = 1e300;
  void validate() const;
};

namespace detail {
struct CascadeHandle;  // owns an ocn_cascades (shared by the grids of a set)
}

// One grid's tables, resident on the device; host copies materialise lazily.
class WaveGrid {
 public:
  WaveGrid() = default;
  int resolution() const { return n_; }
  double length() const { return length_; }
  double band_min() const { return band_min_; }
  double band_max() const { return band_max_; }
  double gravity() const { return gravity_; }
  const WaveVector& wave(int i, int j) const;
  const ComplexField& h0() const;
  const ComplexField& h0_conj_neg() const;
  bool in_band(int i, int j) const;

  // B200 extension: the device tables and this grid's index in them
  ocn_cascades* device_handle() const;
  int device_index() const { return index_; }

  friend WaveGrid generate_h0(const GridConfig&, const SpectrumParams&, uint32_t);
  friend class CascadeSet;

 private:
  struct Host;
  const Host& host() const;
  int n_ = 0, index_ = 0;
  double length_ = 0.0, band_min_ = 0.0, band_max_ = 0.0, gravity_ = kGravity;
  std::shared_ptr<detail::CascadeHandle> dev_;
  std::shared_ptr<Host> host_;
};

WaveGrid generate_h0(const GridConfig& config, const SpectrumParams& params,
                     uint32_t cascade_index = 0);
double h0_variance(const WaveVector& w, double tile_length, const SpectrumParams& params);

}  // namespace ocean

#endif
