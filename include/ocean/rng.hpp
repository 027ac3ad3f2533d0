// ocean/rng.hpp — drop-in for proj/include/ocean/rng.hpp.
//
// Philox4x32-10 as the reference specifies it (128-bit key XOR-folded into
// two round keys, rng.hpp:25-48). The device kernel (csrc/spectrum_math.cuh)
// evaluates the same generator; these host entry points exist for callers and
// studies that draw their own samples.
#ifndef OCEAN_B200_RNG_HPP
#define OCEAN_B200_RNG_HPP

#include <cstdint>

#include "ocean/core.hpp"

namespace ocean {

class Philox {
 public:
  Philox(uint64_t key_lo, uint64_t key_hi) : lo_(key_lo), hi_(key_hi) {}
  struct Block {
    uint32_t v[4];
  };
  Block operator()(uint64_t ctr_lo, uint64_t ctr_hi) const;

 private:
  uint64_t lo_, hi_;
};

// (0, 1]
inline double uniform_open(uint32_t bits) {
  return (static_cast<double>(bits) + 1.0) * (1.0 / 4294967296.0);
}

// Standard complex Gaussian (E|xi|^2 = 1) for (seed, stream, i, j).
cplx gaussian_complex(uint64_t seed, uint32_t stream, uint32_t i, uint32_t j);

class UniformStream {
 public:
  explicit UniformStream(uint64_t seed, uint64_t stream = 0) : gen_(seed, stream) {}
  double next() {
    if (pos_ == 4) {
      block_ = gen_(ctr_++, 0);
      pos_ = 0;
    }
    return uniform_open(block_.v[pos_++]);
  }
  double next(double lo, double hi) { return lo + (hi - lo) * next(); }

 private:
  Philox gen_;
  Philox::Block block_{};
  uint64_t ctr_ = 0;
  int pos_ = 4;
};

}  // namespace ocean

#endif
