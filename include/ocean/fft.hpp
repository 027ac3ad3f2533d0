// ocean/fft.hpp — drop-in for proj/include/ocean/fft.hpp.
//
// Centered unnormalised synthesis transform (storage index s <-> wave index
// s - N/2, exponent +i), run by the sm_100a Stockham kernels (fp32 math,
// fp64 buffers in and out).
#ifndef OCEAN_B200_FFT_HPP
#define OCEAN_B200_FFT_HPP

#include <utility>

#include "ocean/core.hpp"

namespace ocean {

inline int neg_index(int s, int n) { return s == 0 ? 0 : n - s; }
bool is_conjugate_symmetric(const ComplexField& field, double tol = 1e-9);
ComplexField ifft2_centered(ComplexField field);
std::pair<RealField, RealField> ifft2_hermitian_pair(const ComplexField& x, const ComplexField& y,
                                                     bool check = false);

}  // namespace ocean

#endif
