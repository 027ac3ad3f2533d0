// ocean/parallel.hpp — drop-in for proj/include/ocean/parallel.hpp.
//
// On the B200 path the data parallelism lives in the kernels, so the worker
// budget only affects these host utilities. deterministic_sum keeps the
// reference's fixed 1024-chunk order (bit-stable for any thread count).
#ifndef OCEAN_B200_PARALLEL_HPP
#define OCEAN_B200_PARALLEL_HPP

#include <algorithm>
#include <cstddef>
#include <functional>
#include <vector>

namespace ocean {

int worker_count();
void set_worker_count(int n);
void parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn);

template <typename T, typename Fn>
T deterministic_sum(size_t n, T init, Fn term) {
  constexpr size_t kChunk = 1024;
  T total = init;
  for (size_t c0 = 0; c0 < n; c0 += kChunk) {
    T acc = init;
    for (size_t i = c0, e = std::min(n, c0 + kChunk); i < e; ++i) acc += term(i);
    total += acc;
  }
  return total;
}

}  // namespace ocean

#endif
