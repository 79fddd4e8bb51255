// random_fill.hpp -- drop-in for the reference's deterministic fills
// (random_fill.hpp:17-32): mt19937_64, top 53 bits -> [lo, hi); seed streams.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "fftmv_cuda.h"

namespace fftmv {

inline std::vector<double> uniform_fill(std::size_t count, std::uint64_t seed, double lo = -1.0, double hi = 1.0) {
  std::vector<double> v(count);
  fmv_uniform_fill(count, seed, lo, hi, v.data());
  return v;
}

inline std::uint64_t seed_stream(std::uint64_t seed, std::uint64_t stream) { return fmv_seed_stream(seed, stream); }

}  // namespace fftmv
