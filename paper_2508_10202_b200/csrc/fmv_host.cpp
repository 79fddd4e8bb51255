// fmv_host.cpp -- host-side pieces of the reference API that the B200 path
// keeps verbatim in behaviour: deterministic synthetic fills
// (random_fill.hpp:17-32, sweep.hpp:32-46) and the error metric
// (sweep.hpp:49-59). Exported through include/fftmv_cuda.h.
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>

#include "../../include/fftmv_cuda.h"

extern "C" {

uint64_t fmv_seed_stream(uint64_t seed, uint64_t stream) { return seed ^ (0x9E3779B97F4A7C15ull * (stream + 1)); }

void fmv_uniform_fill(size_t count, uint64_t seed, double lo, double hi, double* out) {
  std::mt19937_64 rng(seed);
  const double scale = hi - lo;
  for (size_t i = 0; i < count; ++i) {
    const double u01 = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    out[i] = lo + scale * u01;
  }
}

int fmv_non_representable_fill(size_t count, uint64_t seed, double* out) {
  if (count < 1) return FMV_EINVAL;
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < count; ++i) {
    const uint64_t u = rng();
    double mag = 0.5 + static_cast<double>(u >> 12) * 0x1.0p-53;
    uint64_t bits = std::bit_cast<uint64_t>(mag);
    bits |= (uint64_t{1} << 29) - 1;
    mag = std::bit_cast<double>(bits);
    out[i] = (u & 1u) ? -mag : mag;
  }
  return FMV_OK;
}

int fmv_relative_error(size_t n, const double* x, const double* ref, double* out) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double d = x[i] - ref[i];
    num += d * d;
    den += ref[i] * ref[i];
  }
  if (den == 0.0) return FMV_EINVAL;
  *out = std::sqrt(num) / std::sqrt(den);
  return FMV_OK;
}

}  // extern "C"
