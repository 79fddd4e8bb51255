// fft.hpp -- drop-in for the reference's batched real FFT facade
// (fft.hpp:30-164), executed by the sm_100a Stockham kernels of
// libfftmv_cuda (fmv_fft_r2c / fmv_fft_c2r). Same conventions: unnormalized
// forward with sign -1, half spectrum, inverse with 1/length folded in.
// Host-vector convenience front-end; the matvec pipeline never round-trips
// through it.
#pragma once

#include <complex>
#include <cstddef>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "fftmv/detail_capi.hpp"
#include "fftmv/precision.hpp"

namespace fftmv {

enum class FftDirection : std::uint8_t { Forward, Inverse };

class FftPlan {
 public:
  FftPlan(std::size_t length, std::size_t batch, Precision precision, FftDirection direction)
      : length_(length), batch_(batch), precision_(precision), direction_(direction) {
    if (length < 2 || length % 2 != 0) throw std::invalid_argument("FftPlan: length must be even and >= 2");
    if (batch < 1) throw std::invalid_argument("FftPlan: batch must be >= 1");
    if (precision == Precision::Half) throw std::invalid_argument("FftPlan: fp16 transforms are not supported");
  }
  std::size_t length() const { return length_; }
  std::size_t batch() const { return batch_; }
  Precision precision() const { return precision_; }
  FftDirection direction() const { return direction_; }
  std::size_t n_bins() const { return length_ / 2 + 1; }

 private:
  std::size_t length_, batch_;
  Precision precision_;
  FftDirection direction_;
};

namespace detail {
template <class T>
void check_plan(const FftPlan& p, FftDirection dir, std::size_t got, std::size_t want) {
  if (p.direction() != dir) throw std::invalid_argument("FFT: plan direction mismatch");
  if (p.precision() != precision_of<T>) throw std::invalid_argument("FFT: plan precision mismatch");
  if (got != want)
    throw std::invalid_argument("FFT: length mismatch, got " + std::to_string(got) + " scalars, expected " +
                                std::to_string(want));
}

template <class In, class Out>
std::vector<Out> run_fft(bool forward, const FftPlan& p, std::span<const In> in, std::size_t n_out) {
  DevBuf din(in.size_bytes() + 64), dout(n_out * sizeof(Out) + 64);
  cuda_check(cudaMemcpy(din.p, in.data(), in.size_bytes(), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  const char prec = p.precision() == Precision::Double ? 'd' : 's';
  fmv_ctx* ctx = thread_ctx();
  check(forward ? fmv_fft_r2c(ctx, p.length(), p.batch(), prec, din.p, dout.p)
                : fmv_fft_c2r(ctx, p.length(), p.batch(), prec, din.p, dout.p));
  check(fmv_synchronize(ctx));
  std::vector<Out> out(n_out);
  cuda_check(cudaMemcpy(out.data(), dout.p, n_out * sizeof(Out), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  return out;
}
}  // namespace detail

inline std::vector<std::complex<double>> forward_real_batched(const FftPlan& p, std::span<const double> series) {
  detail::check_plan<double>(p, FftDirection::Forward, series.size(), p.length() * p.batch());
  return detail::run_fft<double, std::complex<double>>(true, p, series, p.n_bins() * p.batch());
}
inline std::vector<std::complex<float>> forward_real_batched(const FftPlan& p, std::span<const float> series) {
  detail::check_plan<float>(p, FftDirection::Forward, series.size(), p.length() * p.batch());
  return detail::run_fft<float, std::complex<float>>(true, p, series, p.n_bins() * p.batch());
}
inline std::vector<double> inverse_real_batched(const FftPlan& p, std::span<const std::complex<double>> bins) {
  detail::check_plan<double>(p, FftDirection::Inverse, bins.size(), p.n_bins() * p.batch());
  return detail::run_fft<std::complex<double>, double>(false, p, bins, p.length() * p.batch());
}
inline std::vector<float> inverse_real_batched(const FftPlan& p, std::span<const std::complex<float>> bins) {
  detail::check_plan<float>(p, FftDirection::Inverse, bins.size(), p.n_bins() * p.batch());
  return detail::run_fft<std::complex<float>, float>(false, p, bins, p.length() * p.batch());
}

// Process-wide plan cache keyed like the reference (fft.hpp:150-164).
inline std::shared_ptr<const FftPlan> shared_plan(std::size_t length, std::size_t batch, Precision precision,
                                                  FftDirection direction) {
  static std::mutex mu;
  static std::map<std::tuple<std::size_t, std::size_t, int, int>, std::shared_ptr<const FftPlan>> cache;
  const auto key = std::make_tuple(length, batch, static_cast<int>(precision), static_cast<int>(direction));
  std::lock_guard<std::mutex> lk(mu);
  auto& slot = cache[key];
  if (!slot) slot = std::make_shared<const FftPlan>(length, batch, precision, direction);
  return slot;
}

}  // namespace fftmv
