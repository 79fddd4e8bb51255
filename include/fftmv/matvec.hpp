// matvec.hpp -- drop-in for the reference's five-phase matvec API
// (matvec.hpp:40-318). The whole pipeline runs in three fused sm_100a
// kernels inside libfftmv_cuda (fmv_matvec): pad+cast+r2c+reorder,
// SBGEMV (+ both reorders and casts), reorder+1/L+c2r+unpad+cast.
// PhaseTimings attribution on B200 (fftmv_cuda.h): [0] H2D of the input,
// [1] r2c kernels, [2] SBGEMV kernels, [3] c2r kernels, [4] D2H of the
// output, each the summed CUDA-event time; the host copies overlap the
// SBGEMV column chunks, so the phases may sum to more than total_s.
#pragma once

#include <array>
#include <chrono>
#include <string>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "fftmv/block_vector.hpp"
#include "fftmv/config.hpp"
#include "fftmv/detail_capi.hpp"
#include "fftmv/gemv.hpp"
#include "fftmv/operator.hpp"

namespace fftmv {

enum class MatvecKind : std::uint8_t { Forward, Adjoint };

struct PhaseTimings {
  std::array<double, 5> phase_s{};
  double total_s = 0.0;
  PhaseTimings& operator+=(const PhaseTimings& o) {
    for (std::size_t i = 0; i < 5; ++i) phase_s[i] += o.phase_s[i];
    total_s += o.total_s;
    return *this;
  }
};

inline const char* phase_name(std::size_t i) {
  static constexpr const char* kNames[5] = {"pad", "fft", "sbgemv", "ifft", "unpad"};
  return kNames[i];
}

struct MatvecResult {
  BlockVector output;
  PhaseTimings timings;
};

namespace detail {

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Working buffer tagged with its precision (the partitioned adjoint's payload).
struct RealBuf {
  Precision prec = Precision::Double;
  std::vector<float> f;
  std::vector<double> d;
  std::size_t size() const { return prec == Precision::Double ? d.size() : f.size(); }
};

inline std::pair<std::vector<double>, PhaseTimings> run_pipeline(const SpectralOperator& op, MatvecKind kind,
                                                                 std::span<const double> input, const RealBuf* payload,
                                                                 PrecisionConfig cfg, const TilingParams& = {}) {
  const bool fwd = kind == MatvecKind::Forward;
  const std::size_t n_in = (fwd ? op.dims.n_m : op.dims.n_d) * op.dims.n_t;
  const std::size_t n_out = (fwd ? op.dims.n_d : op.dims.n_m) * op.dims.n_t;
  const std::string c = cfg.render();
  fmv_phase_times t{};
  fmv_ctx* ctx = thread_ctx(op.device());
  const int k = fwd ? FMV_FORWARD : FMV_ADJOINT;
  auto run = [&](double* dst) {
    if (payload) {
      // payload already rounded to cfg[0] (partition.hpp:196-206): phase 1
      // pads it as is, in its own precision
      if (payload->size() != n_in) throw std::invalid_argument("matvec: input length does not match operator dims");
      if (payload->prec == Precision::Double) {
        check(fmv_matvec_payload(ctx, op.handle(), k, c.c_str(), 'd', payload->d.data(), dst, 0, &t));
      } else if (payload->prec == Precision::Single) {
        check(fmv_matvec_payload(ctx, op.handle(), k, c.c_str(), 's', payload->f.data(), dst, 0, &t));
      } else {  // fp16 extension: the float buffer holds binary16 values exactly
        std::vector<_Float16> h(payload->f.size());
        for (std::size_t i = 0; i < h.size(); ++i) h[i] = static_cast<_Float16>(payload->f[i]);
        check(fmv_matvec_payload(ctx, op.handle(), k, c.c_str(), 'h', h.data(), dst, 0, &t));
      }
    } else {
      if (input.size() != n_in) throw std::invalid_argument("matvec: input length does not match operator dims");
      check(fmv_matvec(ctx, op.handle(), k, c.c_str(), input.data(), dst, 0, &t));
    }
  };
  std::vector<double> out;
  if (n_out * sizeof(double) < (std::size_t(4) << 20)) {
    out.resize(n_out);
    run(out.data());
  } else {
    // A large result (F*: 40 MB at C2) is DMA'd into a pinned buffer while
    // another thread allocates and value-initializes the returned vector
    // (1.4-1.8 ms for 40 MB, as long as the matvec itself); the host pool
    // then copies it over.
    double* pin = static_cast<double*>(thread_pinned_out().ensure(n_out * sizeof(double)));
    HelperThread& helper = thread_helper();
    helper.start([&] { out = std::vector<double>(n_out); });
    try {
      run(pin);
    } catch (...) {
      helper.wait();
      throw;
    }
    helper.wait();
    check(fmv_host_copy(out.data(), pin, n_out * sizeof(double)));
  }
  PhaseTimings pt;
  for (int i = 0; i < 5; ++i) pt.phase_s[i] = t.phase_s[i];
  pt.total_s = t.total_s;
  return {std::move(out), pt};
}

inline void check_matvec_input(const SpectralOperator& op, const BlockVector& v, bool forward) {
  v.validate();
  if (v.precision != Precision::Double) throw std::invalid_argument("matvec: input must be double precision");
  if (v.domain != Domain::Time || v.layout != Layout::SOTI)
    throw std::invalid_argument("matvec: input must be a time-domain SOTI vector");
  if (v.space_extent != (forward ? op.dims.n_m : op.dims.n_d) || v.time_extent != op.dims.n_t)
    throw std::invalid_argument("matvec: input extents do not match operator dims");
}

}  // namespace detail

inline MatvecResult forward_matvec(const SpectralOperator& op, const BlockVector& m, PrecisionConfig cfg,
                                   const TilingParams& tiling = {}) {
  detail::check_matvec_input(op, m, true);
  auto [out, t] = detail::run_pipeline(op, MatvecKind::Forward, m.f64, nullptr, cfg, tiling);
  return {BlockVector::time_double(op.dims.n_d, op.dims.n_t, std::move(out)), t};
}

inline MatvecResult adjoint_matvec(const SpectralOperator& op, const BlockVector& d, PrecisionConfig cfg,
                                   const TilingParams& tiling = {}) {
  detail::check_matvec_input(op, d, false);
  auto [out, t] = detail::run_pipeline(op, MatvecKind::Adjoint, d.f64, nullptr, cfg, tiling);
  return {BlockVector::time_double(op.dims.n_m, op.dims.n_t, std::move(out)), t};
}

// Block (multi-RHS) matvecs -- an addition to the reference API (SURVEY.md §8
// f2; the Hessian-assembly use case): one call applies F or
// F* to every vector in `in`, streaming the operator once per 8 (F) / 4 (F*)
// right-hand sides (fmv_matvec_block). out[r] equals forward_matvec /
// adjoint_matvec of in[r] up to summation order.
namespace detail {
inline std::vector<BlockVector> matvec_block(const SpectralOperator& op, const std::vector<BlockVector>& in,
                                             PrecisionConfig cfg, bool fwd) {
  const std::size_t n_in = (fwd ? op.dims.n_m : op.dims.n_d) * op.dims.n_t;
  const std::size_t n_out = (fwd ? op.dims.n_d : op.dims.n_m) * op.dims.n_t;
  std::vector<double> packed;
  packed.reserve(in.size() * n_in);
  for (const auto& v : in) {
    check_matvec_input(op, v, fwd);
    packed.insert(packed.end(), v.f64.begin(), v.f64.end());
  }
  std::vector<double> out(in.size() * n_out);
  if (!in.empty())
    check(fmv_matvec_block(thread_ctx(op.device()), op.handle(), fwd ? FMV_FORWARD : FMV_ADJOINT, cfg.render().c_str(),
                           in.size(), packed.data(), out.data(), 0));
  std::vector<BlockVector> res;
  res.reserve(in.size());
  for (std::size_t r = 0; r < in.size(); ++r)
    res.push_back(BlockVector::time_double(fwd ? op.dims.n_d : op.dims.n_m, op.dims.n_t,
                                           std::vector<double>(out.begin() + r * n_out, out.begin() + (r + 1) * n_out)));
  return res;
}
}  // namespace detail

inline std::vector<BlockVector> forward_matvec_block(const SpectralOperator& op, const std::vector<BlockVector>& m,
                                                     PrecisionConfig cfg = {}) {
  return detail::matvec_block(op, m, cfg, true);
}
inline std::vector<BlockVector> adjoint_matvec_block(const SpectralOperator& op, const std::vector<BlockVector>& d,
                                                     PrecisionConfig cfg = {}) {
  return detail::matvec_block(op, d, cfg, false);
}

}  // namespace fftmv
