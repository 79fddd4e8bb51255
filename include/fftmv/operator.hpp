// operator.hpp -- drop-in for the reference's BlockColumn / SpectralOperator
// / setup_operator / materialize_single (operator.hpp:26-125).
//
// The spectral bins live on the GPU (fmv_op, owned by libfftmv_cuda):
// setup_operator runs the fp64 r2c of every padded series there. The public
// bins_double field is kept: it is filled from the device when the operator
// is at most host_bins_limit bytes (1 GiB by default) or when requested with
// HostBins::Keep; download_bins() fills it on demand. ensure_single()
// materializes the fp32 bins on the device (the copy the SBGEMV reads) and
// returns a host view of them.
#pragma once

#include <complex>
#include <cstddef>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "fftmv/detail_capi.hpp"
#include "fftmv/dims.hpp"
#include "fftmv/gemv.hpp"
#include "fftmv/precision.hpp"

namespace fftmv {

struct BlockColumn {
  ProblemDims dims;
  std::vector<double> data;  // data[t*n_d*n_m + i + j*n_d]

  BlockColumn() = default;
  BlockColumn(ProblemDims d, std::vector<double> values) : dims(d), data(std::move(values)) {
    if (data.size() != d.n_t * d.n_d * d.n_m) throw std::invalid_argument("BlockColumn: buffer length does not match dims");
  }
  std::size_t block_elems() const { return dims.n_d * dims.n_m; }
  std::span<const double> block(std::size_t t) const {
    return std::span<const double>(data).subspan(t * block_elems(), block_elems());
  }
  double& at(std::size_t t, std::size_t i, std::size_t j) { return data[t * block_elems() + j * dims.n_d + i]; }
  double at(std::size_t t, std::size_t i, std::size_t j) const { return data[t * block_elems() + j * dims.n_d + i]; }
  static BlockColumn zeros(ProblemDims d) { return BlockColumn(d, std::vector<double>(d.n_t * d.n_d * d.n_m)); }
};

enum class HostBins : std::uint8_t { Auto, Keep, Skip };
inline constexpr std::size_t host_bins_limit = std::size_t{1} << 30;

struct SpectralOperator {
  ProblemDims dims;
  std::vector<std::complex<double>> bins_double;  // host mirror (see header comment)

  std::size_t bin_elems() const { return dims.n_d * dims.n_m; }
  fmv_op* handle() const { return dev_ ? dev_->op : nullptr; }

  // Fills bins_double from the device copy (reference layout).
  void download_bins() {
    bins_double.resize(dims.n_bins() * bin_elems());
    detail::check(fmv_op_download_bins(detail::thread_ctx(), handle(), 'd', bins_double.data()));
  }
  MatrixBatch<std::complex<double>> bins_view() const {
    if (bins_double.empty()) throw std::logic_error("SpectralOperator: host bins not kept; call download_bins()");
    return MatrixBatch<std::complex<double>>::tight(bins_double, dims.n_d, dims.n_m, dims.n_bins());
  }
  bool has_single() const { return dev_ && fmv_op_has(dev_->op, 's'); }
  const std::vector<std::complex<float>>& ensure_single() const {
    std::call_once(dev_->single_once, [this] {
      detail::check(fmv_op_materialize(detail::thread_ctx(), dev_->op, 's'));
      dev_->single.resize(dims.n_bins() * bin_elems());
      detail::check(fmv_op_download_bins(detail::thread_ctx(), dev_->op, 's', dev_->single.data()));
      note_cast();
    });
    return dev_->single;
  }
  MatrixBatch<std::complex<float>> bins_single_view() const {
    return MatrixBatch<std::complex<float>>::tight(ensure_single(), dims.n_d, dims.n_m, dims.n_bins());
  }
  // Device-only materialization (no host copy): what the matvec needs.
  void materialize_device(char prec) const { detail::check(fmv_op_materialize(detail::thread_ctx(), dev_->op, prec)); }

 private:
  struct Device {
    fmv_op* op = nullptr;
    std::once_flag single_once;
    std::vector<std::complex<float>> single;
    ~Device() {
      if (op) fmv_op_destroy(op);
    }
  };
  std::shared_ptr<Device> dev_;
  friend SpectralOperator setup_operator(const BlockColumn&, HostBins);
};

inline SpectralOperator setup_operator(const BlockColumn& col, HostBins host = HostBins::Auto) {
  SpectralOperator op;
  op.dims = col.dims;
  op.dev_ = std::make_shared<SpectralOperator::Device>();
  detail::check(fmv_op_create(detail::thread_ctx(), col.dims.n_m, col.dims.n_d, col.dims.n_t, col.data.data(), 0,
                              &op.dev_->op));
  const std::size_t bytes = op.dims.n_bins() * op.bin_elems() * sizeof(std::complex<double>);
  if (host == HostBins::Keep || (host == HostBins::Auto && bytes <= host_bins_limit)) op.download_bins();
  return op;
}

inline const SpectralOperator& materialize_single(const SpectralOperator& op) {
  op.materialize_device('s');
  return op;
}

}  // namespace fftmv
