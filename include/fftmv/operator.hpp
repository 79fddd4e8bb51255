// operator.hpp -- drop-in for the reference's BlockColumn / SpectralOperator
// / setup_operator / materialize_single (operator.hpp:26-125).
//
// The spectral bins live on the GPU (fmv_op, owned by libfftmv_cuda):
// setup_operator runs the fp64 r2c of every padded series there, on the
// device it is given (default 0; one process per GPU passes its local
// device). The public bins_double field is kept and, as in the reference
// (operator.hpp:59), populated by setup_operator -- at C2 that is 8 GB of host
// memory, the reference's own footprint. HostBins::Skip opts out (the device
// copy is all the matvecs need); bins_view() then throws until
// download_bins() fills the field. ensure_single() materializes the fp32 bins
// on the device (the copy the SBGEMV reads) and returns a host view of them.
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

// Auto and Keep populate bins_double (the reference's behaviour); Skip leaves
// it empty.
enum class HostBins : std::uint8_t { Auto, Keep, Skip };

struct SpectralOperator {
  ProblemDims dims;
  std::vector<std::complex<double>> bins_double;  // host mirror (see header comment)

  std::size_t bin_elems() const { return dims.n_d * dims.n_m; }
  fmv_op* handle() const { return dev_ ? dev_->op : nullptr; }
  int device() const { return dev_ ? dev_->device : 0; }

  // Fills bins_double from the device copy (reference layout).
  void download_bins() {
    bins_double.resize(dims.n_bins() * bin_elems());
    detail::check(fmv_op_download_bins(detail::thread_ctx(device()), handle(), 'd', bins_double.data()));
  }
  MatrixBatch<std::complex<double>> bins_view() const {
    if (bins_double.empty())
      throw std::logic_error("SpectralOperator: set up with HostBins::Skip; call download_bins() first");
    return MatrixBatch<std::complex<double>>::tight(bins_double, dims.n_d, dims.n_m, dims.n_bins());
  }
  bool has_single() const { return dev_ && fmv_op_has(dev_->op, 's'); }
  const std::vector<std::complex<float>>& ensure_single() const {
    // (the one logical cast of operator.hpp:72 is counted by the library when
    // the device copy is created, whoever triggers it first)
    std::call_once(dev_->single_once, [this] {
      detail::check(fmv_op_materialize(detail::thread_ctx(device()), dev_->op, 's'));
      dev_->single.resize(dims.n_bins() * bin_elems());
      detail::check(fmv_op_download_bins(detail::thread_ctx(device()), dev_->op, 's', dev_->single.data()));
    });
    return dev_->single;
  }
  MatrixBatch<std::complex<float>> bins_single_view() const {
    return MatrixBatch<std::complex<float>>::tight(ensure_single(), dims.n_d, dims.n_m, dims.n_bins());
  }
  // Device-only materialization (no host copy): what the matvec needs.
  void materialize_device(char prec) const {
    detail::check(fmv_op_materialize(detail::thread_ctx(device()), dev_->op, prec));
  }

 private:
  struct Device {
    fmv_op* op = nullptr;
    int device = 0;
    std::once_flag single_once;
    std::vector<std::complex<float>> single;
    ~Device() {
      if (op) fmv_op_destroy(op);
    }
  };
  std::shared_ptr<Device> dev_;
  friend SpectralOperator setup_operator(const BlockColumn&, HostBins, int);
};

inline SpectralOperator setup_operator(const BlockColumn& col, HostBins host = HostBins::Auto, int device = 0) {
  SpectralOperator op;
  op.dims = col.dims;
  op.dev_ = std::make_shared<SpectralOperator::Device>();
  op.dev_->device = device;
  detail::check(fmv_op_create(detail::thread_ctx(device), col.dims.n_m, col.dims.n_d, col.dims.n_t, col.data.data(), 0,
                              &op.dev_->op));
  if (host != HostBins::Skip) op.download_bins();
  return op;
}

inline const SpectralOperator& materialize_single(const SpectralOperator& op) {
  op.materialize_device('s');
  return op;
}

}  // namespace fftmv
