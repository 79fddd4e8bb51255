// detail_capi.hpp -- error mapping and handle helpers shared by the drop-in
// headers. FMV_EINVAL -> std::invalid_argument (as the reference throws for
// shape/config errors); anything else -> std::runtime_error (fft.hpp:63).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "fftmv_cuda.h"

namespace fftmv::detail {

inline void check(int rc) {
  if (rc == FMV_OK) return;
  const std::string msg = fmv_last_error();
  if (rc == FMV_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("fftmv: " + msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("fftmv: ") + what + ": " + cudaGetErrorString(e));
}

// One context (CUDA stream + workspace) per host thread and device: contexts
// are single-threaded, spectral operators are shared.
inline fmv_ctx* thread_ctx(int device = 0) {
  struct Holder {
    fmv_ctx* c[16] = {};
    ~Holder() {
      for (auto* p : c)
        if (p) fmv_ctx_destroy(p);
    }
  };
  thread_local Holder h;
  if (device < 0 || device >= 16) throw std::invalid_argument("fftmv: device index out of range");
  if (!h.c[device]) check(fmv_ctx_create(device, nullptr, &h.c[device]));
  return h.c[device];
}

// Scoped device buffer.
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace fftmv::detail
