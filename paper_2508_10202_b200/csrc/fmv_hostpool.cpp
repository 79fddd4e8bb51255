// fmv_hostpool.cpp -- a small persistent host thread pool for the library's
// host-side byte moves: copies between caller-owned PAGEABLE buffers (the
// reference API's std::vector I/O, matvec.hpp:305-318) and the context's
// pinned staging buffers, so the DMA engines see pinned memory and the
// pageable side is read / written by several cores at once.
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/fftmv_cuda.h"

namespace fmv {
namespace rt {

namespace {
class Pool {
 public:
  Pool() {
    const char* e = getenv("FMV_HOST_THREADS");
    int n = e && *e ? atoi(e) : (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
    n = std::max(1, std::min(n, 64));
    for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
    size_ = n;
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return size_; }
  // Runs fn(0..n-1) across the pool (the caller takes part); returns when all are done.
  void run(int n, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel region at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      ntask_ = n;
      next_ = 0;
      pending_ = n;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= ntask_) return;
        i = next_++;
        f = fn_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    unsigned long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int ntask_ = 0, next_ = 0, pending_ = 0, size_ = 1;
  unsigned long gen_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static Pool* p = new Pool;  // intentionally leaked: no join at static destruction
  return *p;
}
}  // namespace

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kMinPiece = 256 << 10;
  const int parts = (int)std::min<size_t>((size_t)pool().size(), std::max<size_t>(1, bytes / kMinPiece));
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t piece = (bytes / parts + 63) / 64 * 64;
  pool().run(parts, [&](int i) {
    const size_t off = (size_t)i * piece;
    if (off < bytes)
      std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(piece, bytes - off));
  });
}

}  // namespace rt
}  // namespace fmv

extern "C" int fmv_host_copy(void* dst, const void* src, size_t bytes) {
  if ((!dst || !src) && bytes) return FMV_EINVAL;
  if (bytes) fmv::rt::parallel_memcpy(dst, src, bytes);
  return FMV_OK;
}
