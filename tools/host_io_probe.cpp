// host_io_probe.cpp -- host-side costs of the reference-API (pageable
// std::vector) matvec path on the GPU box: multi-threaded pageable<->pinned
// memcpy, pinned and pageable DMA, and allocating + zeroing a fresh output
// vector (what a by-value std::vector return costs).
//   g++ -O2 -std=c++20 -I/usr/local/cuda/include tools/host_io_probe.cpp -L/usr/local/cuda/lib64 -lcudart -lpthread -o build/host_io_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const size_t n = 5000 * 1000, bytes = n * 8;
  std::vector<double> src(n, 1.0), dst(n, 0.0);
  double *pin = nullptr, *dev = nullptr;
  cudaMallocHost(&pin, bytes);
  cudaMalloc(&dev, bytes);
  std::memset(pin, 0, bytes);
  auto par_copy = [&](void* d, const void* s, int T) {
    std::vector<std::thread> th;
    const size_t per = (bytes + T - 1) / T;
    for (int t = 0; t < T; ++t)
      th.emplace_back([=] {
        const size_t a = t * per, b = std::min(bytes, a + per);
        if (a < b) std::memcpy((char*)d + a, (const char*)s + a, b - a);
      });
    for (auto& x : th) x.join();
  };
  std::printf("{\"cores\": %u", std::thread::hardware_concurrency());
  for (int T : {1, 2, 4, 8, 16}) {
    par_copy(pin, src.data(), T);
    const int R = 10;
    double t0 = now();
    for (int r = 0; r < R; ++r) par_copy(pin, src.data(), T);
    const double in_gbs = bytes * R / (now() - t0) / 1e9;
    t0 = now();
    for (int r = 0; r < R; ++r) par_copy(dst.data(), pin, T);
    const double out_gbs = bytes * R / (now() - t0) / 1e9;
    std::printf(", \"memcpy_to_pinned_T%d_GBs\": %.1f, \"memcpy_from_pinned_T%d_GBs\": %.1f", T, in_gbs, T, out_gbs);
  }
  auto dma = [&](void* d, const void* s, cudaMemcpyKind k) {
    cudaMemcpy(d, s, bytes, k);
    const int R = 10;
    const double t0 = now();
    for (int r = 0; r < R; ++r) cudaMemcpy(d, s, bytes, k);
    return bytes * R / (now() - t0) / 1e9;
  };
  std::printf(", \"h2d_pinned_GBs\": %.1f", dma(dev, pin, cudaMemcpyHostToDevice));
  std::printf(", \"d2h_pinned_GBs\": %.1f", dma(pin, dev, cudaMemcpyDeviceToHost));
  std::printf(", \"h2d_pageable_GBs\": %.1f", dma(dev, src.data(), cudaMemcpyHostToDevice));
  {  // pinned H2D split over k streams (copy engines) at once
    cudaStream_t st[4];
    for (auto& x : st) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    for (int k : {1, 2, 4}) {
      const int R = 10;
      const size_t part = bytes / k;
      cudaDeviceSynchronize();
      const double t0 = now();
      for (int r = 0; r < R; ++r)
        for (int i = 0; i < k; ++i)
          cudaMemcpyAsync((char*)dev + i * part, (char*)pin + i * part, part, cudaMemcpyHostToDevice, st[i]);
      cudaDeviceSynchronize();
      std::printf(", \"h2d_pinned_%dstreams_GBs\": %.1f", k, bytes * R / (now() - t0) / 1e9);
      const double t1 = now();
      for (int r = 0; r < R; ++r)
        for (int i = 0; i < k; ++i)
          cudaMemcpyAsync((char*)pin + i * part, (char*)dev + i * part, part, cudaMemcpyDeviceToHost, st[i]);
      cudaDeviceSynchronize();
      std::printf(", \"d2h_pinned_%dstreams_GBs\": %.1f", k, bytes * R / (now() - t1) / 1e9);
    }
    // H2D and D2H at the same time (F's input while F*'s output drains)
    const int R = 10;
    const double t2 = now();
    for (int r = 0; r < R; ++r) {
      cudaMemcpyAsync(dev, pin, bytes / 2, cudaMemcpyHostToDevice, st[0]);
      cudaMemcpyAsync((char*)pin + bytes / 2, (char*)dev + bytes / 2, bytes / 2, cudaMemcpyDeviceToHost, st[1]);
    }
    cudaDeviceSynchronize();
    std::printf(", \"h2d_plus_d2h_concurrent_GBs_total\": %.1f", bytes * R / (now() - t2) / 1e9);
  }
  std::printf(", \"d2h_pageable_GBs\": %.1f", dma(dst.data(), dev, cudaMemcpyDeviceToHost));
  {  // a 40 MB pinned H2D in flight while T threads copy 40 MB pageable -> pinned
    double* pin2 = nullptr;
    cudaMallocHost(&pin2, bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int T : {1, 4, 8}) {
      const int R = 5;
      double host = 0;
      const double t0 = now();
      for (int r = 0; r < R; ++r) {
        cudaMemcpyAsync(dev, pin, bytes, cudaMemcpyHostToDevice, st);
        const double h0 = now();
        par_copy(pin2, src.data(), T);
        host += now() - h0;
        cudaStreamSynchronize(st);
      }
      std::printf(", \"concurrent_T%d_ms\": %.3f, \"concurrent_T%d_host_ms\": %.3f", T, (now() - t0) / R * 1e3, T,
                  host / R * 1e3);
    }
  }
  {  // pinning the caller's pageable buffer per call: register + DMA + unregister
    const int R = 5;
    double treg = 0, tdma = 0, tun = 0;
    for (int r = 0; r < R; ++r) {
      const double a = now();
      cudaHostRegister(src.data(), bytes, cudaHostRegisterReadOnly);
      const double b = now();
      cudaMemcpy(dev, src.data(), bytes, cudaMemcpyHostToDevice);
      const double c = now();
      cudaHostUnregister(src.data());
      const double d = now();
      treg += b - a;
      tdma += c - b;
      tun += d - c;
    }
    std::printf(", \"register_ms\": %.3f, \"registered_h2d_ms\": %.3f, \"unregister_ms\": %.3f", treg / R * 1e3,
                tdma / R * 1e3, tun / R * 1e3);
  }
  {
    const int R = 10;
    double sink = 0;
    const double t0 = now();
    for (int r = 0; r < R; ++r) {
      std::vector<double> v(n);
      sink += v[n / 2 + r];
    }
    std::printf(", \"alloc_zero_40MB_ms\": %.3f, \"sink\": %g", (now() - t0) / R * 1e3, sink);
  }
  std::printf("}\n");
  return 0;
}
