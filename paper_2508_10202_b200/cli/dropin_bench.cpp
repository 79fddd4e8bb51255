// dropin_bench.cpp -- end-to-end timing through the reference's own C++ API
// (include/fftmv: setup_operator, forward_matvec, adjoint_matvec;
// matvec.hpp:305-318 of the reference), exactly as a reference user calls
// it: std::vector (pageable) host vectors in, BlockVector out, PhaseTimings
// requested. bench.py runs it for the "e2e_dropin" figure.
//
//   fftmv_dropin_bench nm nd nt cfg steps warmup
//
// Prints one JSON line: host wall time per step (one F + one F*), matvecs/s,
// and the bytes copied per step.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "fftmv/matvec.hpp"
#include "fftmv/random_fill.hpp"

using namespace fftmv;

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: %s nm nd nt cfg steps warmup\n", argv[0]);
    return 2;
  }
  const std::size_t nm = std::strtoull(argv[1], nullptr, 10), nd = std::strtoull(argv[2], nullptr, 10),
                    nt = std::strtoull(argv[3], nullptr, 10);
  const PrecisionConfig cfg = parse_precision_config(argv[4]);
  const int steps = std::atoi(argv[5]), warmup = std::atoi(argv[6]);
  try {
    const std::uint64_t S = 20250814;
    const ProblemDims dims(nm, nd, nt);
    BlockColumn col(dims, uniform_fill(nt * nd * nm, seed_stream(S, 0)));
    const BlockVector m = BlockVector::time_double(nm, nt, uniform_fill(nm * nt, seed_stream(S, 1)));
    const BlockVector d = BlockVector::time_double(nd, nt, uniform_fill(nd * nt, seed_stream(S, 2)));
    const SpectralOperator op = setup_operator(col, HostBins::Skip);
    col = BlockColumn();
    double sink = 0;
    auto step = [&] {
      MatvecResult f = forward_matvec(op, m, cfg);
      MatvecResult a = adjoint_matvec(op, d, cfg);
      sink += f.output.f64[0] + a.output.f64[0];
    };
    for (int i = 0; i < warmup; ++i) step();
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps; ++i) step();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const double bytes = 8.0 * (double)(nm * nt + nd * nt);
    // breakdown: a fresh n_m*n_t output vector (what run_pipeline allocates for
    // F*), and the raw C-ABI calls on reused pageable vectors
    auto wall = [](auto&& fn, int reps) {
      const auto a = std::chrono::steady_clock::now();
      for (int i = 0; i < reps; ++i) fn();
      return 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count() / reps;
    };
    const double ms_alloc = wall([&] {
      std::vector<double> v(nm * nt);
      sink += v[nm * nt / 2];
    }, steps);
    std::vector<double> dout(nd * nt), mout(nm * nt);
    fmv_ctx* ctx = detail::thread_ctx(0);
    const std::string c = cfg.render();
    const double ms_f = wall([&] {
      detail::check(fmv_matvec(ctx, op.handle(), FMV_FORWARD, c.c_str(), m.f64.data(), dout.data(), 0, nullptr));
    }, steps);
    const double ms_a = wall([&] {
      detail::check(fmv_matvec(ctx, op.handle(), FMV_ADJOINT, c.c_str(), d.f64.data(), mout.data(), 0, nullptr));
    }, steps);
    std::printf(
        "{\"ms_per_step\": %.6f, \"matvecs_per_s\": %.3f, \"steps\": %d, \"h2d_bytes_per_step\": %.0f, "
        "\"d2h_bytes_per_step\": %.0f, \"ms_alloc_out_vector\": %.4f, \"ms_capi_F_pageable\": %.4f, "
        "\"ms_capi_Fstar_pageable\": %.4f, \"checksum\": %.17g}\n",
        1e3 * s / steps, 2.0 * steps / s, steps, bytes, bytes, ms_alloc, ms_f, ms_a, sink);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "dropin_bench: %s\n", e.what());
    return 1;
  }
  return 0;
}
