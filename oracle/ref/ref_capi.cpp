// C ABI around the UNMODIFIED reference headers (/root/reference/proj/include/fftmv).
// TEST INFRASTRUCTURE ONLY: built into oracle/_ref/libfftmv_ref.so by
// oracle/Makefile, loaded by tests/ (as the checker), by
// __graft_entry__.smoke() and by bench.py's reference / cpu_baseline arm.
// Nothing in the product library (paper_2508_10202_b200/) links or calls it.
//
// Every entry point forwards to the reference function named in its comment;
// exceptions become return codes (-1 invalid_argument, -2 other) with the
// message retrievable through ref_last_error().
#include <algorithm>
#include <atomic>
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fftmv/block_vector.hpp"
#include "fftmv/config.hpp"
#include "fftmv/dense_ref.hpp"
#include "fftmv/dims.hpp"
#include "fftmv/fft.hpp"
#include "fftmv/gemv.hpp"
#include "fftmv/matvec.hpp"
#include "fftmv/operator.hpp"
#include "fftmv/partition.hpp"
#include "fftmv/precision.hpp"
#include "fftmv/random_fill.hpp"
#include "fftmv/sweep.hpp"

using namespace fftmv;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

void put_times(const PhaseTimings& t, double* out6) {
  if (!out6) return;
  for (int i = 0; i < 5; ++i) out6[i] = t.phase_s[i];
  out6[5] = t.total_s;
}

template <class T>
void gemv_dispatch(int impl, GemvMode mode, std::size_t m, std::size_t n, std::size_t batch, std::size_t lda,
                   std::size_t stride_a, const void* A, std::size_t a_len, std::size_t stride_x, const void* x,
                   std::size_t x_len, std::size_t stride_y, void* y, std::size_t y_len, const TilingParams& tp) {
  MatrixBatch<T> Ab{std::span<const T>(static_cast<const T*>(A), a_len), m, n, batch, lda, stride_a};
  const std::size_t xlen = is_transpose(mode) ? m : n;
  const std::size_t ylen = is_transpose(mode) ? n : m;
  VectorBatch<const T> xb{std::span<const T>(static_cast<const T*>(x), x_len), xlen, stride_x, batch};
  VectorBatch<T> yb{std::span<T>(static_cast<T*>(y), y_len), ylen, stride_y, batch};
  if (impl == 0)
    gemv_batched_naive(mode, Ab, xb, yb);
  else if (impl == 1)
    gemv_batched_tiled(mode, Ab, xb, yb, tp);
  else
    gemv_batched_auto(mode, Ab, xb, yb, tp);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// random_fill.hpp:17-27
void ref_uniform_fill(std::size_t count, std::uint64_t seed, double lo, double hi, double* out) {
  const auto v = uniform_fill(count, seed, lo, hi);
  std::memcpy(out, v.data(), count * sizeof(double));
}
// random_fill.hpp:30-32
std::uint64_t ref_seed_stream(std::uint64_t seed, std::uint64_t stream) { return seed_stream(seed, stream); }
// sweep.hpp:32-46
int ref_non_representable_fill(std::size_t count, std::uint64_t seed, double* out) {
  return guarded([&] {
    const auto v = non_representable_fill(count, seed);
    std::memcpy(out, v.data(), count * sizeof(double));
  });
}
// sweep.hpp:49-59
int ref_relative_error(std::size_t n, const double* x, const double* r, double* out) {
  return guarded([&] { *out = relative_error({x, n}, {r, n}); });
}
// gemv.hpp:83-89
int ref_effective_bandwidth(std::size_t m, std::size_t n, std::size_t batch, std::size_t es, double s, double* out) {
  return guarded([&] { *out = effective_bandwidth(m, n, batch, es, s); });
}
// gemv.hpp:74-79 (returns 0 Naive, 1 Tiled)
int ref_select_kernel(std::size_t m, std::size_t n, int mode, std::size_t col_tile, std::size_t row_chunk,
                      double ratio, std::size_t cutoff) {
  return select_kernel(m, n, static_cast<GemvMode>(mode), TilingParams{col_tile, row_chunk, ratio, cutoff}) ==
                 KernelChoice::Tiled
             ? 1
             : 0;
}

// precision.hpp:27-39
std::uint64_t ref_casts_performed() { return casts_performed(); }
void ref_reset_cast_counter() { reset_cast_counter(); }

// config.hpp:36-51; writes the canonical rendering back (round trip)
int ref_parse_config(const char* s, char* out6) {
  return guarded([&] {
    const auto c = parse_precision_config(s);
    std::memcpy(out6, c.render().c_str(), 6);
  });
}
// config.hpp:55-65; 32 x 5 chars
void ref_enumerate_configs(char* out160) {
  const auto all = enumerate_configs();
  for (std::size_t i = 0; i < all.size(); ++i) std::memcpy(out160 + 5 * i, all[i].render().data(), 5);
}

// operator.hpp:99-125
void* ref_setup_operator(std::size_t nm, std::size_t nd, std::size_t nt, const double* col) {
  SpectralOperator* op = nullptr;
  const int rc = guarded([&] {
    const ProblemDims d(nm, nd, nt);
    BlockColumn bc(d, std::vector<double>(col, col + nm * nd * nt));
    op = new SpectralOperator(setup_operator(bc));
  });
  return rc == 0 ? op : nullptr;
}
void ref_op_free(void* op) { delete static_cast<SpectralOperator*>(op); }
// operator.hpp:59 (bin-major, column-major within bin, interleaved re/im)
void ref_op_bins(void* op, double* out) {
  const auto* o = static_cast<SpectralOperator*>(op);
  std::memcpy(out, o->bins_double.data(), o->bins_double.size() * sizeof(std::complex<double>));
}
// operator.hpp:70-75, :90-93
void ref_op_bins_single(void* op, float* out) {
  const auto* o = static_cast<SpectralOperator*>(op);
  const auto& b = materialize_single(*o).ensure_single();
  std::memcpy(out, b.data(), b.size() * sizeof(std::complex<float>));
}
void ref_op_materialize_single(void* op) { materialize_single(*static_cast<SpectralOperator*>(op)); }

// matvec.hpp:305-318 (kind 0 forward, 1 adjoint); phase_s6 = 5 phases + total
int ref_matvec(void* op, int kind, const char* cfg, const double* in, double* out, double* phase_s6) {
  return guarded([&] {
    const auto* o = static_cast<SpectralOperator*>(op);
    const auto c = parse_precision_config(cfg);
    const bool fwd = kind == 0;
    const std::size_t n_in = fwd ? o->dims.n_m : o->dims.n_d;
    const std::size_t n_out = fwd ? o->dims.n_d : o->dims.n_m;
    const auto v = BlockVector::time_double(n_in, o->dims.n_t, std::vector<double>(in, in + n_in * o->dims.n_t));
    const MatvecResult r = fwd ? forward_matvec(*o, v, c) : adjoint_matvec(*o, v, c);
    std::memcpy(out, r.output.f64.data(), n_out * o->dims.n_t * sizeof(double));
    put_times(r.timings, phase_s6);
  });
}

// dense_ref.hpp:30-64
int ref_dense(int kind, std::size_t nm, std::size_t nd, std::size_t nt, const double* col, const double* in,
              double* out) {
  return guarded([&] {
    const ProblemDims d(nm, nd, nt);
    BlockColumn bc(d, std::vector<double>(col, col + nm * nd * nt));
    const std::size_t n_in = kind == 0 ? nm : nd;
    const std::span<const double> x(in, n_in * nt);
    const auto r = kind == 0 ? dense_forward(bc, x) : dense_adjoint(bc, x);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// fft.hpp:110-148. prec: 0 single, 1 double. Buffers interleaved complex.
int ref_fft_forward(std::size_t L, std::size_t batch, int prec, const void* in, void* out) {
  return guarded([&] {
    const auto p = shared_plan(L, batch, prec ? Precision::Double : Precision::Single, FftDirection::Forward);
    if (prec) {
      const auto r = forward_real_batched(*p, std::span<const double>(static_cast<const double*>(in), L * batch));
      std::memcpy(out, r.data(), r.size() * sizeof(r[0]));
    } else {
      const auto r = forward_real_batched(*p, std::span<const float>(static_cast<const float*>(in), L * batch));
      std::memcpy(out, r.data(), r.size() * sizeof(r[0]));
    }
  });
}
int ref_fft_inverse(std::size_t L, std::size_t batch, int prec, const void* in, void* out) {
  return guarded([&] {
    const std::size_t nb = L / 2 + 1;
    const auto p = shared_plan(L, batch, prec ? Precision::Double : Precision::Single, FftDirection::Inverse);
    if (prec) {
      const auto* b = static_cast<const std::complex<double>*>(in);
      const auto r = inverse_real_batched(*p, std::span<const std::complex<double>>(b, nb * batch));
      std::memcpy(out, r.data(), r.size() * sizeof(r[0]));
    } else {
      const auto* b = static_cast<const std::complex<float>*>(in);
      const auto r = inverse_real_batched(*p, std::span<const std::complex<float>>(b, nb * batch));
      std::memcpy(out, r.data(), r.size() * sizeof(r[0]));
    }
  });
}

// gemv.hpp:206-240. impl 0 naive, 1 tiled, 2 auto; dtype 's','d','c','z'; lengths in elements.
int ref_gemv(int impl, int mode, char dtype, std::size_t m, std::size_t n, std::size_t batch, std::size_t lda,
             std::size_t stride_a, const void* A, std::size_t a_len, std::size_t stride_x, const void* x,
             std::size_t x_len, std::size_t stride_y, void* y, std::size_t y_len, std::size_t col_tile,
             std::size_t row_chunk, double ratio, std::size_t cutoff) {
  return guarded([&] {
    const TilingParams tp{col_tile, row_chunk, ratio, cutoff};
    const auto md = static_cast<GemvMode>(mode);
    switch (dtype) {
      case 's': gemv_dispatch<float>(impl, md, m, n, batch, lda, stride_a, A, a_len, stride_x, x, x_len, stride_y, y, y_len, tp); break;
      case 'd': gemv_dispatch<double>(impl, md, m, n, batch, lda, stride_a, A, a_len, stride_x, x, x_len, stride_y, y, y_len, tp); break;
      case 'c': gemv_dispatch<std::complex<float>>(impl, md, m, n, batch, lda, stride_a, A, a_len, stride_x, x, x_len, stride_y, y, y_len, tp); break;
      case 'z': gemv_dispatch<std::complex<double>>(impl, md, m, n, batch, lda, stride_a, A, a_len, stride_x, x, x_len, stride_y, y, y_len, tp); break;
      default: throw std::invalid_argument("ref_gemv: dtype must be s/d/c/z");
    }
  });
}

// partition.hpp:27-40 -> 2*p size_t [begin,end)
int ref_grid_split(std::size_t p, std::size_t nm, std::size_t* ranges) {
  return guarded([&] {
    const auto g = Grid1xP::split(p, nm);
    for (std::size_t w = 0; w < p; ++w) {
      ranges[2 * w] = g.shard_ranges[w].first;
      ranges[2 * w + 1] = g.shard_ranges[w].second;
    }
  });
}
// partition.hpp:128-132; bufs = p contiguous vectors of n
int ref_tree_reduce(std::size_t p, std::size_t n, const double* bufs, int prec, double* out) {
  return guarded([&] {
    std::vector<std::vector<double>> b(p);
    for (std::size_t w = 0; w < p; ++w) b[w].assign(bufs + w * n, bufs + (w + 1) * n);
    const auto r = tree_reduce(b, prec ? Precision::Double : Precision::Single);
    std::memcpy(out, r.data(), n * sizeof(double));
  });
}
// partition.hpp:141-147
void* ref_setup_partitioned(std::size_t nm, std::size_t nd, std::size_t nt, const double* col, std::size_t p) {
  PartitionedOperator* pop = nullptr;
  const int rc = guarded([&] {
    const ProblemDims d(nm, nd, nt);
    BlockColumn bc(d, std::vector<double>(col, col + nm * nd * nt));
    pop = new PartitionedOperator(setup_partitioned(bc, Grid1xP::split(p, nm)));
  });
  return rc == 0 ? pop : nullptr;
}
void ref_pop_free(void* p) { delete static_cast<PartitionedOperator*>(p); }
// partition.hpp:157-217. forward_matvec_partitioned throws for p>=2 (its input
// check compares the full m against the shard dims, partition.hpp:159), so
// the forward body (:164-181) is restated here around the verbatim
// run_pipeline and tree_reduce; the adjoint calls the reference directly.
int ref_matvec_partitioned(void* pp, int kind, const char* cfg, const double* in, double* out, double* phase_s6) {
  return guarded([&] {
    const auto* pop = static_cast<PartitionedOperator*>(pp);
    const auto c = parse_precision_config(cfg);
    const std::size_t nt = pop->dims.n_t;
    if (kind == 0) {
      PhaseTimings total;
      std::vector<std::vector<double>> partials;
      for (std::size_t w = 0; w < pop->grid.p; ++w) {
        const auto [lo, hi] = pop->grid.shard_ranges[w];
        auto [part, t] = detail::run_pipeline(pop->workers[w], MatvecKind::Forward,
                                              std::span<const double>(in + lo * nt, (hi - lo) * nt), nullptr, c, {});
        total += t;
        partials.push_back(std::move(part));
      }
      const auto comm = CommSpec::forward_reduce(c, pop->dims);
      const auto d = tree_reduce(partials, comm.precision);
      std::memcpy(out, d.data(), d.size() * sizeof(double));
      put_times(total, phase_s6);
    } else {
      const auto d =
          BlockVector::time_double(pop->dims.n_d, nt, std::vector<double>(in, in + pop->dims.n_d * nt));
      const auto r = adjoint_matvec_partitioned(*pop, d, c);
      std::memcpy(out, r.output.f64.data(), r.output.f64.size() * sizeof(double));
      put_times(r.timings, phase_s6);
    }
  });
}

// sweep.hpp:108-119 + make_report (:169-179). rows: 32 x {mean,min,max,err}.
int ref_sweep(void* op, int kind, const double* in, int reps, int warmup, double tol, double* rows, char* chosen6) {
  return guarded([&] {
    const auto* o = static_cast<SpectralOperator*>(op);
    const std::size_t n_in = kind == 0 ? o->dims.n_m : o->dims.n_d;
    auto res = sweep_configs(*o, std::span<const double>(in, n_in * o->dims.n_t),
                             kind == 0 ? MatvecKind::Forward : MatvecKind::Adjoint, reps, warmup);
    for (std::size_t i = 0; i < res.size(); ++i) {
      rows[4 * i] = res[i].mean_s;
      rows[4 * i + 1] = res[i].min_s;
      rows[4 * i + 2] = res[i].max_s;
      rows[4 * i + 3] = res[i].rel_error;
    }
    const auto rep = make_report(o->dims, kind == 0 ? MatvecKind::Forward : MatvecKind::Adjoint, reps, tol, res);
    std::memcpy(chosen6, rep.chosen.render().c_str(), 6);
  });
}

static std::vector<ConfigResult> rows_from(std::size_t n, const double* mean, const double* err, const char* cfgs) {
  std::vector<ConfigResult> r(n);
  for (std::size_t i = 0; i < n; ++i) {
    r[i].config = parse_precision_config(std::string_view(cfgs + 5 * i, 5));
    r[i].mean_s = r[i].min_s = r[i].max_s = mean[i];
    r[i].rel_error = err[i];
  }
  return r;
}
// sweep.hpp:127-139 -> mask[i] = 1 iff row i is on the front
int ref_pareto(std::size_t n, const double* mean, const double* err, const char* cfgs, int* mask) {
  return guarded([&] {
    const auto rows = rows_from(n, mean, err, cfgs);
    const auto front = pareto_front(rows);
    for (std::size_t i = 0; i < n; ++i) {
      mask[i] = 0;
      for (const auto& f : front)
        if (f.config == rows[i].config && f.mean_s == rows[i].mean_s && f.rel_error == rows[i].rel_error) mask[i] = 1;
    }
  });
}
// sweep.hpp:143-156
int ref_optimal(std::size_t n, const double* mean, const double* err, const char* cfgs, double tol, char* out6) {
  return guarded([&] {
    const auto c = optimal_config(rows_from(n, mean, err, cfgs), tol);
    std::memcpy(out6, c.render().c_str(), 6);
  });
}

// CPU baseline: `threads` std::threads each run `per_thread` matvecs of the
// given kind concurrently on the shared operator (reentrant per SPEC.md:291).
// Returns wall seconds for the whole batch.
int ref_throughput(void* op, int kind, const char* cfg, const double* in, int threads, int per_thread,
                   double* seconds) {
  return guarded([&] {
    const auto* o = static_cast<SpectralOperator*>(op);
    const auto c = parse_precision_config(cfg);
    materialize_single(*o);
    const bool fwd = kind == 0;
    const std::size_t n_in = fwd ? o->dims.n_m : o->dims.n_d;
    const auto v = BlockVector::time_double(n_in, o->dims.n_t, std::vector<double>(in, in + n_in * o->dims.n_t));
    std::atomic<int> failures{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        try {
          for (int i = 0; i < per_thread; ++i) (void)(fwd ? forward_matvec(*o, v, c) : adjoint_matvec(*o, v, c));
        } catch (...) {
          failures.fetch_add(1);
        }
      });
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (failures.load()) throw std::runtime_error("ref_throughput: a worker thread failed");
  });
}

// CPU reference arm: `threads` std::threads run concurrently on the shared
// operator, even-numbered threads one forward matvec each, odd-numbered one
// adjoint matvec each. Wall seconds of the whole batch.
int ref_throughput_mixed(void* op, const char* cfg, const double* m, const double* d, int threads, double* seconds) {
  return guarded([&] {
    const auto* o = static_cast<SpectralOperator*>(op);
    const auto c = parse_precision_config(cfg);
    materialize_single(*o);
    const auto vm = BlockVector::time_double(o->dims.n_m, o->dims.n_t, std::vector<double>(m, m + o->dims.n_m * o->dims.n_t));
    const auto vd = BlockVector::time_double(o->dims.n_d, o->dims.n_t, std::vector<double>(d, d + o->dims.n_d * o->dims.n_t));
    std::atomic<int> failures{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        try {
          if (t % 2 == 0)
            (void)forward_matvec(*o, vm, c);
          else
            (void)adjoint_matvec(*o, vd, c);
        } catch (...) {
          failures.fetch_add(1);
        }
      });
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (failures.load()) throw std::runtime_error("ref_throughput_mixed: a worker thread failed");
  });
}

}  // extern "C"
