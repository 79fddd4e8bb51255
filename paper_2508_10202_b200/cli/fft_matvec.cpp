// fft_matvec -- command-line harness of the B200 FFTMatvec (SPEC.md cli
// module), written over the drop-in C++ API
// (include/fftmv/*.hpp -> libfftmv_cuda.so).
//
//   fft_matvec [-nm N] [-nd N] [-Nt N] [-prec CFG] [-rand] [-raw] [-s DIR]
//              [-p WORKERS] [-reps N] [-warmup N] [-tol X] [-sweep] [-seed S]
//
// Builds a synthetic block column (non-representable fill with -rand, else
// seeded uniform [-1,1)), then either times forward and adjoint matvecs in
// one precision config (per-phase mean/min/max; -raw: CSV
// `matvec,phase,mean_s,min_s,max_s`, 5 phase rows + a total row per matvec)
// or, with -sweep, all 32 configs (-raw: CSV `config,mean_s,min_s,max_s,rel_error`
// per direction, plus the chosen config under -tol). -p runs the 1 x p
// partition; -s saves the output vectors as FMV1 files. Exit codes: 0 ok,
// 2 usage error (message names the bad flag / config position), 1 runtime or
// I/O failure.
#include <algorithm>
#include <cstdio>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "fftmv/config.hpp"
#include "fftmv/matvec.hpp"
#include "fftmv/operator.hpp"
#include "fftmv/partition.hpp"
#include "fftmv/random_fill.hpp"
#include "fftmv/sweep.hpp"
#include "fftmv/vector_io.hpp"

using namespace fftmv;

namespace {

struct RunArgs {  // SPEC.md RunArgs defaults
  std::size_t n_m = 5000, n_d = 100, n_t = 1000;
  std::string prec = "ddddd";
  bool rand = false, raw = false, sweep = false;
  std::string save_dir;
  std::size_t workers = 1;
  int reps = 100, warmup = 2;
  double tol = 1e-7;
  std::uint64_t seed = 20250814;
};

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

const char* kUsage =
    "usage: fft_matvec [-nm N] [-nd N] [-Nt N] [-prec CFG] [-rand] [-raw] [-s DIR] [-p WORKERS]\n"
    "                  [-reps N] [-warmup N] [-tol X] [-sweep] [-seed S]\n";

std::uint64_t parse_uint(const std::string& flag, const char* v, std::uint64_t lo) {
  if (!v) throw Usage(flag + ": missing value");
  char* end = nullptr;
  errno = 0;
  const unsigned long long x = std::strtoull(v, &end, 10);
  if (errno || !end || *end || v[0] == '-' || x < lo) throw Usage(flag + ": invalid value '" + v + "'");
  return x;
}

RunArgs parse(int argc, char** argv) {
  RunArgs a;
  for (int i = 1; i < argc; ++i) {
    const std::string f = argv[i];
    const char* v = i + 1 < argc ? argv[i + 1] : nullptr;
    auto take = [&] { ++i; };
    if (f == "-nm") a.n_m = parse_uint(f, v, 1), take();
    else if (f == "-nd") a.n_d = parse_uint(f, v, 1), take();
    else if (f == "-Nt") a.n_t = parse_uint(f, v, 1), take();
    else if (f == "-p") a.workers = parse_uint(f, v, 1), take();
    else if (f == "-reps") a.reps = (int)parse_uint(f, v, 1), take();
    else if (f == "-warmup") a.warmup = (int)parse_uint(f, v, 0), take();
    else if (f == "-seed") a.seed = parse_uint(f, v, 0), take();
    else if (f == "-prec") {
      if (!v) throw Usage("-prec: missing value");
      try {
        (void)parse_precision_config(v);
      } catch (const std::invalid_argument& e) {
        throw Usage(std::string("-prec: ") + e.what());
      }
      a.prec = v;
      take();
    } else if (f == "-tol") {
      if (!v) throw Usage("-tol: missing value");
      char* end = nullptr;
      a.tol = std::strtod(v, &end);
      if (!end || *end || !(a.tol > 0)) throw Usage(std::string("-tol: invalid value '") + v + "'");
      take();
    } else if (f == "-s") {
      if (!v) throw Usage("-s: missing directory");
      a.save_dir = v;
      take();
    } else if (f == "-rand") a.rand = true;
    else if (f == "-raw") a.raw = true;
    else if (f == "-sweep") a.sweep = true;
    else throw Usage("unknown flag '" + f + "'");
  }
  if (a.workers > a.n_m) throw Usage("-p: more workers than parameter columns");
  return a;
}

struct Stat {
  double mean = 0, mn = std::numeric_limits<double>::infinity(), mx = 0;
  void add(double x) {
    mean += x;
    mn = std::min(mn, x);
    mx = std::max(mx, x);
  }
};

int run(const RunArgs& a) {
  const ProblemDims dims(a.n_m, a.n_d, a.n_t);
  auto fill = [&](std::size_t n, std::uint64_t k) {
    return a.rand ? non_representable_fill(n, seed_stream(a.seed, k)) : uniform_fill(n, seed_stream(a.seed, k));
  };
  BlockColumn col(dims, fill(dims.n_t * dims.n_d * dims.n_m, 0));
  const auto m = fill(dims.n_m * dims.n_t, 1);
  const auto d = fill(dims.n_d * dims.n_t, 2);
  const BlockVector mv = BlockVector::time_double(dims.n_m, dims.n_t, m);
  const BlockVector dv = BlockVector::time_double(dims.n_d, dims.n_t, d);
  const PrecisionConfig cfg = parse_precision_config(a.prec);

  if (a.sweep) {
    if (a.workers != 1) throw Usage("-sweep runs on the unpartitioned operator (drop -p)");
    const SpectralOperator op = setup_operator(col, HostBins::Skip);
    for (MatvecKind k : {MatvecKind::Forward, MatvecKind::Adjoint}) {
      auto rows = sweep_configs(op, k == MatvecKind::Forward ? std::span<const double>(m) : std::span<const double>(d),
                                k, a.reps, a.warmup);
      const SweepReport rep = make_report(dims, k, a.reps, a.tol, rows);
      if (a.raw) {
        std::cout << "# " << kind_name(k) << " chosen=" << rep.chosen.render() << " tol=" << a.tol << '\n'
                  << to_csv(rep);
      } else {
        std::printf("%s sweep (%zu x %zu x %zu, reps %d): chosen %s at tol %.3g\n", kind_name(k), dims.n_m,
                    dims.n_d, dims.n_t, a.reps, rep.chosen.render().c_str(), a.tol);
        std::printf("  %-7s %12s %12s %12s %12s\n", "config", "mean_s", "min_s", "max_s", "rel_error");
        for (const auto& r : rep.rows)
          std::printf("  %-7s %12.6e %12.6e %12.6e %12.4e\n", r.config.render().c_str(), r.mean_s, r.min_s, r.max_s,
                      r.rel_error);
      }
    }
    return 0;
  }

  std::vector<Stat> fs(6), as(6);
  BlockVector fo, ao;
  auto once = [&](bool record) {
    PhaseTimings tf, ta;
    if (a.workers == 1) {
      static const SpectralOperator op = setup_operator(col, HostBins::Skip);
      auto F = forward_matvec(op, mv, cfg);
      auto A = adjoint_matvec(op, dv, cfg);
      tf = F.timings, ta = A.timings, fo = std::move(F.output), ao = std::move(A.output);
    } else {
      static const PartitionedOperator pop = setup_partitioned(col, Grid1xP::split(a.workers, dims.n_m));
      auto F = forward_matvec_partitioned(pop, mv, cfg);
      auto A = adjoint_matvec_partitioned(pop, dv, cfg);
      tf = F.timings, ta = A.timings, fo = std::move(F.output), ao = std::move(A.output);
    }
    if (!record) return;
    for (int i = 0; i < 5; ++i) fs[i].add(tf.phase_s[i]), as[i].add(ta.phase_s[i]);
    fs[5].add(tf.total_s), as[5].add(ta.total_s);
  };
  for (int w = 0; w < a.warmup; ++w) once(false);
  for (int r = 0; r < a.reps; ++r) once(true);
  auto emit = [&](const char* name, std::vector<Stat>& st) {
    for (int i = 0; i < 6; ++i) {
      const char* ph = i < 5 ? phase_name(i) : "total";
      const double mean = st[i].mean / a.reps;
      if (a.raw)
        std::printf("%s,%s,%.9e,%.9e,%.9e\n", name, ph, mean, st[i].mn, st[i].mx);
      else
        std::printf("  %-8s %-10s mean %11.6f ms  min %11.6f ms  max %11.6f ms\n", name, ph, mean * 1e3,
                    st[i].mn * 1e3, st[i].mx * 1e3);
    }
  };
  if (a.raw) std::printf("matvec,phase,mean_s,min_s,max_s\n");
  else
    std::printf("fft_matvec %zu x %zu x %zu, cfg %s, p=%zu, reps %d (B200, libfftmv_cuda)\n", dims.n_m, dims.n_d,
                dims.n_t, a.prec.c_str(), a.workers, a.reps);
  emit("forward", fs);
  emit("adjoint", as);
  if (!a.save_dir.empty()) {
    std::error_code ec;
    std::filesystem::create_directories(a.save_dir, ec);
    if (ec) throw std::runtime_error("-s: cannot create " + a.save_dir + ": " + ec.message());
    save_vector(a.save_dir + "/forward_output.fmv", fo);
    save_vector(a.save_dir + "/adjoint_output.fmv", ao);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  RunArgs a;
  try {
    a = parse(argc, argv);
  } catch (const Usage& e) {
    std::fprintf(stderr, "fft_matvec: %s\n%s", e.what(), kUsage);
    return 2;
  }
  try {
    return run(a);
  } catch (const Usage& e) {
    std::fprintf(stderr, "fft_matvec: %s\n%s", e.what(), kUsage);
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "fft_matvec: %s\n", e.what());
    return 1;
  }
}
